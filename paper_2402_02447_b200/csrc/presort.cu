// H2 / K3 — per-pool stable sort by (-length, id) + raster/snake deal (sm_100a).
//
// Reference: assign_local_presort (balance.py:158-184) pools each node's GPU
// draws in GPU order (:179-182), sorts them with key (-length, id) using a
// stable sort (_sorted_desc, :73-75), deals rows of `lanes` items, reversing
// odd rows for SNAKE (_deal, :59-70), and sums lengths per lane
// (_from_per_gpu, :54-56).  assign_global_presort (:83-88) is the same with a
// single pool.
//
// The composite key ((max_len - len) << id_bits) | id orders exactly like
// (-len, id); equal keys are identical samples, so the order among them
// cannot change the output.  Three paths, all equal to the reference:
//   * counting sort, one warp per pool (lengths <= 1024, the pool fills at
//     least half the length bins, e.g. 384-key pools): length histogram with
//     ranks from the atomics, warp scan, scatter, ids ordered inside
//     equal-length bins;
//   * bitonic network, one warp per pool (pools <= 512, e.g. 128-key pools):
//     64-bit composite keys in registers, shuffles across lanes;
//   * stable LSD radix sort, one CTA per pool (any pool <= 4096, and the only
//     path that also returns each sample's input slot): cub::BlockRadixSort
//     limited to the bits the key actually spans.
// Each sorted slot is dealt to (lane, row) and staged in shared memory so the
// [lanes][rows] output tile is written with consecutive addresses; token sums
// read the staged lengths.
#include "bitonic.cuh"
#include "common.cuh"

#include <cub/block/block_radix_sort.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

namespace b2 {
namespace {

constexpr int kMaxSeg = 4096;

struct PresortParams {
  const int32_t* ids;
  const int32_t* lens;
  int64_t nseg;
  int seg_len, lanes, rows, snake;
  int32_t max_len, max_id;
  int id_bits, end_bit;
  int32_t* out_ids;
  int32_t* out_pos;  // optional: flat input index of each dealt sample
  int64_t* tokens;
  int64_t* bad;
};

template <int T, int I, bool POS>
__global__ void __launch_bounds__(T) k_presort_deal(const __grid_constant__ PresortParams p) {
  // POS: carry each sample's input slot through the sort (a stable LSD radix
  // sort keeps equal keys in input order, exactly like Timsort at :75)
  using Sort = cub::BlockRadixSort<unsigned long long, T, I, typename std::conditional<POS, int32_t, cub::NullType>::type>;
  __shared__ union {
    typename Sort::TempStorage sort;
    struct {
      int32_t ids[T * I];   // dealt layout [lane][row]
      int32_t lens[T * I];
      int16_t pos[POS ? T * I : 1];  // slot within the pool (< 4096)
    } stage;
  } sm;
  const unsigned long long idmask = (1ull << p.id_bits) - 1ull;
  for (int64_t seg = blockIdx.x; seg < p.nseg; seg += gridDim.x) {
    const int64_t base = seg * p.seg_len;
    unsigned long long key[I];
    int32_t slot[I];
    long long first_bad = -1;
#pragma unroll
    for (int j = 0; j < I; ++j) {
      const int i = threadIdx.x * I + j;  // blocked: keeps input order for stability
      slot[j] = i;
      if (i < p.seg_len) {
        const int32_t L = p.lens[base + i], D = p.ids[base + i];
        const bool ok = L >= 1 && L <= p.max_len && D >= 0 && D <= p.max_id;
        if (!ok && first_bad < 0) first_bad = base + i;
        key[j] = ((unsigned long long)(uint32_t)(p.max_len - L) << p.id_bits) | (unsigned long long)(uint32_t)D;
      } else {
        key[j] = ~0ull;  // padding sorts last (stable: after any equal real key)
      }
    }
    if (first_bad >= 0 && p.bad) atomicMin(reinterpret_cast<unsigned long long*>(p.bad), (unsigned long long)first_bad);
    if constexpr (POS) Sort(sm.sort).Sort(key, slot, 0, p.end_bit);
    else Sort(sm.sort).Sort(key, 0, p.end_bit);
    __syncthreads();  // sort temp storage -> staging buffer
#pragma unroll
    for (int j = 0; j < I; ++j) {
      const int pos = threadIdx.x * I + j;
      if (pos < p.seg_len) {
        const int r = pos / p.lanes, c = pos - r * p.lanes;
        const int lane = (p.snake && (r & 1)) ? p.lanes - 1 - c : c;  // balance.py:66-67
        const int32_t id = (int32_t)(key[j] & idmask);
        const int32_t len = p.max_len - (int32_t)(key[j] >> p.id_bits);
        sm.stage.ids[lane * p.rows + r] = id;
        sm.stage.lens[lane * p.rows + r] = len;
        if constexpr (POS) sm.stage.pos[lane * p.rows + r] = (int16_t)slot[j];
      }
    }
    __syncthreads();
    int32_t* out = p.out_ids + base;
    for (int i = threadIdx.x; i < p.seg_len; i += T) out[i] = sm.stage.ids[i];
    if constexpr (POS)
      for (int i = threadIdx.x; i < p.seg_len; i += T) p.out_pos[base + i] = (int32_t)base + sm.stage.pos[i];
    if (p.tokens)
      for (int l = threadIdx.x; l < p.lanes; l += T) {
        int64_t s = 0;  // per-lane token sum (_from_per_gpu, balance.py:54-56)
        for (int r = 0; r < p.rows; ++r) s += sm.stage.lens[l * p.rows + r];
        p.tokens[seg * p.lanes + l] = s;
      }
    __syncthreads();  // staging / tok reused by the next pool
  }
}

// Warp-per-pool bitonic sort (pools <= 32*K keys, K keys per lane, blocked:
// element i = lane*K + j).  The composite key is unique per (len, id), so an
// unstable network yields exactly the reference's stable order whenever the
// caller does not need input slots (out_pos); ties of identical samples are
// indistinguishable.  Padding keys (all ones) sort last.
template <int K, int WARPS>
__global__ void __launch_bounds__(32 * WARPS) k_presort_deal_warp(const __grid_constant__ PresortParams p) {
  constexpr int n = 32 * K;
  __shared__ int32_t s_ids[WARPS][n];
  __shared__ int32_t s_lens[WARPS][n];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned long long idmask = (1ull << p.id_bits) - 1ull;
  const int64_t nwarps = (int64_t)gridDim.x * WARPS;
  for (int64_t seg = (int64_t)blockIdx.x * WARPS + w; seg < p.nseg; seg += nwarps) {
    const int64_t base = seg * p.seg_len;
    unsigned long long key[K];
    long long first_bad = -1;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int i = lane * K + j;
      if (i < p.seg_len) {
        const int32_t L = p.lens[base + i], D = p.ids[base + i];
        const bool ok = L >= 1 && L <= p.max_len && D >= 0 && D <= p.max_id;
        if (!ok && first_bad < 0) first_bad = base + i;
        key[j] = ((unsigned long long)(uint32_t)(p.max_len - L) << p.id_bits) | (unsigned long long)(uint32_t)D;
      } else {
        key[j] = ~0ull;
      }
    }
    if (first_bad >= 0 && p.bad) atomicMin(reinterpret_cast<unsigned long long*>(p.bad), (unsigned long long)first_bad);
    warp_bitonic_sort<K>(key, lane);
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int pos = lane * K + j;
      if (pos < p.seg_len) {
        const int r = pos / p.lanes, c = pos - r * p.lanes;
        const int ln = (p.snake && (r & 1)) ? p.lanes - 1 - c : c;  // balance.py:66-67
        s_ids[w][ln * p.rows + r] = (int32_t)(key[j] & idmask);
        s_lens[w][ln * p.rows + r] = p.max_len - (int32_t)(key[j] >> p.id_bits);
      }
    }
    __syncwarp();
    int32_t* out = p.out_ids + base;
    for (int i = lane; i < p.seg_len; i += 32) out[i] = s_ids[w][i];
    if (p.tokens)
      for (int l = lane; l < p.lanes; l += 32) {
        int64_t sum = 0;  // per-lane token sum (_from_per_gpu, balance.py:54-56)
        for (int r = 0; r < p.rows; ++r) sum += s_lens[w][l * p.rows + r];
        p.tokens[seg * p.lanes + l] = sum;
      }
    __syncwarp();
  }
}

// Warp-per-pool COUNTING sort (lengths are small integers): histogram of the
// pool's lengths in shared memory (the atomic's return value ranks each key
// inside its bin), one warp scan over the bins, a scatter into sorted order,
// then ids ordered inside each multi-key bin (equal lengths; a handful of
// keys on real data).  O(pool) work instead of the bitonic network's
// O(pool log^2 pool) 64-bit compare-exchanges; (-len, id) is unique per
// sample, so the output is the same.  Pools <= 512 keys, lengths <= 1024.
constexpr int kCntBins = 1024;
constexpr int kCntMaxSeg = 512;

template <int WARPS>
__global__ void __launch_bounds__(32 * WARPS) k_presort_deal_count(const __grid_constant__ PresortParams p) {
  __shared__ int s_hist[WARPS][kCntBins];         // counts, then bin starts
  __shared__ int32_t s_sid[WARPS][kCntMaxSeg];    // sorted ids
  __shared__ int16_t s_slen[WARPS][kCntMaxSeg];   // sorted lengths
  __shared__ int32_t s_oid[WARPS][kCntMaxSeg];    // dealt [lane][row]
  __shared__ int16_t s_olen[WARPS][kCntMaxSeg];
  constexpr int KM = kCntMaxSeg / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int M = p.max_len, P = p.seg_len;
  const int per = (M + 31) / 32;  // bins per lane in the scan
  int* hist = s_hist[w];
  const int64_t nwarps = (int64_t)gridDim.x * WARPS;
  for (int64_t seg = (int64_t)blockIdx.x * WARPS + w; seg < p.nseg; seg += nwarps) {
    const int64_t base = seg * P;
    for (int b = lane; b < M; b += 32) hist[b] = 0;
    __syncwarp();
    int32_t id[KM];
    int16_t len[KM], rk[KM];
    long long first_bad = -1;
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      const int i = j * 32 + lane;  // striped: coalesced loads
      if (i < P) {
        int32_t L = p.lens[base + i];
        const int32_t D = p.ids[base + i];
        if (!(L >= 1 && L <= M && D >= 0 && D <= p.max_id)) {
          if (first_bad < 0) first_bad = base + i;
          L = L < 1 ? 1 : (L > M ? M : L);  // keep the slot well-formed; the caller raises
        }
        id[j] = D;
        len[j] = (int16_t)L;
        rk[j] = (int16_t)atomicAdd(&hist[M - L], 1);  // bin 0 = longest
      }
    }
    if (first_bad >= 0 && p.bad) atomicMin(reinterpret_cast<unsigned long long*>(p.bad), (unsigned long long)first_bad);
    __syncwarp();
    {  // exclusive scan over the M bins: `per` contiguous bins per lane
      const int b0 = lane * per, b1 = min(b0 + per, M);
      int sum = 0;
      for (int b = b0; b < b1; ++b) sum += hist[b];
      int inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      int ex = inc - sum;
      for (int b = b0; b < b1; ++b) {
        const int c = hist[b];
        hist[b] = ex;
        ex += c;
      }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      const int i = j * 32 + lane;
      if (i < P) {
        const int pos = hist[M - len[j]] + rk[j];
        s_sid[w][pos] = id[j];
        s_slen[w][pos] = len[j];
      }
    }
    __syncwarp();
    {  // equal lengths: ids ascending inside each bin (insertion sort; bins are tiny)
      const int b0 = lane * per, b1 = min(b0 + per, M);
      for (int b = b0; b < b1; ++b) {
        const int st = hist[b], en = b + 1 < M ? hist[b + 1] : P;
        for (int x = st + 1; x < en; ++x) {
          const int32_t v = s_sid[w][x];
          int y = x - 1;
          while (y >= st && s_sid[w][y] > v) {
            s_sid[w][y + 1] = s_sid[w][y];
            --y;
          }
          s_sid[w][y + 1] = v;
        }
      }
    }
    __syncwarp();
    for (int q = lane; q < P; q += 32) {  // deal (balance.py:59-70)
      const int r = q / p.lanes, c = q - r * p.lanes;
      const int ln = (p.snake && (r & 1)) ? p.lanes - 1 - c : c;
      s_oid[w][ln * p.rows + r] = s_sid[w][q];
      s_olen[w][ln * p.rows + r] = s_slen[w][q];
    }
    __syncwarp();
    int32_t* out = p.out_ids + base;
    for (int i = lane; i < P; i += 32) out[i] = s_oid[w][i];
    if (p.tokens)
      for (int l = lane; l < p.lanes; l += 32) {
        int64_t sum = 0;  // per-lane token sum (_from_per_gpu, balance.py:54-56)
        for (int r = 0; r < p.rows; ++r) sum += s_olen[w][l * p.rows + r];
        p.tokens[seg * p.lanes + l] = sum;
      }
    __syncwarp();
  }
}

template <int WARPS>
int launch_count(const PresortParams& p, cudaStream_t st) {
  const DeviceInfo& di = device_info();
  const int64_t blocks = (p.nseg + WARPS - 1) / WARPS;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)di.sm_count * 16));
  k_presort_deal_count<WARPS><<<grid, 32 * WARPS, 0, st>>>(p);
  B2_CHECK(cudaGetLastError());
  return B2_OK;
}

template <int K, int WARPS>
int launch_warp(const PresortParams& p, cudaStream_t st) {
  const DeviceInfo& di = device_info();
  const int64_t blocks = (p.nseg + WARPS - 1) / WARPS;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)di.sm_count * 16));
  k_presort_deal_warp<K, WARPS><<<grid, 32 * WARPS, 0, st>>>(p);
  B2_CHECK(cudaGetLastError());
  return B2_OK;
}

int bits_for(int64_t v) {  // bits needed to represent 0..v
  int b = 0;
  while (b < 63 && (1ll << b) <= v) ++b;
  return b;
}

template <int T, int I>
int launch(const PresortParams& p, cudaStream_t st) {
  const DeviceInfo& di = device_info();
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(p.nseg, (int64_t)di.sm_count * 32));
  if (p.out_pos) k_presort_deal<T, I, true><<<grid, T, 0, st>>>(p);
  else k_presort_deal<T, I, false><<<grid, T, 0, st>>>(p);
  B2_CHECK(cudaGetLastError());
  return B2_OK;
}

}  // namespace
}  // namespace b2

using namespace b2;

extern "C" int b2_presort_deal(const int32_t* ids, const int32_t* lens, int64_t nseg, int seg_len,
                               int lanes, int scan, int32_t max_len, int32_t max_id,
                               int32_t* out_ids, int32_t* out_pos, int64_t* tokens, int64_t* bad,
                               void* stream) {
  B2_REQUIRE(lanes >= 1, B2_ERR_INVALID, "lanes must be >= 1, got %d", lanes);
  B2_REQUIRE(seg_len >= 0, B2_ERR_INVALID, "seg_len must be >= 0");
  B2_REQUIRE(seg_len % lanes == 0, B2_ERR_INDIVISIBLE, "%d items do not divide over %d GPUs", seg_len, lanes);
  B2_REQUIRE(seg_len <= kMaxSeg, B2_ERR_UNSUPPORTED, "seg_len %d exceeds %d", seg_len, kMaxSeg);
  B2_REQUIRE(max_len >= 1 && max_id >= 0, B2_ERR_INVALID, "max_len must be >= 1 and max_id >= 0");
  B2_REQUIRE(scan == B2_SCAN_RASTER || scan == B2_SCAN_SNAKE, B2_ERR_INVALID, "bad scan %d", scan);
  cudaStream_t st = (cudaStream_t)stream;
  if (bad) B2_CHECK(cudaMemsetAsync(bad, 0xff, sizeof(int64_t), st));
  if (nseg <= 0 || seg_len == 0) return B2_OK;
  B2_REQUIRE(ids && lens && out_ids, B2_ERR_INVALID, "NULL pointer argument");
  PresortParams p{};
  p.ids = ids;
  p.lens = lens;
  p.nseg = nseg;
  p.seg_len = seg_len;
  p.lanes = lanes;
  p.rows = seg_len / lanes;
  p.snake = scan == B2_SCAN_SNAKE;
  p.max_len = max_len;
  p.max_id = max_id;
  p.id_bits = std::max(1, bits_for(max_id));
  p.end_bit = p.id_bits + std::max(1, bits_for((int64_t)max_len - 1));
  p.out_ids = out_ids;
  p.out_pos = out_pos;
  p.tokens = tokens;
  p.bad = bad;
  B2_REQUIRE(p.end_bit <= 64, B2_ERR_UNSUPPORTED, "key does not fit 64 bits");
  static int variant = -1;  // B2_PRESORT_PATH=bitonic forces the network (A/B runs, tests)
  if (variant < 0) {
    const char* e = getenv("B2_PRESORT_PATH");
    variant = (e && !strcmp(e, "bitonic")) ? 1 : 0;
  }
  // counting sort pays when the pool fills at least half of the length bins
  // (lb48: 384 keys / 512 bins, 1.37x over the network); smaller pools sort
  // faster in registers than the bins can be cleared and scanned (lb16: 3x)
  if (!out_pos && variant == 0 && seg_len <= kCntMaxSeg && max_len <= kCntBins && 2 * seg_len >= max_len)
    return launch_count<4>(p, st);
  if (!out_pos) {  // no input slots needed: warp-per-pool bitonic network
    if (seg_len <= 64) return launch_warp<2, 8>(p, st);
    if (seg_len <= 128) return launch_warp<4, 8>(p, st);
    if (seg_len <= 256) return launch_warp<8, 4>(p, st);
    if (seg_len <= 512) return launch_warp<16, 2>(p, st);
  }
  if (seg_len <= 128) return launch<32, 4>(p, st);
  if (seg_len <= 512) return launch<128, 4>(p, st);
  if (seg_len <= 2048) return launch<256, 8>(p, st);
  return launch<512, 8>(p, st);
}
