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

// Warp-per-pool COUNTING sort (lengths are small integers), sized for
// occupancy (~2.8 KB of shared memory per warp, two registers per key).
// Per pool:
//   1. length histogram, two 16-bit bins per word; the packed atomic's old
//      value ranks each key inside its bin (bin 0 = longest);
//   2. one warp scan turns the packed counts into packed bin starts;
//   3. each id is scattered to start+rank of its bin.  Every key of a bin has
//      the same length, so the bin's contribution to each GPU lane's token sum
//      (_from_per_gpu, balance.py:54-56) is fixed by the bin's slots alone and
//      is added here, before the order inside the bin is known;
//   4. each bin is put in id order (the reference's (-len, id) key,
//      balance.py:73-75): bins of 2+ keys are listed by their second key and
//      insertion-sorted in place, one lane per bin (bins hold ~1 key on real
//      data); bins above kCntBig keys are ranked by the whole warp instead.  Equal (len, id) pairs are identical
//      samples, so their order is immaterial;
//   5. the deal is a GATHER: output slot o = lane*rows + r reads sorted
//      position r*lanes + c (c mirrored on odd rows for SNAKE,
//      balance.py:59-70), so the [lanes][rows] tile is written with
//      consecutive addresses and no staging buffer.
// The next pool's lines are prefetched into L2 while this one is sorted.
// Input order inside a pool is irrelevant to the result, so VEC loads 4
// consecutive keys per lane.
constexpr int kCntWarps = 4;
constexpr int kCntBins = 1024;   // max_len limit of the counting path
constexpr int kCntMaxSeg = 512;  // pool limit of the counting path
constexpr int kCntTok = 64;      // lanes whose token sums stay in shared memory (more: global atomics)
constexpr int kCntBig = 24;      // bins above this many keys are sorted by the whole warp

template <int KM, int HW, int MINB, bool VEC>
__global__ void __launch_bounds__(32 * kCntWarps, MINB) k_presort_deal_count(const __grid_constant__ PresortParams p) {
  constexpr int PM = 32 * KM;    // pool capacity
  constexpr int WPL = HW / 32;   // histogram words per lane in the scan (2 bins each)
  __shared__ __align__(16) uint32_t s_hist[kCntWarps][HW];  // packed counts, then packed starts
  __shared__ int32_t s_srt[kCntWarps][PM];                  // ids grouped by bin, then sorted
  __shared__ int32_t s_tok[kCntWarps][kCntTok];             // per-lane token sums
  __shared__ int16_t s_mul[kCntWarps][PM / 2];              // bins with 2+ keys; big bins from the top
  __shared__ int s_cnt[kCntWarps][2];                       // list lengths
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int M = p.max_len, P = p.seg_len, rows = p.rows, lanes = p.lanes;
  uint32_t* hist = s_hist[w];
  int32_t* srt = s_srt[w];
  int32_t* stok = s_tok[w];
  int16_t* smul = s_mul[w];
  const bool tok_smem = lanes <= kCntTok;
  const float inv_lanes = 1.0f / (float)lanes;
  const int ln0 = lane / rows, r0 = lane - ln0 * rows;  // deal coordinates of output slot `lane`
  const int dq = 32 / rows, dr = 32 - dq * rows;        // ... and their step per 32 slots
  const int64_t nwarps = (int64_t)gridDim.x * kCntWarps;
  for (int k = lane; k < kCntTok; k += 32) stok[k] = 0;
  if (lane < 2) s_cnt[w][lane] = 0;
  __syncwarp();
  for (int64_t seg = (int64_t)blockIdx.x * kCntWarps + w; seg < p.nseg; seg += nwarps) {
    const int64_t base = seg * P;
    if (KM > 4 && seg + nwarps < p.nseg) {  // next pool of this warp -> L2 (128-key pools: other warps hide the
      // loads and the prefetch only costs instructions, 75.8 -> 69.6 us at lb16)
      const int64_t nb = base + nwarps * P;
      const int nl = (P * 4 + 127) / 128 + 1;
      for (int k = lane; k < 2 * nl; k += 32) {
        const int32_t* a0 = (k < nl ? p.lens : p.ids) + nb;
        const int32_t* a = a0 + (int64_t)(k < nl ? k : k - nl) * 32;
        if (a < a0 + P) asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
      }
    }
#pragma unroll
    for (int k = lane; k < HW / 4; k += 32) reinterpret_cast<uint4*>(hist)[k] = make_uint4(0, 0, 0, 0);
    if (!tok_smem && p.tokens)
      for (int k = lane; k < lanes; k += 32) p.tokens[seg * lanes + k] = 0;
    __syncwarp();
    uint32_t kb[KM];  // (bin << 16) | rank in bin
    int32_t kd[KM];   // ids
    long long first_bad = -1;
    auto add_key = [&](int j, int64_t flat, int32_t L, int32_t D) {
      if (!(L >= 1 && L <= M && D >= 0 && D <= p.max_id)) {
        if (first_bad < 0 || flat < first_bad) first_bad = flat;
        L = L < 1 ? 1 : (L > M ? M : L);  // keep the slot well-formed; the caller raises
      }
      const uint32_t bin = (uint32_t)(M - L), sh = (bin & 1u) << 4;
      B2_DASSERT((int)(bin >> 1) < HW);
      const uint32_t old = atomicAdd(&hist[bin >> 1], 1u << sh);
      kb[j] = (bin << 16) | ((old >> sh) & 0xffffu);
      kd[j] = D;
    };
    auto live = [&](int j) { return VEC ? ((j / 4) * 32 + lane) * 4 < P : j * 32 + lane < P; };
    if constexpr (VEC) {
#pragma unroll
      for (int j4 = 0; j4 < KM / 4; ++j4) {
        const int i = (j4 * 32 + lane) * 4;
        if (i < P) {
          const int4 L4 = __ldg(reinterpret_cast<const int4*>(p.lens + base + i));
          const int4 D4 = __ldg(reinterpret_cast<const int4*>(p.ids + base + i));
          add_key(4 * j4 + 0, base + i + 0, L4.x, D4.x);
          add_key(4 * j4 + 1, base + i + 1, L4.y, D4.y);
          add_key(4 * j4 + 2, base + i + 2, L4.z, D4.z);
          add_key(4 * j4 + 3, base + i + 3, L4.w, D4.w);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < KM; ++j) {
        const int i = j * 32 + lane;  // striped: coalesced loads
        if (i < P) add_key(j, base + i, __ldg(p.lens + base + i), __ldg(p.ids + base + i));
      }
    }
    if (first_bad >= 0 && p.bad) atomicMin(reinterpret_cast<unsigned long long*>(p.bad), (unsigned long long)first_bad);
    __syncwarp();
    {  // packed exclusive scan: lane owns WPL consecutive words = bins [2*WPL*lane, 2*WPL*(lane+1))
      uint32_t v[WPL];
#pragma unroll
      for (int k = 0; k < WPL / 4; ++k) {
        const uint4 q = reinterpret_cast<const uint4*>(hist)[lane * (WPL / 4) + k];
        v[4 * k] = q.x, v[4 * k + 1] = q.y, v[4 * k + 2] = q.z, v[4 * k + 3] = q.w;
      }
      uint32_t tot = 0;
#pragma unroll
      for (int k = 0; k < WPL; ++k) tot += (v[k] & 0xffffu) + (v[k] >> 16);
      uint32_t inc = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      uint32_t ex = inc - tot;
#pragma unroll
      for (int k = 0; k < WPL; ++k) {
        const uint32_t lo = v[k] & 0xffffu, hi = v[k] >> 16;
        v[k] = ex | ((ex + lo) << 16);
        ex += lo + hi;
      }
#pragma unroll
      for (int k = 0; k < WPL / 4; ++k)
        reinterpret_cast<uint4*>(hist)[lane * (WPL / 4) + k] = make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
    }
    __syncwarp();
    int32_t* out = p.out_ids + base;
    // bins with 2+ keys are listed by their second key: above 128-key pools by a warp
    // ballot (no same-address shared atomics; 71.7 -> 68 us at lb48), for 128-key pools
    // by one shared atomic (the ballots cost more there: 69.6 -> 71.7 us at lb16)
    constexpr bool kBallotList = KM > 4;
    int nm = 0;  // warp-uniform count (ballot form)
#pragma unroll
    for (int j = 0; j < KM; ++j) {  // ids into their bins; the bin's slots fix its token shares
      const bool lvj = live(j);
      unsigned second = 0;
      if constexpr (kBallotList) second = __ballot_sync(0xffffffffu, lvj && (kb[j] & 0xffffu) == 1u);
      if (lvj) {
        const uint32_t bin = kb[j] >> 16, rk = kb[j] & 0xffffu;
        const int pos = (int)(((hist[bin >> 1] >> ((bin & 1u) << 4)) & 0xffffu) + rk);
        B2_DASSERT(pos >= 0 && pos < P);
        srt[pos] = kd[j];
        if (rk == 1) {  // the bin holds 2+ keys
          const int q = kBallotList ? nm + __popc(second & ((1u << lane) - 1u)) : atomicAdd(&s_cnt[w][0], 1);
          B2_DASSERT(q < PM / 2);
          smul[q] = (int16_t)bin;
        }
        if (p.tokens) {  // the GPU lane slot `pos` is dealt to
          const int r = __float2int_rd(((float)pos + 0.5f) * inv_lanes), c = pos - r * lanes;
          const int g = (p.snake && (r & 1)) ? lanes - 1 - c : c;
          const int L = M - (int)bin;
          B2_DASSERT(g >= 0 && g < lanes);
          if (tok_smem) atomicAdd(&stok[g], L);
          else atomicAdd(reinterpret_cast<unsigned long long*>(p.tokens + seg * lanes + g), (unsigned long long)L);
        }
      }
      if constexpr (kBallotList) nm += __popc(second);
    }
    if (kBallotList && lane == 0) s_cnt[w][0] = nm;
    __syncwarp();
    // bins with 2+ keys (listed by their second key in the scatter) are put in id order,
    // spread over the lanes; bins above kCntBig keys go to a second list for the whole warp
    const int nmulti = s_cnt[w][0];
    auto bstart = [&](int b) { return b < M ? (int)((hist[b >> 1] >> ((b & 1) << 4)) & 0xffffu) : P; };
    for (int q = lane; q < nmulti; q += 32) {
      const int b = smul[q], st = bstart(b), e = bstart(b + 1);
      if (e - st > kCntBig) {
        const int qb = PM / 2 - 1 - atomicAdd(&s_cnt[w][1], 1);  // big list grows from the top
        B2_DASSERT(qb >= nmulti);
        smul[qb] = (int16_t)b;
        continue;
      }
      for (int x = st + 1; x < e; ++x) {  // insertion sort, ids ascending
        const int32_t val = srt[x];
        int y = x - 1;
        int32_t prev = srt[y];
        while (prev > val) {
          srt[y + 1] = prev;
          if (--y < st) break;
          prev = srt[y];
        }
        srt[y + 1] = val;
      }
    }
    __syncwarp();
    const int nbig = s_cnt[w][1];
    for (int q = 0; q < nbig; ++q) {
      // rank every element by (id, slot) against the bin; stage the sorted bin in this pool's
      // own output rows (global, rewritten by the gather below)
      const int b = smul[PM / 2 - 1 - q], st = bstart(b), e = bstart(b + 1);
      for (int x = st + lane; x < e; x += 32) {
        const int32_t me = srt[x];
        int f = st;
        for (int y = st; y < e; ++y) {
          const int32_t o = srt[y];
          f += (o < me) || (o == me && y < x);
        }
        B2_DASSERT(f >= st && f < e);
        out[f] = me;
      }
      __syncwarp();
      for (int x = st + lane; x < e; x += 32) srt[x] = out[x];
      __syncwarp();
    }
    if (lane == 0) s_cnt[w][0] = s_cnt[w][1] = 0;
    __syncwarp();
    int ln = ln0, r = r0;
#pragma unroll 4
    for (int o = lane; o < P; o += 32) {  // the deal as a gather (balance.py:59-70)
      const int c = (p.snake && (r & 1)) ? lanes - 1 - ln : ln;
      B2_DASSERT(r < rows && c >= 0 && c < lanes && r * lanes + c < P);
      out[o] = srt[r * lanes + c];
      r += dr;
      ln += dq;
      if (r >= rows) {
        r -= rows;
        ++ln;
      }
    }
    if (tok_smem && p.tokens) {
      __syncwarp();
      for (int k = lane; k < lanes; k += 32) {
        p.tokens[seg * lanes + k] = stok[k];
        stok[k] = 0;
      }
    }
    __syncwarp();  // shared buffers are reused by the next pool
  }
}

template <int KM, int HW>
int launch_count(const PresortParams& p, cudaStream_t st) {
  // CTAs per SM from the shared-memory footprint (+1 KB reserved per CTA)
  constexpr int kSmem = kCntWarps * (HW * 4 + 32 * KM * 5 + kCntTok * 4 + 8);
  // and registers: 64 per thread (8 CTAs) keeps the unrolled loads spill-free;
  // the 256-bin pools up to 384 keys fit 48 (10 CTAs)
  constexpr int kRegB = 8;
  constexpr int kSmemB = (220 * 1024) / (kSmem + 1024);
  constexpr int kMinB = kSmemB < kRegB ? kSmemB : kRegB;
  const DeviceInfo& di = device_info();
  const int64_t blocks = (p.nseg + kCntWarps - 1) / kCntWarps;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)di.sm_count * kMinB));
  const bool vec = KM % 4 == 0 && p.seg_len % 4 == 0 && ((uintptr_t)p.ids & 15) == 0 && ((uintptr_t)p.lens & 15) == 0;
  if (vec) k_presort_deal_count<KM, HW, kMinB, true><<<grid, 32 * kCntWarps, 0, st>>>(p);
  else k_presort_deal_count<KM, HW, kMinB, false><<<grid, 32 * kCntWarps, 0, st>>>(p);
  B2_CHECK(cudaGetLastError());
  return B2_OK;
}

template <int HW>
int launch_count_km(const PresortParams& p, cudaStream_t st) {
  if (p.seg_len <= 128) return launch_count<4, HW>(p, st);
  if (p.seg_len <= 256) return launch_count<8, HW>(p, st);
  if (p.seg_len <= 384) return launch_count<12, HW>(p, st);
  return launch_count<16, HW>(p, st);
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
  // B2_PRESORT_PATH=bitonic|count forces one warp path (A/B runs, tests)
  static int variant = -1;
  if (variant < 0) {
    const char* e = getenv("B2_PRESORT_PATH");
    variant = (e && !strcmp(e, "bitonic")) ? 1 : (e && !strcmp(e, "count")) ? 2 : 0;
  }
  const bool count_ok = !out_pos && seg_len <= kCntMaxSeg && max_len <= kCntBins;
  // counting sort pays when the pool is not tiny next to the length bins
  if (count_ok && (variant == 2 || (variant == 0 && 4 * seg_len >= max_len)))
    return max_len <= 512 ? launch_count_km<256>(p, st) : launch_count_km<512>(p, st);
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
