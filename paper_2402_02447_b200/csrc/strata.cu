// H2 / K2 — stratum histogram + stable partition (sm_100a).
//
// Reference: stratify (strata.py:61-83): stratum of a sample is
// searchsorted(bounds, length, side='left') (:74), samples are appended to
// their stratum in input order (:81), probs = count/N (:82; host side).
//
// Two launches for ALL rank shards at once (HBM/L2-streaming, 8 B/key
// algorithmic: 4 B length read, 4 B id written; +4 B if explicit ids are read):
//   k_strata_count  : one CTA per 4096-key tile -> per-tile per-stratum counts
//                     (striped loads, #{len > bound} per bound, differenced;
//                     + the shard's first bad index via atomicMin)
//                     and, in the LAST tile of each shard to finish (atomic
//                     ticket), the shard's exclusive per-tile prefixes (in
//                     place over the tile counts) and per-stratum totals —
//                     no scan launch, no O(tiles^2) re-summing
//   k_strata_scatter: one CTA per tile reads its prefix row + the shard totals,
//                     then places its keys with stable in-tile ranks from a
//                     single packed block scan (4 strata x 16-bit fields per
//                     u64), staged through shared memory so each stratum's run
//                     is written with consecutive addresses.
#include "common.cuh"

#include <cub/block/block_load.cuh>
#include <cub/block/block_scan.cuh>

#include <algorithm>

namespace b2 {
namespace {

constexpr int kMaxStrata = 16;
constexpr int kT = 256;            // threads per tile CTA
constexpr int kItems = 16;         // keys per thread
constexpr int kTile = kT * kItems; // 4096 keys per tile (fits 16-bit fields)

constexpr int kMaxShards = 64;  // shards (segments) per launch

struct StrataParams {
  const int32_t* len;
  const int32_t* ids;  // may be null: id = index within the shard
  int nb, nshard;
  int32_t bounds[kMaxStrata];
  int64_t shard_off[kMaxShards + 1];  // element offset of each shard
  int32_t tile_off[kMaxShards + 1];   // first tile of each shard
  int32_t* tile_counts;               // [T][kMaxStrata]: counts, then exclusive in-shard prefixes
  unsigned* shard_done;               // [kMaxShards] tiles counted per shard (zeroed per launch)
  int64_t* counts;                    // [nshard][nb] totals
  int64_t* bad;                       // [nshard] first bad index within the shard (u64 min), pre-set to -1
  int32_t* ids_out;                   // same offsets as the input
};

template <int NB>
__device__ __forceinline__ int stratum_of(int32_t len, const StrataParams& p) {
  int k = 0;
#pragma unroll
  for (int j = 0; j < NB; ++j) k += (len > p.bounds[j]);  // == searchsorted(..., 'left'); unused bounds are INT32_MAX
  return k;
}

__device__ __forceinline__ int shard_of_tile(const StrataParams& p, int tile) {
  int g = 0;
  while (g + 1 < p.nshard && p.tile_off[g + 1] <= tile) ++g;
  return g;
}

template <int NW>
struct Packed {
  unsigned long long w[NW];
  __device__ __forceinline__ Packed operator+(const Packed& o) const {
    Packed r;
#pragma unroll
    for (int i = 0; i < NW; ++i) r.w[i] = w[i] + o.w[i];
    return r;
  }
  __device__ __forceinline__ unsigned field(int k) const {
    return (unsigned)((w[k >> 2] >> ((k & 3) * 16)) & 0xffffull);
  }
};

using LoadT = cub::BlockLoad<int32_t, kT, kItems, cub::BLOCK_LOAD_WARP_TRANSPOSE>;

// pass 1: per-tile stratum counts (+ first bad sample of the shard).  Order
// is irrelevant for counting, so keys load striped (direct coalesced loads),
// and each thread counts #{len > bound_j} per bound with the bounds in
// registers; stratum counts are differences of those (stratum 0 also drops
// lengths < 1; lengths beyond the last bound cancel out).  Bad samples only
// cost a block OR unless one exists.
template <int NB>
__global__ void __launch_bounds__(kT) k_strata_count(const __grid_constant__ StrataParams p) {
  __shared__ int cnt[kMaxStrata + 1];  // [NB] strata, [NB] = valid keys >= 1
  const int tile = blockIdx.x;
  const int g = shard_of_tile(p, tile);
  const int64_t sbeg = p.shard_off[g], send = p.shard_off[g + 1];
  const int64_t lbase = (int64_t)(tile - p.tile_off[g]) * kTile;  // within the shard
  const int valid = (int)min64(kTile, send - sbeg - lbase);
  if (threadIdx.x <= kMaxStrata) cnt[threadIdx.x] = 0;
  const int32_t* L = p.len + sbeg + lbase;
  int32_t bnd[NB];
#pragma unroll
  for (int q = 0; q < NB; ++q) bnd[q] = p.bounds[q];
  const int32_t blast = p.bounds[p.nb - 1];
  int32_t v[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int idx = j * kT + threadIdx.x;
    v[j] = idx < valid ? L[idx] : 1;  // padding: a length that counts nowhere (fixed below)
  }
  int gt[NB];
#pragma unroll
  for (int q = 0; q < NB; ++q) gt[q] = 0;
  int pos = 0, anybad = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int32_t x = v[j];
    pos += (x >= 1);
#pragma unroll
    for (int q = 0; q < NB; ++q) gt[q] += (x > bnd[q]);
    anybad |= (x < 1) | (x > blast);
  }
  // padding slots were given length 1: they count in `pos` only; remove them
  pos -= kItems - (valid > threadIdx.x ? (valid - 1 - (int)threadIdx.x) / kT + 1 : 0);
  __syncthreads();  // cnt zeroed
  if (__syncthreads_or(anybad)) {  // rare: locate the tile's first bad sample
    long long first_bad = -1;
#pragma unroll
    for (int j = kItems - 1; j >= 0; --j) {  // keeps the smallest index
      const int idx = j * kT + threadIdx.x;
      if (idx < valid && (v[j] < 1 || v[j] > blast)) first_bad = lbase + idx;
    }
    if (first_bad >= 0) atomicMin(reinterpret_cast<unsigned long long*>(p.bad + g), (unsigned long long)first_bad);
  }
  // stratum q < nb: gt[q-1] - gt[q] (q = 0: pos - gt[0]); warp sums, then one smem add per warp
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    int c = (q == 0 ? pos : gt[q - 1]) - gt[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c && q < p.nb) atomicAdd(&cnt[q], c);
  }
  __syncthreads();
  if (threadIdx.x < NB) p.tile_counts[(int64_t)tile * kMaxStrata + threadIdx.x] = threadIdx.x < p.nb ? cnt[threadIdx.x] : 0;

  // the shard's last tile to finish turns its tile counts into exclusive
  // prefixes (in place) and publishes the shard totals
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned nt = (unsigned)(p.tile_off[g + 1] - p.tile_off[g]);
    s_last = atomicAdd(&p.shard_done[g], 1u) == nt - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int t0 = p.tile_off[g], t1 = p.tile_off[g + 1], nt = t1 - t0;
  const int per = (nt + kT - 1) / kT;  // contiguous tiles per thread
  const int a = min(t0 + (int)threadIdx.x * per, t1), b = min(a + per, t1);
  using Scan = cub::BlockScan<int, kT>;
  __shared__ typename Scan::TempStorage scan;
  __shared__ int64_t s_tot[NB];
  for (int k = 0; k < NB; ++k) {
    int sum = 0;
    for (int t = a; t < b; ++t) sum += __ldcg(&p.tile_counts[(int64_t)t * kMaxStrata + k]);
    int ex, agg;
    Scan(scan).ExclusiveSum(sum, ex, agg);
    for (int t = a; t < b; ++t) {
      int32_t* c = &p.tile_counts[(int64_t)t * kMaxStrata + k];
      const int v = __ldcg(c);
      *c = ex;
      ex += v;
    }
    if (threadIdx.x == 0) s_tot[k] = agg;
    __syncthreads();  // scan storage reuse
  }
  if (threadIdx.x < p.nb) p.counts[(int64_t)g * p.nb + threadIdx.x] = s_tot[threadIdx.x];
}

// pass 2: each tile sums the counts of the earlier tiles of its shard (one L2
// round trip, no separate scan launch), then scatters with stable in-tile
// ranks from a single packed block scan, staged so runs are written coalesced
template <int NB>
__global__ void __launch_bounds__(kT) k_strata_scatter(const __grid_constant__ StrataParams p) {
  constexpr int NW = (NB + 3) / 4;
  using Scan = cub::BlockScan<Packed<NW>, kT>;
  __shared__ union {
    typename LoadT::TempStorage ld;
    typename Scan::TempStorage scan;
    int32_t stage[kTile];
  } sm;
  __shared__ int32_t s_kof[kTile];       // stratum of each staged slot
  __shared__ int64_t s_dst[kMaxStrata];  // global start of this tile's run, per stratum
  __shared__ int32_t s_lstart[kMaxStrata + 1];
  __shared__ unsigned long long s_pre[kMaxStrata], s_tot[kMaxStrata];
  const int tile = blockIdx.x;
  const int g = shard_of_tile(p, tile);
  const int64_t sbeg = p.shard_off[g], send = p.shard_off[g + 1];
  const int64_t lbase = (int64_t)(tile - p.tile_off[g]) * kTile;
  const int valid = (int)min64(kTile, send - sbeg - lbase);
  if (threadIdx.x < kMaxStrata) {  // this tile's exclusive prefix + the shard totals (from pass 1)
    const bool in = threadIdx.x < p.nb;
    s_pre[threadIdx.x] = in ? (unsigned long long)p.tile_counts[(int64_t)tile * kMaxStrata + threadIdx.x] : 0ull;
    s_tot[threadIdx.x] = in ? (unsigned long long)p.counts[(int64_t)g * p.nb + threadIdx.x] : 0ull;
  }
  int32_t v[kItems];
  LoadT(sm.ld).Load(p.len + sbeg + lbase, v, valid, 1);
  __syncthreads();
  int32_t id[kItems];
  if (p.ids) {
    LoadT(sm.ld).Load(p.ids + sbeg + lbase, id, valid, 0);
    __syncthreads();
  } else {
#pragma unroll
    for (int j = 0; j < kItems; ++j) id[j] = (int32_t)(lbase + threadIdx.x * kItems + j);
  }
  int8_t kk[kItems];
  Packed<NW> mine;
#pragma unroll
  for (int i = 0; i < NW; ++i) mine.w[i] = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int idx = threadIdx.x * kItems + j;
    int k = -1;
    if (idx < valid) {
      k = stratum_of<NB>(v[j], p);
      if (k >= p.nb || v[j] < 1) k = -1;  // bad samples are reported, not placed
    }
    kk[j] = (int8_t)k;
    if (k >= 0) mine.w[k >> 2] += 1ull << ((k & 3) * 16);
  }
  Packed<NW> ex, agg;
  Scan(sm.scan).ExclusiveSum(mine, ex, agg);
  if (threadIdx.x == 0) {
    int acc = 0;
    int64_t gbase = sbeg;
    for (int k = 0; k < p.nb; ++k) {
      s_lstart[k] = acc;
      acc += (int)agg.field(k);
      s_dst[k] = gbase + (int64_t)s_pre[k];
      gbase += (int64_t)s_tot[k];
    }
    s_lstart[p.nb] = acc;
  }
  __syncthreads();  // also retires the scan temp storage before staging
  unsigned run[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) run[k] = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int k = kk[j];
    if (k >= 0) {
      unsigned r = 0;
#pragma unroll
      for (int q = 0; q < NB; ++q)
        if (q == k) {
          r = run[q];
          run[q] = r + 1;
        }
      const int slot = s_lstart[k] + (int)ex.field(k) + (int)r;
      sm.stage[slot] = id[j];
      s_kof[slot] = k;
    }
  }
  __syncthreads();
  const int placed = s_lstart[p.nb];
  for (int slot = threadIdx.x; slot < placed; slot += kT) {
    const int k = s_kof[slot];
    p.ids_out[s_dst[k] + (slot - s_lstart[k])] = sm.stage[slot];
  }
}

}  // namespace
}  // namespace b2

using namespace b2;

static inline int64_t strata_tiles(int64_t n) { return (n + kTile - 1) / kTile; }

extern "C" size_t b2_strata_workspace_bytes(int64_t n) {
  if (n < 1) n = 1;
  // per-shard tile tickets; per-tile counts (+ one partial tile per shard boundary)
  return kMaxShards * sizeof(unsigned) + (size_t)(strata_tiles(n) + kMaxShards) * kMaxStrata * sizeof(int32_t);
}

extern "C" int b2_strata_partition_shards(const int32_t* lengths, const int32_t* ids, const int64_t* shard_off,
                                          int nshard, const int32_t* bounds, int nb, int32_t* ids_out,
                                          int64_t* counts, int64_t* bad, void* workspace, size_t workspace_bytes,
                                          void* stream) {
  B2_REQUIRE(lengths && ids_out && counts && bad && bounds && shard_off, B2_ERR_INVALID, "NULL pointer argument");
  B2_REQUIRE(nshard >= 1 && nshard <= kMaxShards, B2_ERR_UNSUPPORTED, "nshard must be in [1, %d]", kMaxShards);
  B2_REQUIRE(nb >= 1 && nb <= kMaxStrata, B2_ERR_UNSUPPORTED, "nb must be in [1, %d], got %d", kMaxStrata, nb);
  B2_REQUIRE(bounds[0] >= 1, B2_ERR_INVALID, "boundaries must be >= 1");
  for (int k = 1; k < nb; ++k)
    B2_REQUIRE(bounds[k - 1] < bounds[k], B2_ERR_INVALID, "boundaries must be strictly ascending");
  StrataParams p{};
  p.len = lengths;
  p.ids = ids;
  p.nb = nb;
  p.nshard = nshard;
  for (int k = 0; k < kMaxStrata; ++k) p.bounds[k] = k < nb ? bounds[k] : INT32_MAX;
  int64_t T = 0;
  p.shard_off[0] = shard_off[0];
  for (int g = 0; g < nshard; ++g) {
    const int64_t n = shard_off[g + 1] - shard_off[g];
    B2_REQUIRE(n >= 1 && n <= INT32_MAX, B2_ERR_INVALID, "shard %d must hold 1..2^31-1 samples", g);
    p.shard_off[g + 1] = shard_off[g + 1];
    p.tile_off[g] = (int32_t)T;
    T += strata_tiles(n);
  }
  p.tile_off[nshard] = (int32_t)T;
  const size_t need = kMaxShards * sizeof(unsigned) + (size_t)T * kMaxStrata * sizeof(int32_t);
  B2_REQUIRE(workspace && workspace_bytes >= need, B2_ERR_INVALID, "strata workspace needs %zu bytes", need);
  p.shard_done = static_cast<unsigned*>(workspace);
  p.tile_counts = reinterpret_cast<int32_t*>(static_cast<char*>(workspace) + kMaxShards * sizeof(unsigned));
  p.counts = counts;
  p.bad = bad;
  p.ids_out = ids_out;
  cudaStream_t st = (cudaStream_t)stream;
  B2_CHECK(cudaMemsetAsync(bad, 0xff, sizeof(int64_t) * nshard, st));
  B2_CHECK(cudaMemsetAsync(p.shard_done, 0, sizeof(unsigned) * nshard, st));
  if (nb <= 4) {
    k_strata_count<4><<<(unsigned)T, kT, 0, st>>>(p);
    B2_CHECK(cudaGetLastError());
    k_strata_scatter<4><<<(unsigned)T, kT, 0, st>>>(p);
  } else if (nb <= 8) {
    k_strata_count<8><<<(unsigned)T, kT, 0, st>>>(p);
    B2_CHECK(cudaGetLastError());
    k_strata_scatter<8><<<(unsigned)T, kT, 0, st>>>(p);
  } else {
    k_strata_count<16><<<(unsigned)T, kT, 0, st>>>(p);
    B2_CHECK(cudaGetLastError());
    k_strata_scatter<16><<<(unsigned)T, kT, 0, st>>>(p);
  }
  B2_CHECK(cudaGetLastError());
  return B2_OK;
}

extern "C" int b2_strata_partition(const int32_t* lengths, const int32_t* ids, int64_t n,
                                   const int32_t* bounds, int nb, int32_t* ids_out, int64_t* counts,
                                   int64_t* bad, void* workspace, size_t workspace_bytes, void* stream) {
  B2_REQUIRE(n >= 1 && n <= INT32_MAX, B2_ERR_INVALID, "n must be in [1, 2^31-1], got %lld", (long long)n);
  const int64_t off[2] = {0, n};
  return b2_strata_partition_shards(lengths, ids, off, 1, bounds, nb, ids_out, counts, bad, workspace,
                                    workspace_bytes, stream);
}
