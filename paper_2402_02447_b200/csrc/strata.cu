// H2 / K2 — stratum histogram + stable partition (sm_100a).
//
// Reference: stratify (strata.py:61-83): stratum of a sample is
// searchsorted(bounds, length, side='left') (:74), samples are appended to
// their stratum in input order (:81), probs = count/N (:82; host side).
//
// Three launches for ALL rank shards at once.  Algorithmic traffic is 8 B/key
// (4 B length read, 4 B id written; +4 B if explicit ids are read); the
// launches move 8.5 B/key (2-bit stratum codes, 4-bit above 4 strata):
//   k_strata_count  : one CTA per 4096-key tile reads the lengths once (16 B
//                     vector loads, all issued up front), writes each key's
//                     stratum CODE packed 16 per word (0.25 B/key) and the
//                     tile's per-stratum counts — no tail, so CTAs retire as
//                     soon as their stores are issued;
//   k_strata_scan   : one CTA per shard turns the tile counts into exclusive
//                     in-shard prefixes and writes the shard totals;
//   k_strata_scatter: one CTA per tile, one warp per 512 keys, reads only the
//                     codes.  A warp counts its words with bit tricks, the
//                     tile's warps are offset through shared memory; with <= 4
//                     strata each lane then holds, for its word, the first
//                     output slot of every code, and a key's slot is that
//                     slot (four shuffles + a select) + the count of its code
//                     in the earlier fields of its word; with more strata a
//                     round's ranks come from one ballot per code bit.  Each
//                     id is stored straight to its final slot (a round writes
//                     <= nb contiguous runs: coalesced, no staging).
// A bad sample (length < 1 or above the last bound) is reported through
// `bad` (the wrapper raises like the reference); it is placed in an edge
// stratum, so ids_out/counts of that shard are unspecified.
#include "common.cuh"

#include <cub/block/block_scan.cuh>

#include <algorithm>

namespace b2 {
namespace {

constexpr int kMaxStrata = 16;
constexpr int kT = 256;            // threads per tile CTA
constexpr int kTile = 4096;        // keys per tile (8 warps x 512)
constexpr int kWarpKeys = 512;     // keys per warp in the scatter
constexpr int kMaxShards = 64;     // shards (segments) per launch
constexpr int kScanT = 1024;       // threads of the per-shard tile-count scan

struct StrataParams {
  const int32_t* len;
  const int32_t* ids;  // may be null: id = index within the shard
  int nb, nshard;
  int32_t bounds[kMaxStrata];
  int shift;  // >= 0: bounds are (q+1) << shift (the count pass shifts instead of comparing)
  int64_t shard_off[kMaxShards + 1];  // element offset of each shard
  int32_t tile_off[kMaxShards + 1];   // first tile of each shard
  int32_t* tile_counts;               // [T][kMaxStrata]: counts, then the tile's first in-shard slot per stratum
  uint32_t* codes;                    // [T][kTile * CB / 32] packed stratum codes
  int64_t* counts;                    // [nshard][nb] totals
  int64_t* bad;                       // [nshard] first bad index within the shard (u64 min), pre-set to -1
  int32_t* ids_out;                   // same offsets as the input
};

template <int NB>
__host__ __device__ constexpr int code_bits() { return NB <= 4 ? 2 : 4; }

__device__ __forceinline__ int shard_of_tile(const StrataParams& p, int tile) {
  int lo = 0, hi = p.nshard - 1;  // last g with tile_off[g] <= tile (binary search, <= 6 steps)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.tile_off[mid] <= tile) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// pass 1: codes + per-tile counts (+ the shard's first bad sample).  The code is
// sum_{q < nb-1} (len > bound_q): a length above the last bound lands in the
// last stratum and one below 1 in the first (the last with shift codes), so
// bad samples need no branch.
template <int NB, bool UNIFORM>
__global__ void __launch_bounds__(kT) k_strata_count(const __grid_constant__ StrataParams p) {
  pdl_trigger();  // the scan may launch now (it waits for this grid before reading)
  constexpr int CB = code_bits<NB>();
  constexpr int WPT = kTile * CB / 32;   // code words per tile
  constexpr int QPW = 32 / (4 * CB);     // 4-key quads per word (4 or 2)
  __shared__ int cnt[kMaxStrata];
  const int tile = blockIdx.x;
  const int g = shard_of_tile(p, tile);
  const int64_t sbeg = p.shard_off[g], send = p.shard_off[g + 1];
  const int64_t lbase = (int64_t)(tile - p.tile_off[g]) * kTile;  // within the shard
  const int valid = (int)min64(kTile, send - sbeg - lbase);
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < kMaxStrata) cnt[threadIdx.x] = 0;
  const int32_t* L = p.len + sbeg + lbase;
  const bool vec = (((uintptr_t)L) & 15) == 0 && valid == kTile;
  int32_t bnd[NB - 1 > 0 ? NB - 1 : 1];
#pragma unroll
  for (int q = 0; q < NB - 1; ++q) bnd[q] = q < p.nb - 1 ? p.bounds[q] : INT32_MAX;
  const uint32_t blast = (uint32_t)p.bounds[p.nb - 1];
  // per-thread counts: quads counted from their packed codes
  int c[NB];
#pragma unroll
  for (int q = 0; q < NB; ++q) c[q] = 0;
  bool anybad = false;
  uint32_t* cw = p.codes + (int64_t)tile * WPT;
  constexpr int R = kTile / (4 * kT);  // rounds of 4 consecutive keys per thread
  int32_t xs[R][4];
#pragma unroll
  for (int it = 0; it < R; ++it) {  // every load issued before any use
    const int i0 = (it * kT + threadIdx.x) * 4;
    if (vec) {
      const int4 q = __ldcs(reinterpret_cast<const int4*>(L + i0));
      xs[it][0] = q.x, xs[it][1] = q.y, xs[it][2] = q.z, xs[it][3] = q.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) xs[it][e] = i0 + e < valid ? __ldcs(L + i0 + e) : 1;
    }
  }
#pragma unroll
  for (int it = 0; it < R; ++it) {
    const int i0 = (it * kT + threadIdx.x) * 4;
    const int32_t* x = xs[it];
    uint32_t packed = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int k = 0;
      if constexpr (UNIFORM) {
        // bounds (q+1) * 2^shift: searchsorted(..., 'left') = (len-1) >> shift, clamped (a
        // length below 1 wraps to the last stratum: bad, the shard's output is unspecified)
        k = (int)min((uint32_t)(x[e] - 1) >> p.shift, (uint32_t)(p.nb - 1));
      } else {
#pragma unroll
        for (int q = 0; q < NB - 1; ++q) k += (x[e] > bnd[q]);  // == searchsorted(..., 'left')
      }
      anybad |= (uint32_t)(x[e] - 1) >= blast;               // len < 1 or len > last bound
      packed |= (uint32_t)k << (e * CB);
    }
    const int nv = vec ? 4 : max(0, min(4, valid - i0));  // keys of this quad inside the tile
    if (CB == 2) {  // counts of codes 1..3 from the 2-bit fields; code 0 = the rest
      const uint32_t lo = packed & 0x55u, hi = (packed >> 1) & 0x55u;
      c[1] += __popc(lo & ~hi);
      if (NB > 2) c[2] += __popc(hi & ~lo);
      if (NB > 3) c[3] += __popc(lo & hi);
      c[0] += nv;  // minus the others at the end
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (e < nv) {
          const int k = (int)((packed >> (e * CB)) & 15u);
#pragma unroll
          for (int q = 0; q < NB; ++q) c[q] += (k == q);
        }
    }
    // lanes QPW*m .. QPW*m + QPW-1 hold one word's quads
#pragma unroll
    for (int o = 1; o < QPW; o <<= 1) packed |= __shfl_down_sync(0xffffffffu, packed, o) << (o * 4 * CB);
    B2_DASSERT((i0 / 4) / QPW < WPT);
    if ((lane & (QPW - 1)) == 0) cw[(i0 / 4) / QPW] = packed;
  }
  if (CB == 2) c[0] -= c[1] + (NB > 2 ? c[2] : 0) + (NB > 3 ? c[3] : 0);
  if (__syncthreads_or(anybad)) {  // rare: the tile's first bad sample (smallest index)
    long long first_bad = -1;
    for (int i = (int)threadIdx.x; i < valid && first_bad < 0; i += kT) {
      const int32_t x = L[i];
      if ((uint32_t)(x - 1) >= blast) first_bad = lbase + i;
    }
    if (first_bad >= 0) atomicMin(reinterpret_cast<unsigned long long*>(p.bad + g), (unsigned long long)first_bad);
  }
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    const int v = (int)__reduce_add_sync(0xffffffffu, (unsigned)c[q]);  // one REDUX per stratum
    if (lane == 0 && v && q < p.nb) atomicAdd(&cnt[q], v);
  }
  __syncthreads();
  if (threadIdx.x < NB) p.tile_counts[(int64_t)tile * kMaxStrata + threadIdx.x] = threadIdx.x < p.nb ? cnt[threadIdx.x] : 0;
}

// pass 1b: one CTA per shard turns its tile counts into each tile's first
// in-shard slot per stratum (exclusive prefix + the earlier strata's totals,
// in place) and writes the shard totals.  Each thread owns a run
// of consecutive tiles and reads each tile's count row once (16 B vectors);
// the NB block scans run back to back on register sums.
template <int NB>
__global__ void __launch_bounds__(kScanT) k_strata_scan(const __grid_constant__ StrataParams p) {
  pdl_trigger();
  pdl_wait();  // the count grid's tile counts are complete and visible
  using Scan = cub::BlockScan<int, kScanT>;
  __shared__ typename Scan::TempStorage scan;
  const int g = blockIdx.x;
  const int t0 = p.tile_off[g], t1 = p.tile_off[g + 1], nt = t1 - t0;
  const int per = (nt + kScanT - 1) / kScanT;  // contiguous tiles per thread
  const int a = min(t0 + (int)threadIdx.x * per, t1), b = min(a + per, t1);
  int sum[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) sum[k] = 0;
  for (int t = a; t < b; ++t) {
    const int4* row = reinterpret_cast<const int4*>(p.tile_counts + (int64_t)t * kMaxStrata);
#pragma unroll
    for (int q = 0; q < NB / 4; ++q) {
      const int4 v = row[q];
      sum[4 * q] += v.x, sum[4 * q + 1] += v.y, sum[4 * q + 2] += v.z, sum[4 * q + 3] += v.w;
    }
  }
  int ex[NB];
  int base = 0;  // slots of the earlier strata in this shard: the prefixes are final in-shard slots
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    int agg;
    if (k) __syncthreads();  // scan storage reuse
    Scan(scan).ExclusiveSum(sum[k], ex[k], agg);
    if (threadIdx.x == 0 && k < p.nb) p.counts[(int64_t)g * p.nb + k] = agg;
    ex[k] += base;
    base += agg;
  }
  for (int t = a; t < b; ++t) {
    int4* row = reinterpret_cast<int4*>(p.tile_counts + (int64_t)t * kMaxStrata);
#pragma unroll
    for (int q = 0; q < NB / 4; ++q) {
      const int4 v = row[q];
      row[q] = make_int4(ex[4 * q], ex[4 * q + 1], ex[4 * q + 2], ex[4 * q + 3]);
      ex[4 * q] += v.x, ex[4 * q + 1] += v.y, ex[4 * q + 2] += v.z, ex[4 * q + 3] += v.w;
    }
  }
}

// pass 2: scatter from the codes.  A warp owns 512 consecutive keys; the
// tile's warps are offset by a shared-memory scan of their per-stratum
// counts; inside a warp, 16 rounds of 32 keys in input order.  Lane k < nb
// carries stratum k's next output slot (32-bit, within the shard).
template <int NB, bool IDS, bool FULL>
__device__ __forceinline__ void scatter_rounds(const StrataParams& p, const uint32_t (&word)[(kWarpKeys * code_bits<NB>() / 32) / 32],
                                               int next, int32_t* out, const int32_t* ids, int wbase, int valid,
                                               int shard_n) {
  constexpr int CB = code_bits<NB>();
  constexpr int WPL = (kWarpKeys * CB / 32) / 32;  // code words per lane (1 or 2)
  constexpr int KPW = 32 / CB;                     // keys per word
  constexpr uint32_t CMASK = (1u << CB) - 1u;
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  const int shift = (lane % KPW) * CB;  // field of this lane's key in its word (32 % KPW == 0)
  uint32_t inv[CB];                     // lane k's code bits, as select masks
#pragma unroll
  for (int b = 0; b < CB; ++b) inv[b] = ((lane >> b) & 1) ? 0u : 0xffffffffu;
#pragma unroll
  for (int j = 0; j < kWarpKeys / 32; ++j) {
    const int key = j * 32 + lane;   // warp-local key of this lane in round j
    const int wi = key / KPW;        // its word (warp-local)
    uint32_t wsel;
    if constexpr (WPL == 1) {
      wsel = __shfl_sync(0xffffffffu, word[0], wi);
    } else {
      const uint32_t a0 = __shfl_sync(0xffffffffu, word[0], wi >> 1), a1 = __shfl_sync(0xffffffffu, word[WPL - 1], wi >> 1);
      wsel = (wi & 1) ? a1 : a0;
    }
    const bool ok = FULL || wbase + key < valid;
    const int code = (int)((wsel >> shift) & CMASK);
    const uint32_t live = FULL ? 0xffffffffu : __ballot_sync(0xffffffffu, ok);
    uint32_t diff = 0, mk = live;  // lanes whose code differs from mine; lanes with code == lane
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      const uint32_t bits = __ballot_sync(0xffffffffu, (code >> b) & 1);
      diff |= bits ^ (((code >> b) & 1) ? 0xffffffffu : 0u);
      mk &= bits ^ inv[b];
    }
    const int base = __shfl_sync(0xffffffffu, next, code);
    B2_DASSERT(!ok || (base + __popc(~diff & live & lt) >= 0 && base + __popc(~diff & live & lt) < shard_n));
    if (ok) out[base + __popc(~diff & live & lt)] = IDS ? __ldcs(ids + wbase + key) : wbase + key;
    next += __popc(mk);
  }
}

// NB <= 4 (2-bit codes, one word of 16 keys per lane): the lane holding word
// wi writes, for each code c, the slot of the first key of code c in that
// word (stratum base + count of code c in earlier words of the warp) to a
// shared [word][code] table; a key's slot is its (word, code) entry + the
// count of its code in the earlier fields of the word.  No per-round
// ballots, scans or base updates.
template <bool IDS, bool FULL>
__device__ __forceinline__ void scatter_rounds_prefix(uint32_t word, const int* slot_tab, int32_t* out,
                                                      const int32_t* ids, int wbase, int valid, int shard_n) {
  constexpr uint32_t LOW = 0x55555555u;
  const int lane = threadIdx.x & 31;
  const int f = lane & 15, half = lane >> 4;
  const uint32_t below = LOW & ((1u << (2 * f)) - 1u);  // low bits of the fields before this lane's field
#pragma unroll
  for (int j = 0; j < kWarpKeys / 32; ++j) {
    const int wi = 2 * j + half;  // word of this lane's key in round j
    const int key = j * 32 + lane;
    const uint32_t wv = __shfl_sync(0xffffffffu, word, wi);
    const uint32_t code = (wv >> (2 * f)) & 3u;
    const uint32_t y = wv ^ (LOW * code);
    const int inword = __popc(~(y | (y >> 1)) & below);
    const int sc = slot_tab[wi * 4 + (int)code];
    B2_DASSERT(!(FULL || wbase + key < valid) || (sc + inword >= 0 && sc + inword < shard_n));
    // unsigned in-shard slot: one IMAD.WIDE.U32 per address instead of a 64-bit add + shifts
    if (FULL || wbase + key < valid)
      out[(uint32_t)(sc + inword)] = IDS ? __ldcs(ids + (uint32_t)(wbase + key)) : wbase + key;
  }
}

template <int NB>
__global__ void __launch_bounds__(kT) k_strata_scatter(const __grid_constant__ StrataParams p) {
  pdl_wait();  // codes, tile prefixes and shard totals are complete and visible
  constexpr int CB = code_bits<NB>();
  constexpr int WPT = kTile * CB / 32;           // code words per tile
  constexpr int WPW = kWarpKeys * CB / 32;       // code words per warp (32 or 64)
  constexpr int WPL = WPW / 32;                  // ... per lane (1 or 2)
  constexpr int KPW = 32 / CB;                   // keys per word
  __shared__ int s_wcnt[kT / 32][kMaxStrata];
  __shared__ int s_dst[kMaxStrata];
  __shared__ __align__(16) int s_slot[kT / 32][CB == 2 ? 32 * 4 : 1];  // [word][code] first slots (<= 4 strata)
  __shared__ int s_g;
  const int tile = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wbeg = w * kWarpKeys;  // first key of this warp in the tile
  uint32_t word[WPL];
  const uint32_t* cw = p.codes + (int64_t)tile * WPT + w * WPW;
#pragma unroll
  for (int i = 0; i < WPL; ++i) word[i] = __ldcs(cw + lane * WPL + i);  // in flight during the lookup below
  if (threadIdx.x < NB) s_dst[threadIdx.x] = p.tile_counts[(int64_t)tile * kMaxStrata + threadIdx.x];  // first in-shard slot per stratum
  if (threadIdx.x == 0) s_g = shard_of_tile(p, tile);  // the tile's shard: one lookup per CTA
  __syncthreads();
  const int g = s_g;
  const int64_t sbeg = p.shard_off[g], send = p.shard_off[g + 1];
  const int64_t lbase = (int64_t)(tile - p.tile_off[g]) * kTile;
  const int valid = (int)min64(kTile, send - sbeg - lbase);
  if constexpr (CB == 2) {
    // per-word counts of codes 0..2 (keys beyond `valid` masked out), packed 10 bits each
    constexpr uint32_t LOW = 0x55555555u;
    const int k0 = wbeg + lane * 16;
    const int nv = max(0, min(16, valid - k0));
    const uint32_t vmask = nv >= 16 ? 0xffffffffu : ((1u << (nv * 2)) - 1u);
    uint32_t pk = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const uint32_t y = word[0] ^ (LOW * (uint32_t)k);
      pk |= (uint32_t)__popc(~(y | (y >> 1)) & LOW & vmask) << (10 * k);
    }
    uint32_t inc = pk;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
    const int wkeys = max(0, min(kWarpKeys, valid - wbeg));
    if (lane < 4) {
      const int t0 = (int)(tot & 1023u), t1 = (int)((tot >> 10) & 1023u), t2 = (int)(tot >> 20);
      s_wcnt[w][lane] = lane == 0 ? t0 : lane == 1 ? t1 : lane == 2 ? t2 : wkeys - t0 - t1 - t2;
    }
    __syncthreads();
    int next = 0;  // lane k < nb: first slot of stratum k for this warp (within the shard)
    if (lane < p.nb) {
      int off = s_dst[lane];
#pragma unroll
      for (int u = 0; u < kT / 32 - 1; ++u)
        if (u < w) off += s_wcnt[u][lane];
      next = off;
    }
    int32_t* out = opaque(p.ids_out + sbeg);  // one base register: slot addresses are one IMAD.WIDE.U32
    const int wbase = (int)lbase + wbeg;  // shard-local index of this warp's first key
    const int32_t* ids = p.ids ? p.ids + sbeg : nullptr;
    const int wvalid = (int)lbase + valid;
    const uint32_t ex = inc - pk;  // codes 0..2 in the warp's earlier words
    const int e0 = (int)(ex & 1023u), e1 = (int)((ex >> 10) & 1023u), e2 = (int)(ex >> 20);
    // this word's first slot per code (stratum base + the code's keys in earlier words)
    int* tab = s_slot[w];
    reinterpret_cast<int4*>(tab)[lane] = make_int4(
        __shfl_sync(0xffffffffu, next, 0) + e0, __shfl_sync(0xffffffffu, next, 1) + e1,
        __shfl_sync(0xffffffffu, next, 2) + e2,
        __shfl_sync(0xffffffffu, next, 3) + 16 * lane - e0 - e1 - e2);  // earlier words are full
    __syncwarp();
    if (wbeg + kWarpKeys <= valid) {
      if (ids) scatter_rounds_prefix<true, true>(word[0], tab, out, ids, wbase, wvalid, (int)(send - sbeg));
      else scatter_rounds_prefix<false, true>(word[0], tab, out, ids, wbase, wvalid, (int)(send - sbeg));
    } else {
      if (ids) scatter_rounds_prefix<true, false>(word[0], tab, out, ids, wbase, wvalid, (int)(send - sbeg));
      else scatter_rounds_prefix<false, false>(word[0], tab, out, ids, wbase, wvalid, (int)(send - sbeg));
    }
    return;
  } else {
    // per-stratum counts of this warp's keys (keys beyond `valid` masked out)
  int mine[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) mine[k] = 0;
#pragma unroll
  for (int i = 0; i < WPL; ++i) {
    const int k0 = wbeg + (lane * WPL + i) * KPW;  // first key of this word
    const int nv = max(0, min(KPW, valid - k0));
    const uint32_t vmask = nv >= KPW ? 0xffffffffu : ((1u << (nv * CB)) - 1u);
    uint32_t low = 0;
#pragma unroll
    for (int f = 0; f < KPW; ++f) low |= 1u << (f * CB);
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      // fields equal to k: XOR with k replicated, then fields that are all-zero
      const uint32_t y = word[i] ^ (low * (uint32_t)k);
      uint32_t z = y;
#pragma unroll
      for (int b = 1; b < CB; ++b) z |= y >> b;  // low bit of each field = OR of the field's bits
      mine[k] += __popc(~z & low & vmask);
    }
  }
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    const int v = (int)__reduce_add_sync(0xffffffffu, (unsigned)mine[k]);
    if (lane == k) s_wcnt[w][k] = v;
  }
  __syncthreads();
  int next = 0;  // lane k < nb: next output slot of stratum k for this warp (within the shard)
  if (lane < p.nb) {
    int off = s_dst[lane];
#pragma unroll
    for (int u = 0; u < kT / 32 - 1; ++u)
      if (u < w) off += s_wcnt[u][lane];
    next = off;
  }
  int32_t* out = p.ids_out + sbeg;
  const int wbase = (int)lbase + wbeg;  // shard-local index of this warp's first key
  const int32_t* ids = p.ids ? p.ids + sbeg : nullptr;
  const int wvalid = (int)lbase + valid;
  const bool full = wbeg + kWarpKeys <= valid;
  if (full) {
    if (ids) scatter_rounds<NB, true, true>(p, word, next, out, ids, wbase, wvalid, (int)(send - sbeg));
    else scatter_rounds<NB, false, true>(p, word, next, out, ids, wbase, wvalid, (int)(send - sbeg));
  } else {
    if (ids) scatter_rounds<NB, true, false>(p, word, next, out, ids, wbase, wvalid, (int)(send - sbeg));
    else scatter_rounds<NB, false, false>(p, word, next, out, ids, wbase, wvalid, (int)(send - sbeg));
  }
  }
}

}  // namespace
}  // namespace b2

using namespace b2;

static inline int64_t strata_tiles(int64_t n) { return (n + kTile - 1) / kTile; }

template <int NB>
static cudaError_t launch_all(const StrataParams& p, int64_t T, cudaStream_t st) {
  // the scan and the scatter are programmatic dependents: their launch overlaps
  // the previous kernel's tail, and they wait (griddepcontrol.wait) before reading
  if (p.shift >= 0) k_strata_count<NB, true><<<(unsigned)T, kT, 0, st>>>(p);
  else k_strata_count<NB, false><<<(unsigned)T, kT, 0, st>>>(p);
  cudaError_t e = launch_pdl(k_strata_scan<NB>, dim3((unsigned)p.nshard), dim3(kScanT), 0, st, p);
  if (e != cudaSuccess) return e;
  e = launch_pdl(k_strata_scatter<NB>, dim3((unsigned)T), dim3(kT), 0, st, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

static inline size_t strata_ws_bytes(int64_t tiles) {
  // per-tile counts; per-tile codes (4 bits/key: room for 16 strata)
  return (size_t)tiles * kMaxStrata * sizeof(int32_t) + (size_t)tiles * (kTile / 2);
}

extern "C" size_t b2_strata_workspace_bytes(int64_t n) {
  if (n < 1) n = 1;
  return strata_ws_bytes(strata_tiles(n) + kMaxShards);  // + one partial tile per shard boundary
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
  p.shift = -1;  // uniform power-of-two strata (e.g. the default 128/256/384/512)?
  for (int sh = 0; sh < 31 && p.shift < 0; ++sh) {
    bool ok = true;
    for (int k = 0; k < nb && ok; ++k) ok = (int64_t)bounds[k] == ((int64_t)(k + 1) << sh);
    if (ok) p.shift = sh;
  }
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
  const size_t need = strata_ws_bytes(T);
  B2_REQUIRE(workspace && workspace_bytes >= need, B2_ERR_INVALID, "strata workspace needs %zu bytes", need);
  p.tile_counts = static_cast<int32_t*>(workspace);
  p.codes = reinterpret_cast<uint32_t*>(p.tile_counts + T * kMaxStrata);
  p.counts = counts;
  p.bad = bad;
  p.ids_out = ids_out;
  cudaStream_t st = (cudaStream_t)stream;
  B2_CHECK(cudaMemsetAsync(bad, 0xff, sizeof(int64_t) * nshard, st));
  if (nb <= 4) B2_CHECK(launch_all<4>(p, T, st));
  else if (nb <= 8) B2_CHECK(launch_all<8>(p, T, st));
  else B2_CHECK(launch_all<16>(p, T, st));
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
