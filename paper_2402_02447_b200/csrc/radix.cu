// H2 / K5 — device-wide stable LSD radix sort by (-length, id) + raster/snake
// deal, for pools of ANY size (sm_100a).
//
// Reference: _sorted_desc (balance.py:73-75) is Python's stable Timsort with
// key (-length, id); _deal (:59-70) deals rows of `lanes` items (odd rows
// reversed for SNAKE); _from_per_gpu (:54-56) sums lengths per lane.
// assign_global_presort (:83-88) applies them to one pool of b*G samples and
// the per-rank shard sort of the local presort (north_star: "a stable per-rank
// radix sort on length keys") to a whole 1.25M-sample shard.  K3
// (presort.cu) sorts pools of <= 4096 keys inside one CTA; this file is the
// multi-CTA path for larger pools.
//
// Key: ((max_len - len) << id_bits) | id orders exactly like (-len, id); the
// sort is stable LSD, so samples with equal (len, id) keep input order exactly
// like Timsort, and each sample's input slot can ride along (out_pos).
//
// Launches (per call, every segment at once):
//   k_radix_hist<false> (upsweep): one read of (id, len), kept in L2: validates,
//                     counts the length digits' histograms per segment
//                     (shared-memory histograms, flushed once per run of
//                     tiles), detects whether ids are already non-decreasing
//                     inside every segment, zeroes the look-back state and
//                     the token sums.
//   k_radix_hist<true>: the id digits' histograms; returns at once when the
//                     ids are already ordered.
//   k_radix_pass x P: onesweep -- one read + one write per key per pass.  A
//                     persistent grid takes tiles (4096 keys, never
//                     straddling segments) by atomic ticket, round-robin over
//                     the segments.  A tile ranks its keys stably (per-bit
//                     warp ballots give each key's peer group; the group's
//                     leader takes its slots from the warp's digit counter
//                     with one shared atomic), publishes per-digit counts
//                     and resolves its global per-digit offsets by decoupled
//                     look-back over the preceding tiles of its segment
//                     (ticket order, so a predecessor is always running or
//                     done), stages the tile digit-sorted in shared memory
//                     and writes runs with consecutive addresses.  The last
//                     pass writes the deal directly: sorted slot q of a
//                     segment -> row q / lanes, lane (snake-reversed on odd
//                     rows) -> out_ids[seg][lane][row]; token sums per lane.
// If the upsweep finds ids non-decreasing inside every segment (a rank shard
// in id order, the stratified shard of K2, ...) the id-digit passes are
// skipped on the device (no host round trip): a stable sort by length alone
// then IS the (-len, id) order.  Algorithmic bytes: 8 B/key read (id, len) +
// 4 B/key written (dealt id), +4 B with input slots.
#include "common.cuh"

#include <algorithm>

namespace b2 {
namespace {

constexpr int RT = 256;            // threads per tile
constexpr int RI = 16;             // keys per thread
constexpr int TILE = RT * RI;      // 4096 keys per tile
constexpr int RW = RT / 32;        // warps per tile
constexpr int WKEYS = TILE / RW;   // 512 keys per warp
constexpr int RBITS = 9;           // widest digit
constexpr int RBINS = 1 << RBITS;  // 512 bins
constexpr int MAX_PASS = 8;
constexpr int TOK_SMEM = 256;      // lanes whose token sums are staged in shared memory
constexpr int kLookBack = 16;      // predecessor status words per look-back round trip

constexpr uint32_t ST_AGG = 1u << 30, ST_PRE = 2u << 30, ST_VAL = (1u << 30) - 1u;

struct RadixParams {
  const int32_t* ids;
  const int32_t* lens;
  int64_t nseg;
  int seg_len, tps;  // tiles per segment
  int64_t ntiles;
  int32_t max_len, max_id;
  int id_bits;
  int npass, npass_id;  // passes (LSD order); the first npass_id sort id bits
  int shift[MAX_PASS], bits[MAX_PASS];
  uint32_t* hist;       // [npass][nseg][RBINS]
  uint32_t* status[2];  // [ntiles][RBINS] look-back words, alternating by pass
  uint16_t* tcnt;       // [ntiles][RBINS] first length digit per tile, input order (upsweep)
  uint32_t* tbase;      // [ntiles][RBINS] its tile bases in the segment (k_radix_tscan)
  uint32_t* counters;   // [MAX_PASS] tile tickets
  int32_t* flags;       // [0]: 1 if some segment's ids decrease somewhere
  unsigned long long* keys[2];
  int32_t* pos[2];
  int lanes, rows, snake;
  int32_t* out_ids;
  int32_t* out_pos;
  int64_t* tokens;
  int64_t* bad;
};

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// 4 B load that asks L2 to keep the line (evict_last): the upsweep's reads of
// (id, len) stay resident for the first pass, which reads them again
__device__ __forceinline__ int32_t ld_keep(const int32_t* a, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void prefetch_l2(const void* a) { asm volatile("prefetch.global.L2 [%0];" ::"l"(a)); }

__device__ __forceinline__ unsigned long long make_key(const RadixParams& p, int32_t L, int32_t D) {
  L = L < 1 ? 1 : (L > p.max_len ? p.max_len : L);  // out-of-range samples are reported via bad
  D = D < 0 ? 0 : (D > p.max_id ? p.max_id : D);
  return ((unsigned long long)(uint32_t)(p.max_len - L) << p.id_bits) | (unsigned long long)(uint32_t)D;
}

// Block-wide exclusive scan of two values per thread (bins 2t, 2t+1).
// Returns the exclusive prefix of (a) for bin 2t; bin 2t+1's is that + a0.
__device__ __forceinline__ void block_scan2(uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1, uint32_t& ea,
                                            uint32_t& eb, uint32_t* s_warp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t xa = a0 + a1, xb = b0 + b1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t ya = __shfl_up_sync(0xffffffffu, xa, o), yb = __shfl_up_sync(0xffffffffu, xb, o);
    if (lane >= o) {
      xa += ya;
      xb += yb;
    }
  }
  if (lane == 31) {
    s_warp[w] = xa;
    s_warp[RW + w] = xb;
  }
  __syncthreads();
  uint32_t pa = 0, pb = 0;
  for (int i = 0; i < w; ++i) {
    pa += s_warp[i];
    pb += s_warp[RW + i];
  }
  ea = pa + xa - (a0 + a1);
  eb = pb + xb - (b0 + b1);
  __syncthreads();  // s_warp reusable
}

// ---------------------------------------------------------------- upsweep
// Two histogram launches, UKEYS (len, id) loads in flight per thread per tile
// round (no barrier inside a round, so they issue back to back):
//   k_radix_hist<false> (the upsweep proper): validates, detects whether ids
//     are non-decreasing inside every segment, zeroes the look-back state and
//     the token sums, and builds the LENGTH digits' histograms;
//   k_radix_hist<true>: the id digits' histograms -- only needed when some
//     segment's ids decrease, so an ordered shard (the stratified rank shard)
//     returns at once and never pays for them.
constexpr int UKEYS = 16;
static_assert(UKEYS * RT == TILE, "one upsweep round covers a tile");
template <bool IDS>
__global__ void __launch_bounds__(RT, 4) k_radix_hist(const __grid_constant__ RadixParams p, int64_t tiles_per_cta) {
  __shared__ uint32_t s_h[MAX_PASS][RBINS];
  __shared__ uint32_t s_t[RBINS];  // this tile's counts of the first executed digit (-> tcnt)
  __shared__ int s_unsorted;
  const int t = threadIdx.x, lane = t & 31;
  static_assert(UKEYS * 32 == WKEYS, "a warp covers its 512 keys in UKEYS rounds");
  if constexpr (IDS) {
    pdl_wait();  // the upsweep's sortedness flag
    pdl_trigger();
    if (*(volatile const int32_t*)p.flags == 0) return;
  } else {
    pdl_trigger();  // the next launch may start; it waits for this grid before reading
  }
  const int q0 = IDS ? 0 : p.npass_id, q1 = IDS ? p.npass_id : p.npass;  // digits counted here
  const int64_t gt = (int64_t)blockIdx.x * RT + t, gs = (int64_t)gridDim.x * RT;
  if constexpr (!IDS) {
    for (int64_t i = gt; i < p.ntiles * RBINS; i += gs) {
      p.status[0][i] = 0u;
      p.status[1][i] = 0u;
    }
    if (p.tokens)
      for (int64_t i = gt; i < p.nseg * p.lanes; i += gs) p.tokens[i] = 0;
    if (gt < MAX_PASS) p.counters[gt] = 0u;
    if (t == 0) s_unsorted = 0;
  }
  for (int i = t; i < MAX_PASS * RBINS; i += RT) (&s_h[0][0])[i] = 0u;
  for (int i = t; i < RBINS; i += RT) s_t[i] = 0u;
  __syncthreads();
  auto flush = [&](int64_t seg) {
    for (int i = q0 * RBINS + t; i < q1 * RBINS; i += RT) {
      const uint32_t c = (&s_h[0][0])[i];
      if (c) {
        atomicAdd(&p.hist[((size_t)(i / RBINS) * p.nseg + seg) * RBINS + (i % RBINS)], c);
        (&s_h[0][0])[i] = 0u;
      }
    }
  };
  const int64_t tile0 = (int64_t)blockIdx.x * tiles_per_cta;
  const int64_t tile1 = min64(tile0 + tiles_per_cta, p.ntiles);
  int64_t cur_seg = tile0 < tile1 ? tile0 / p.tps : -1;
  long long first_bad = -1;
  int unsorted = 0;
  for (int64_t tile = tile0; tile < tile1; ++tile) {
    const int64_t seg = tile / p.tps;
    if (seg != cur_seg) {  // flush the finished segment's histograms
      __syncthreads();
      flush(cur_seg);
      __syncthreads();
      cur_seg = seg;
    }
    const int64_t sbase = seg * (int64_t)p.seg_len;
    const int in0 = (int)(tile - seg * p.tps) * TILE;
    const int n = min(TILE, p.seg_len - in0);
    // warp w owns keys [w*512, w*512+512) of the tile, lane-striped rounds:
    // the key after lane 31's is lane 0's of the next round (a shuffle)
    const int w = t >> 5;
    int32_t L[UKEYS], D[UKEYS];
    const uint64_t pol = policy_evict_last();
    const int32_t* idp = p.ids + sbase + in0 + w * WKEYS + lane;
    const int32_t* lnp = p.lens + sbase + in0 + w * WKEYS + lane;
    const int nw = n - w * WKEYS;  // keys of this warp (may be <= 0)
#pragma unroll
    for (int j = 0; j < UKEYS; ++j) {  // coalesced, all loads in flight
      L[j] = 1;
      D[j] = 0;
      if (j * 32 + lane < nw) {
        if constexpr (IDS) {
          D[j] = __ldg(idp + j * 32);
        } else {
          D[j] = ld_keep(idp + j * 32, pol);
          L[j] = ld_keep(lnp + j * 32, pol);
        }
      }
    }
    if constexpr (!IDS) {
      // the key after the warp's last: the next warp's / tile's first (an L1/L2 hit)
      const int last_i = in0 + w * WKEYS + min(nw, WKEYS);  // in-segment index after the warp's keys
      const int32_t after = (nw > 0 && last_i < p.seg_len) ? __ldg(p.ids + sbase + last_i) : 0x7fffffff;
#pragma unroll
      for (int j = 0; j < UKEYS; ++j) {
        const int iw = j * 32 + lane;
        const bool valid = iw < nw;
        const int32_t nx0 = __shfl_down_sync(0xffffffffu, D[j], 1);
        const int32_t nx1 = __shfl_sync(0xffffffffu, j + 1 < UKEYS ? D[j + 1 < UKEYS ? j + 1 : j] : 0, 0);
        int32_t nxt = lane < 31 ? nx0 : (j + 1 < UKEYS ? nx1 : after);
        if (iw + 1 == nw) nxt = after;  // the warp's last key
        if (valid) {
          if (!(L[j] >= 1 && L[j] <= p.max_len && D[j] >= 0 && D[j] <= p.max_id) && first_bad < 0)
            first_bad = sbase + in0 + w * WKEYS + iw;
          if (nxt < D[j]) unsorted = 1;
          // length digits from 32-bit arithmetic: shift >= id_bits for every length pass
          const uint32_t lk = (uint32_t)(p.max_len - (L[j] < 1 ? 1 : (L[j] > p.max_len ? p.max_len : L[j])));
          atomicAdd(&s_t[(lk >> (p.shift[q0] - p.id_bits)) & ((1u << p.bits[q0]) - 1u)], 1u);
          for (int q = q0 + 1; q < q1; ++q) atomicAdd(&s_h[q][(lk >> (p.shift[q] - p.id_bits)) & ((1u << p.bits[q]) - 1u)], 1u);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < UKEYS; ++j)
        if (j * 32 + lane < nw) {
          const uint32_t dk = (uint32_t)(D[j] < 0 ? 0 : (D[j] > p.max_id ? p.max_id : D[j]));
          atomicAdd(&s_t[(dk >> p.shift[0]) & ((1u << p.bits[0]) - 1u)], 1u);
          for (int q = 1; q < q1; ++q) atomicAdd(&s_h[q][(dk >> p.shift[q]) & ((1u << p.bits[q]) - 1u)], 1u);
        }
    }
    // the tile's counts of the first executed digit (ids unordered: the first
    // id digit, overwriting the upsweep's length counts): to tcnt for
    // k_radix_tscan, and into the segment histogram
    __syncthreads();
    for (int b = t; b < RBINS; b += RT) {
      const uint32_t c = s_t[b];
      p.tcnt[(size_t)tile * RBINS + b] = (uint16_t)c;
      s_h[q0][b] += c;
      s_t[b] = 0u;
    }
    __syncthreads();
  }
  if constexpr (!IDS) {
    if (unsorted) s_unsorted = 1;
    if (first_bad >= 0 && p.bad) atomicMin(reinterpret_cast<unsigned long long*>(p.bad), (unsigned long long)first_bad);
  }
  __syncthreads();
  if (cur_seg >= 0) flush(cur_seg);
  if constexpr (!IDS)
    if (t == 0 && s_unsorted) atomicOr(p.flags, 1);
}

// ---------------------------------------------------------------- tile bases
// The first executed pass (the first length pass when ids are ordered, else
// the first id pass) reads the input order, whose per-tile digit counts the
// histogram launches wrote to tcnt: every tile's per-digit base in its
// segment is known before that pass, so it needs no look-back.  CTA (segment, 32 digits), 1024
// threads: warp w sums its run of tiles per digit (lane), the runs are
// scanned in shared memory, then each run is walked again writing bases.
constexpr int TS_T = 1024, TS_W = TS_T / 32;
__global__ void __launch_bounds__(TS_T) k_radix_tscan(const __grid_constant__ RadixParams p) {
  pdl_wait();
  pdl_trigger();
  const bool unsorted = *(volatile const int32_t*)p.flags != 0;
  __shared__ uint32_t s_run[TS_W][32];
  __shared__ uint32_t s_tot[RBINS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t seg = blockIdx.x / (RBINS / 32);
  const int d = (int)(blockIdx.x % (RBINS / 32)) * 32 + lane;
  const int q = unsorted ? 0 : p.npass_id;  // the first executed pass
  const uint32_t* hseg = p.hist + ((size_t)q * p.nseg + seg) * RBINS;
  const int per = (p.tps + TS_W - 1) / TS_W;
  const int k0 = min(w * per, p.tps), k1 = min(k0 + per, p.tps);
  const uint16_t* tc = p.tcnt + (size_t)seg * p.tps * RBINS + d;
  uint32_t sum = 0;
#pragma unroll 8
  for (int k = k0; k < k1; ++k) sum += tc[(size_t)k * RBINS];
  s_run[w][lane] = sum;
  if (w == 0) {  // exclusive prefix of the segment's digit totals: 16 per lane + a warp scan
    uint32_t v[RBINS / 32], run = 0;
#pragma unroll
    for (int i = 0; i < RBINS / 32; ++i) {
      v[i] = hseg[lane * (RBINS / 32) + i];
      run += v[i];
    }
    uint32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    x -= run;
#pragma unroll
    for (int i = 0; i < RBINS / 32; ++i) {
      s_tot[lane * (RBINS / 32) + i] = x;
      x += v[i];
    }
  }
  __syncthreads();
  uint32_t base = s_tot[d];  // digits before d in the segment (the sort is by digit first)
  for (int i = 0; i < w; ++i) base += s_run[i][lane];
  uint32_t* tb = p.tbase + (size_t)seg * p.tps * RBINS + d;
  for (int k = k0; k < k1; ++k) {
    B2_DASSERT(base <= (uint32_t)p.seg_len);
    tb[(size_t)k * RBINS] = base;
    base += tc[(size_t)k * RBINS];
  }
}

// ---------------------------------------------------------------- onesweep pass
template <bool POS>
struct PassSmem {
  unsigned long long key[TILE];  // tile, digit-sorted
  int32_t pos[POS ? TILE : 1];
  // per-warp digit counts, then per-warp exclusive prefixes: 16-bit fields
  // (<= 4096 per tile), two per 32-bit word for the ranking atomics
  union {
    uint16_t whist[RW][RBINS];
    uint32_t whist2[RW][RBINS / 2];
  };
  uint32_t off[RBINS];           // tile-local digit starts
  uint32_t gbase[RBINS];         // global (segment) offset of this tile's first key of each digit
  long long tok[TOK_SMEM];       // per-lane token sums of this tile (last pass)
  uint32_t warp_tot[2 * RW];
  int tile;
};

template <bool POS>
__device__ __forceinline__ void radix_tile(const RadixParams& p, int pass, bool unsorted, int64_t ticket,
                                           PassSmem<POS>& sm) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int exec = unsorted ? pass : pass - p.npass_id;  // index among the executed passes
  const bool from_input = exec == 0, last = pass == p.npass - 1;
  const int shift = p.shift[pass];
  const int nbits = p.bits[pass];
  const uint32_t mask = (1u << nbits) - 1u;
  // tickets go round-robin over the segments (ticket = tin * nseg + seg): a
  // tile's predecessor in its segment holds an earlier ticket, and the tiles in
  // flight per segment -- the depth of a look-back walk -- are ~grid / nseg
  const int64_t tin64 = ticket / p.nseg;
  const int64_t seg = ticket - tin64 * p.nseg;
  const int tin = (int)tin64;
  const int64_t tile = seg * p.tps + tin;  // status row
  if (pass + 1 < p.npass)
    for (int d = t; d < RBINS; d += RT) p.status[(pass + 1) & 1][(size_t)tile * RBINS + d] = 0u;
  const int64_t sbase = seg * (int64_t)p.seg_len;
  const int in0 = tin * TILE;
  const int n = min(TILE, p.seg_len - in0);
  const unsigned long long* kin = p.keys[(exec - 1) & 1];
  const int32_t* pin = p.pos[(exec - 1) & 1];

  for (int i = t; i < RW * RBINS / 2; i += RT) (&sm.whist2[0][0])[i] = 0u;
  if (last && p.tokens && p.lanes <= TOK_SMEM)
    for (int i = t; i < p.lanes; i += RT) sm.tok[i] = 0;

  // load (warp w owns keys [w*512, w*512+512) of the tile, lane-striped): every
  // load of the tile is issued before the first use
  unsigned long long key[RI];
  int32_t pos[RI];
  uint32_t rank[RI];
#pragma unroll
  for (int j = 0; j < RI; ++j) {
    const int i = w * WKEYS + j * 32 + lane;
    const int64_t g = sbase + in0 + i;
    key[j] = 0ull;
    pos[j] = 0;
    if (i < n) {
      if (from_input) {
        key[j] = make_key(p, __ldg(p.lens + g), __ldg(p.ids + g));
        pos[j] = (int32_t)g;
      } else {
        key[j] = __ldcs(kin + g);
        if constexpr (POS) pos[j] = __ldcs(pin + g);
      }
    }
  }
  // warm L2 with the tile a CTA of the next round will take (ticket + grid):
  // one 128 B line per thread of the pass's input; the tile's own loads above
  // are already in flight
  {
    const int64_t nt = ticket + gridDim.x;
    if (nt < p.ntiles) {
      const int64_t ntin = nt / p.nseg, nseg_ = nt - ntin * p.nseg;
      const int nin0 = (int)ntin * TILE;
      const int nn = min(TILE, p.seg_len - nin0);
      const int64_t g0 = nseg_ * (int64_t)p.seg_len + nin0;
      if (from_input) {  // 2 x 4 B per key: lens lines, then ids lines
        const int per = 32;  // keys per 128 B line
        const int lines = (nn + per - 1) / per;
        if (t < lines) prefetch_l2(p.lens + g0 + t * per);
        else if (t - lines < lines) prefetch_l2(p.ids + g0 + (t - lines) * per);
      } else {  // 8 B keys
        const int lines = (nn + 15) / 16;
        for (int l = t; l < lines; l += RT) prefetch_l2(kin + g0 + l * 16);
      }
    }
  }
  __syncthreads();  // whist cleared
  // rank stably: inside a warp by (iteration, lane) = input order.  The peer
  // group's leader takes the group's slots with one shared atomic; a warp's
  // atomics are performed in issue order, so the rounds need no barrier
  // between them and their atomics pipeline.
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < RI; ++j) {
    const int i = w * WKEYS + j * 32 + lane;
    const bool valid = i < n;
    const uint32_t d = valid ? (uint32_t)(key[j] >> shift) & mask : 0u;
    // lanes with this lane's digit: one ballot per digit bit (MATCH.ANY costs a
    // pass per distinct value, ~30 for a random 9-bit digit)
    uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < RBITS; ++b) {
      if (b < nbits) {
        const bool bit = (d >> b) & 1u;
        const uint32_t m = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? m : ~m;
      }
    }
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (valid && lane == leader)
      base = (atomicAdd(&sm.whist2[w][d >> 1], (uint32_t)__popc(peers) << (16 * (d & 1))) >> (16 * (d & 1))) & 0xffffu;
    rank[j] = __shfl_sync(0xffffffffu, base, leader) + __popc(peers & lt);
  }
  __syncthreads();

  // per digit (thread t owns bins 2t, 2t+1): exclusive prefix over warps and
  // the tile total; then the tile-local digit starts and the segment's global
  // digit starts (one block scan of both)
  uint32_t tot[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int d = 2 * t + h;
    uint32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < RW; ++ww) {
      const uint32_t c = sm.whist[ww][d];
      sm.whist[ww][d] = (uint16_t)run;
      run += c;
    }
    tot[h] = run;
  }
  // publish this tile's per-digit counts (the first tile of a segment has its
  // inclusive prefix at once)
  // ids ordered and this is the first length pass: the tile bases are tabled
  // (k_radix_tscan), no publish and no look-back
  const bool tabled = pass == (unsorted ? 0 : p.npass_id);
  uint32_t* st = p.status[pass & 1] + (size_t)tile * RBINS;
  uint32_t h0 = 0, h1 = 0, tb0 = 0, tb1 = 0;
  if (tabled) {
    tb0 = p.tbase[(size_t)tile * RBINS + 2 * t];
    tb1 = p.tbase[(size_t)tile * RBINS + 2 * t + 1];
    B2_DASSERT(tile < p.ntiles && tb0 + tot[0] <= (uint32_t)p.seg_len && tb1 + tot[1] <= (uint32_t)p.seg_len);
  } else {
#pragma unroll
    for (int h = 0; h < 2; ++h) st_relaxed_u32(&st[2 * t + h], (tin == 0 ? ST_PRE : ST_AGG) | tot[h]);
    const uint32_t* hseg = p.hist + ((size_t)pass * p.nseg + seg) * RBINS;
    h0 = hseg[2 * t];
    h1 = hseg[2 * t + 1];
  }
  uint32_t eloc, eglob;
  block_scan2(tot[0], tot[1], h0, h1, eloc, eglob, sm.warp_tot);
  sm.off[2 * t] = eloc;
  sm.off[2 * t + 1] = eloc + tot[0];
  if (tabled) {
    sm.gbase[2 * t] = tb0;
    sm.gbase[2 * t + 1] = tb1;
  } else {
  // decoupled look-back over the preceding tiles of this segment, kLookBack
  // predecessors per round trip (their status words are loaded together, then
  // folded newest-first until an inclusive prefix is met; an unpublished
  // word is re-polled on its own)
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int d = 2 * t + h;
    uint32_t excl = 0;
    if (tin > 0) {
      const uint32_t* sp = p.status[pass & 1] + d;
      int64_t k = tile - 1;
      const int64_t kmin = tile - tin;  // first tile of the segment (always publishes ST_PRE)
      bool done = false;
      while (!done) {
        uint32_t v[kLookBack];
#pragma unroll
        for (int u = 0; u < kLookBack; ++u) v[u] = k - u >= kmin ? ld_relaxed_u32(sp + (size_t)(k - u) * RBINS) : ST_PRE;
#pragma unroll
        for (int u = 0; u < kLookBack; ++u) {
          if (done) break;
          uint32_t x = v[u];
          while ((x & ~ST_VAL) == 0u) x = ld_relaxed_u32(sp + (size_t)(k - u) * RBINS);  // not published yet
          excl += x & ST_VAL;
          if (x & ST_PRE) done = true;
        }
        k -= kLookBack;
      }
      st_relaxed_u32(&st[d], ST_PRE | (excl + tot[h]));
    }
    sm.gbase[d] = (eglob + (h ? h0 : 0u)) + excl;
  }
  }
  __syncthreads();

  // last pass: deal each key straight to its output slot (balance.py:59-70)
  const unsigned long long idmask = (1ull << p.id_bits) - 1ull;
  const bool tok_smem = p.tokens && p.lanes <= TOK_SMEM;
  // q / lanes = umul64hi(q, floor(2^64 / lanes) + 1), exact for q * lanes < 2^64
  const unsigned long long lanes_magic = ~0ull / (unsigned long long)p.lanes + 1ull;
  // lanes of a warp that deal to the same GPU lane add their lengths first (one atomic per
  // group); with lanes = 1 every key lands on one counter: a register sum
  const bool tok_redux = p.max_len < (1 << 26);
  unsigned long long tsum = 0;
  auto deal = [&](bool v, unsigned long long k, int32_t pv, uint32_t q) {  // q: sorted slot in the segment
    int ln = -1;
    int32_t len = 0;
    if (v) {
      const uint32_t r = p.lanes == 1 ? q : (uint32_t)__umul64hi((unsigned long long)q, lanes_magic);
      const int c = (int)(q - r * (uint32_t)p.lanes);
      ln = (p.snake && (r & 1u)) ? p.lanes - 1 - c : c;  // balance.py:66-67
      const int64_t o = sbase + (int64_t)ln * p.rows + r;
      B2_DASSERT(ln >= 0 && ln < p.lanes && (int)r < p.rows);
      p.out_ids[o] = (int32_t)(k & idmask);
      if constexpr (POS) p.out_pos[o] = pv;
      len = p.max_len - (int32_t)(k >> p.id_bits);
    }
    if (!p.tokens) return;
    if (p.lanes == 1) {
      tsum += (unsigned long long)len;
    } else if (tok_redux) {
      const unsigned grp = __match_any_sync(0xffffffffu, ln);
      const unsigned sum = __reduce_add_sync(grp, (unsigned)len);
      if (v && lane == __ffs(grp) - 1) {
        if (tok_smem) atomicAdd(reinterpret_cast<unsigned long long*>(&sm.tok[ln]), (unsigned long long)sum);
        else atomicAdd(reinterpret_cast<unsigned long long*>(&p.tokens[seg * p.lanes + ln]), (unsigned long long)sum);
      }
    } else if (v) {
      if (tok_smem) atomicAdd(reinterpret_cast<unsigned long long*>(&sm.tok[ln]), (unsigned long long)len);
      else atomicAdd(reinterpret_cast<unsigned long long*>(&p.tokens[seg * p.lanes + ln]), (unsigned long long)len);
    }
  };
  auto flush_tokens = [&]() {
    if (p.tokens && p.lanes == 1) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, o);
      if (lane == 0 && tsum) atomicAdd(reinterpret_cast<unsigned long long*>(&p.tokens[seg]), tsum);
    } else if (tok_smem) {
      __syncthreads();
      for (int l = t; l < p.lanes; l += RT)  // per-lane token sums (_from_per_gpu, balance.py:54-56)
        if (sm.tok[l]) atomicAdd(reinterpret_cast<unsigned long long*>(&p.tokens[seg * p.lanes + l]), (unsigned long long)sm.tok[l]);
    }
  };
#ifdef B2_K5_DIRECT
  if (last) {  // each key knows its slot: gbase + the warp's prefix + its rank; no staging
#pragma unroll
    for (int j = 0; j < RI; ++j) {
      const int i = w * WKEYS + j * 32 + lane;
      const bool v = i < n;
      const uint32_t d = (uint32_t)(key[j] >> shift) & mask;
      deal(v, key[j], pos[j], v ? sm.gbase[d] + sm.whist[w][d] + rank[j] : 0u);
    }
    flush_tokens();
    return;
  }
#endif

  // stage the tile digit-sorted
#pragma unroll
  for (int j = 0; j < RI; ++j) {
    const int i = w * WKEYS + j * 32 + lane;
    if (i < n) {
      const uint32_t d = (uint32_t)(key[j] >> shift) & mask;
      const uint32_t lp = sm.off[d] + sm.whist[w][d] + rank[j];
      B2_DASSERT(d < RBINS && lp < (uint32_t)n);
      sm.key[lp] = key[j];
      if constexpr (POS) sm.pos[lp] = pos[j];
    }
  }
  __syncthreads();

  if (!last) {
    unsigned long long* kout = p.keys[exec & 1];
    int32_t* pout = p.pos[exec & 1];
    for (int i = t; i < n; i += RT) {
      const unsigned long long k = sm.key[i];
      const uint32_t d = (uint32_t)(k >> shift) & mask;
      const int64_t o = sbase + sm.gbase[d] + (i - sm.off[d]);
      B2_DASSERT(o >= sbase && o < sbase + p.seg_len);
      kout[o] = k;
      if constexpr (POS) pout[o] = sm.pos[i];
    }
    return;
  }
  for (int i0 = 0; i0 < n; i0 += RT) {
    const int i = i0 + t;
    const bool v = i < n;
    unsigned long long k = 0ull;
    uint32_t q = 0u;
    int32_t pv = 0;
    if (v) {
      k = sm.key[i];
      const uint32_t d = (uint32_t)(k >> shift) & mask;
      q = sm.gbase[d] + (uint32_t)(i - sm.off[d]);
      if constexpr (POS) pv = sm.pos[i];
    }
    deal(v, k, pv, q);
  }
  flush_tokens();
}

// Persistent: grid = resident CTAs; each CTA takes tiles by atomic ticket
// until none are left (ticket order = look-back order, so a predecessor tile
// is always held by a running CTA).  A skipped pass costs one flag read per CTA.
template <bool POS>
__global__ void __launch_bounds__(RT, 4) k_radix_pass(const __grid_constant__ RadixParams p, int pass) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PassSmem<POS>& sm = *reinterpret_cast<PassSmem<POS>*>(smem_raw);
  pdl_wait();     // the previous pass (or the upsweep) has completed and its writes are visible
  pdl_trigger();  // the next pass may launch; it waits for this grid in turn
  const bool unsorted = *(volatile const int32_t*)p.flags != 0;
  if (!unsorted && pass < p.npass_id) return;  // ids already ordered: length passes only
  for (;;) {
    __syncthreads();  // the previous tile's shared-memory reads are done
    if (threadIdx.x == 0) sm.tile = (int)atomicAdd(&p.counters[pass], 1u);
    __syncthreads();
    const int64_t ticket = sm.tile;
    if (ticket >= p.ntiles) return;
    radix_tile<POS>(p, pass, unsorted, ticket, sm);
  }
}

int bits_for(int64_t v) {  // bits needed to represent 0..v
  int b = 0;
  while (b < 63 && (1ll << b) <= v) ++b;
  return b;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct Plan {
  int id_bits, len_bits, npass, npass_id;
  int shift[MAX_PASS], bits[MAX_PASS];
  int tps;
  int64_t ntiles, n;
  size_t off_keys[2], off_pos[2], off_hist, off_status[2], off_tcnt, off_tbase, off_counters, off_flags, total;
};

// digits of <= 9 bits: the id bits first (LSD), then the length bits
bool make_plan(Plan& pl, int64_t nseg, int seg_len, int32_t max_len, int32_t max_id, bool with_pos) {
  pl.id_bits = std::max(1, bits_for(max_id));
  pl.len_bits = std::max(1, bits_for((int64_t)max_len - 1));
  if (pl.id_bits + pl.len_bits > 62) return false;
  int np = 0;
  auto split = [&](int lo, int nbits) {
    const int k = (nbits + RBITS - 1) / RBITS;
    int at = lo;
    for (int i = 0; i < k; ++i) {
      const int w = (nbits - (at - lo) + (k - i) - 1) / (k - i);  // even split
      pl.shift[np] = at;
      pl.bits[np] = w;
      at += w;
      ++np;
    }
  };
  split(0, pl.id_bits);
  pl.npass_id = np;
  split(pl.id_bits, pl.len_bits);
  pl.npass = np;
  if (np > MAX_PASS) return false;
  pl.tps = (seg_len + TILE - 1) / TILE;
  pl.ntiles = nseg * pl.tps;
  pl.n = nseg * (int64_t)seg_len;
  size_t o = 0;
  for (int b = 0; b < 2; ++b) {
    pl.off_keys[b] = o;
    o = align256(o + (size_t)pl.n * 8);
  }
  for (int b = 0; b < 2; ++b) {
    pl.off_pos[b] = o;
    if (with_pos) o = align256(o + (size_t)pl.n * 4);
  }
  pl.off_hist = o;
  o = align256(o + (size_t)pl.npass * nseg * RBINS * 4);
  for (int b = 0; b < 2; ++b) {
    pl.off_status[b] = o;
    o = align256(o + (size_t)pl.ntiles * RBINS * 4);
  }
  pl.off_tcnt = o;
  o = align256(o + (size_t)pl.ntiles * RBINS * 2);
  pl.off_tbase = o;
  o = align256(o + (size_t)pl.ntiles * RBINS * 4);
  pl.off_counters = o;
  o = align256(o + MAX_PASS * 4);
  pl.off_flags = o;
  o = align256(o + 16);
  pl.total = o;
  return true;
}

}  // namespace
}  // namespace b2

using namespace b2;

extern "C" size_t b2_presort_workspace_bytes(int64_t nseg, int seg_len, int32_t max_len, int32_t max_id,
                                             int with_pos) {
  if (nseg <= 0 || seg_len <= 4096 || max_len < 1 || max_id < 0) return 0;
  Plan pl;
  if (!make_plan(pl, nseg, seg_len, max_len, max_id, with_pos != 0)) return 0;
  return pl.total;
}

extern "C" int b2_presort_sort_deal(const int32_t* ids, const int32_t* lens, int64_t nseg, int seg_len, int lanes,
                                    int scan, int32_t max_len, int32_t max_id, int32_t* out_ids, int32_t* out_pos,
                                    int64_t* tokens, int64_t* bad, void* workspace, size_t workspace_bytes,
                                    void* stream) {
  if (seg_len <= 4096)  // one pool per CTA (K3)
    return b2_presort_deal(ids, lens, nseg, seg_len, lanes, scan, max_len, max_id, out_ids, out_pos, tokens, bad,
                           stream);
  B2_REQUIRE(lanes >= 1, B2_ERR_INVALID, "lanes must be >= 1, got %d", lanes);
  B2_REQUIRE(seg_len % lanes == 0, B2_ERR_INDIVISIBLE, "%d items do not divide over %d GPUs", seg_len, lanes);
  B2_REQUIRE(seg_len < (1 << 30), B2_ERR_UNSUPPORTED, "pool of %d samples exceeds 2^30", seg_len);
  B2_REQUIRE(max_len >= 1 && max_id >= 0, B2_ERR_INVALID, "max_len must be >= 1 and max_id >= 0");
  B2_REQUIRE(scan == B2_SCAN_RASTER || scan == B2_SCAN_SNAKE, B2_ERR_INVALID, "bad scan %d", scan);
  cudaStream_t st = (cudaStream_t)stream;
  if (bad) B2_CHECK(cudaMemsetAsync(bad, 0xff, sizeof(int64_t), st));
  if (nseg <= 0) return B2_OK;
  B2_REQUIRE(ids && lens && out_ids, B2_ERR_INVALID, "NULL pointer argument");
  Plan pl;
  B2_REQUIRE(make_plan(pl, nseg, seg_len, max_len, max_id, out_pos != nullptr), B2_ERR_UNSUPPORTED,
             "key (%d id bits + length bits) does not fit the radix plan", bits_for(max_id));
  B2_REQUIRE(workspace && workspace_bytes >= pl.total, B2_ERR_INVALID, "presort workspace needs %zu bytes",
             pl.total);
  char* ws = static_cast<char*>(workspace);
  RadixParams p{};
  p.ids = ids;
  p.lens = lens;
  p.nseg = nseg;
  p.seg_len = seg_len;
  p.tps = pl.tps;
  p.ntiles = pl.ntiles;
  p.max_len = max_len;
  p.max_id = max_id;
  p.id_bits = pl.id_bits;
  p.npass = pl.npass;
  p.npass_id = pl.npass_id;
  for (int i = 0; i < pl.npass; ++i) {
    p.shift[i] = pl.shift[i];
    p.bits[i] = pl.bits[i];
  }
  p.hist = reinterpret_cast<uint32_t*>(ws + pl.off_hist);
  for (int b = 0; b < 2; ++b) {
    p.status[b] = reinterpret_cast<uint32_t*>(ws + pl.off_status[b]);
    p.keys[b] = reinterpret_cast<unsigned long long*>(ws + pl.off_keys[b]);
    p.pos[b] = out_pos ? reinterpret_cast<int32_t*>(ws + pl.off_pos[b]) : nullptr;
  }
  p.tcnt = reinterpret_cast<uint16_t*>(ws + pl.off_tcnt);
  p.tbase = reinterpret_cast<uint32_t*>(ws + pl.off_tbase);
  p.counters = reinterpret_cast<uint32_t*>(ws + pl.off_counters);
  p.flags = reinterpret_cast<int32_t*>(ws + pl.off_flags);
  p.lanes = lanes;
  p.rows = seg_len / lanes;
  p.snake = scan == B2_SCAN_SNAKE;
  p.out_ids = out_ids;
  p.out_pos = out_pos;
  p.tokens = tokens;
  p.bad = bad;
  // histograms and the sortedness flag start at zero (one small memset)
  B2_CHECK(cudaMemsetAsync(ws + pl.off_hist, 0, (size_t)pl.npass * nseg * RBINS * 4, st));
  B2_CHECK(cudaMemsetAsync(ws + pl.off_flags, 0, 16, st));
  const DeviceInfo& di = device_info();
  const int64_t ctas = std::min<int64_t>(pl.ntiles, (int64_t)di.sm_count * 8);
  const int64_t per = (pl.ntiles + ctas - 1) / ctas;
  const int64_t grid_up = (pl.ntiles + per - 1) / per;
  k_radix_hist<false><<<(unsigned)grid_up, RT, 0, st>>>(p, per);
  B2_CHECK(cudaGetLastError());
  if (pl.npass_id > 0) B2_CHECK(launch_pdl(k_radix_hist<true>, dim3((unsigned)grid_up), dim3(RT), 0, st, p, per));
  B2_CHECK(launch_pdl(k_radix_tscan, dim3((unsigned)(nseg * (RBINS / 32))), dim3(TS_T), 0, st, p));
  const size_t smem = out_pos ? sizeof(PassSmem<true>) : sizeof(PassSmem<false>);
  static int occ_cached[64][2] = {};
  const bool pos = out_pos != nullptr;
  int& occ = occ_cached[di.device & 63][pos];
  if (occ == 0) {
    if (pos) {
      B2_CHECK(cudaFuncSetAttribute((const void*)k_radix_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      B2_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_radix_pass<true>, RT, smem));
    } else {
      B2_CHECK(cudaFuncSetAttribute((const void*)k_radix_pass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      B2_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_radix_pass<false>, RT, smem));
    }
    B2_REQUIRE(occ >= 1, B2_ERR_CUDA, "radix pass cannot be resident");
  }
  // persistent: one wave of resident CTAs takes the tiles by ticket
  const unsigned grid = (unsigned)std::min<int64_t>(pl.ntiles, (int64_t)di.sm_count * occ);
  for (int q = 0; q < pl.npass; ++q) {
    // programmatic dependents: each pass launches under the previous kernel's tail
    if (pos) B2_CHECK(launch_pdl(k_radix_pass<true>, dim3(grid), dim3(RT), smem, st, p, q));
    else B2_CHECK(launch_pdl(k_radix_pass<false>, dim3(grid), dim3(RT), smem, st, p, q));
    B2_CHECK(cudaGetLastError());
  }
  return B2_OK;
}
