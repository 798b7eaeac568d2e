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
//   k_radix_upsweep : one read of (id, len): validates, counts every pass's
//                     digit histogram per segment (shared-memory histograms,
//                     flushed once per run of tiles), detects whether ids are
//                     already non-decreasing inside every segment, and zeroes
//                     the first pass's look-back state and the token sums.
//   k_radix_pass x P: onesweep — one read + one write per key per pass.  A
//                     tile (4096 keys, never straddling segments) ranks its
//                     keys stably (warp match_any + per-warp digit counters),
//                     publishes per-digit counts and resolves its global
//                     per-digit offsets by decoupled look-back over the
//                     preceding tiles of its segment (tile order = atomic
//                     ticket order, so a predecessor is always running or
//                     done), stages the tile digit-sorted in shared memory
//                     and writes runs with consecutive addresses.  The last
//                     pass writes the deal directly: sorted slot q of a
//                     segment -> row q / lanes, lane (snake-reversed on odd
//                     rows) -> out_ids[seg][lane][row]; token sums are
//                     accumulated per tile in shared memory.
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
constexpr int TOK_SMEM = 1024;     // lanes whose token sums are staged in shared memory
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
__global__ void __launch_bounds__(RT) k_radix_upsweep(const __grid_constant__ RadixParams p, int64_t tiles_per_cta) {
  pdl_trigger();  // the first pass may launch now (it waits for this grid before reading)
  __shared__ uint32_t s_h[MAX_PASS][RBINS];
  __shared__ int s_unsorted;
  const int t = threadIdx.x;
  const int64_t gt = (int64_t)blockIdx.x * RT + t, gs = (int64_t)gridDim.x * RT;
  for (int64_t i = gt; i < p.ntiles * RBINS; i += gs) {
    p.status[0][i] = 0u;
    p.status[1][i] = 0u;
  }
  if (p.tokens)
    for (int64_t i = gt; i < p.nseg * p.lanes; i += gs) p.tokens[i] = 0;
  if (gt < MAX_PASS) p.counters[gt] = 0u;
  if (t == 0) s_unsorted = 0;
  for (int i = t; i < p.npass * RBINS; i += RT) (&s_h[0][0])[i] = 0u;
  __syncthreads();
  const int64_t tile0 = (int64_t)blockIdx.x * tiles_per_cta;
  const int64_t tile1 = min64(tile0 + tiles_per_cta, p.ntiles);
  int64_t cur_seg = tile0 < tile1 ? tile0 / p.tps : -1;
  long long first_bad = -1;
  int unsorted = 0;
  for (int64_t tile = tile0; tile < tile1; ++tile) {
    const int64_t seg = tile / p.tps;
    if (seg != cur_seg) {  // flush the finished segment's histograms
      __syncthreads();
      for (int i = t; i < p.npass * RBINS; i += RT) {
        const uint32_t c = (&s_h[0][0])[i];
        if (c) {
          atomicAdd(&p.hist[((size_t)(i / RBINS) * p.nseg + cur_seg) * RBINS + (i % RBINS)], c);
          (&s_h[0][0])[i] = 0u;
        }
      }
      __syncthreads();
      cur_seg = seg;
    }
    const int64_t sbase = seg * (int64_t)p.seg_len;
    const int in0 = (int)(tile - seg * p.tps) * TILE;
    const int n = min(TILE, p.seg_len - in0);
    for (int i = t; i < n; i += RT) {  // striped: coalesced
      const int64_t g = sbase + in0 + i;
      const int32_t L = p.lens[g], D = p.ids[g];
      if (!(L >= 1 && L <= p.max_len && D >= 0 && D <= p.max_id) && first_bad < 0) first_bad = g;
      if (in0 + i + 1 < p.seg_len && p.ids[g + 1] < D) unsorted = 1;  // neighbour: an L1/L2 hit
      const unsigned long long k = make_key(p, L, D);
      for (int q = 0; q < p.npass; ++q)
        atomicAdd(&s_h[q][(uint32_t)(k >> p.shift[q]) & ((1u << p.bits[q]) - 1u)], 1u);
    }
  }
  if (unsorted) s_unsorted = 1;
  if (first_bad >= 0 && p.bad) atomicMin(reinterpret_cast<unsigned long long*>(p.bad), (unsigned long long)first_bad);
  __syncthreads();
  if (cur_seg >= 0)
    for (int i = t; i < p.npass * RBINS; i += RT) {
      const uint32_t c = (&s_h[0][0])[i];
      if (c) atomicAdd(&p.hist[((size_t)(i / RBINS) * p.nseg + cur_seg) * RBINS + (i % RBINS)], c);
    }
  if (t == 0 && s_unsorted) atomicOr(p.flags, 1);
}

// ---------------------------------------------------------------- onesweep pass
template <bool POS>
struct PassSmem {
  unsigned long long key[TILE];  // tile, digit-sorted
  int32_t pos[POS ? TILE : 1];
  uint32_t whist[RW][RBINS];     // per-warp digit counts, then per-warp exclusive prefixes
  uint32_t off[RBINS];           // tile-local digit starts
  uint32_t gbase[RBINS];         // global (segment) offset of this tile's first key of each digit
  long long tok[TOK_SMEM];       // per-lane token sums of this tile (last pass)
  uint32_t warp_tot[2 * RW];
  int tile;
};

template <bool POS>
__global__ void __launch_bounds__(RT) k_radix_pass(const __grid_constant__ RadixParams p, int pass) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PassSmem<POS>& sm = *reinterpret_cast<PassSmem<POS>*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  pdl_wait();     // the previous pass (or the upsweep) has completed and its writes are visible
  pdl_trigger();  // the next pass may launch; it waits for this grid in turn
  if (t == 0) sm.tile = (int)atomicAdd(&p.counters[pass], 1u);
  __syncthreads();
  const int64_t tile = sm.tile;
  const bool unsorted = *(volatile const int32_t*)p.flags != 0;
  if (!unsorted && pass < p.npass_id) return;  // ids already ordered: length passes only
  if (pass + 1 < p.npass)
    for (int d = t; d < RBINS; d += RT) p.status[(pass + 1) & 1][(size_t)tile * RBINS + d] = 0u;
  const int exec = unsorted ? pass : pass - p.npass_id;  // index among the executed passes
  const bool from_input = exec == 0, last = pass == p.npass - 1;
  const int shift = p.shift[pass];
  const uint32_t mask = (1u << p.bits[pass]) - 1u;
  const int64_t seg = tile / p.tps;
  const int tin = (int)(tile - seg * p.tps);
  const int64_t sbase = seg * (int64_t)p.seg_len;
  const int in0 = tin * TILE;
  const int n = min(TILE, p.seg_len - in0);
  const unsigned long long* kin = p.keys[(exec - 1) & 1];
  const int32_t* pin = p.pos[(exec - 1) & 1];

  for (int i = t; i < RW * RBINS; i += RT) (&sm.whist[0][0])[i] = 0u;
  if (last && p.tokens && p.lanes <= TOK_SMEM)
    for (int i = t; i < p.lanes; i += RT) sm.tok[i] = 0;
  __syncthreads();

  // load (warp w owns keys [w*512, w*512+512) of the tile, lane-striped) and
  // rank stably: inside a warp by (iteration, lane) = input order
  unsigned long long key[RI];
  int32_t pos[RI];
  uint32_t rank[RI];
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < RI; ++j) {
    const int i = w * WKEYS + j * 32 + lane;
    const bool valid = i < n;
    const int64_t g = sbase + in0 + i;
    if (valid) {
      if (from_input) {
        key[j] = make_key(p, p.lens[g], p.ids[g]);
        pos[j] = (int32_t)g;
      } else {
        key[j] = kin[g];
        if constexpr (POS) pos[j] = pin[g];
      }
    }
    const uint32_t d = valid ? (uint32_t)(key[j] >> shift) & mask : 0xffffffffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t cnt = 0;
    if (valid) cnt = sm.whist[w][d];
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) sm.whist[w][d] = cnt + __popc(peers);
    __syncwarp();
    rank[j] = cnt + __popc(peers & lt);
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
      sm.whist[ww][d] = run;
      run += c;
    }
    tot[h] = run;
  }
  // publish this tile's per-digit counts (the first tile of a segment has its
  // inclusive prefix at once)
  uint32_t* st = p.status[pass & 1] + (size_t)tile * RBINS;
#pragma unroll
  for (int h = 0; h < 2; ++h) st_relaxed_u32(&st[2 * t + h], (tin == 0 ? ST_PRE : ST_AGG) | tot[h]);
  const uint32_t* hseg = p.hist + ((size_t)pass * p.nseg + seg) * RBINS;
  const uint32_t h0 = hseg[2 * t], h1 = hseg[2 * t + 1];
  uint32_t eloc, eglob;
  block_scan2(tot[0], tot[1], h0, h1, eloc, eglob, sm.warp_tot);
  sm.off[2 * t] = eloc;
  sm.off[2 * t + 1] = eloc + tot[0];
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
  __syncthreads();

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
  // last pass: deal straight from the sorted slot (balance.py:59-70)
  const unsigned long long idmask = (1ull << p.id_bits) - 1ull;
  const bool tok_smem = p.tokens && p.lanes <= TOK_SMEM;
  // q / lanes = umul64hi(q, floor(2^64 / lanes) + 1), exact for q * lanes < 2^64
  const unsigned long long lanes_magic = ~0ull / (unsigned long long)p.lanes + 1ull;
  // lanes of a warp that deal to the same GPU lane add their lengths first (one atomic per
  // group; with lanes = 1 every key of the tile lands on one counter)
  const bool tok_redux = p.max_len < (1 << 26);
  for (int i0 = 0; i0 < n; i0 += RT) {
    const int i = i0 + t;
    const bool v = i < n;
    int ln = -1;
    int32_t len = 0;
    if (v) {
      const unsigned long long k = sm.key[i];
      const uint32_t d = (uint32_t)(k >> shift) & mask;
      const int64_t q = (int64_t)sm.gbase[d] + (i - sm.off[d]);  // sorted slot inside the segment
      const int64_t r = p.lanes == 1 ? q : (int64_t)__umul64hi((unsigned long long)q, lanes_magic);
      const int c = (int)(q - r * p.lanes);
      ln = (p.snake && (r & 1)) ? p.lanes - 1 - c : c;  // balance.py:66-67
      const int64_t o = sbase + (int64_t)ln * p.rows + r;
      B2_DASSERT(ln >= 0 && ln < p.lanes && r >= 0 && r < p.rows);
      p.out_ids[o] = (int32_t)(k & idmask);
      if constexpr (POS) p.out_pos[o] = sm.pos[i];
      len = p.max_len - (int32_t)(k >> p.id_bits);
    }
    if (!p.tokens) continue;
    if (tok_redux) {
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
  }
  if (tok_smem) {
    __syncthreads();
    for (int l = t; l < p.lanes; l += RT)  // per-lane token sums (_from_per_gpu, balance.py:54-56)
      if (sm.tok[l]) atomicAdd(reinterpret_cast<unsigned long long*>(&p.tokens[seg * p.lanes + l]), (unsigned long long)sm.tok[l]);
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
  size_t off_keys[2], off_pos[2], off_hist, off_status[2], off_counters, off_flags, total;
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
  const int64_t ctas = std::min<int64_t>(pl.ntiles, (int64_t)di.sm_count * 4);
  const int64_t per = (pl.ntiles + ctas - 1) / ctas;
  const int64_t grid_up = (pl.ntiles + per - 1) / per;
  k_radix_upsweep<<<(unsigned)grid_up, RT, 0, st>>>(p, per);
  B2_CHECK(cudaGetLastError());
  const size_t smem = out_pos ? sizeof(PassSmem<true>) : sizeof(PassSmem<false>);
  static bool configured[64][2] = {};
  const bool pos = out_pos != nullptr;
  if (!configured[di.device & 63][pos]) {
    if (pos) B2_CHECK(cudaFuncSetAttribute((const void*)k_radix_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    else B2_CHECK(cudaFuncSetAttribute((const void*)k_radix_pass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured[di.device & 63][pos] = true;
  }
  for (int q = 0; q < pl.npass; ++q) {
    // programmatic dependents: each pass launches under the previous kernel's tail
    if (pos) B2_CHECK(launch_pdl(k_radix_pass<true>, dim3((unsigned)pl.ntiles), dim3(RT), smem, st, p, q));
    else B2_CHECK(launch_pdl(k_radix_pass<false>, dim3((unsigned)pl.ntiles), dim3(RT), smem, st, p, q));
    B2_CHECK(cudaGetLastError());
  }
  return B2_OK;
}
