// Monte-Carlo balance engine, device side: per-trial
// per-GPU token counts and their min / max, for every trial in one launch.
//
// Reference: mcsim._trial_token_counts (mcsim.py:182-213) and _run
// (:284-300).  Input: the (b, G) length matrix of each trial, row-major (the
// host draws, b2_mc_draw).  Per strategy:
//   NONE, STRATIFIED  column sums (:186-188, :198-199);
//   LOCAL_PRESORT     per node: the pool (rows x that node's gpn columns, row
//                     order) sorted descending by value, dealt back as (b, gpn)
//                     rows, odd rows reversed under SNAKE, column sums
//                     (:201-212, _snake_flip :160-163);
//   GLOBAL_PRESORT    the same over all b*G values at once (:190-196).
// Only values are sorted (np.sort), so ties need no tie-break.  Sums are
// exact int64.  Layout: one CTA per trial (grid-stride), per-GPU counts in
// shared memory; LOCAL pools of <= 512 values sort in one warp (bitonic,
// registers); GLOBAL pools use a counting sort (lengths lie in [1, max_len])
// whose descending positions are resolved by binary search.
#include "bitonic.cuh"
#include "common.cuh"
#include "rng.h"

#include <algorithm>
#include <climits>

namespace b2 {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxGpus = 2048;   // per-CTA int64 counts in shared memory: 16 KB
constexpr int kMaxLenBins = 4096;

struct McParams {
  const int32_t* mat;
  int64_t ntrials;
  int b, G, gpn, strategy, snake, max_len;
  int64_t* counts;  // [ntrials][G] or null
  int64_t* mins;
  int64_t* maxs;
  int* bad;         // set to 1 if a length is outside [1, max_len]
};

__device__ __forceinline__ void block_minmax(int64_t& mn, int64_t& mx, int64_t* s_mn, int64_t* s_mx) {
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mn, o));
    mx = max(mx, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mx, o));
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_mn[w] = mn;
    s_mx[w] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < kThreads / 32; ++i) {
      s_mn[0] = min(s_mn[0], s_mn[i]);
      s_mx[0] = max(s_mx[0], s_mx[i]);
    }
  }
  __syncthreads();
  mn = s_mn[0];
  mx = s_mx[0];
}

template <int K>
__global__ void __launch_bounds__(kThreads) k_mc_counts(const __grid_constant__ McParams p) {
  __shared__ unsigned long long s_cnt[kMaxGpus];
  __shared__ int s_hist[kMaxLenBins + 1];
  __shared__ int64_t s_mn[kThreads / 32], s_mx[kThreads / 32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int b = p.b, G = p.G, P = b * G;
  // LOCAL_PRESORT: slot i = lane*K + j of a node pool is row i / gpn, column i % gpn of
  // the trial matrix (offset moff without the node's first column; -1 past the pool), and
  // sorted position i is dealt to GPU column lnj (snake-flipped on odd rows) -- the same
  // for every pool and trial, so the divisions are done once
  int moff[K], lnj[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int i = lane * K + j;
    const int gpn = p.gpn > 0 ? p.gpn : 1, r = i / gpn, c = i - r * gpn;
    const bool in = p.strategy == 2 && i < b * gpn;
    moff[j] = in ? r * G + c : -1;
    lnj[j] = in ? ((p.snake && (r & 1)) ? gpn - 1 - c : c) : -1;
  }
  for (int64_t tr = blockIdx.x; tr < p.ntrials; tr += gridDim.x) {
    const int32_t* m = p.mat + tr * (int64_t)P;
    for (int g = t; g < G; g += kThreads) s_cnt[g] = 0ull;
    __syncthreads();
    if (p.strategy <= 1) {  // NONE / STRATIFIED: column sums of the (b, G) matrix
      for (int g = t; g < G; g += kThreads) {
        long long s = 0;
        for (int r = 0; r < b; ++r) {
          const int v = m[(int64_t)r * G + g];
          if (v < 1 || v > p.max_len) *p.bad = 1;
          s += v;
        }
        s_cnt[g] = (unsigned long long)s;
      }
    } else if (p.strategy == 2) {  // LOCAL_PRESORT: one warp per node pool
      const int gpn = p.gpn, nodes = G / gpn;
      for (int nd = w; nd < nodes; nd += kThreads / 32) {
        uint32_t key[K];
#pragma unroll
        for (int j = 0; j < K; ++j) {
          if (moff[j] >= 0) {  // pool order: row r, then the node's columns
            const int v = m[(int64_t)moff[j] + nd * gpn];
            if (v < 1 || v > p.max_len) *p.bad = 1;
            key[j] = (uint32_t)(p.max_len - v);  // ascending key = descending length
          } else {
            key[j] = 0xffffffffu;
          }
        }
        warp_bitonic_sort<K>(key, lane);
        // the node's column sums by warp reductions: this warp alone owns columns
        // nd*gpn .. +gpn (plain stores; per-key 64-bit shared atomics into gpn addresses
        // were half the kernel's time).  A column sum <= b * max_len fits 32 bits.
        uint32_t lv[K];
#pragma unroll
        for (int j = 0; j < K; ++j) lv[j] = (uint32_t)(p.max_len - (int)key[j]);
        for (int col = 0; col < gpn; ++col) {
          uint32_t part = 0;
#pragma unroll
          for (int j = 0; j < K; ++j) part += lnj[j] == col ? lv[j] : 0u;
          const uint32_t tot = __reduce_add_sync(0xffffffffu, part);
          if (lane == (col & 31)) s_cnt[nd * gpn + col] = (unsigned long long)tot;
        }
      }
    } else {  // GLOBAL_PRESORT: counting sort of all b*G values
      for (int v = t; v <= p.max_len; v += kThreads) s_hist[v] = 0;
      __syncthreads();
      for (int i = t; i < P; i += kThreads) {
        const int v = m[i];
        if (v < 1 || v > p.max_len) {
          *p.bad = 1;
          continue;
        }
        atomicAdd(&s_hist[p.max_len - v], 1);  // bin 0 = longest
      }
      __syncthreads();
      if (t == 0) {  // exclusive prefix over <= 4097 bins (one pass, tiny next to the sums)
        int acc = 0;
        for (int v = 0; v <= p.max_len; ++v) {
          const int c = s_hist[v];
          s_hist[v] = acc;
          acc += c;
        }
      }
      __syncthreads();
      for (int pos = t; pos < P; pos += kThreads) {
        int lo = 0, hi = p.max_len;  // last bin whose start <= pos
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_hist[mid] <= pos) lo = mid;
          else hi = mid - 1;
        }
        const int v = p.max_len - lo;
        const int r = pos / G, c = pos - r * G;
        const int ln = (p.snake && (r & 1)) ? G - 1 - c : c;
        atomicAdd(&s_cnt[ln], (unsigned long long)v);
      }
    }
    __syncthreads();
    int64_t mn = LLONG_MAX, mx = LLONG_MIN;
    for (int g = t; g < G; g += kThreads) {
      const int64_t c = (int64_t)s_cnt[g];
      mn = min(mn, c);
      mx = max(mx, c);
      if (p.counts) p.counts[tr * G + g] = c;
    }
    block_minmax(mn, mx, s_mn, s_mx);
    if (t == 0) {
      p.mins[tr] = mn;
      p.maxs[tr] = mx;
    }
    __syncthreads();
  }
}

template <int K>
int launch(const McParams& p, cudaStream_t st) {
  const DeviceInfo& di = device_info();
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(p.ntrials, (int64_t)di.sm_count * 8));
  k_mc_counts<K><<<grid, kThreads, 0, st>>>(p);
  B2_CHECK(cudaGetLastError());
  return B2_OK;
}

// ---------------------------------------------------------------- device draws
// Trial t's draws (derive_rng(seed, t); per stratum choice(pool, need,
// replace=False) in the Floyd branch + numpy's final shuffle) for many trials
// at once: one warp per trial.  Floyd's algorithm is a sequential chain of
// bounded draws, so lane 0 runs it against an open-addressing set in shared
// memory (membership is all that matters for the output, so any exact set
// gives numpy's bits) and then the shuffle; the warp clears the set and
// gathers the picked lengths.  The tail-shuffle branch (pop > 10000 and
// need > pop/50) needs a population-sized array and stays on the host.
constexpr int kMaxStrataDraw = 16;
struct McDrawParams {
  const int32_t* lens;  // pool lengths, strata concatenated (device)
  int32_t* out;         // [ntrials][per_trial]
  uint64_t seed;
  int64_t first_trial, ntrials, per_trial;
  int nstrata;
  int64_t off[kMaxStrataDraw], pop[kMaxStrataDraw], need[kMaxStrataDraw];
  int bits[kMaxStrataDraw];  // log2 of the set size per stratum
  int set_cap, pick_cap;     // shared-memory words for the set and the picks
  int rbits;                 // compact kernel: value bits above the home slot (entry = probe << rbits | rest)
  int redo_only;             // 32-bit kernel: only trials the compact kernel marked (out row [0] == kRedo)
  int pmax_cap;              // > 0: a lower probe-index cap for the compact kernel (tests force the redo path)
};
constexpr int32_t kRedo = INT_MIN;  // compact kernel's mark: redo this trial with the 32-bit set

__global__ void __launch_bounds__(32) k_mc_draw(const __grid_constant__ McDrawParams q) {
  // one shared region per trial: the Floyd set, then (reloaded) the picks for
  // the shuffle; during Floyd the picks go straight to the trial's output
  // rows in global memory (fire-and-forget stores, off the critical path)
  extern __shared__ uint32_t sm[];
  uint32_t* set = sm;    // [set_cap] during Floyd
  uint32_t* picks = sm;  // [need] during the shuffle
  const int lane = threadIdx.x;
  constexpr uint32_t kEmpty = 0xffffffffu;
  for (int64_t tr = blockIdx.x; tr < q.ntrials; tr += gridDim.x) {
    if (q.redo_only && q.out[tr * q.per_trial] != kRedo) continue;  // warp-uniform
    const uint64_t key = (uint64_t)(q.first_trial + tr);
    rng::Pcg64 g(rng::SeedSeq(q.seed, &key, 1));  // used by lane 0 only
    int64_t row = 0;
    for (int k = 0; k < q.nstrata; ++k) {
      const int64_t need = q.need[k];
      if (need == 0) continue;
      const int bits = q.bits[k];
      const uint32_t hmask = (1u << bits) - 1u;
      for (int i = lane; i <= (int)hmask; i += 32) set[i] = kEmpty;
      __syncwarp();
      int32_t* o = q.out + tr * q.per_trial + row;  // this stratum's output rows (scratch first)
      if (lane == 0) {
        const int64_t pop = q.pop[k];
        for (int64_t j = pop - need; j < pop; ++j) {  // Floyd (numpy _generator choice)
          const uint32_t val = (uint32_t)g.bounded((uint64_t)j);
          // triangular probing (h + i(i+1)/2 visits every slot of a power-of-two table):
          // fewer probes than linear probing near the 0.75 load factor, same membership
          uint32_t h = (val * 2654435761u) >> (32 - bits), step = 0;
          uint32_t cur = set[h];
          while (cur != kEmpty && cur != val) {
            h = (h + ++step) & hmask;
            cur = set[h];
          }
          uint32_t pick = val;
          if (cur == kEmpty) {
            set[h] = val;
          } else {  // val already drawn: take j itself (never in the set yet)
            pick = (uint32_t)j;
            uint32_t h2 = ((uint32_t)j * 2654435761u) >> (32 - bits), step2 = 0;
            while (set[h2] != kEmpty) h2 = (h2 + ++step2) & hmask;
            set[h2] = pick;
          }
          o[j - pop + need] = (int32_t)pick;
        }
      }
      __syncwarp();  // orders lane 0's global stores before the warp's reload
      for (int64_t i = lane; i < need; i += 32) picks[i] = (uint32_t)o[i];
      __syncwarp();
      if (lane == 0) {
        for (int64_t i = need - 1; i >= 1; --i) {  // _shuffle_int(size, 1, idx)
          const int64_t j = (int64_t)g.bounded((uint64_t)i);
          const uint32_t t0 = picks[j];
          picks[j] = picks[i];
          picks[i] = t0;
        }
      }
      __syncwarp();
      const int32_t* L = q.lens + q.off[k];
      for (int64_t i = lane; i < need; i += 32) o[i] = L[picks[i]];
      __syncwarp();
      row += need;
    }
  }
}


// The same draws with half the shared memory per trial, so twice the trials
// (independent serial chains) are resident per SM.  The Floyd set holds 16-bit
// entries: a value's home slot is its low `bits` bits, and the entry keeps
// the rest of the value (rbits) plus the triangular-probe index at which it
// was stored, which together give the value back -- membership is exact.  The
// shuffle permutes 16-bit indices into the picks (numpy's swaps applied to
// positions), and the gathered lengths land in the same 16-bit slots.  A probe
// index or a length that does not fit marks the trial (row[0] = kRedo) for
// the 32-bit kernel, launched behind this one; redoing a trial is always
// exact, so the marks only cost time.
__global__ void __launch_bounds__(32) k_mc_draw16(const __grid_constant__ McDrawParams q) {
  extern __shared__ uint16_t sm16[];
  const int lane = threadIdx.x;
  constexpr uint16_t kEmpty16 = 0xffffu;
  uint32_t pmax = (1u << (16 - q.rbits)) - 2u;  // largest storable probe index (all-ones = empty)
  if (q.pmax_cap > 0 && (uint32_t)q.pmax_cap < pmax) pmax = (uint32_t)q.pmax_cap;
  for (int64_t tr = blockIdx.x; tr < q.ntrials; tr += gridDim.x) {
    const uint64_t key = (uint64_t)(q.first_trial + tr);
    rng::Pcg64 g(rng::SeedSeq(q.seed, &key, 1));  // used by lane 0 only
    int64_t row = 0;
    int redo = 0;
    for (int k = 0; k < q.nstrata && !redo; ++k) {
      const int64_t need = q.need[k];
      if (need == 0) continue;
      const int bits = q.bits[k];
      const uint32_t hmask = (1u << bits) - 1u;
      for (int i = lane; i <= (int)hmask; i += 32) sm16[i] = kEmpty16;
      __syncwarp();
      int32_t* o = q.out + tr * q.per_trial + row;
      if (lane == 0) {
        const int64_t pop = q.pop[k];
        for (int64_t j = pop - need; j < pop; ++j) {  // Floyd (numpy _generator choice)
          const uint32_t val = (uint32_t)g.bounded((uint64_t)j);
          uint32_t h = val & hmask, i = 0;
          const uint16_t want = (uint16_t)(val >> bits);
          bool found = false;
          for (;;) {  // triangular probing: home + i(i+1)/2 visits every slot
            if (i > pmax) break;  // entries are stored at probe index <= pmax: not there, and no room
            const uint16_t e = sm16[h];
            if (e == kEmpty16) break;
            if (e == (uint16_t)((i << q.rbits) | want)) {
              found = true;
              break;
            }
            h = (h + ++i) & hmask;
          }
          uint32_t pick = val;
          if (found) {  // val already drawn: take j itself (never in the set yet)
            pick = (uint32_t)j;
            h = pick & hmask;
            i = 0;
            while (i <= pmax && sm16[h] != kEmpty16) h = (h + ++i) & hmask;
          }
          if (i > pmax) {
            redo = 1;
            break;
          }
          sm16[h] = (uint16_t)((i << q.rbits) | (pick >> bits));
          o[j - pop + need] = (int32_t)pick;
        }
      }
      redo = __shfl_sync(0xffffffffu, redo, 0);
      if (redo) break;
      // shuffle 16-bit positions instead of the picks: numpy's swaps, same bits
      for (int64_t i = lane; i < need; i += 32) sm16[i] = (uint16_t)i;
      __syncwarp();
      if (lane == 0) {
        for (int64_t i = need - 1; i >= 1; --i) {  // _shuffle_int(size, 1, idx)
          const int64_t jj = (int64_t)g.bounded((uint64_t)i);
          const uint16_t t0 = sm16[jj];
          sm16[jj] = sm16[i];
          sm16[i] = t0;
        }
      }
      __syncwarp();
      // slot i: the pick at position perm[i] -> its length, kept in the same slot
      const int32_t* L = q.lens + q.off[k];
      int big = 0;
      for (int64_t i = lane; i < need; i += 32) {
        const int32_t v = L[o[sm16[i]]];
        big |= (uint32_t)v > 0xffffu;
        sm16[i] = (uint16_t)v;
      }
      if (__any_sync(0xffffffffu, big)) {
        redo = 1;
        break;
      }
      __syncwarp();  // every pick is read before the row is overwritten
      for (int64_t i = lane; i < need; i += 32) o[i] = (int32_t)sm16[i];
      __syncwarp();
      row += need;
    }
    if (redo && lane == 0) q.out[tr * q.per_trial] = kRedo;
    __syncwarp();
  }
}

}  // namespace
}  // namespace b2

using namespace b2;

extern "C" int b2_mc_draw_device(const int32_t* pool_lens, const int64_t* pool_sizes, int nstrata,
                                 const int64_t* counts, int num_gpus, uint64_t seed, int64_t first_trial,
                                 int64_t ntrials, int32_t* out, void* stream) {
  B2_REQUIRE(pool_lens && pool_sizes && counts && out, B2_ERR_INVALID, "NULL argument");
  B2_REQUIRE(nstrata >= 1 && nstrata <= kMaxStrataDraw, B2_ERR_UNSUPPORTED, "nstrata must be in [1, %d]",
             kMaxStrataDraw);
  B2_REQUIRE(num_gpus >= 1 && ntrials >= 0 && first_trial >= 0, B2_ERR_INVALID, "bad shape");
  McDrawParams q{};
  q.lens = pool_lens;
  q.out = out;
  q.seed = seed;
  q.first_trial = first_trial;
  q.ntrials = ntrials;
  q.nstrata = nstrata;
  int64_t off = 0, per = 0, maxneed = 0;
  int maxbits = 5;
  for (int k = 0; k < nstrata; ++k) {
    const int64_t need = counts[k] * (int64_t)num_gpus, pop = pool_sizes[k];
    B2_REQUIRE(counts[k] >= 0 && need <= pop, B2_ERR_INVALID,
               "corpus exhausted within a trial: a stratum holds %lld samples but the trial needs %lld",
               (long long)pop, (long long)need);
    B2_REQUIRE(pop < (int64_t)0xffffffffll, B2_ERR_UNSUPPORTED, "stratum %d too large for device draws", k);
    B2_REQUIRE(!(need > 0 && pop > 10000 && need > pop / 50), B2_ERR_UNSUPPORTED,
               "stratum %d uses numpy's tail-shuffle branch (host draws only)", k);
    int bits = 5;  // set of >= need / 0.75 slots, power of two
    while ((int64_t)(1ll << bits) * 3 < need * 4) ++bits;
    q.off[k] = off;
    q.pop[k] = pop;
    q.need[k] = need;
    q.bits[k] = bits;
    off += pop;
    per += need;
    maxneed = std::max(maxneed, need);
    maxbits = std::max(maxbits, bits);
  }
  q.per_trial = per;
  q.set_cap = 1 << maxbits;
  q.pick_cap = (int)std::max<int64_t>(1, maxneed);
  const size_t smem = sizeof(uint32_t) * (size_t)std::max<int64_t>(q.set_cap, q.pick_cap);
  B2_REQUIRE(smem <= 200 * 1024, B2_ERR_UNSUPPORTED, "trial too large for device draws (%zu B of shared memory)", smem);
  if (ntrials == 0) return B2_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const DeviceInfo& di = device_info();
  // compact 16-bit set (k_mc_draw16) when every stratum's values leave >= 4 bits of probe index
  // and positions fit 16 bits; the 32-bit kernel then redoes only the trials it marked
  static int env16 = -1;
  if (env16 < 0) {
    const char* e = getenv("B2_MC_DRAW16");
    env16 = e ? atoi(e) : 1;
  }
  bool compact = env16 != 0 && per > 0;
  int rbits = 0;
  for (int k = 0; k < nstrata; ++k) {
    if (q.need[k] == 0) continue;
    int vb = 0;  // bits of the largest value, pop - 1
    while ((1ll << vb) < q.pop[k]) ++vb;
    rbits = std::max(rbits, std::max(0, vb - q.bits[k]));
    compact = compact && q.need[k] <= 0xffff;
  }
  compact = compact && 16 - rbits >= 4;
  if (compact) {
    q.rbits = rbits;
    const char* pc = getenv("B2_MC_DRAW16_PMAX");  // test hook: force probe overflows -> redo path
    q.pmax_cap = pc ? atoi(pc) : 0;
    const size_t smem16 = sizeof(uint16_t) * (size_t)std::max<int64_t>(q.set_cap, q.pick_cap);
    B2_CHECK(cudaFuncSetAttribute(k_mc_draw16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem16));
    int occ16 = 0;
    B2_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ16, k_mc_draw16, 32, smem16));
    B2_REQUIRE(occ16 >= 1, B2_ERR_UNSUPPORTED, "device draw kernel cannot be resident");
    const unsigned g16 = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ntrials, (int64_t)di.sm_count * occ16));
    k_mc_draw16<<<g16, 32, smem16, st>>>(q);
    B2_CHECK(cudaGetLastError());
    q.redo_only = 1;
  }
  B2_CHECK(cudaFuncSetAttribute(k_mc_draw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  B2_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mc_draw, 32, smem));
  B2_REQUIRE(occ >= 1, B2_ERR_UNSUPPORTED, "device draw kernel cannot be resident");
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ntrials, (int64_t)di.sm_count * occ));
  k_mc_draw<<<grid, 32, smem, st>>>(q);
  B2_CHECK(cudaGetLastError());
  return B2_OK;
}

extern "C" int b2_mc_token_counts(const int32_t* mat, int64_t ntrials, int b, int num_gpus, int gpus_per_node,
                                  int strategy, int scan, int32_t max_len, int64_t* counts, int64_t* mins,
                                  int64_t* maxs, int32_t* bad, void* stream) {
  B2_REQUIRE(b >= 1 && num_gpus >= 1 && gpus_per_node >= 1 && num_gpus % gpus_per_node == 0, B2_ERR_INVALID,
             "bad shape: b=%d G=%d gpn=%d", b, num_gpus, gpus_per_node);
  B2_REQUIRE(strategy >= 0 && strategy <= 3, B2_ERR_INVALID, "bad strategy %d", strategy);
  B2_REQUIRE(scan == B2_SCAN_RASTER || scan == B2_SCAN_SNAKE, B2_ERR_INVALID, "bad scan %d", scan);
  B2_REQUIRE(num_gpus <= kMaxGpus, B2_ERR_UNSUPPORTED, "at most %d GPUs per trial", kMaxGpus);
  B2_REQUIRE(max_len >= 1 && max_len <= kMaxLenBins, B2_ERR_UNSUPPORTED, "max_len must be in [1, %d]", kMaxLenBins);
  B2_REQUIRE(strategy != 2 || b * gpus_per_node <= 512, B2_ERR_UNSUPPORTED,
             "local presort pools of %d samples exceed 512", b * gpus_per_node);
  B2_REQUIRE(ntrials >= 0, B2_ERR_INVALID, "ntrials must be >= 0");
  B2_REQUIRE(mins && maxs && bad, B2_ERR_INVALID, "NULL output");
  cudaStream_t st = (cudaStream_t)stream;
  B2_CHECK(cudaMemsetAsync(bad, 0, sizeof(int32_t), st));
  if (ntrials == 0) return B2_OK;
  B2_REQUIRE(mat, B2_ERR_INVALID, "NULL matrix");
  McParams p{};
  p.mat = mat;
  p.ntrials = ntrials;
  p.b = b;
  p.G = num_gpus;
  p.gpn = gpus_per_node;
  p.strategy = strategy;
  p.snake = scan == B2_SCAN_SNAKE;
  p.max_len = max_len;
  p.counts = counts;
  p.mins = mins;
  p.maxs = maxs;
  p.bad = bad;
  const int pp = strategy == 2 ? b * gpus_per_node : 32;
  if (pp <= 32) return launch<1>(p, st);
  if (pp <= 64) return launch<2>(p, st);
  if (pp <= 128) return launch<4>(p, st);
  if (pp <= 256) return launch<8>(p, st);
  return launch<16>(p, st);
}
