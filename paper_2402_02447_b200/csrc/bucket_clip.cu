// H1 — bucket-wise gradient clipping before allreduce (sm_100a).
//
// K1  k_bucket_clip : fused per-bucket L2 norm -> clip coefficient -> scale +
//                     cast into the communication buffer.
//                     Reference: clip_by_norm (gradsync.py:106-116) applied per
//                     (worker, bucket) by sync_bucketwise (gradsync.py:148-162).
// K1b k_weighted_mean: single-process K-worker mean of clipped buckets with the
//                     reference's pairwise tree (gradsync.py:119-128).
//
// K1 design (HBM-bound: 4 B read + 2/4 B write per element):
//   one persistent cooperative grid (2 CTAs/SM) walks the list of segments
//   (buckets) with two streams per CTA — A: norm pass over bucket s (128-bit
//   loads, L2 evict_last), B: scale pass over bucket s-1 (L2 re-read,
//   evict_first) — so the grid-wide norm dependency of a bucket is hidden
//   behind a whole bucket of A work.  Several buckets per launch: A and B are
//   concurrent warp groups of every CTA (k_bucket_clip_ws, 256 + 256
//   threads; small buckets form CTA groups, each owning every R-th bucket);
//   a lone bucket (the DDP-hook shape): the time-sliced k_bucket_clip_l2lag.  Partials are published fire-and-forget
//   and every CTA folds them in one fixed order (bit-deterministic, identical
//   coefficient grid-wide).  A TMA-ring variant (cp.async.bulk into a
//   shared-memory ring) measured slower on B200 because the ring must either
//   hold the bucket through the barrier or lose its L2 residency.
#include "clip_common.cuh"

#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace b2 {
namespace {
using namespace clip;

// ----------------------------------------------------------------------------
// K1 (L2-lag): the production variant.  Persistent cooperative grid of CPS
// CTAs per SM; each CTA owns one contiguous chunk of every bucket.
//   stream A (norm): 128-bit loads with an L2 evict_last policy, UA in flight
//     per thread; fp32 mini-sums promoted to fp64; one partial per
//     (bucket, CTA) published fire-and-forget (red.release).
//   stream B (scale), LAG buckets behind: every CTA folds the bucket's
//     partials in one fixed order (bit-identical coefficient grid-wide),
//     re-reads its chunk - an L2 hit, A touched it one bucket ago - with an
//     evict_first policy (last use) and stores cast(g * coef * post_scale).
// The grid-wide norm dependency is hidden behind a whole bucket of A work,
// and HBM sees the algorithmic 4 B read + out-dtype write per element.
template <typename Tin, typename Tout, int THREADS, int CPS, int LAG, int UA, int UB, int BNC>
__global__ void __launch_bounds__(THREADS, CPS) k_bucket_clip_l2lag(const __grid_constant__ ClipParams p) {
  using V = typename VecOf<Tin>::V;
  constexpr int N = VecOf<Tin>::N;
  constexpr bool kF64 = std::is_same<Tin, double>::value;
  using Acc = typename std::conditional<std::is_same<Tin, double>::value || std::is_same<Tout, double>::value,
                                        double, float>::type;
  __shared__ double s_coef[2];
  __shared__ double red[32];
  // lone-bucket launches are programmatic dependents (launch_l2lag): the
  // launch overlaps the previous kernel's tail, every read waits for it.  A
  // no-op otherwise.  Triggering here is safe: a dependent can only start once
  // every CTA of this grid has triggered, i.e. is resident.
  pdl_wait();
  pdl_trigger();
  const int G = gridDim.x, c = blockIdx.x, t = threadIdx.x;
  const bool scale = p.out != nullptr;
  const uint64_t pol_keep = scale ? l2_policy_evict_last() : l2_policy_evict_first();
  const uint64_t pol_drop = l2_policy_evict_first();

  // block-wide fixed-order fold of the G partials of segment s -> coefficient
  // (one L2 round trip: each thread loads <= ceil(G/THREADS) partials)
  auto fold = [&](int s, bool publish) -> double {
    if (t == 0) {
      unsigned ns = 32;
      while (ld_acquire_u32(&p.counters[s]) < (unsigned)G) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
      }
    }
    __syncthreads();
    double v = 0.0;
    for (int j = t; j < G; j += THREADS) v += __ldcg(&p.partials[(size_t)s * G + j]);
    const double total = block_sum<THREADS>(v, red);
    if (t == 0) {
      const double norm = sqrt(total);
      const double coef = (norm >= p.limit) ? p.limit / norm : 1.0;  // gradsync.py:114-116
      if (publish) {
        if (p.norms) p.norms[s] = norm;
        if (p.coefs) p.coefs[s] = coef;
        if (p.nonfinite) p.nonfinite[s] = (kF64 ? isnan(total) : !isfinite(total)) ? 1 : 0;
      }
      s_coef[s & 1] = coef;
    }
    __syncthreads();
    return s_coef[s & 1];
  };

  auto norm_pass = [&](int s) {
    const Seg sg = p.seg[s];
    const Tin* in = static_cast<const Tin*>(p.in) + sg.in_off;
    double acc[N];
#pragma unroll
    for (int u = 0; u < N; ++u) acc[u] = 0.0;
    bool bad = false;
    auto add = [&](const V& x) {
      double e[N];
      unpack(x, e);
#pragma unroll
      for (int u = 0; u < N; ++u) {
        if constexpr (kF64) bad |= !isfinite(e[u]);
        acc[u] = fma(e[u], e[u], acc[u]);
      }
    };
    if (sg.vec) {
      const V* vin = reinterpret_cast<const V*>(in + sg.head);
      const int64_t v0 = min64((int64_t)c * sg.per, sg.nv), v1 = min64(v0 + sg.per, sg.nv);
      for (int64_t v = v0 + t; v < v1; v += (int64_t)THREADS * UA) {
        V x[UA];
#pragma unroll
        for (int u = 0; u < UA; ++u) {
          const int64_t vi = v + (int64_t)u * THREADS;
          x[u] = vi < v1 ? ld_a<0>(vin + vi, pol_keep) : V{};
        }
        if constexpr (kF64) {
#pragma unroll
          for (int u = 0; u < UA; ++u) add(x[u]);
        } else {
          // f32: <= 32 squares summed in fp32 (rel. error < 2e-6), promoted
          // once; a mini-sum outside [2^-100, 2^100] (underflow, overflow,
          // inf, nan) with a non-zero element is redone exactly in fp64
#pragma unroll
          for (int h = 0; h < UA; h += 8) {
            float m = 0.0f;
            unsigned nz = 0;
#pragma unroll
            for (int u = h; u < h + 8 && u < UA; ++u) {
              m = fmaf(x[u].x, x[u].x, m);
              m = fmaf(x[u].y, x[u].y, m);
              m = fmaf(x[u].z, x[u].z, m);
              m = fmaf(x[u].w, x[u].w, m);
              nz |= __float_as_uint(x[u].x) | __float_as_uint(x[u].y) | __float_as_uint(x[u].z) |
                    __float_as_uint(x[u].w);
            }
            if (m >= 0x1p-100f && m <= 0x1p100f) {
              acc[0] += (double)m;
            } else if ((nz << 1) != 0u) {
#pragma unroll
              for (int u = h; u < h + 8 && u < UA; ++u) add(x[u]);
            }
          }
        }
      }
      const int64_t tail0 = sg.head + sg.nv * N;
      if (c == 0 && t < sg.head) acc[0] += sq_of(in[t], bad);
      if (c == G - 1 && t < sg.n - tail0) acc[N - 1] += sq_of(in[tail0 + t], bad);
    } else {
      const int64_t per = (sg.n + G - 1) / G;
      const int64_t e0 = min64((int64_t)c * per, sg.n), e1 = min64(e0 + per, sg.n);
      for (int64_t e = e0 + t; e < e1; e += THREADS) acc[0] += sq_of(in[e], bad);
    }
    double part = 0.0;
#pragma unroll
    for (int u = 0; u < N; ++u) part += acc[u];
    double tot = block_sum<THREADS>(part, red);
    if constexpr (kF64) {
      if (__syncthreads_or(bad)) tot = __longlong_as_double(0x7ff8000000000000ll);  // NaN marks inf/nan input
    }
    if (t == 0) {
      B2_DASSERT(s < kMaxSegs && c < G && (size_t)s * G + c < (size_t)kMaxSegs * kMaxGrid);
      p.partials[(size_t)s * G + c] = tot;
      red_release_u32(&p.counters[s], 1u);  // fire-and-forget arrival
    }
  };

  auto scale_pass = [&](int s) {
    const Seg sg = p.seg[s];
    const Tin* in = static_cast<const Tin*>(p.in) + sg.in_off;
    Tout* out = static_cast<Tout*>(p.out) + sg.out_off;
    const V* vin = reinterpret_cast<const V*>(in + sg.head);
    const int64_t v0 = sg.vec ? min64((int64_t)c * sg.per, sg.nv) : 0;
    const int64_t v1 = sg.vec ? min64(v0 + sg.per, sg.nv) : 0;
    // the chunk's first UB vectors load while the bucket's partials are awaited and folded
    V x[UB];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int64_t vi = v0 + t + (int64_t)u * THREADS;
      if (vi < v1) x[u] = ld_b<BNC>(vin + vi, pol_drop);
    }
    const Acc cf = static_cast<Acc>(fold(s, c == 0) * p.post_scale);
    if (sg.vec) {
      Tout* vout = out + sg.head;
      for (int64_t v = v0 + t; v < v1; v += (int64_t)THREADS * UB) {
        if (v != v0 + t) {
#pragma unroll
          for (int u = 0; u < UB; ++u) {
            const int64_t vi = v + (int64_t)u * THREADS;
            if (vi < v1) x[u] = ld_b<BNC>(vin + vi, pol_drop);
          }
        }
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int64_t vi = v + (int64_t)u * THREADS;
          if (vi < v1) {
            Acc y[N];
            if constexpr (kF64) {
              y[0] = x[u].x * cf;
              y[1] = x[u].y * cf;
            } else {  // f32 in: scale in the output's working precision
              y[0] = static_cast<Acc>(x[u].x) * cf;
              y[1] = static_cast<Acc>(x[u].y) * cf;
              y[2] = static_cast<Acc>(x[u].z) * cf;
              y[3] = static_cast<Acc>(x[u].w) * cf;
            }
            put_vec<Tout, N, Acc>(vout + vi * N, y);
          }
        }
      }
      const int64_t tail0 = sg.head + sg.nv * N;
      if (c == 0 && t < sg.head) put1(out + t, static_cast<Acc>(in[t]) * cf);
      if (c == G - 1 && t < sg.n - tail0) put1(out + tail0 + t, static_cast<Acc>(in[tail0 + t]) * cf);
    } else {
      const int64_t per = (sg.n + G - 1) / G;
      const int64_t e0 = min64((int64_t)c * per, sg.n), e1 = min64(e0 + per, sg.n);
      for (int64_t e = e0 + t; e < e1; e += THREADS) put1(out + e, static_cast<Acc>(in[e]) * cf);
    }
  };

  for (int it = 0; it < p.nseg + (scale ? LAG : 0); ++it) {
    if (it < p.nseg) norm_pass(it);
    if (scale && it >= LAG) scale_pass(it - LAG);
  }
  if (!scale)  // norm-only: publish every segment, spread over CTAs
    for (int s = c; s < p.nseg; s += G) fold(s, true);

  __syncthreads();
  if (t == 0) {
    if (atom_add_acq_rel_u32(&p.counters[kMaxSegs], 1u) == (unsigned)G - 1) {
      for (int s = 0; s < p.nseg; ++s) p.counters[s] = 0u;
      p.counters[kMaxSegs] = 0u;
      __threadfence();
    }
  }
}

template <typename Tin, typename Tout, int THREADS, int CPS, int LAG, int UA, int UB, int BNC>
int launch_l2lag(ClipParams& p, cudaStream_t stream) {
  auto kern = k_bucket_clip_l2lag<Tin, Tout, THREADS, CPS, LAG, UA, UB, BNC>;
  const DeviceInfo& di = device_info();
  B2_REQUIRE(di.coop, B2_ERR_CUDA, "device does not support cooperative launch");
  static int occ_cached[64] = {};
  int& occ = occ_cached[di.device & 63];
  if (occ == 0) {
    B2_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, THREADS, 0));
    B2_REQUIRE(occ >= 1, B2_ERR_CUDA, "clip kernel cannot be resident");
  }
  int64_t total = 0;
  for (int s = 0; s < p.nseg; ++s) total += p.seg[s].n;
  const int64_t want = (total + 16384 - 1) / 16384;  // small problems: fewer CTAs
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>({(int64_t)di.sm_count * std::min(CPS, occ), want, (int64_t)kMaxGrid}));
  const int N = p.seg_vec_elems;
  for (int s = 0; s < p.nseg; ++s) {
    Seg& sg = p.seg[s];
    sg.nv = sg.vec ? (sg.n - sg.head) / N : 0;
    sg.per = (sg.nv + grid - 1) / grid;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  // A lone bucket (the DDP-hook / reducer shape, one launch per bucket) is
  // launch-bound: it goes out as a programmatic dependent launch, which a
  // cooperative launch cannot be (~2 us of the 12 us; DESIGN K1).  The grid
  // is sized to what is co-resident, and a dependent of this grid can only
  // start once all of its CTAs are resident, so the spin on the partials
  // still sees every CTA.  Several buckets per launch stay cooperative.
  static int pdl_env = -1;
  if (pdl_env < 0) {
    const char* e = getenv("B2_CLIP_PDL");
    pdl_env = e ? atoi(e) : 1;
  }
  if (p.nseg == 1 && p.out != nullptr && pdl_env) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
  } else {
    attr[0].id = cudaLaunchAttributeCooperative;  // CTAs wait on each other's partials
    attr[0].val.cooperative = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  B2_CHECK(cudaLaunchKernelEx(&cfg, kern, p));
  return B2_OK;
}

// ----------------------------------------------------------------------------
// K1 (warp-specialised L2-lag): the same two streams as k_bucket_clip_l2lag,
// but run CONCURRENTLY by two warp groups of every CTA: AT threads stream the
// norm pass of bucket s while BT threads scale bucket s-1 out of L2.  The
// groups sync only through named barriers of their own and one shared
// counter (A may run at most LAG+1 buckets ahead of B, which bounds the L2
// footprint to ~2 buckets), so HBM reads (A), L2 re-reads and HBM writes (B)
// overlap instead of alternating.
template <typename Tin, typename Tout, int AT, int BT, int CPS, int LAG, int UA, int UB>
__global__ void __launch_bounds__(AT + BT, CPS) k_bucket_clip_ws(const __grid_constant__ ClipParams p) {
  using V = typename VecOf<Tin>::V;
  constexpr int N = VecOf<Tin>::N;
  constexpr bool kF64 = std::is_same<Tin, double>::value;
  using Acc = typename std::conditional<std::is_same<Tin, double>::value || std::is_same<Tout, double>::value,
                                        double, float>::type;
  constexpr int kBarA = 1, kBarB = 2;
  __shared__ double redA[32], redB[32];
  __shared__ double s_coef;
  __shared__ volatile int s_bdone;  // buckets the B group has finished
  // CTA groups (p.ngroups): this CTA serves buckets gid, gid+R, ... as member gr of Gc CTAs
  const int R = p.ngroups, gid = blockIdx.x % R, gr = blockIdx.x / R;
  const int Gc = group_size(gridDim.x, R, gid), t = threadIdx.x;
  const int G = Gc, c = gr;
  const bool scale = p.out != nullptr;
  if (t == 0) s_bdone = 0;
  __syncthreads();

  // fixed-order fold of segment s's G partials by a group of NTH threads
  auto fold = [&](auto nth, int gt, int bar, double* scratch, int s, bool publish) -> double {
    constexpr int NTH = decltype(nth)::value;
    if (gt == 0) {
      unsigned ns = 32;
      while (ld_acquire_u32(&p.counters[s]) < (unsigned)G) {
        __nanosleep(ns);
        if (ns < 32) ns <<= 1;
      }
    }
    group_sync<NTH>(bar);
    double v = 0.0;
    for (int j = gt; j < G; j += NTH) v += __ldcg(&p.partials[(size_t)s * kMaxGrid + j]);
    const double total = group_sum<NTH>(v, scratch, gt, bar);
    double coef = 1.0;
    if (gt == 0) {
      const double norm = sqrt(total);
      coef = (norm >= p.limit) ? p.limit / norm : 1.0;  // gradsync.py:114-116
      if (publish) {
        if (p.norms) p.norms[s] = norm;
        if (p.coefs) p.coefs[s] = coef;
        if (p.nonfinite) p.nonfinite[s] = (kF64 ? isnan(total) : !isfinite(total)) ? 1 : 0;
      }
    }
    return coef;  // valid in gt == 0
  };

  if (t < AT) {
    // ================= A group: norm pass, bucket after bucket
    const int gt = t;
    const uint64_t pol_keep = scale ? l2_policy_evict_last() : l2_policy_evict_first();
    for (int i = 0, s = gid; s < p.nseg; ++i, s += R) {
      const Seg sg = p.seg[s];
      const Tin* in = static_cast<const Tin*>(p.in) + sg.in_off;
      const V* vin = reinterpret_cast<const V*>(in + sg.head);
      const int64_t v0 = sg.vec ? min64((int64_t)c * sg.per, sg.nv) : 0;
      const int64_t v1 = sg.vec ? min64(v0 + sg.per, sg.nv) : 0;
      auto wait_b = [&]() {
        if (scale && i > LAG) {  // L2 footprint bound: wait until B finished this group's bucket i-LAG-1
          if (gt == 0) {
            unsigned ns = 32;
            while (s_bdone < i - LAG) {
              __nanosleep(ns);
              if (ns < 32) ns <<= 1;
            }
          }
          group_sync<AT>(kBarA);
        }
      };
      // bf16 out: the chunk's first UA vectors are requested before the L2-footprint wait
      // (32 KB per CTA more in flight; the wait overlaps their latency): 370 -> 351 us.
      // With 4 B outputs all UA early cost more than they hide (485 -> 515 us); half of
      // them early measured 485 -> 482 us.
      constexpr int kPreA = sizeof(Tout) <= 2 ? UA : UA / 2;  // vectors requested before the wait
      V x[UA];
#pragma unroll
      for (int u = 0; u < kPreA; ++u) {
        const int64_t vi = v0 + gt + (int64_t)u * AT;
        x[u] = vi < v1 ? ld_a<0>(vin + vi, pol_keep) : V{};
      }
      wait_b();
#pragma unroll
      for (int u = kPreA; u < UA; ++u) {
        const int64_t vi = v0 + gt + (int64_t)u * AT;
        x[u] = vi < v1 ? ld_a<0>(vin + vi, pol_keep) : V{};
      }
      double acc[N];
#pragma unroll
      for (int u = 0; u < N; ++u) acc[u] = 0.0;
      bool bad = false;
      auto add = [&](const V& x) {
        double e[N];
        unpack(x, e);
#pragma unroll
        for (int u = 0; u < N; ++u) {
          if constexpr (kF64) bad |= !isfinite(e[u]);
          acc[u] = fma(e[u], e[u], acc[u]);
        }
      };
      if (sg.vec) {
        for (int64_t v = v0 + gt; v < v1; v += (int64_t)AT * UA) {
          if (v != v0 + gt) {
#pragma unroll
            for (int u = 0; u < UA; ++u) {
              const int64_t vi = v + (int64_t)u * AT;
              x[u] = vi < v1 ? ld_a<0>(vin + vi, pol_keep) : V{};
            }
          }
          if constexpr (kF64) {
#pragma unroll
            for (int u = 0; u < UA; ++u) add(x[u]);
          } else {
            // f32: <= 32 squares summed in fp32 (rel. error < 2e-6), promoted
            // once; a mini-sum outside [2^-100, 2^100] with a non-zero element
            // (underflow, overflow, inf, nan) is redone exactly in fp64
#pragma unroll
            for (int h = 0; h < UA; h += 8) {
              float m = 0.0f;
              unsigned nz = 0;
#pragma unroll
              for (int u = h; u < h + 8 && u < UA; ++u) {
                m = fmaf(x[u].x, x[u].x, m);
                m = fmaf(x[u].y, x[u].y, m);
                m = fmaf(x[u].z, x[u].z, m);
                m = fmaf(x[u].w, x[u].w, m);
                nz |= __float_as_uint(x[u].x) | __float_as_uint(x[u].y) | __float_as_uint(x[u].z) |
                      __float_as_uint(x[u].w);
              }
              if (m >= 0x1p-100f && m <= 0x1p100f) {
                acc[0] += (double)m;
              } else if ((nz << 1) != 0u) {
#pragma unroll
                for (int u = h; u < h + 8 && u < UA; ++u) add(x[u]);
              }
            }
          }
        }
        const int64_t tail0 = sg.head + sg.nv * N;
        if (c == 0 && gt < sg.head) acc[0] += sq_of(in[gt], bad);
        if (c == G - 1 && gt < sg.n - tail0) acc[N - 1] += sq_of(in[tail0 + gt], bad);
      } else {
        const int64_t per = (sg.n + G - 1) / G;
        const int64_t e0 = min64((int64_t)c * per, sg.n), e1 = min64(e0 + per, sg.n);
        for (int64_t e = e0 + gt; e < e1; e += AT) acc[0] += sq_of(in[e], bad);
      }
      double part = 0.0;
#pragma unroll
      for (int u = 0; u < N; ++u) part += acc[u];
      if constexpr (kF64) part = __any_sync(0xffffffffu, bad) ? __longlong_as_double(0x7ff8000000000000ll) : part;
      const double tot = group_sum<AT>(part, redA, gt, kBarA);  // NaN propagates: marks inf/nan input
      if (gt == 0) {
        B2_DASSERT(s < kMaxSegs && c < kMaxGrid);
        p.partials[(size_t)s * kMaxGrid + c] = tot;
        red_release_u32(&p.counters[s], 1u);  // fire-and-forget arrival
      }
    }
    if (!scale && c == 0)  // norm-only: the group's first CTA publishes its buckets
      for (int s = gid; s < p.nseg; s += R) fold(std::integral_constant<int, AT>{}, gt, kBarA, redA, s, true);
  } else if (scale) {
    // ================= B group: scale pass, one bucket behind
    const int gt = t - AT;
    const uint64_t pol_drop = l2_policy_evict_first();
    for (int i = 0, s = gid; s < p.nseg; ++i, s += R) {
      const Seg sg = p.seg[s];
      const Tin* in = static_cast<const Tin*>(p.in) + sg.in_off;
      Tout* out = static_cast<Tout*>(p.out) + sg.out_off;
      const V* vin = reinterpret_cast<const V*>(in + sg.head);
      const int64_t v0 = sg.vec ? min64((int64_t)c * sg.per, sg.nv) : 0;
      const int64_t v1 = sg.vec ? min64(v0 + sg.per, sg.nv) : 0;
      // the chunk's first UB vectors are loaded before the coefficient is known (they do
      // not depend on it): their L2 latency overlaps the wait for the bucket's partials
      V x[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int64_t vi = v0 + gt + (int64_t)u * BT;
        if (vi < v1) x[u] = ld_b<0>(vin + vi, pol_drop);
      }
      const double coef = fold(std::integral_constant<int, BT>{}, gt, kBarB, redB, s, c == 0);
      if (gt == 0) s_coef = coef;
      group_sync<BT>(kBarB);
      const Acc cf = static_cast<Acc>(s_coef * p.post_scale);
      if (sg.vec) {
        Tout* vout = out + sg.head;
        for (int64_t v = v0 + gt; v < v1; v += (int64_t)BT * UB) {
          if (v != v0 + gt) {
#pragma unroll
            for (int u = 0; u < UB; ++u) {
              const int64_t vi = v + (int64_t)u * BT;
              if (vi < v1) x[u] = ld_b<0>(vin + vi, pol_drop);
            }
          }
#pragma unroll
          for (int u = 0; u < UB; ++u) {
            const int64_t vi = v + (int64_t)u * BT;
            if (vi < v1) {
              Acc y[N];
              if constexpr (kF64) {
                y[0] = x[u].x * cf;
                y[1] = x[u].y * cf;
              } else {
                y[0] = static_cast<Acc>(x[u].x) * cf;
                y[1] = static_cast<Acc>(x[u].y) * cf;
                y[2] = static_cast<Acc>(x[u].z) * cf;
                y[3] = static_cast<Acc>(x[u].w) * cf;
              }
              put_vec<Tout, N, Acc>(vout + vi * N, y);
            }
          }
        }
        const int64_t tail0 = sg.head + sg.nv * N;
        if (c == 0 && gt < sg.head) put1(out + gt, static_cast<Acc>(in[gt]) * cf);
        if (c == G - 1 && gt < sg.n - tail0) put1(out + tail0 + gt, static_cast<Acc>(in[tail0 + gt]) * cf);
      } else {
        const int64_t per = (sg.n + G - 1) / G;
        const int64_t e0 = min64((int64_t)c * per, sg.n), e1 = min64(e0 + per, sg.n);
        for (int64_t e = e0 + gt; e < e1; e += BT) put1(out + e, static_cast<Acc>(in[e]) * cf);
      }
      group_sync<BT>(kBarB);  // whole group done with bucket s (also retires s_coef)
      if (gt == 0) s_bdone = i + 1;
    }
  }

  __syncthreads();
  if (t == 0) {
    if (atom_add_acq_rel_u32(&p.counters[kMaxSegs], 1u) == gridDim.x - 1) {
      for (int s = 0; s < p.nseg; ++s) p.counters[s] = 0u;
      p.counters[kMaxSegs] = 0u;
      __threadfence();
    }
  }
}

template <typename Tin, typename Tout, int AT, int BT, int CPS, int LAG, int UA, int UB>
int launch_ws(ClipParams& p, cudaStream_t stream) {
  auto kern = k_bucket_clip_ws<Tin, Tout, AT, BT, CPS, LAG, UA, UB>;
  const DeviceInfo& di = device_info();
  B2_REQUIRE(di.coop, B2_ERR_CUDA, "device does not support cooperative launch");
  static int occ_cached[64] = {};
  int& occ = occ_cached[di.device & 63];
  if (occ == 0) {
    B2_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, AT + BT, 0));
    B2_REQUIRE(occ >= 1, B2_ERR_CUDA, "clip kernel cannot be resident");
  }
  int64_t total = 0;
  for (int s = 0; s < p.nseg; ++s) total += p.seg[s].n;
  const int64_t want = (total + 16384 - 1) / 16384;  // small problems: fewer CTAs
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>({(int64_t)di.sm_count * std::min(CPS, occ), want, (int64_t)kMaxGrid}));
  const int N = p.seg_vec_elems;
  p.ngroups = choose_groups(p, grid, sizeof(Tin));
  for (int s = 0; s < p.nseg; ++s) {
    Seg& sg = p.seg[s];
    const int gs = group_size(grid, p.ngroups, s % p.ngroups);
    sg.nv = sg.vec ? (sg.n - sg.head) / N : 0;
    sg.per = (sg.nv + gs - 1) / gs;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(AT + BT);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // CTAs wait on each other's partials
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  B2_CHECK(cudaLaunchKernelEx(&cfg, kern, p));
  return B2_OK;
}

// K1 configuration (tools/clip_bench.py sweeps; measurements in DESIGN.md):
// several buckets per launch -> warp-specialised two-stream kernel
// (256 norm + 256 scale threads, 8 vectors in flight per thread in both, 2
// CTAs/SM, each stream requesting its next chunk's first vectors before it
// waits: 351 us timed alone / 378 us at the power cap for BERT-large bf16 out,
// vs 382 / 401 for round 1's 192 + 320 with 4 scale vectors,
// tools/step_timing_probe.py); a lone bucket (DDP-hook shape) -> the
// time-sliced L2-lag kernel, which has the shorter critical path.
// (The measured alternatives — a TMA shared-memory ring and other warp
// splits — live in git history, commit 4cd4b3b, not in the product library.)
template <typename Tin, typename Tout>
int launch_clip_k1(ClipParams& p, cudaStream_t stream) {
  // norm-only launches have no scale stream: the time-sliced kernel puts every thread on the norm
  if (p.nseg >= 2 && p.out != nullptr) return launch_ws<Tin, Tout, 256, 256, 2, 1, 8, 8>(p, stream);
  return launch_l2lag<Tin, Tout, 384, 2, 1, 8, 4, 0>(p, stream);
}

// ---------------------------------------------------------------- K1b
constexpr int kCoefSmem = 256;  // coefficients staged in shared memory (more: read through L1)
constexpr int kMeanThreads = 256;

struct MeanParams {
  const void* G;
  void* out;
  const double* coef;  // [K][B_total]
  int64_t K, ld;
  int B_total, b0, nb;  // this launch covers buckets b0 .. b0+nb-1
  int64_t bounds[kMaxSegs + 1];
};

// The reference's pairwise tree (gradsync.py:123-127: each round merges
// (0,1),(2,3).., an odd tail is carried) equals a binary-counter stack walk in
// ascending worker order: push each value as a block of size 1, merge the top
// two while they have equal sizes, and at the end fold the stack from the top
// (right to left).  Every addition has the same operands in the same order,
// so the result is bit-identical for any K, with a stack of log2(K)+1 slots
// instead of K registers.
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kMeanThreads) k_weighted_mean(const __grid_constant__ MeanParams p) {
  __shared__ double cf[kCoefSmem];
  const int b = p.b0 + blockIdx.y;
  const int64_t K = p.K;
  for (int k = threadIdx.x; k < K && k < kCoefSmem; k += kMeanThreads) cf[k] = p.coef[(int64_t)k * p.B_total + b];
  __syncthreads();
  const int64_t lo = p.bounds[blockIdx.y], hi = p.bounds[blockIdx.y + 1];
  const Tin* g = static_cast<const Tin*>(p.G);
  Tout* out = static_cast<Tout*>(p.out);
  for (int64_t i = lo + (int64_t)blockIdx.x * kMeanThreads + threadIdx.x; i < hi;
       i += (int64_t)gridDim.x * kMeanThreads) {
    double st[64];
    int64_t sz[64];
    int top = 0;
    for (int64_t k = 0; k < K; ++k) {
      const double c = k < kCoefSmem ? cf[k] : __ldg(&p.coef[k * p.B_total + b]);
      double v = static_cast<double>(g[k * p.ld + i]) * c;
      int64_t n = 1;
      while (top > 0 && sz[top - 1] == n) {  // equal blocks: one tree merge
        v = st[--top] + v;
        n <<= 1;
      }
      st[top] = v;
      sz[top++] = n;
    }
    double v = st[--top];
    while (top > 0) v = st[--top] + v;  // odd tails, folded right to left
    out[i] = static_cast<Tout>(v / (double)K);  // mean, not sum (:128)
  }
}

}  // namespace
}  // namespace b2

using namespace b2;
using namespace b2::clip;

extern "C" size_t b2_clip_workspace_bytes(void) { return WsLayout::bytes; }

extern "C" int b2_clip_workspace_init(void* ws, size_t bytes, void* stream) {
  B2_REQUIRE(ws != nullptr && bytes >= WsLayout::bytes, B2_ERR_INVALID,
             "clip workspace needs %zu bytes", (size_t)WsLayout::bytes);
  B2_CHECK(cudaMemsetAsync(ws, 0, WsLayout::bytes, (cudaStream_t)stream));
  return B2_OK;
}

extern "C" int b2_bucket_clip_cast(const void* in, int in_dtype, void* out, int out_dtype,
                                   const int64_t* seg_in_off, const int64_t* seg_out_off,
                                   const int64_t* seg_len, int nseg, double limit,
                                   double post_scale, double* norms, double* coefs,
                                   int32_t* nonfinite, void* workspace, size_t workspace_bytes,
                                   int ctas_per_sm, void* stream) {
  B2_REQUIRE(in != nullptr, B2_ERR_INVALID, "input pointer is NULL");
  B2_REQUIRE(nseg >= 0, B2_ERR_INVALID, "nseg must be >= 0");
  B2_REQUIRE(nseg == 0 || (seg_in_off && seg_len && (out == nullptr || seg_out_off)), B2_ERR_INVALID,
             "segment arrays are NULL");
  B2_REQUIRE(limit > 0.0, B2_ERR_INVALID, "limit must be > 0, got %g", limit);
  B2_REQUIRE(workspace != nullptr && workspace_bytes >= WsLayout::bytes, B2_ERR_INVALID,
             "clip workspace needs %zu bytes", (size_t)WsLayout::bytes);
  B2_REQUIRE(in_dtype == B2_F32 || in_dtype == B2_F64, B2_ERR_INVALID, "in_dtype must be F32 or F64");
  B2_REQUIRE(out == nullptr || out_dtype == B2_F32 || out_dtype == B2_BF16 || out_dtype == B2_F64,
             B2_ERR_INVALID, "bad out_dtype %d", out_dtype);
  B2_REQUIRE(!(in_dtype == B2_F64 && out != nullptr && out_dtype != B2_F64), B2_ERR_INVALID,
             "f64 input supports f64 output only");
  if (nseg == 0) return B2_OK;
  for (int s0 = 0; s0 < nseg; s0 += kMaxSegs) {
    ClipParams p;
    int rc = fill_params(p, in, in_dtype, out, out_dtype, seg_in_off, seg_out_off, seg_len, s0, nseg, limit,
                         post_scale, norms, coefs, nonfinite, workspace);
    if (rc != B2_OK) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (in_dtype == B2_F64) rc = launch_clip_k1<double, double>(p, st);
    else if (out == nullptr || out_dtype == B2_F32) rc = launch_clip_k1<float, float>(p, st);
    else if (out_dtype == B2_BF16) rc = launch_clip_k1<float, __nv_bfloat16>(p, st);
    else rc = launch_clip_k1<float, double>(p, st);
    if (rc != B2_OK) return rc;
  }
  return B2_OK;
}

extern "C" int b2_weighted_mean(const void* G, int in_dtype, int64_t K, int64_t D, int64_t ld,
                                const double* coef, const int64_t* bounds, int B, void* out,
                                int out_dtype, void* stream) {
  B2_REQUIRE(G && coef && bounds && out, B2_ERR_INVALID, "NULL pointer argument");
  B2_REQUIRE(K >= 1, B2_ERR_INVALID, "K must be >= 1, got %lld", (long long)K);
  B2_REQUIRE(B >= 1 && D >= 1 && ld >= D, B2_ERR_INVALID, "bad shape");
  B2_REQUIRE(bounds[0] == 0 && bounds[B] == D, B2_ERR_INVALID, "bounds must cover [0, D)");
  B2_REQUIRE(in_dtype == B2_F32 || in_dtype == B2_F64, B2_ERR_INVALID, "bad in_dtype");
  B2_REQUIRE(out_dtype == B2_F32 || out_dtype == B2_F64, B2_ERR_INVALID, "bad out_dtype");
  cudaStream_t st = (cudaStream_t)stream;
  for (int b0 = 0; b0 < B; b0 += kMaxSegs) {
    MeanParams p{};
    p.G = G;
    p.out = out;
    p.coef = coef;
    p.K = K;
    p.ld = ld;
    p.B_total = B;
    p.b0 = b0;
    p.nb = std::min(kMaxSegs, B - b0);
    int64_t maxlen = 0;
    for (int i = 0; i <= p.nb; ++i) p.bounds[i] = bounds[b0 + i];
    for (int i = 0; i < p.nb; ++i) {
      B2_REQUIRE(p.bounds[i + 1] > p.bounds[i], B2_ERR_INVALID, "bounds must be increasing");
      maxlen = std::max(maxlen, p.bounds[i + 1] - p.bounds[i]);
    }
    const int gx = (int)std::min<int64_t>((maxlen + kMeanThreads - 1) / kMeanThreads, 4096);
    dim3 grid(gx, p.nb);
    if (in_dtype == B2_F64 && out_dtype == B2_F64) k_weighted_mean<double, double><<<grid, kMeanThreads, 0, st>>>(p);
    else if (in_dtype == B2_F64) k_weighted_mean<double, float><<<grid, kMeanThreads, 0, st>>>(p);
    else if (out_dtype == B2_F64) k_weighted_mean<float, double><<<grid, kMeanThreads, 0, st>>>(p);
    else k_weighted_mean<float, float><<<grid, kMeanThreads, 0, st>>>(p);
    B2_CHECK(cudaGetLastError());
  }
  return B2_OK;
}
