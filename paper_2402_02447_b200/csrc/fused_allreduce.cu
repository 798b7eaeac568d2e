// H1 fused across ranks: bucket-wise clip + allreduce in ONE persistent kernel
// per GPU, the transfer running over NVLink peer memory (no NCCL).
//
// Reference semantics: sync_bucketwise (gradsync.py:148-162) with rank r as
// worker row r — each worker's bucket is clipped at c/sqrt(B) (:155, local,
// no norm collective), then averaged over workers (allreduce_mean, :119-128).
//
// Every rank owns a symmetric bf16 stage buffer (the comm buffer) mapped into
// every peer (CUDA IPC).  Three warp groups per CTA, 2 CTAs per SM:
//   A (256 thr): norm pass of bucket s (128-bit loads, L2 evict_last), one
//                fp64 partial per (bucket, CTA), fire-and-forget;
//   B (128 thr): bucket s-1: fixed-order fold -> coefficient, L2 re-read,
//                scale, cast, store into the LOCAL stage; the last CTA to
//                finish raises ready[rank][s] in every peer's flag area;
//   C (128 thr): two-shot allreduce of bucket s: once every rank's bucket s is
//                staged, this rank reduces its 1/N slice — 16 B loads from all
//                N stages (peer loads go over NVLink), fp32 sum in rank order,
//                x 1/N, bf16 — and stores the result into all N stages; after
//                the last bucket one system-scope release per CTA, and the
//                last CTA raises done[rank] everywhere.
// The launch ends when this rank has seen every done flag, so the local stage
// then holds the averaged clipped gradient.  Per-rank NVLink traffic per
// bucket is (N-1)/N of it in and out — the ring's volume without its
// 2(N-1) latency steps.  Flags carry a per-launch epoch (no resets); every
// cross-GPU wait is bounded (trap after 30 s instead of a hang).
#include "clip_common.cuh"

#include <cuda_bf16.h>

#include <cstdlib>
#include <cstring>

namespace b2 {
namespace {
using namespace clip;

constexpr int kMaxRanks = 8;
constexpr int kBarA = 1, kBarB = 2, kBarC = 3;
constexpr uint64_t kSpinTimeoutNs = 30ull * 1000 * 1000 * 1000;

struct FusedParams {
  ClipParams p;                        // in/out/limit/segments; p.out = local stage
  __nv_bfloat16* stage[kMaxRanks];     // every rank's stage (index = rank)
  uint32_t* flags[kMaxRanks];          // every rank's flag area [2][kMaxRanks][kMaxSegs]
  unsigned* pcount;                    // local arrival counters [2][kMaxSegs]
  unsigned* epoch;                     // launches so far (device; this launch is *epoch + 1)
  __nv_bfloat16* mc;                   // NVLS: multicast address of the stage buffers (or null)
  int nranks, rank;
  float inv_n;
};

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// wait until *p has reached `epoch` (wrap-safe), bounded
__device__ __forceinline__ void wait_epoch(const uint32_t* p, uint32_t epoch) {
  const uint64_t t0 = global_ns();
  unsigned ns = 32;
  while ((int32_t)(ld_acquire_sys(p) - epoch) < 0) {
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
    if (global_ns() - t0 > kSpinTimeoutNs) __trap();  // a peer never arrived: fail, do not hang
  }
}
// timeline stamps (ns) in the unused partial rows kMaxSegs-1-k of the
// workspace, read back by tools/k4_timeline.py (only when nseg leaves them free)
__device__ __forceinline__ void stamp(const ClipParams& p, int k) {
  if (p.nseg <= kMaxSegs - 8) reinterpret_cast<uint64_t*>(p.partials)[(size_t)(kMaxSegs - 1 - k) * kMaxGrid + blockIdx.x] = global_ns();
}
__device__ __forceinline__ uint32_t* flag(const FusedParams& f, int owner, int kind, int src, int s) {
  return f.flags[owner] + ((size_t)kind * kMaxRanks + src) * kMaxSegs + s;
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& v, float (&x)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    x[2 * i] = f.x;
    x[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ uint4 f32_to_bf16x8(const float (&x)[8]) {
  uint4 v;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(x[2 * i], x[2 * i + 1]);
  return v;
}

__device__ __forceinline__ uint32_t ld_acquire_cta_shared(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_shared(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}

template <int kAT, int kBT, int kCT, int UA, int UB, int UC, int RMAX, int CV, bool MC, bool FLAT, int THR>
__global__ void __launch_bounds__(kAT + kBT + kCT, 2) k_clip_allreduce_p2p(const __grid_constant__ FusedParams f) {
  using V = float4;
  constexpr int N = 4;
  const ClipParams& p = f.p;
  __shared__ double redA[32], redB[32];
  __shared__ double s_coef;
  __shared__ volatile int s_bdone;
  __shared__ volatile int s_cprog;  // FLAT: the bucket (local index) C is working on
  __shared__ uint32_t s_epoch;
  // CTA groups (p.ngroups): this CTA serves buckets gid, gid+R, ... as member c of G CTAs
  const int R = p.ngroups, gid = blockIdx.x % R;
  const int G = group_size(gridDim.x, R, gid), c = blockIdx.x / R, t = threadIdx.x;
  if (t == 0) {
    s_bdone = 0;
    s_cprog = 0;
    s_epoch = *f.epoch + 1u;  // read from device memory: CUDA-graph replays advance it too
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;
  if (t == 0) stamp(p, 0);

  if (t < kAT) {
    // ================= A: norm pass (bucket s), at most 2 buckets ahead of B
    const int gt = t;
    const uint64_t pol_keep = l2_policy_evict_last();
    for (int i = 0, s = gid; s < p.nseg; ++i, s += R) {
      if (i > 1) {
        if (gt == 0) {
          unsigned ns = 32;
          while (s_bdone < i - 1) {
            __nanosleep(ns);
            if (ns < 256) ns <<= 1;
          }
        }
        group_sync<kAT>(kBarA);
      }
      const Seg sg = p.seg[s];
      const float* in = static_cast<const float*>(p.in) + sg.in_off;
      double acc = 0.0;
      const V* vin = reinterpret_cast<const V*>(in + sg.head);
      const int64_t v0 = min64((int64_t)c * sg.per, sg.nv), v1 = min64(v0 + sg.per, sg.nv);
      for (int64_t v = v0 + gt; v < v1; v += (int64_t)kAT * UA) {
        V x[UA];
#pragma unroll
        for (int u = 0; u < UA; ++u) {
          const int64_t vi = v + (int64_t)u * kAT;
          x[u] = vi < v1 ? ld_a<0>(vin + vi, pol_keep) : V{};
        }
        // fp32 mini-sum of <= 4*UA squares promoted to fp64; out-of-range -> exact fp64
        float m = 0.0f;
        unsigned nz = 0;
#pragma unroll
        for (int u = 0; u < UA; ++u) {
          m = fmaf(x[u].x, x[u].x, m);
          m = fmaf(x[u].y, x[u].y, m);
          m = fmaf(x[u].z, x[u].z, m);
          m = fmaf(x[u].w, x[u].w, m);
          nz |= __float_as_uint(x[u].x) | __float_as_uint(x[u].y) | __float_as_uint(x[u].z) | __float_as_uint(x[u].w);
        }
        if (m >= 0x1p-100f && m <= 0x1p100f) {
          acc += (double)m;
        } else if ((nz << 1) != 0u) {
#pragma unroll
          for (int u = 0; u < UA; ++u)
            acc += (double)x[u].x * x[u].x + (double)x[u].y * x[u].y + (double)x[u].z * x[u].z +
                   (double)x[u].w * x[u].w;
        }
      }
      const int64_t tail0 = sg.head + sg.nv * N;
      if (c == 0 && gt < sg.head) acc += (double)in[gt] * in[gt];
      if (c == G - 1 && gt < sg.n - tail0) acc += (double)in[tail0 + gt] * in[tail0 + gt];
      const double tot = group_sum<kAT>(acc, redA, gt, kBarA);
      if (gt == 0) {
        p.partials[(size_t)s * kMaxGrid + c] = tot;
        red_release_u32(&p.counters[s], 1u);
      }
    }
  } else if (t < kAT + kBT) {
    // ================= B: coefficient + scale + cast into the local stage
    const int gt = t - kAT;
    const uint64_t pol_drop = l2_policy_evict_first();
    __nv_bfloat16* stage = f.stage[f.rank];
    for (int i = 0, s = gid; s < p.nseg; ++i, s += R) {
      if (gt == 0) {
        unsigned ns = 32;
        if constexpr (FLAT && THR > 0) {
          // the clip only has to stay ahead of the NVLink-bound reduce: running
          // further ahead just competes with it for HBM and issue slots
          while (i > s_cprog + THR) {
            __nanosleep(ns);
            if (ns < 256) ns <<= 1;
          }
          ns = 32;
        }
        while (ld_acquire_u32(&p.counters[s]) < (unsigned)G) {
          __nanosleep(ns);
          if (ns < 256) ns <<= 1;
        }
      }
      group_sync<kBT>(kBarB);
      double v = 0.0;
      for (int j = gt; j < G; j += kBT) v += __ldcg(&p.partials[(size_t)s * kMaxGrid + j]);
      const double total = group_sum<kBT>(v, redB, gt, kBarB);
      if (gt == 0) {
        const double norm = sqrt(total);
        const double coef = (norm >= p.limit) ? p.limit / norm : 1.0;  // gradsync.py:114-116
        if (c == 0) {
          if (p.norms) p.norms[s] = norm;
          if (p.nonfinite) p.nonfinite[s] = !isfinite(total) ? 1 : 0;
        }
        s_coef = coef;
      }
      group_sync<kBT>(kBarB);
      // NVLS stages clip * 1/N: the in-switch sum of the stages is then the mean
      const float cf = MC ? (float)(s_coef * (double)f.inv_n) : (float)s_coef;
      const Seg sg = p.seg[s];
      const float* in = static_cast<const float*>(p.in) + sg.in_off;
      __nv_bfloat16* out = stage + sg.out_off;
      const V* vin = reinterpret_cast<const V*>(in + sg.head);
      const int64_t v0 = min64((int64_t)c * sg.per, sg.nv), v1 = min64(v0 + sg.per, sg.nv);
      for (int64_t v = v0 + gt; v < v1; v += (int64_t)kBT * UB) {
        V x[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int64_t vi = v + (int64_t)u * kBT;
          if (vi < v1) x[u] = ld_b<0>(vin + vi, pol_drop);
        }
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int64_t vi = v + (int64_t)u * kBT;
          if (vi < v1) {
            float y[4] = {x[u].x * cf, x[u].y * cf, x[u].z * cf, x[u].w * cf};
            put_vec<__nv_bfloat16, 4, float>(out + sg.head + vi * N, y);
          }
        }
      }
      const int64_t tail0 = sg.head + sg.nv * N;
      if (c == 0 && gt < sg.head) out[gt] = __float2bfloat16_rn(in[gt] * cf);
      if (c == G - 1 && gt < sg.n - tail0) out[tail0 + gt] = __float2bfloat16_rn(in[tail0 + gt] * cf);
      group_sync<kBT>(kBarB);
      if (gt == 0) {
        // local stage writes -> gpu-scope release; the last CTA's system-scope
        // release to the peers is cumulative over the whole chain
        __threadfence();
        if (atomicAdd(&f.pcount[s], 1u) == (unsigned)G - 1) {
          __threadfence_system();
          for (int q = 0; q < f.nranks; ++q) st_release_sys(flag(f, q, 0, f.rank, s), epoch);
        }
        s_bdone = i + 1;
      }
    }
    if (gt == 0) stamp(p, 1);
  } else if constexpr (FLAT) {
    // ================= C (flat): this CTA's slices of all its buckets as ONE
    // stream — no per-bucket barrier or ragged tail; a bucket's ready flags
    // are acquired by the first thread that reaches it and cached in smem
    const int gt = t - kAT - kBT;
    const int NR = f.nranks;
    __shared__ int64_t s_beg[kMaxSegs + 1], s_voff[kMaxSegs];
    __shared__ uint32_t s_rdy[kMaxSegs];
    __shared__ int s_sid[kMaxSegs];
    int nb = 0;
    for (int s = gid; s < p.nseg; s += R) ++nb;
    if (gt == 0) {
      int64_t acc = 0;
      for (int i = 0; i < nb; ++i) {
        const int s = gid + i * R;
        const Seg sg = p.seg[s];
        const int64_t nv8 = sg.n / 8;
        const int64_t per_r = (nv8 + NR - 1) / NR;
        const int64_t r0 = min64((int64_t)f.rank * per_r, nv8), r1 = min64(r0 + per_r, nv8);
        const int64_t per_c = (r1 - r0 + G - 1) / G;
        const int64_t c0 = min64(r0 + (int64_t)c * per_c, r1), c1 = min64(c0 + per_c, r1);
        s_beg[i] = acc;
        s_voff[i] = sg.out_off / 8 + c0 - acc;  // stage vector index = flat index + s_voff
        s_sid[i] = s;
        s_rdy[i] = 0u;
        acc += c1 - c0;
      }
      s_beg[nb] = acc;
    }
    group_sync<kCT>(kBarC);
    const int64_t M = s_beg[nb];
    int cur = 0;
    for (int64_t f0 = gt; f0 < M; f0 += (int64_t)kCT * UC) {
      uint4 x[UC][RMAX];
      int64_t vix[UC];
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        const int64_t fi = f0 + (int64_t)u * kCT;
        vix[u] = -1;
        if (fi < M) {
          while (fi >= s_beg[cur + 1]) {
            ++cur;
            if (THR > 0 && gt == 0) s_cprog = cur;
          }
          if (ld_acquire_cta_shared(&s_rdy[cur]) == 0u) {
            for (int q = 0; q < NR; ++q) wait_epoch(flag(f, f.rank, 0, q, s_sid[cur]), epoch);
            st_release_cta_shared(&s_rdy[cur], 1u);
            if (cur == 0 && gt == 0) stamp(p, 2);
          }
          vix[u] = fi + s_voff[cur];
          if constexpr (MC) {
            // NVSwitch sums the N stages (fp32 accumulate; the stages hold clip/N)
            asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                         : "=r"(x[u][0].x), "=r"(x[u][0].y), "=r"(x[u][0].z), "=r"(x[u][0].w)
                         : "l"(reinterpret_cast<const uint4*>(f.mc) + vix[u])
                         : "memory");
          } else {
#pragma unroll
            for (int q = 0; q < RMAX; ++q)
              if (q < NR) {
                const uint4* src = reinterpret_cast<const uint4*>(f.stage[q]) + vix[u];
                x[u][q] = CV ? __ldcv(src) : __ldcg(src);
              }
          }
        }
      }
      if constexpr (MC) {
#pragma unroll
        for (int u = 0; u < UC; ++u)
          if (vix[u] >= 0)  // one store, multicast to every rank's stage
            asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(
                             reinterpret_cast<uint4*>(f.mc) + vix[u]),
                         "f"(__uint_as_float(x[u][0].x)), "f"(__uint_as_float(x[u][0].y)),
                         "f"(__uint_as_float(x[u][0].z)), "f"(__uint_as_float(x[u][0].w))
                         : "memory");
      } else {
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        if (vix[u] >= 0) {
          float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int q = 0; q < RMAX; ++q) {
            if (q < NR) {  // fixed rank order: identical bits on every rank
              float e[8];
              bf16x8_to_f32(x[u][q], e);
#pragma unroll
              for (int i = 0; i < 8; ++i) acc[i] += e[i];
            }
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] *= f.inv_n;  // mean, not sum (gradsync.py:128)
          const uint4 y = f32_to_bf16x8(acc);
#pragma unroll
          for (int q = 0; q < RMAX; ++q)
            if (q < NR) __stcg(reinterpret_cast<uint4*>(f.stage[q]) + vix[u], y);
        }
      }
      }  // P2P
    }
    if (THR > 0 && gt == 0) s_cprog = nb;
    group_sync<kCT>(kBarC);
    if (gt == 0) stamp(p, 3);
    if (gt == 0) {
      __threadfence_system();
      if (atomicAdd(&f.pcount[kMaxSegs], 1u) == gridDim.x - 1) {
        __threadfence_system();
        for (int q = 0; q < NR; ++q) st_release_sys(flag(f, q, 1, f.rank, 0), epoch);
      }
      if (blockIdx.x == 0)
        for (int q = 0; q < NR; ++q) wait_epoch(flag(f, f.rank, 1, q, 0), epoch);
    }
  } else {
    // ================= C: two-shot allreduce of bucket s over NVLink
    const int gt = t - kAT - kBT;
    const int NR = f.nranks;
    for (int s = gid; s < p.nseg; s += R) {
      if (gt == 0)
        for (int q = 0; q < NR; ++q) wait_epoch(flag(f, f.rank, 0, q, s), epoch);
      group_sync<kCT>(kBarC);
      const Seg sg = p.seg[s];
      const int64_t nv8 = sg.n / 8;                   // 16 B = 8 bf16 (host guarantees n % 8 == 0)
      const int64_t per_r = (nv8 + NR - 1) / NR;
      const int64_t r0 = min64((int64_t)f.rank * per_r, nv8), r1 = min64(r0 + per_r, nv8);
      const int64_t per_c = (r1 - r0 + G - 1) / G;
      const int64_t c0 = min64(r0 + (int64_t)c * per_c, r1), c1 = min64(c0 + per_c, r1);
      if constexpr (MC) {
        // NVSwitch reduction: one multimem load-reduce (fp32 accumulate) and one
        // multimem store (broadcast to every rank) per 16 B
        const char* mcb = reinterpret_cast<const char*>(f.mc + sg.out_off);
        for (int64_t v = c0 + gt; v < c1; v += (int64_t)kCT * UC) {
          uint32_t r[UC][4];
#pragma unroll
          for (int u = 0; u < UC; ++u) {
            const int64_t vi = v + (int64_t)u * kCT;
            if (vi < c1)
              asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                           : "=r"(r[u][0]), "=r"(r[u][1]), "=r"(r[u][2]), "=r"(r[u][3])
                           : "l"(mcb + vi * 16)
                           : "memory");
          }
#pragma unroll
          for (int u = 0; u < UC; ++u) {
            const int64_t vi = v + (int64_t)u * kCT;
            if (vi < c1)
              asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mcb + vi * 16),
                           "f"(__uint_as_float(r[u][0])), "f"(__uint_as_float(r[u][1])),
                           "f"(__uint_as_float(r[u][2])), "f"(__uint_as_float(r[u][3]))
                           : "memory");
          }
        }
      } else {
      for (int64_t v = c0 + gt; v < c1; v += (int64_t)kCT * UC) {
        uint4 x[UC][RMAX];
#pragma unroll
        for (int u = 0; u < UC; ++u) {
          const int64_t vi = v + (int64_t)u * kCT;
          if (vi < c1) {
#pragma unroll
            for (int q = 0; q < RMAX; ++q)
              if (q < NR) {
                const uint4* src = reinterpret_cast<const uint4*>(f.stage[q] + sg.out_off) + vi;
                x[u][q] = CV ? __ldcv(src) : __ldcg(src);
              }
          }
        }
#pragma unroll
        for (int u = 0; u < UC; ++u) {
          const int64_t vi = v + (int64_t)u * kCT;
          if (vi < c1) {
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int q = 0; q < RMAX; ++q) {
              if (q < NR) {  // fixed rank order: identical bits on every rank
                float e[8];
                bf16x8_to_f32(x[u][q], e);
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i] += e[i];
              }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] *= f.inv_n;  // mean, not sum (gradsync.py:128)
            const uint4 y = f32_to_bf16x8(acc);
#pragma unroll
            for (int q = 0; q < RMAX; ++q)
              if (q < NR) __stcg(reinterpret_cast<uint4*>(f.stage[q] + sg.out_off) + vi, y);
          }
        }
      }
      }  // P2P two-shot
    }
    // one system-scope release per CTA for all of its remote stores, one
    // done flag per rank; the launch completes only once every rank's slices
    // of every bucket have landed here
    group_sync<kCT>(kBarC);
    if (gt == 0) {
      __threadfence_system();
      if (atomicAdd(&f.pcount[kMaxSegs], 1u) == gridDim.x - 1) {
        __threadfence_system();
        for (int q = 0; q < NR; ++q) st_release_sys(flag(f, q, 1, f.rank, 0), epoch);
      }
      if (blockIdx.x == 0)
        for (int q = 0; q < NR; ++q) wait_epoch(flag(f, f.rank, 1, q, 0), epoch);
    }
  }

  __syncthreads();
  if (t == 0) {
    stamp(p, 4);
    if (atom_add_acq_rel_u32(&p.counters[kMaxSegs], 1u) == gridDim.x - 1) {
      for (int s = 0; s < p.nseg; ++s) {
        p.counters[s] = 0u;
        f.pcount[s] = 0u;
      }
      f.pcount[kMaxSegs] = 0u;
      p.counters[kMaxSegs] = 0u;
      *f.epoch = epoch;  // every CTA read it at entry; the next launch sees epoch + 1
      __threadfence();
    }
  }
}

template <int AT, int BT, int CT, int UA, int UB, int UC, int RMAX, int CV, bool MC = false, bool FLAT = false,
          int THR = 0>
int launch_p2p(FusedParams& f, cudaStream_t stream) {
  constexpr int kAT = AT, kBT = BT, kCT = CT;
  auto kern = k_clip_allreduce_p2p<AT, BT, CT, UA, UB, UC, RMAX, CV, MC, FLAT, THR>;
  const DeviceInfo& di = device_info();
  B2_REQUIRE(di.coop, B2_ERR_CUDA, "device does not support cooperative launch");
  static int occ_cached[64] = {};
  int& occ = occ_cached[di.device & 63];
  if (occ == 0) {
    B2_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kAT + kBT + kCT, 0));
    B2_REQUIRE(occ >= 1, B2_ERR_CUDA, "fused kernel cannot be resident");
  }
  const int grid = std::min(di.sm_count * std::min(2, occ), kMaxGrid);
  f.p.ngroups = choose_groups(f.p, grid, sizeof(float));
  for (int s = 0; s < f.p.nseg; ++s) {
    Seg& sg = f.p.seg[s];
    const int gs = group_size(grid, f.p.ngroups, s % f.p.ngroups);
    sg.nv = (sg.n - sg.head) / 4;
    sg.per = (sg.nv + gs - 1) / gs;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kAT + kBT + kCT);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // CTAs wait on each other's partials
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  B2_CHECK(cudaLaunchKernelEx(&cfg, kern, f));
  return B2_OK;
}

typedef int (*PMemGetAddressRange)(unsigned long long*, size_t*, unsigned long long);

}  // namespace
}  // namespace b2

using namespace b2;
using namespace b2::clip;

extern "C" size_t b2_p2p_flag_bytes(void) { return sizeof(uint32_t) * 2 * kMaxRanks * kMaxSegs; }

extern "C" int b2_ipc_export(const void* ptr, void* handle64, int64_t* offset) {
  B2_REQUIRE(ptr && handle64 && offset, B2_ERR_INVALID, "NULL argument");
  // the IPC handle names the whole allocation: find its base (driver entry point, no -lcuda)
  static PMemGetAddressRange get_range = nullptr;
  if (!get_range) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    B2_CHECK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
    B2_REQUIRE(fn && q == cudaDriverEntryPointSuccess, B2_ERR_CUDA, "cuMemGetAddressRange unavailable");
    get_range = (PMemGetAddressRange)fn;
  }
  unsigned long long base = 0;
  size_t size = 0;
  B2_REQUIRE(get_range(&base, &size, (unsigned long long)ptr) == 0, B2_ERR_CUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  B2_CHECK(cudaIpcGetMemHandle(&h, (void*)base));
  memcpy(handle64, &h, sizeof(h));
  *offset = (int64_t)((unsigned long long)ptr - base);
  return B2_OK;
}

extern "C" int b2_ipc_import(const void* handle64, int64_t offset, void** base, void** ptr) {
  B2_REQUIRE(handle64 && base && ptr, B2_ERR_INVALID, "NULL argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  B2_CHECK(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
  *ptr = static_cast<char*>(*base) + offset;
  return B2_OK;
}

extern "C" int b2_ipc_close(void* base) {
  B2_CHECK(cudaIpcCloseMemHandle(base));
  return B2_OK;
}

static int clip_allreduce_impl(const void* in, void* const* stages, void* mc_stage, uint32_t* const* flags,
                               int nranks, int rank, const int64_t* seg_off, const int64_t* seg_len, int nseg,
                               double limit, double* norms, int32_t* nonfinite, void* workspace,
                               size_t workspace_bytes, void* stream);

extern "C" int b2_bucket_clip_allreduce_nvls(const void* in, void* const* stages, void* mc_stage,
                                             uint32_t* const* flags, int nranks, int rank, const int64_t* seg_off,
                                             const int64_t* seg_len, int nseg, double limit, double* norms,
                                             int32_t* nonfinite, void* workspace, size_t workspace_bytes,
                                             void* stream) {
  B2_REQUIRE(mc_stage != nullptr && reinterpret_cast<uintptr_t>(mc_stage) % 16 == 0, B2_ERR_INVALID,
             "NVLS needs a 16 B aligned multicast address");
  return clip_allreduce_impl(in, stages, mc_stage, flags, nranks, rank, seg_off, seg_len, nseg, limit, norms,
                             nonfinite, workspace, workspace_bytes, stream);
}

extern "C" int b2_bucket_clip_allreduce_p2p(const void* in, void* const* stages, uint32_t* const* flags, int nranks,
                                            int rank, const int64_t* seg_off, const int64_t* seg_len, int nseg,
                                            double limit, double* norms, int32_t* nonfinite, void* workspace,
                                            size_t workspace_bytes, void* stream) {
  return clip_allreduce_impl(in, stages, nullptr, flags, nranks, rank, seg_off, seg_len, nseg, limit, norms,
                             nonfinite, workspace, workspace_bytes, stream);
}

static int clip_allreduce_impl(const void* in, void* const* stages, void* mc_stage, uint32_t* const* flags,
                               int nranks, int rank, const int64_t* seg_off, const int64_t* seg_len, int nseg,
                               double limit, double* norms, int32_t* nonfinite, void* workspace,
                               size_t workspace_bytes, void* stream) {
  B2_REQUIRE(in && stages && flags && seg_off && seg_len, B2_ERR_INVALID, "NULL argument");
  B2_REQUIRE(nranks >= 1 && nranks <= kMaxRanks && rank >= 0 && rank < nranks, B2_ERR_UNSUPPORTED,
             "nranks must be in [1, %d]", kMaxRanks);
  B2_REQUIRE(nseg >= 1 && nseg <= kMaxSegs, B2_ERR_UNSUPPORTED, "nseg must be in [1, %d]", kMaxSegs);
  B2_REQUIRE(limit > 0.0, B2_ERR_INVALID, "limit must be > 0, got %g", limit);
  B2_REQUIRE(workspace && workspace_bytes >= WsLayout::bytes, B2_ERR_INVALID, "clip workspace needs %zu bytes",
             (size_t)WsLayout::bytes);
  for (int s = 0; s < nseg; ++s)
    B2_REQUIRE(seg_off[s] % 8 == 0 && seg_len[s] % 8 == 0, B2_ERR_UNSUPPORTED,
               "fused allreduce needs 8-element aligned buckets (bucket %d)", s);
  for (int q = 0; q < nranks; ++q)
    B2_REQUIRE(reinterpret_cast<uintptr_t>(stages[q]) % 16 == 0, B2_ERR_INVALID, "stage %d not 16 B aligned", q);
  FusedParams f{};
  int rc = fill_params(f.p, in, B2_F32, stages[rank], B2_BF16, seg_off, seg_off, seg_len, 0, nseg, limit, 1.0, norms,
                       nullptr, nonfinite, workspace);
  if (rc != B2_OK) return rc;
  for (int s = 0; s < nseg; ++s)
    B2_REQUIRE(f.p.seg[s].vec, B2_ERR_UNSUPPORTED, "fused allreduce needs 16 B aligned gradients");
  for (int q = 0; q < nranks; ++q) {
    f.stage[q] = static_cast<__nv_bfloat16*>(stages[q]);
    f.flags[q] = flags[q];
  }
  f.pcount = reinterpret_cast<unsigned*>(static_cast<char*>(workspace) + WsLayout::pcounters);
  f.epoch = reinterpret_cast<unsigned*>(static_cast<char*>(workspace) + WsLayout::epoch);
  f.nranks = nranks;
  f.rank = rank;
  f.inv_n = 1.0f / (float)nranks;
  f.mc = static_cast<__nv_bfloat16*>(mc_stage);

  // the reduce group keeps UC x RMAX 16 B vectors in flight: 32 registers
  cudaStream_t st = (cudaStream_t)stream;
  static int cfg = -1;  // tuning knob: B2_FUSED_CFG selects the warp-group split (A/B/C threads)
  if (cfg < 0) {
    const char* e = getenv("B2_FUSED_CFG");
    cfg = e ? atoi(e) : 0;
  }
  if (mc_stage) {  // RMAX 1: one multimem load per vector
    switch (cfg) {
      case 1: return launch_p2p<256, 128, 128, 8, 4, 4, 1, 1, true>(f, st);
      case 2: return launch_p2p<128, 256, 128, 8, 4, 8, 1, 1, true, true>(f, st);
      case 3: return launch_p2p<128, 256, 128, 8, 4, 16, 1, 1, true, true>(f, st);
      default: return launch_p2p<128, 256, 128, 8, 4, 8, 1, 1, true, true>(f, st);
    }
  }
  if (nranks <= 2) {
    switch (cfg) {
      case 1: return launch_p2p<128, 128, 256, 8, 4, 4, 2, 1>(f, st);
      case 2: return launch_p2p<256, 128, 128, 8, 4, 4, 2, 0>(f, st);
      case 5: return launch_p2p<192, 192, 128, 8, 4, 4, 2, 1>(f, st);
      case 6: return launch_p2p<160, 224, 128, 8, 4, 4, 2, 1>(f, st);
      case 7: return launch_p2p<192, 160, 160, 8, 4, 4, 2, 1>(f, st);
      case 10: return launch_p2p<256, 128, 128, 8, 4, 4, 2, 1, false, true>(f, st);
      case 11: return launch_p2p<256, 128, 128, 8, 4, 8, 2, 1, false, true>(f, st);
      case 12: return launch_p2p<256, 128, 128, 8, 4, 4, 2, 0, false, true>(f, st);
      case 13: return launch_p2p<192, 160, 160, 8, 4, 4, 2, 1, false, true>(f, st);
      case 18: return launch_p2p<192, 192, 128, 8, 4, 8, 2, 1, false, true>(f, st);
      case 19: return launch_p2p<128, 256, 128, 8, 4, 8, 2, 1, false, true>(f, st);
      case 20: return launch_p2p<256, 128, 128, 8, 8, 8, 2, 1, false, true>(f, st);
      case 21: return launch_p2p<192, 192, 128, 8, 8, 8, 2, 1, false, true>(f, st);
      case 22: return launch_p2p<160, 224, 128, 8, 4, 8, 2, 1, false, true>(f, st);
      case 9: return launch_p2p<256, 128, 128, 8, 4, 4, 2, 1>(f, st);  // per-bucket C (round-1 v1)
      default: return launch_p2p<128, 256, 128, 8, 4, 8, 2, 1, false, true>(f, st);
    }
  }
  if (nranks <= 4) {
    switch (cfg) {
      case 5: return launch_p2p<192, 192, 128, 8, 4, 2, 4, 1>(f, st);
      case 6: return launch_p2p<160, 224, 128, 8, 4, 2, 4, 1>(f, st);
      case 7: return launch_p2p<192, 160, 160, 8, 4, 2, 4, 1>(f, st);
      case 10: return launch_p2p<256, 128, 128, 8, 4, 2, 4, 1, false, true>(f, st);
      case 11: return launch_p2p<256, 128, 128, 8, 4, 4, 4, 1, false, true>(f, st);
      case 12: return launch_p2p<128, 256, 128, 8, 4, 4, 4, 1, false, true>(f, st);
      case 13: return launch_p2p<192, 192, 128, 8, 4, 4, 4, 1, false, true>(f, st);
      case 14: return launch_p2p<128, 256, 128, 8, 4, 2, 4, 1, false, true>(f, st);
      case 9: return launch_p2p<256, 128, 128, 8, 4, 2, 4, 1>(f, st);  // per-bucket C (round-1 v1)
      default: return launch_p2p<128, 256, 128, 8, 4, 4, 4, 1, false, true>(f, st);
    }
  }
  return launch_p2p<128, 256, 128, 8, 4, 2, 8, 1, false, true>(f, st);
}
