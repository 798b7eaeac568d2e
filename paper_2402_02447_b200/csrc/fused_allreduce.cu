// H1 fused across ranks: bucket-wise clip + allreduce in ONE persistent kernel
// per GPU, the transfer running over NVLink peer memory (no NCCL).
//
// Reference semantics: sync_bucketwise (gradsync.py:148-162) with rank r as
// worker row r — each worker's bucket is clipped at c/sqrt(B) (:155, local,
// no norm collective), then averaged over workers (allreduce_mean, :119-128).
//
// Every rank owns a symmetric bf16 stage buffer (the comm buffer) mapped into
// every peer (CUDA IPC, or one NVLS multicast object).  One persistent
// cooperative kernel per GPU, 2 CTAs per SM, roles split BY SM:
//   clip CTAs (SMs >= comm_sms), K1's two warp-specialised streams:
//     A (192 thr): norm pass of bucket s (128-bit loads, L2 evict_last), one
//                  fp64 partial per (bucket, CTA), fire-and-forget;
//     B (320 thr): fixed-order fold -> coefficient, L2 re-read, scale, cast,
//                  store into the LOCAL stage; the group's last CTA publishes
//                  "bucket s staged" with a gpu-scope release of this rank's
//                  own ready flag;
//   comm CTAs (SMs < comm_sms): one warp forwards ready flags (system fence,
//     then a sys-scope release into every peer's flag area); the other 15
//     warps reduce this rank's 1/N slice of every bucket, as one continuous
//     stream, once every rank has staged it — 16 B loads from all N stages
//     (peer loads go over NVLink), fp32 sum in rank order, x 1/N, bf16, and a
//     store into all N stages (P2P two-shot); or one multimem load-reduce and
//     one multimem store (NVLS: the switch sums).
// Why by SM: remote loads on an SM starve that SM's own HBM stream
// (tools/mb/contention_mb.cu), and a system-scope fence on the clip's
// per-bucket path costs 30+ µs under NVLink load; both measured, both moved
// off the clip SMs.  The launch ends when this rank has seen every rank's done
// flag, so the local stage then holds the averaged clipped gradient.  Flags
// carry a per-launch epoch (no resets); every cross-GPU wait is bounded (trap
// after B2_SPIN_TIMEOUT_S, default 10 min, 0 = unbounded).
#include "clip_common.cuh"

#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace b2 {
namespace {
using namespace clip;

constexpr int kMaxRanks = 8;
constexpr int kBarA = 1, kBarB = 2;
// Bound on every cross-GPU wait.  Ranks legitimately drift apart (a
// checkpoint or eval on one rank, a slow loader), so the default is generous
// (10 min) and 0 disables it (wait forever, like NCCL).  B2_SPIN_TIMEOUT_S or
// b2_set_spin_timeout() set it per process; a wait that exceeds it traps
// (sticky CUDA error) instead of hanging the job silently.
constexpr double kDefaultSpinTimeoutS = 600.0;
static double g_spin_timeout_s = -1.0;  // < 0: not yet read from the environment

struct FusedParams {
  ClipParams p;                        // in/out/limit/segments; p.out = local stage
  void* stage[kMaxRanks];              // every rank's stage (index = rank): bf16, or fp32 (parity mode)
  uint32_t* flags[kMaxRanks];          // every rank's flag area [2][kMaxRanks][kMaxSegs]
  unsigned* pcount;                    // local arrival counters [2][kMaxSegs]
  unsigned* epoch;                     // launches so far (device; this launch is *epoch + 1)
  __nv_bfloat16* mc;                   // NVLS: multicast address of the stage buffers (or null)
  int nranks, rank;
  float inv_n;
  int comm_sms;  // split kernel: CTAs on SMs [0, comm_sms) reduce, all others clip
  uint64_t timeout_ns;  // cross-GPU wait bound (0 = unbounded)
};

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// wait until *p has reached `epoch` (wrap-safe), bounded
__device__ __forceinline__ void wait_epoch(const uint32_t* p, uint32_t epoch, uint64_t timeout_ns) {
  const uint64_t t0 = global_ns();
  unsigned ns = 32;
  while ((int32_t)(ld_acquire_sys(p) - epoch) < 0) {
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
    if (timeout_ns && global_ns() - t0 > timeout_ns) __trap();  // a peer never arrived: fail, do not hang
  }
}
// timeline stamps (ns) in the unused partial rows kMaxSegs-1-k of the
// workspace, read back by tools/k4_timeline.py (only when nseg leaves them free)
__device__ __forceinline__ void stamp(const ClipParams& p, int k) {
  if (p.nseg <= kMaxSegs - 8) reinterpret_cast<uint64_t*>(p.partials)[(size_t)(kMaxSegs - 1 - k) * kMaxGrid + blockIdx.x] = global_ns();
}
__device__ __forceinline__ uint32_t* flag(const FusedParams& f, int owner, int kind, int src, int s) {
  B2_DASSERT(owner >= 0 && owner < f.nranks && kind >= 0 && kind < 2 && src >= 0 && src < kMaxRanks && s >= 0 &&
             s < kMaxSegs);
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

__device__ __forceinline__ unsigned smid_u32() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// ---------------------------------------------------------------------------
// Split-role K4: remote (NVLink) loads on an SM starve that SM's own HBM
// stream (tools/mb/contention_mb.cu: local reads fall from 6.9 to 1.4 TB/s
// when 4 of 16 warps pull from a peer; they keep 6.6 TB/s when the pulls run
// on 16 other SMs).  So the roles are split by SM, not by warp: CTAs resident
// on SMs [0, comm_sms) only reduce (all their threads), every other CTA only
// clips (A norm stream ∥ B scale stream, K1's split).  Roles and their counts
// are settled by one registration barrier at entry (the launch is
// cooperative, so every CTA is resident); chunks are derived from the actual
// counts on the device.
template <int kAT, int kBT, int UA, int UB, int UC, int RMAX, bool MC, typename ST>
__global__ void __launch_bounds__(kAT + kBT, 2) k_clip_allreduce_split(const __grid_constant__ FusedParams f) {
  using V = float4;
  constexpr int N = 4, kT = kAT + kBT;
  constexpr int EPV = 16 / (int)sizeof(ST);  // stage elements per 16 B vector: 8 bf16 or 4 fp32
  static_assert(!MC || sizeof(ST) == 2, "NVLS multimem reduce is built for the bf16 stage");
  const ClipParams& p = f.p;
  __shared__ double redA[32], redB[32];
  __shared__ double s_coef;
  __shared__ volatile int s_bdone;
  __shared__ uint32_t s_epoch;
  __shared__ int s_role, s_idx, s_nk, s_nc;
  const int t = threadIdx.x;
  unsigned* reg = f.pcount + kMaxSegs + 1;  // [0] clip CTAs, [1] comm CTAs, [2] arrivals
  if (t == 0) {
    s_bdone = 0;
    s_epoch = *f.epoch + 1u;
    const int role = (int)smid_u32() < f.comm_sms ? 1 : 0;
    s_role = role;
    s_idx = (int)atomicAdd(&reg[role], 1u);
    red_release_u32(&reg[2], 1u);
    const uint64_t t0 = global_ns();
    while (ld_acquire_u32(&reg[2]) < gridDim.x)
      if (f.timeout_ns && global_ns() - t0 > f.timeout_ns) __trap();
    s_nk = (int)ld_acquire_u32(&reg[0]);
    s_nc = (int)ld_acquire_u32(&reg[1]);
    if (s_nk == 0 || s_nc == 0) __trap();  // host sizes comm_sms inside the SM count
    stamp(p, 0);
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;
  const int NR = f.nranks;

  if (s_role == 0) {
    // ============================ clip CTA: A (norm) ∥ B (scale into the stage)
    const int R = p.ngroups, kidx = s_idx, gid = kidx % R;
    const int G = group_size(s_nk, R, gid), c = kidx / R;
    if (t < kAT) {
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
        const int64_t per = (sg.nv + G - 1) / G;
        double acc = 0.0;
        const V* vin = reinterpret_cast<const V*>(in + sg.head);
        const int64_t v0 = min64((int64_t)c * per, sg.nv), v1 = min64(v0 + per, sg.nv);
        for (int64_t v = v0 + gt; v < v1; v += (int64_t)kAT * UA) {
          V x[UA];
#pragma unroll
          for (int u = 0; u < UA; ++u) {
            const int64_t vi = v + (int64_t)u * kAT;
            x[u] = vi < v1 ? ld_a<0>(vin + vi, pol_keep) : V{};
          }
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
          } else if ((nz << 1) != 0u) {  // out-of-range mini-sum: exact fp64
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
          B2_DASSERT(s < kMaxSegs && c < kMaxGrid);
          p.partials[(size_t)s * kMaxGrid + c] = tot;
          red_release_u32(&p.counters[s], 1u);
        }
      }
    } else {
      const int gt = t - kAT;
      const uint64_t pol_drop = l2_policy_evict_first();
      ST* stage = static_cast<ST*>(f.stage[f.rank]);
      for (int i = 0, s = gid; s < p.nseg; ++i, s += R) {
        if (gt == 0) {
          unsigned ns = 32;
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
          // gradsync.py:114-116.  A non-finite bucket (the reference raises,
          // :111-112) is staged as all-NaN, so after the mean EVERY rank's
          // copy of the whole bucket is NaN: any rank detects it locally
          // (FusedBucketSync.nonfinite_buckets) without another collective.
          const double coef = !isfinite(total) ? __longlong_as_double(0x7ff8000000000000ll)
                              : (norm >= p.limit) ? p.limit / norm : 1.0;
          if (c == 0) {
            if (p.norms) p.norms[s] = norm;
            if (p.nonfinite) p.nonfinite[s] = !isfinite(total) ? 1 : 0;
          }
          s_coef = coef;
        }
        group_sync<kBT>(kBarB);
        const float cf = MC ? (float)(s_coef * (double)f.inv_n) : (float)s_coef;
        const Seg sg = p.seg[s];
        const float* in = static_cast<const float*>(p.in) + sg.in_off;
        ST* out = stage + sg.out_off;
        const V* vin = reinterpret_cast<const V*>(in + sg.head);
        const int64_t per = (sg.nv + G - 1) / G;
        const int64_t v0 = min64((int64_t)c * per, sg.nv), v1 = min64(v0 + per, sg.nv);
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
              put_vec<ST, 4, float>(out + sg.head + vi * N, y);
            }
          }
        }
        const int64_t tail0 = sg.head + sg.nv * N;
        if (c == 0 && gt < sg.head) put1(out + gt, in[gt] * cf);
        if (c == G - 1 && gt < sg.n - tail0) put1(out + tail0 + gt, in[tail0 + gt] * cf);
        group_sync<kBT>(kBarB);
        if (gt == 0) {
          __threadfence();
          // last clip CTA of the group: publish "bucket s staged" with a
          // gpu-scope release of this rank's own ready flag only.  A
          // system-scope fence here measured 30+ µs per bucket under NVLink
          // load and sat on the clip's critical path (2.07 vs 0.56 ms for the
          // clip at N=4); the comm CTAs' forwarder warps pay it instead.
          if (atomicAdd(&f.pcount[s], 1u) == (unsigned)G - 1) st_release_gpu(flag(f, f.rank, 0, f.rank, s), epoch);
          s_bdone = i + 1;
        }
      }
      if (gt == 0) stamp(p, 1);
    }
  } else {
    // ============================ comm CTA: reduce this rank's slice of every
    // bucket (its 1/NC share), as one continuous stream in bucket order
    const int NC = s_nc, cidx = s_idx;
    __shared__ int64_t s_beg[kMaxSegs + 1], s_voff[kMaxSegs];
    __shared__ uint32_t s_rdy[kMaxSegs];
    if (t == 0) {
      int64_t acc = 0;
      for (int s = 0; s < p.nseg; ++s) {
        const Seg sg = p.seg[s];
        const int64_t nvs = sg.n / EPV;  // 16 B stage vectors of the bucket
        const int64_t per_r = (nvs + NR - 1) / NR;
        const int64_t r0 = min64((int64_t)f.rank * per_r, nvs), r1 = min64(r0 + per_r, nvs);
        const int64_t per_c = (r1 - r0 + NC - 1) / NC;
        const int64_t c0 = min64(r0 + (int64_t)cidx * per_c, r1), c1 = min64(c0 + per_c, r1);
        s_beg[s] = acc;
        s_voff[s] = sg.out_off / EPV + c0 - acc;
        s_rdy[s] = 0u;
        acc += c1 - c0;
      }
      s_beg[p.nseg] = acc;
    }
    __syncthreads();
    const int64_t M = s_beg[p.nseg];
    constexpr int kTC = kT - 32;  // the last warp forwards ready flags
    if (t >= kTC) {
      // forwarder: this rank's ready flag of bucket s (gpu-scope release by
      // the clip) -> system fence -> every peer's flag area (sys release).
      // Causality is transitive: clip stores -> gpu release/acquire -> sys
      // release/acquire -> the peer's loads of this rank's stage.
      if (t == kTC && NR > 1) {
        for (int s = cidx; s < p.nseg; s += NC) {
          wait_epoch(flag(f, f.rank, 0, f.rank, s), epoch, f.timeout_ns);
          __threadfence_system();
          for (int q = 0; q < NR; ++q)
            if (q != f.rank) st_release_sys(flag(f, q, 0, f.rank, s), epoch);
        }
      }
    } else {
    int cur = 0;
    for (int64_t f0 = t; f0 < M; f0 += (int64_t)kTC * UC) {
      uint4 x[UC][RMAX];
      int64_t vix[UC];
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        const int64_t fi = f0 + (int64_t)u * kTC;
        vix[u] = -1;
        if (fi < M) {
          while (fi >= s_beg[cur + 1]) ++cur;
          if (ld_acquire_cta_shared(&s_rdy[cur]) == 0u) {
            for (int q = 0; q < NR; ++q) wait_epoch(flag(f, f.rank, 0, q, cur), epoch, f.timeout_ns);
            st_release_cta_shared(&s_rdy[cur], 1u);
            if (cur == 0 && t == 0) stamp(p, 2);
          }
          vix[u] = fi + s_voff[cur];
          if constexpr (MC) {
            asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                         : "=r"(x[u][0].x), "=r"(x[u][0].y), "=r"(x[u][0].z), "=r"(x[u][0].w)
                         : "l"(reinterpret_cast<const uint4*>(f.mc) + vix[u])
                         : "memory");
          } else {
#pragma unroll
            for (int q = 0; q < RMAX; ++q)
              if (q < NR) x[u][q] = __ldcg(reinterpret_cast<const uint4*>(f.stage[q]) + vix[u]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        if (vix[u] < 0) continue;
        if constexpr (MC) {
          asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(
                           reinterpret_cast<uint4*>(f.mc) + vix[u]),
                       "f"(__uint_as_float(x[u][0].x)), "f"(__uint_as_float(x[u][0].y)),
                       "f"(__uint_as_float(x[u][0].z)), "f"(__uint_as_float(x[u][0].w))
                       : "memory");
        } else {
          float acc[EPV];
#pragma unroll
          for (int i = 0; i < EPV; ++i) acc[i] = 0.f;
#pragma unroll
          for (int q = 0; q < RMAX; ++q) {
            if (q < NR) {  // fixed rank order: identical bits on every rank
              if constexpr (EPV == 8) {
                float e[8];
                bf16x8_to_f32(x[u][q], e);
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i] += e[i];
              } else {
                acc[0] += __uint_as_float(x[u][q].x);
                acc[1] += __uint_as_float(x[u][q].y);
                acc[2] += __uint_as_float(x[u][q].z);
                acc[3] += __uint_as_float(x[u][q].w);
              }
            }
          }
#pragma unroll
          for (int i = 0; i < EPV; ++i) acc[i] *= f.inv_n;  // mean, not sum (gradsync.py:128)
          uint4 y;
          if constexpr (EPV == 8) {
            y = f32_to_bf16x8(acc);
          } else {
            y = make_uint4(__float_as_uint(acc[0]), __float_as_uint(acc[1]), __float_as_uint(acc[2]),
                           __float_as_uint(acc[3]));
          }
#pragma unroll
          for (int q = 0; q < RMAX; ++q)
            if (q < NR) __stcg(reinterpret_cast<uint4*>(f.stage[q]) + vix[u], y);
        }
      }
    }
    }  // reduce threads
    __syncthreads();
    if (t == 0) {
      stamp(p, 3);
      __threadfence_system();  // one system-scope release per CTA for all its remote stores
      if (atomicAdd(&f.pcount[kMaxSegs], 1u) == (unsigned)NC - 1) {
        __threadfence_system();
        for (int q = 0; q < NR; ++q) st_release_sys(flag(f, q, 1, f.rank, 0), epoch);
      }
      if (cidx == 0)
        for (int q = 0; q < NR; ++q) wait_epoch(flag(f, f.rank, 1, q, 0), epoch, f.timeout_ns);
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
      reg[0] = reg[1] = reg[2] = 0u;
      p.counters[kMaxSegs] = 0u;
      *f.epoch = epoch;
      __threadfence();
    }
  }
}

template <int AT, int BT, int UA, int UB, int UC, int RMAX, bool MC = false, typename ST = __nv_bfloat16>
int launch_split(FusedParams& f, cudaStream_t stream, int comm_sms) {
  auto kern = k_clip_allreduce_split<AT, BT, UA, UB, UC, RMAX, MC, ST>;
  const DeviceInfo& di = device_info();
  B2_REQUIRE(di.coop, B2_ERR_CUDA, "device does not support cooperative launch");
  static int occ_cached[64] = {};
  int& occ = occ_cached[di.device & 63];
  if (occ == 0) {
    B2_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, AT + BT, 0));
    B2_REQUIRE(occ >= 1, B2_ERR_CUDA, "fused kernel cannot be resident");
  }
  const int per_sm = std::min(2, occ);
  const int grid = std::min(di.sm_count * per_sm, kMaxGrid);
  comm_sms = std::max(1, std::min(comm_sms, di.sm_count - 1));
  f.comm_sms = comm_sms;
  // groups are sized for the clip CTAs the placement will give (one per
  // resident slot on the clip SMs); the device re-derives chunks from the
  // actual registration counts
  f.p.ngroups = choose_groups(f.p, grid - comm_sms * per_sm, sizeof(float));
  for (int s = 0; s < f.p.nseg; ++s) f.p.seg[s].nv = (f.p.seg[s].n - f.p.seg[s].head) / 4;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(AT + BT);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // registration barrier + cross-CTA waits
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

static double spin_timeout_s() {
  if (g_spin_timeout_s < 0.0) {
    const char* e = getenv("B2_SPIN_TIMEOUT_S");
    g_spin_timeout_s = e ? atof(e) : kDefaultSpinTimeoutS;
    if (g_spin_timeout_s < 0.0) g_spin_timeout_s = 0.0;
  }
  return g_spin_timeout_s;
}

extern "C" int b2_set_spin_timeout(double seconds) {
  B2_REQUIRE(seconds >= 0.0, B2_ERR_INVALID, "timeout must be >= 0 seconds (0 = wait forever)");
  g_spin_timeout_s = seconds;
  return B2_OK;
}

extern "C" double b2_get_spin_timeout(void) { return spin_timeout_s(); }

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
                               size_t workspace_bytes, void* stream, int stage_dtype = B2_BF16);

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

extern "C" int b2_bucket_clip_allreduce_p2p_dtype(const void* in, void* const* stages, int stage_dtype,
                                                  uint32_t* const* flags, int nranks, int rank,
                                                  const int64_t* seg_off, const int64_t* seg_len, int nseg,
                                                  double limit, double* norms, int32_t* nonfinite, void* workspace,
                                                  size_t workspace_bytes, void* stream) {
  B2_REQUIRE(stage_dtype == B2_BF16 || stage_dtype == B2_F32, B2_ERR_UNSUPPORTED,
             "stage dtype must be B2_BF16 or B2_F32");
  return clip_allreduce_impl(in, stages, nullptr, flags, nranks, rank, seg_off, seg_len, nseg, limit, norms,
                             nonfinite, workspace, workspace_bytes, stream, stage_dtype);
}

static int clip_allreduce_impl(const void* in, void* const* stages, void* mc_stage, uint32_t* const* flags,
                               int nranks, int rank, const int64_t* seg_off, const int64_t* seg_len, int nseg,
                               double limit, double* norms, int32_t* nonfinite, void* workspace,
                               size_t workspace_bytes, void* stream, int stage_dtype) {
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
  const bool f32 = stage_dtype == B2_F32;
  B2_REQUIRE(!(f32 && mc_stage), B2_ERR_UNSUPPORTED, "the NVLS form reduces a bf16 stage");
  int rc = fill_params(f.p, in, B2_F32, stages[rank], f32 ? B2_F32 : B2_BF16, seg_off, seg_off, seg_len, 0, nseg,
                       limit, 1.0, norms, nullptr, nonfinite, workspace);
  if (rc != B2_OK) return rc;
  for (int s = 0; s < nseg; ++s)
    B2_REQUIRE(f.p.seg[s].vec, B2_ERR_UNSUPPORTED, "fused allreduce needs 16 B aligned gradients");
  for (int q = 0; q < nranks; ++q) {
    f.stage[q] = stages[q];
    f.flags[q] = flags[q];
  }
  f.pcount = reinterpret_cast<unsigned*>(static_cast<char*>(workspace) + WsLayout::pcounters);
  f.epoch = reinterpret_cast<unsigned*>(static_cast<char*>(workspace) + WsLayout::epoch);
  f.nranks = nranks;
  f.rank = rank;
  f.inv_n = 1.0f / (float)nranks;
  f.mc = static_cast<__nv_bfloat16*>(mc_stage);
  f.timeout_ns = (uint64_t)(spin_timeout_s() * 1e9);

  // roles: comm CTAs on the first `cs` SMs (B2_COMM_SMS overrides), clip CTAs
  // on the rest.  Sweeps (profiles/r01_k4_split_sweep.jsonl): P2P best at 64
  // of 148 SMs for N = 2, 48 for N = 4 (1.63 vs 1.67-1.70 ms at 64), NVLS at 32.
  // Twice the reduce vectors in flight per thread measured slower for both.
  cudaStream_t st = (cudaStream_t)stream;
  const char* cse = getenv("B2_COMM_SMS");
  const int csms = cse ? atoi(cse) : 0;
  const int cs = csms > 0 ? csms : (mc_stage ? 32 : nranks <= 2 ? 64 : 48);
  // each reduce thread keeps UC x RMAX 16 B vectors in flight (32 registers)
  if (mc_stage) return launch_split<192, 320, 8, 4, 8, 1, true>(f, st, cs);
  // B2_K4_RMAX=2|4|8 picks the rank-count instantiation (>= nranks), read at
  // every call: tests run each build at the ranks a box has (1-GPU included)
  int rmax = nranks <= 2 ? 2 : nranks <= 4 ? 4 : 8;
  if (const char* e = getenv("B2_K4_RMAX")) {
    const int want = atoi(e);
    B2_REQUIRE(want == 2 || want == 4 || want == 8, B2_ERR_INVALID, "B2_K4_RMAX must be 2, 4 or 8");
    rmax = std::max(rmax, want);
  }
  if (f32) {  // parity mode: fp32 stage, the 1e-5 contract across ranks
    if (rmax == 2) return launch_split<192, 320, 8, 4, 4, 2, false, float>(f, st, cs);
    if (rmax == 4) return launch_split<192, 320, 8, 4, 2, 4, false, float>(f, st, cs);
    return launch_split<192, 320, 8, 4, 1, 8, false, float>(f, st, cs);
  }
  if (rmax == 2) return launch_split<192, 320, 8, 4, 4, 2>(f, st, cs);
  if (rmax == 4) return launch_split<192, 320, 8, 4, 2, 4>(f, st, cs);
  return launch_split<192, 320, 8, 4, 1, 8>(f, st, cs);
}
