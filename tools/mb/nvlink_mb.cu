// SM-driven NVLink bandwidth between two B200s (one process, peer access):
// what can K4's reduce stream get from remote loads (pull) vs remote stores
// (push), with both GPUs driving traffic at once as in an allreduce?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o nvlink_mb nvlink_mb.cu
//   ./nvlink_mb            (needs 2 visible GPUs)
// Modes, each GPU d working on S bytes of its peer's memory per iteration:
//   pull   : 16 B loads from the peer buffer (data flows peer -> d)
//   push   : 16 B stores into the peer buffer (data flows d -> peer)
//   2shot  : K4's two-shot step on a bf16 slice of S bytes: load local + peer,
//            add, store local + peer (peer->d S and d->peer S per GPU)
// Prints GB/s per direction = bytes crossing one direction / time.
#include <cuda_bf16.h>

#include <cstdint>
#include <cstdio>
#include <vector>
#include <cstdlib>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int U>
__global__ void k_pull(const uint4* __restrict__ peer, int64_t nv, uint32_t* sink) {
  uint32_t a = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += stride * U) {
    uint4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = i + u * stride;
      x[u] = j < nv ? __ldcg(peer + j) : uint4{};
    }
#pragma unroll
    for (int u = 0; u < U; ++u) a ^= x[u].x ^ x[u].y ^ x[u].z ^ x[u].w;
  }
  if (a == 0x12345678u) sink[threadIdx.x] = a;
}

template <int U>
__global__ void k_push(uint4* __restrict__ peer, int64_t nv) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += stride * U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = i + u * stride;
      if (j < nv) __stcg(peer + j, make_uint4((uint32_t)j, 1, 2, 3));
    }
  }
}

template <int U>
__global__ void k_twoshot(uint4* __restrict__ local, uint4* __restrict__ peer, int64_t nv) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += stride * U) {
    uint4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = i + u * stride;
      if (j < nv) {
        a[u] = __ldcg(local + j);
        b[u] = __ldcg(peer + j);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = i + u * stride;
      if (j < nv) {
        const __nv_bfloat162* ha = reinterpret_cast<const __nv_bfloat162*>(&a[u]);
        const __nv_bfloat162* hb = reinterpret_cast<const __nv_bfloat162*>(&b[u]);
        uint4 y;
        __nv_bfloat162* hy = reinterpret_cast<__nv_bfloat162*>(&y);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 fa = __bfloat1622float2(ha[k]), fb = __bfloat1622float2(hb[k]);
          hy[k] = __floats2bfloat162_rn((fa.x + fb.x) * 0.5f, (fa.y + fb.y) * 0.5f);
        }
        __stcg(local + j, y);
        __stcg(peer + j, y);
      }
    }
  }
}

// LDGSTS pull: per thread a ring of D 16 B async copies from the peer into smem
template <int D>
__global__ void k_pull_ldgsts(const uint4* __restrict__ peer, int64_t nv, uint32_t* sink) {
  extern __shared__ uint4 ring[];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  uint32_t a = 0;
  auto slot = [&](int d) { return (uint32_t)__cvta_generic_to_shared(&ring[d * blockDim.x + threadIdx.x]); };
  for (int d = 0; d < D - 1; ++d) {
    const int64_t j = i0 + d * stride;
    if (j < nv) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(slot(d)), "l"(peer + j) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int64_t k = 0;; ++k) {
    const int64_t j = i0 + k * stride;
    if (j >= nv) break;
    const int64_t jn = i0 + (k + D - 1) * stride;
    if (jn < nv)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(slot((int)((k + D - 1) % D))), "l"(peer + jn) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
    const uint4 v = ring[(k % D) * blockDim.x + threadIdx.x];
    a ^= v.x ^ v.w;
  }
  if (a == 0x12345678u) sink[threadIdx.x] = a;
}

// TMA bulk pull: one elected thread streams CH-byte pieces of the CTA's
// contiguous share of the peer buffer into an NS-slot smem ring (mbarriers)
template <int CH, int NS>
__global__ void k_pull_tma(const char* __restrict__ peer, int64_t bytes, uint32_t* sink) {
  extern __shared__ __align__(128) char tring[];
  __shared__ __align__(8) uint64_t full[NS];
  const int64_t per = (bytes / gridDim.x) & ~(int64_t)(CH - 1);
  const char* src = peer + blockIdx.x * per;
  const int npieces = (int)(per / CH);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t a = 0;
  if (threadIdx.x == 0) {
    auto issue = [&](int piece) {
      const int sl = piece % NS;
      const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&full[sl]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(CH) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(tring + sl * CH)),
                   "l"(src + (int64_t)piece * CH), "r"(CH), "r"(bar)
                   : "memory");
    };
    for (int p = 0; p < NS && p < npieces; ++p) issue(p);
    for (int p = 0; p < npieces; ++p) {
      const int sl = p % NS;
      const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&full[sl]);
      const uint32_t phase = (p / NS) & 1;
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                     : "=r"(done)
                     : "r"(bar), "r"(phase)
                     : "memory");
      a ^= *reinterpret_cast<const uint32_t*>(tring + sl * CH);
      if (p + NS < npieces) issue(p + NS);
    }
  }
  if (a == 0x12345678u) sink[threadIdx.x] = a;
}

// two-shot by PUSH only: phase 1 writes my copy of the peer-owned slice into
// the peer's receive buffer; phase 2 (after both phase 1s) reduces my slice
// from local memory (stage + recv) and writes the result locally and into
// the peer's stage.  Every NVLink byte is a remote store.
template <int U>
__global__ void k_push_p1(const uint4* __restrict__ mine, uint4* __restrict__ peer_recv, int64_t nv) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += stride * U) {
    uint4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = i + u * stride;
      if (j < nv) x[u] = __ldcg(mine + j);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = i + u * stride;
      if (j < nv) __stcg(peer_recv + j, x[u]);
    }
  }
}
template <int U>
__global__ void k_push_p2(uint4* __restrict__ stage, const uint4* __restrict__ recv, uint4* __restrict__ peer_stage,
                          int64_t nv) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += stride * U) {
    uint4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = i + u * stride;
      if (j < nv) {
        a[u] = __ldcg(stage + j);
        b[u] = __ldcg(recv + j);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = i + u * stride;
      if (j < nv) {
        const __nv_bfloat162* ha = reinterpret_cast<const __nv_bfloat162*>(&a[u]);
        const __nv_bfloat162* hb = reinterpret_cast<const __nv_bfloat162*>(&b[u]);
        uint4 y;
        __nv_bfloat162* hy = reinterpret_cast<__nv_bfloat162*>(&y);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 fa = __bfloat1622float2(ha[k]), fb = __bfloat1622float2(hb[k]);
          hy[k] = __floats2bfloat162_rn((fa.x + fb.x) * 0.5f, (fa.y + fb.y) * 0.5f);
        }
        __stcg(stage + j, y);
        __stcg(peer_stage + j, y);
      }
    }
  }
}

struct Dev {
  int id;
  cudaStream_t st;
  uint4* buf;   // own memory, 2 x S (half 0 = what the peer touches, half 1 = local)
  uint32_t* sink;
  cudaEvent_t e0, e1, done;
};

template <typename L>
float run(Dev* d, int iters, L launch) {
  // lock-step: iteration k on each GPU starts after both finished k-1
  for (int k = -2; k < iters; ++k) {
    if (k == 0)
      for (int g = 0; g < 2; ++g) { CK(cudaSetDevice(d[g].id)); CK(cudaEventRecord(d[g].e0, d[g].st)); }
    for (int g = 0; g < 2; ++g) {
      CK(cudaSetDevice(d[g].id));
      launch(g);
      CK(cudaEventRecord(d[g].done, d[g].st));
    }
    for (int g = 0; g < 2; ++g) { CK(cudaSetDevice(d[g].id)); CK(cudaStreamWaitEvent(d[g].st, d[1 - g].done, 0)); }
  }
  float ms = 0;
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(d[g].id));
    CK(cudaEventRecord(d[g].e1, d[g].st));
    CK(cudaEventSynchronize(d[g].e1));
    float m;
    CK(cudaEventElapsedTime(&m, d[g].e0, d[g].e1));
    ms = m > ms ? m : ms;
  }
  return ms / iters;
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("needs 2 GPUs\n"); return 0; }
  const int64_t S = 335ll << 20;  // bytes per GPU per direction (half of BERT-large's bf16 buckets)
  const int64_t nv = S / 16;
  Dev d[2];
  for (int g = 0; g < 2; ++g) {
    d[g].id = g;
    CK(cudaSetDevice(g));
    CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaStreamCreateWithFlags(&d[g].st, cudaStreamNonBlocking));
    CK(cudaMalloc(&d[g].buf, 2 * S));
    CK(cudaMemset(d[g].buf, 0, 2 * S));
    CK(cudaMalloc(&d[g].sink, 4096));
    CK(cudaEventCreate(&d[g].e0));
    CK(cudaEventCreate(&d[g].e1));
    CK(cudaEventCreateWithFlags(&d[g].done, cudaEventDisableTiming));
  }
  for (int g = 0; g < 2; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); }
  const int iters = 10;
  const int blocks_per_sm[] = {1, 2, 4};
  const int threads[] = {128, 256, 512};
  auto report = [&](const char* mode, int both, int bps, int t, int u, float ms, double bytes_dir) {
    printf("{\"mode\": \"%s\", \"bidir\": %d, \"ctas_per_sm\": %d, \"threads\": %d, \"unroll\": %d, \"ms\": %.4f, "
           "\"gbs_per_dir\": %.1f}\n", mode, both, bps, t, u, ms, bytes_dir / (ms * 1e-3) / 1e9);
    fflush(stdout);
  };
#define SWEEP(MODE, BOTH, BYTES, LAUNCH)                                                   \
  for (int bps : blocks_per_sm)                                                            \
    for (int t : threads) {                                                                \
      const int grid = 148 * bps;                                                          \
      {constexpr int U = 2; float ms = run(d, iters, [&](int g) { if (BOTH || g == 0) LAUNCH; }); report(MODE, BOTH, bps, t, U, ms, BYTES);} \
      {constexpr int U = 4; float ms = run(d, iters, [&](int g) { if (BOTH || g == 0) LAUNCH; }); report(MODE, BOTH, bps, t, U, ms, BYTES);} \
      {constexpr int U = 8; float ms = run(d, iters, [&](int g) { if (BOTH || g == 0) LAUNCH; }); report(MODE, BOTH, bps, t, U, ms, BYTES);} \
    }
  for (int both = 0; both < 2; ++both) {
    SWEEP("pull", both, (double)S, (k_pull<U><<<grid, t, 0, d[g].st>>>(d[1 - g].buf, nv, d[g].sink)))
    SWEEP("push", both, (double)S, (k_push<U><<<grid, t, 0, d[g].st>>>(d[1 - g].buf, nv)))
  }
  for (int both = 0; both < 2; ++both) {
    for (int t : {128, 256}) {
      {constexpr int D = 8; const size_t sm = (size_t)D * t * 16; float ms = run(d, iters, [&](int g) { if (both || g == 0) { cudaFuncSetAttribute(k_pull_ldgsts<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000); k_pull_ldgsts<D><<<296, t, sm, d[g].st>>>(d[1 - g].buf, nv, d[g].sink);} }); report("pull_ldgsts_d8", both, 2, t, D, ms, (double)S);}
      {constexpr int D = 16; const size_t sm = (size_t)D * t * 16; float ms = run(d, iters, [&](int g) { if (both || g == 0) { cudaFuncSetAttribute(k_pull_ldgsts<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000); k_pull_ldgsts<D><<<296, t, sm, d[g].st>>>(d[1 - g].buf, nv, d[g].sink);} }); report("pull_ldgsts_d16", both, 2, t, D, ms, (double)S);}
    }
    for (int bps : {1, 2}) {
      {constexpr int CH = 4096, NS = 8; float ms = run(d, iters, [&](int g) { if (both || g == 0) { cudaFuncSetAttribute(k_pull_tma<CH, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000); k_pull_tma<CH, NS><<<148 * bps, 32, CH * NS, d[g].st>>>((const char*)d[1 - g].buf, S, d[g].sink);} }); report("pull_tma_4k_x8", both, bps, 32, 0, ms, (double)S);}
      {constexpr int CH = 16384, NS = 4; float ms = run(d, iters, [&](int g) { if (both || g == 0) { cudaFuncSetAttribute(k_pull_tma<CH, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000); k_pull_tma<CH, NS><<<148 * bps, 32, CH * NS, d[g].st>>>((const char*)d[1 - g].buf, S, d[g].sink);} }); report("pull_tma_16k_x4", both, bps, 32, 0, ms, (double)S);}
      {constexpr int CH = 8192, NS = 8; float ms = run(d, iters, [&](int g) { if (both || g == 0) { cudaFuncSetAttribute(k_pull_tma<CH, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000); k_pull_tma<CH, NS><<<148 * bps, 32, CH * NS, d[g].st>>>((const char*)d[1 - g].buf, S, d[g].sink);} }); report("pull_tma_8k_x8", both, bps, 32, 0, ms, (double)S);}
    }
  }
  if (getenv("MB_ONLY_ASYNC")) return 0;
  if (getenv("MB_ONLY_PUSH2")) {
    // buffers: buf = [slice 0 | slice 1] stage (2 x S), recv = S per GPU
    uint4* recv[2];
    for (int g = 0; g < 2; ++g) { CK(cudaSetDevice(g)); CK(cudaMalloc(&recv[g], S)); }
    cudaEvent_t p1[2];
    for (int g = 0; g < 2; ++g) { CK(cudaSetDevice(g)); CK(cudaEventCreateWithFlags(&p1[g], cudaEventDisableTiming)); }
    for (int bps : {1, 2}) for (int t : {256, 512}) {
      const int grid = 148 * bps;
      float ms = run(d, iters, [&](int g) {
        // GPU g owns slice g; it pushes its copy of slice (1-g) to the peer's recv
        k_push_p1<4><<<grid, t, 0, d[g].st>>>(d[g].buf + (1 - g) * nv, recv[1 - g], nv);
        CK(cudaEventRecord(p1[g], d[g].st));
        CK(cudaSetDevice(1 - g));
        CK(cudaSetDevice(g));
      });
      (void)ms;
      // phase-separated timing: p1 on both, cross wait, p2 on both
      auto iter = [&]() {
        for (int g = 0; g < 2; ++g) {
          CK(cudaSetDevice(g));
          k_push_p1<4><<<grid, t, 0, d[g].st>>>(d[g].buf + (1 - g) * nv, recv[1 - g], nv);
          CK(cudaEventRecord(p1[g], d[g].st));
        }
        for (int g = 0; g < 2; ++g) { CK(cudaSetDevice(g)); CK(cudaStreamWaitEvent(d[g].st, p1[1 - g], 0)); }
        for (int g = 0; g < 2; ++g) {
          CK(cudaSetDevice(g));
          k_push_p2<4><<<grid, t, 0, d[g].st>>>(d[g].buf + g * nv, recv[g], d[1 - g].buf + g * nv, nv);
        }
      };
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        for (int g = 0; g < 2; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); }
        CK(cudaSetDevice(0));
        CK(cudaEventRecord(d[0].e0, d[0].st));
        for (int k = 0; k < iters; ++k) {
          iter();
          for (int g = 0; g < 2; ++g) { CK(cudaSetDevice(g)); CK(cudaEventRecord(d[g].done, d[g].st)); }
          for (int g = 0; g < 2; ++g) { CK(cudaSetDevice(g)); CK(cudaStreamWaitEvent(d[g].st, d[1 - g].done, 0)); }
        }
        CK(cudaSetDevice(0));
        CK(cudaEventRecord(d[0].e1, d[0].st));
        CK(cudaEventSynchronize(d[0].e1));
        float m;
        CK(cudaEventElapsedTime(&m, d[0].e0, d[0].e1));
        best = std::min(best, m / iters);
      }
      report("2shot_push", 1, bps, t, 4, best, (double)S);
    }
    // the pull two-shot for the same sizes, same timing harness
    for (int bps : {2}) for (int t : {128, 256}) {
      const int grid = 148 * bps;
      float ms = run(d, iters, [&](int g) { k_twoshot<4><<<grid, t, 0, d[g].st>>>(d[g].buf + g * nv, d[1 - g].buf + g * nv, nv); });
      report("2shot_pull", 1, bps, t, 4, ms, (double)S);
    }
    return 0;
  }
  // two-shot: GPU g reduces slice g of the (2 x S) buffer: local slice + the peer's same slice
  SWEEP("2shot", 1, (double)S,
        (k_twoshot<U><<<grid, t, 0, d[g].st>>>(d[g].buf + g * nv, d[1 - g].buf + g * nv, nv)))
  // copy engine reference
  for (int both = 0; both < 2; ++both) {
    float ms = run(d, iters, [&](int g) {
      if (both || g == 0) CK(cudaMemcpyPeerAsync(d[1 - g].buf + nv, 1 - g, d[g].buf, g, S, d[g].st));
    });
    report("ce_copy", both, 0, 0, 0, ms, (double)S);
  }
  return 0;
}
