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
