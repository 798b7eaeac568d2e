// Fixed costs of a lone-bucket K1 launch on B200 (decides the DDP-hook-shape design).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o launch_mb launch_mb.cu
// Back-to-back launches (CUDA events over 200), 296 CTAs x 512 threads:
//   empty       : nothing (launch + ramp + drain)
//   coop_empty  : the same, cooperative attribute
//   barrier     : one grid-wide arrive/spin (the fold's dependency), cooperative
//   read26      : each CTA reads its 88 KB chunk of a 26 MB fp32 buffer (vector loads), no barrier
//   read_write  : read 26 MB + write 13 MB (bf16), no barrier
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_empty() {}

__global__ void k_empty_pdl() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
}

__global__ void k_rw_pdl(const float4* x, int64_t nv, uint2* y) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t per = (nv + gridDim.x - 1) / gridDim.x;
  const int64_t v0 = blockIdx.x * per, v1 = min(v0 + per, nv);
  for (int64_t v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
    float4 a = x[v];
    __nv_bfloat162 p = __floats2bfloat162_rn(a.x * 0.5f, a.y * 0.5f), q = __floats2bfloat162_rn(a.z * 0.5f, a.w * 0.5f);
    y[v] = make_uint2(*reinterpret_cast<unsigned*>(&p), *reinterpret_cast<unsigned*>(&q));
  }
}

__global__ void k_barrier(unsigned* ctr, unsigned* exitc) {
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(ctr, 1u);
    while (atomicAdd(ctr, 0u) < gridDim.x) __nanosleep(32);
    if (atomicAdd(exitc, 1u) == gridDim.x - 1) { *ctr = 0; *exitc = 0; __threadfence(); }
  }
  __syncthreads();
}

__global__ void k_read(const float4* x, int64_t nv, float* sink) {
  const int64_t per = (nv + gridDim.x - 1) / gridDim.x;
  const int64_t v0 = blockIdx.x * per, v1 = min(v0 + per, nv);
  float s = 0;
  for (int64_t v = v0 + threadIdx.x; v < v1; v += blockDim.x) { float4 a = x[v]; s += a.x * a.x + a.y * a.y + a.z * a.z + a.w * a.w; }
  if (s == 1234.5f) sink[0] = s;
}

__global__ void k_rw(const float4* x, int64_t nv, uint2* y) {
  const int64_t per = (nv + gridDim.x - 1) / gridDim.x;
  const int64_t v0 = blockIdx.x * per, v1 = min(v0 + per, nv);
  for (int64_t v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
    float4 a = x[v];
    __nv_bfloat162 p = __floats2bfloat162_rn(a.x * 0.5f, a.y * 0.5f), q = __floats2bfloat162_rn(a.z * 0.5f, a.w * 0.5f);
    y[v] = make_uint2(*reinterpret_cast<unsigned*>(&p), *reinterpret_cast<unsigned*>(&q));
  }
}

template <typename F>
float timeit(F f, int reps = 200) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 10; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;
}

int main() {
  const int grid = 296, thr = 512;
  const int64_t n = 6553600, nv = n / 4;
  float4* x; uint2* y; float* sink; unsigned* ctr;
  CK(cudaMalloc(&x, n * 4)); CK(cudaMalloc(&y, n * 2)); CK(cudaMalloc(&sink, 4)); CK(cudaMalloc(&ctr, 8));
  CK(cudaMemset(x, 0, n * 4)); CK(cudaMemset(ctr, 0, 8));
  // big buffers so each launch reads cold data (126 MB L2): rotate over 8 x 26 MB
  float4* xs; CK(cudaMalloc(&xs, n * 4 * 8)); CK(cudaMemset(xs, 0, n * 4 * 8));
  int rot = 0;
  printf("empty      %.2f us\n", timeit([&] { k_empty<<<grid, thr>>>(); }));
  cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(grid); cfg.blockDim = dim3(thr);
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1; cfg.attrs = at; cfg.numAttrs = 1;
  printf("coop_empty %.2f us\n", timeit([&] { cudaLaunchKernelEx(&cfg, k_empty); }));
  printf("barrier    %.2f us\n", timeit([&] { cudaLaunchKernelEx(&cfg, k_barrier, ctr, ctr + 1); }));
  printf("read26     %.2f us\n", timeit([&] { k_read<<<grid, thr>>>(xs + (rot++ % 8) * nv, nv, sink); }));
  printf("read_write %.2f us\n", timeit([&] { k_rw<<<grid, thr>>>(xs + (rot++ % 8) * nv, nv, y); }));
  cudaLaunchConfig_t pc = {}; pc.gridDim = dim3(grid); pc.blockDim = dim3(thr);
  cudaLaunchAttribute pa[1]; pa[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; pa[0].val.programmaticStreamSerializationAllowed = 1;
  pc.attrs = pa; pc.numAttrs = 1;
  printf("empty_pdl  %.2f us\n", timeit([&] { cudaLaunchKernelEx(&pc, k_empty_pdl); }));
  printf("rw_pdl     %.2f us\n", timeit([&] { cudaLaunchKernelEx(&pc, k_rw_pdl, (const float4*)(xs + (rot++ % 8) * nv), nv, y); }));
  for (int g2 : {148, 296, 592}) for (int t2 : {256, 512, 1024}) {
    if (g2 * t2 > 296 * 1024) continue;
    printf("empty %4dx%-4d %.2f us   rw %.2f us\n", g2, t2, timeit([&] { k_empty<<<g2, t2>>>(); }),
           timeit([&] { k_rw<<<g2, t2>>>(xs + (rot++ % 8) * nv, nv, y); }));
  }
  {
    cudaLaunchConfig_t cc = {}; cc.gridDim = dim3(grid); cc.blockDim = dim3(thr);
    cudaLaunchAttribute ca[2];
    ca[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; ca[0].val.programmaticStreamSerializationAllowed = 1;
    ca[1].id = cudaLaunchAttributeCooperative; ca[1].val.cooperative = 1;
    cc.attrs = ca; cc.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cc, k_rw_pdl, (const float4*)xs, nv, y);
    printf("coop+pdl launch: %s\n", cudaGetErrorString(e));
    cudaDeviceSynchronize();
    if (e == cudaSuccess) printf("coop+pdl rw %.2f us\n", timeit([&] { cudaLaunchKernelEx(&cc, k_rw_pdl, (const float4*)(xs + (rot++ % 8) * nv), nv, y); }));
  }
  // graph of 52 rw launches (the hook-shape loop)
  cudaStream_t s; cudaStreamCreate(&s);
  cudaGraph_t gr; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 52; ++i) k_rw<<<grid, thr, 0, s>>>(xs + (i % 8) * nv, nv, y);
  cudaStreamEndCapture(s, &gr); cudaGraphInstantiate(&ge, gr, 0);
  printf("graph52 rw  %.2f us per launch\n", timeit([&] { cudaGraphLaunch(ge, s); }, 20) / 52);
  CK(cudaGetLastError());
  return 0;
}
