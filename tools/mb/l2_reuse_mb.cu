// Does a 26 MB bucket survive in B200's L2 across other streaming traffic?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o l2_reuse_mb l2_reuse_mb.cu
// Pattern: read X (flavour F) ; stream Y (gap MB) ; re-read X (timed).  A fast
// re-read means L2 hits.  Flavours: 0 ld.global, 1 ld.global.nc.L1::no_allocate,
// 2 ld + L2::evict_last policy, 3 ld.global.cs (evict-first).
#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int F>
__device__ __forceinline__ float4 ld(const float4* p) {
  float4 v;
  if (F == 0) asm volatile("ld.global.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  if (F == 1) asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  if (F == 2) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  }
  if (F == 3) asm volatile("ld.global.cs.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

template <int F>
__global__ void k_read(const float4* __restrict__ x, int64_t nv, float* out) {
  float a = 0;
  for (int64_t i = blockIdx.x * 512ll + threadIdx.x; i < nv; i += (int64_t)gridDim.x * 512) {
    float4 v = ld<F>(x + i);
    a += v.x + v.y + v.z + v.w;
  }
  if (a == 1234.5f) out[threadIdx.x] = a;
}

__global__ void k_write(float4* __restrict__ y, int64_t nv) {
  for (int64_t i = blockIdx.x * 512ll + threadIdx.x; i < nv; i += (int64_t)gridDim.x * 512) y[i] = make_float4(1, 2, 3, 4);
}

int main() {
  const int64_t bx = 26214400, nvx = bx / 16;
  const int64_t by = 1ll << 30;
  float4 *x, *y, *flush; float* o;
  CK(cudaMalloc(&x, bx)); CK(cudaMalloc(&y, by)); CK(cudaMalloc(&flush, 512ll << 20)); CK(cudaMalloc(&o, 8192));
  CK(cudaMemset(x, 1, bx)); CK(cudaMemset(y, 1, by));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int g = sms * 4;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto reread = [&](int flavour, int64_t gap_mb, bool gap_write) -> float {
    k_write<<<g, 512>>>(flush, (512ll << 20) / 16);  // evict everything
    if (flavour == 0) k_read<0><<<g, 512>>>(x, nvx, o);
    if (flavour == 1) k_read<1><<<g, 512>>>(x, nvx, o);
    if (flavour == 2) k_read<2><<<g, 512>>>(x, nvx, o);
    if (flavour == 3) k_read<3><<<g, 512>>>(x, nvx, o);
    if (gap_mb > 0) {
      if (gap_write) k_write<<<g, 512>>>(y, (gap_mb << 20) / 16);
      else k_read<1><<<g, 512>>>(y, (gap_mb << 20) / 16, o);
    }
    cudaEventRecord(a);
    k_read<0><<<g, 512>>>(x, nvx, o);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e3f;
  };
  printf("cold re-read baseline (flush only): %.2f us\n", reread(3, 0, false));
  for (int f = 0; f < 4; ++f)
    for (int64_t gap : {0, 13, 26, 52, 78, 104})
      for (int w = 0; w < 2; ++w) {
        float t = 0;
        for (int r = 0; r < 3; ++r) t += reread(f, gap, w) / 3;
        printf("flavour=%d gap=%3lld MB (%s): re-read 26 MB in %6.2f us = %6.0f GB/s\n", f, (long long)gap, w ? "write" : "read ", t, bx / (t * 1e-6) / 1e9);
      }
  return 0;
}
