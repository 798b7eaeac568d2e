// Streaming micro-benchmarks that decide K1's inner loop on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_mb stream_mb.cu
// Reads 1.34 GB fp32 (BERT-large gradient size, > L2), prints GB/s per variant.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int U>
__global__ void __launch_bounds__(512) k_sumsq_f64(const float4* __restrict__ x, int64_t nv, double* out) {
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int64_t i = blockIdx.x * 512ll + threadIdx.x; i < nv; i += (int64_t)gridDim.x * 512 * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { int64_t j = i + (int64_t)u * gridDim.x * 512; v[u] = j < nv ? __ldcs(x + j) : make_float4(0, 0, 0, 0); }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a0 = fma((double)v[u].x, (double)v[u].x, a0); a1 = fma((double)v[u].y, (double)v[u].y, a1);
      a2 = fma((double)v[u].z, (double)v[u].z, a2); a3 = fma((double)v[u].w, (double)v[u].w, a3);
    }
  }
  double r = a0 + a1 + a2 + a3;
  if (r == 12345.0) out[threadIdx.x] = r;
}

template <int U>
__global__ void __launch_bounds__(512) k_sumsq_f32(const float4* __restrict__ x, int64_t nv, double* out) {
  float a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int64_t i = blockIdx.x * 512ll + threadIdx.x; i < nv; i += (int64_t)gridDim.x * 512 * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { int64_t j = i + (int64_t)u * gridDim.x * 512; v[u] = j < nv ? __ldcs(x + j) : make_float4(0, 0, 0, 0); }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a0 = fmaf(v[u].x, v[u].x, a0); a1 = fmaf(v[u].y, v[u].y, a1);
      a2 = fmaf(v[u].z, v[u].z, a2); a3 = fmaf(v[u].w, v[u].w, a3);
    }
  }
  double r = (double)a0 + a1 + a2 + a3;
  if (r == 12345.0) out[threadIdx.x] = r;
}

template <int U>
__global__ void __launch_bounds__(512) k_scale_bf16(const float4* __restrict__ x, int64_t nv, uint2* __restrict__ y, float c) {
  for (int64_t i = blockIdx.x * 512ll + threadIdx.x; i < nv; i += (int64_t)gridDim.x * 512 * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { int64_t j = i + (int64_t)u * gridDim.x * 512; if (j < nv) v[u] = __ldcs(x + j); }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t j = i + (int64_t)u * gridDim.x * 512;
      if (j < nv) {
        __nv_bfloat162 a = __floats2bfloat162_rn(v[u].x * c, v[u].y * c), b = __floats2bfloat162_rn(v[u].z * c, v[u].w * c);
        uint2 w; w.x = *reinterpret_cast<unsigned*>(&a); w.y = *reinterpret_cast<unsigned*>(&b);
        y[j] = w;
      }
    }
  }
}

// 256-bit variants (LDG.E.ENL2.256 on sm_100a): 8 fp32 per load, 16 B bf16 stores
struct __align__(32) F8 { float a[8]; };
__device__ __forceinline__ F8 ld8(const F8* p) {
  F8 v;
  asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
    : "=f"(v.a[0]),"=f"(v.a[1]),"=f"(v.a[2]),"=f"(v.a[3]),"=f"(v.a[4]),"=f"(v.a[5]),"=f"(v.a[6]),"=f"(v.a[7]) : "l"(p));
  return v;
}
template <int U>
__global__ void __launch_bounds__(512) k_sumsq8(const F8* __restrict__ x, int64_t n8, double* out) {
  float a0 = 0, a1 = 0;
  for (int64_t i = blockIdx.x * 512ll + threadIdx.x; i < n8; i += (int64_t)gridDim.x * 512 * U) {
    F8 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { int64_t j = i + (int64_t)u * gridDim.x * 512; if (j < n8) v[u] = ld8(x + j); else for (int k = 0; k < 8; ++k) v[u].a[k] = 0; }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < 8; k += 2) { a0 = fmaf(v[u].a[k], v[u].a[k], a0); a1 = fmaf(v[u].a[k + 1], v[u].a[k + 1], a1); }
  }
  double r = (double)a0 + a1;
  if (r == 12345.0) out[threadIdx.x] = r;
}
template <int U>
__global__ void __launch_bounds__(512) k_scale8_bf16(const F8* __restrict__ x, int64_t n8, uint4* __restrict__ y, float c) {
  for (int64_t i = blockIdx.x * 512ll + threadIdx.x; i < n8; i += (int64_t)gridDim.x * 512 * U) {
    F8 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { int64_t j = i + (int64_t)u * gridDim.x * 512; if (j < n8) v[u] = ld8(x + j); }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t j = i + (int64_t)u * gridDim.x * 512;
      if (j < n8) {
        uint4 w;
        unsigned* pw = &w.x;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          __nv_bfloat162 h = __floats2bfloat162_rn(v[u].a[2 * k] * c, v[u].a[2 * k + 1] * c);
          pw[k] = *reinterpret_cast<unsigned*>(&h);
        }
        y[j] = w;
      }
    }
  }
}

template <typename F>
float timeit(F f, int iters) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) f();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / iters;
}

int main() {
  const int64_t n = 335141888, nv = n / 4;
  float4* x; uint2* y; double* o;
  CK(cudaMalloc(&x, n * 4)); CK(cudaMalloc(&y, n * 2)); CK(cudaMalloc(&o, 4096));
  CK(cudaMemset(x, 0, n * 4));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per : {1, 2, 4}) {
    int g = sms * per;
    float t;
    t = timeit([&] { k_sumsq_f64<4><<<g, 512>>>(x, nv, o); }, 10); printf("sumsq_f64 U4  ctas/sm=%d %.1f us %.0f GB/s\n", per, t * 1e3, n * 4 / (t * 1e-3) / 1e9);
    t = timeit([&] { k_sumsq_f64<8><<<g, 512>>>(x, nv, o); }, 10); printf("sumsq_f64 U8  ctas/sm=%d %.1f us %.0f GB/s\n", per, t * 1e3, n * 4 / (t * 1e-3) / 1e9);
    t = timeit([&] { k_sumsq_f32<4><<<g, 512>>>(x, nv, o); }, 10); printf("sumsq_f32 U4  ctas/sm=%d %.1f us %.0f GB/s\n", per, t * 1e3, n * 4 / (t * 1e-3) / 1e9);
    t = timeit([&] { k_sumsq_f32<8><<<g, 512>>>(x, nv, o); }, 10); printf("sumsq_f32 U8  ctas/sm=%d %.1f us %.0f GB/s\n", per, t * 1e3, n * 4 / (t * 1e-3) / 1e9);
    t = timeit([&] { k_scale_bf16<4><<<g, 512>>>(x, nv, y, 0.5f); }, 10); printf("scale_bf16 U4 ctas/sm=%d %.1f us %.0f GB/s\n", per, t * 1e3, n * 6 / (t * 1e-3) / 1e9);
    t = timeit([&] { k_scale_bf16<8><<<g, 512>>>(x, nv, y, 0.5f); }, 10); printf("scale_bf16 U8 ctas/sm=%d %.1f us %.0f GB/s\n", per, t * 1e3, n * 6 / (t * 1e-3) / 1e9);
    t = timeit([&] { k_sumsq8<4><<<g, 512>>>((const F8*)x, n / 8, o); }, 10); printf("sumsq v8 U4 ctas/sm=%d %.1f us %.0f GB/s\n", per, t * 1e3, n * 4 / (t * 1e-3) / 1e9);
    t = timeit([&] { k_scale8_bf16<2><<<g, 512>>>((const F8*)x, n / 8, (uint4*)y, 0.5f); }, 10); printf("scale_bf16 v8 U2 ctas/sm=%d %.1f us %.0f GB/s\n", per, t * 1e3, n * 6 / (t * 1e-3) / 1e9);
    t = timeit([&] { k_scale8_bf16<4><<<g, 512>>>((const F8*)x, n / 8, (uint4*)y, 0.5f); }, 10); printf("scale_bf16 v8 U4 ctas/sm=%d %.1f us %.0f GB/s\n", per, t * 1e3, n * 6 / (t * 1e-3) / 1e9);
  }
  float t = timeit([&] { cudaMemcpyAsync(y, x, n * 2, cudaMemcpyDeviceToDevice); }, 10);
  printf("memcpy d2d %.1f us %.0f GB/s (r+w)\n", t * 1e3, n * 4 / (t * 1e-3) / 1e9);
  return 0;
}
