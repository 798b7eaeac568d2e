// TMA ring streaming micro-benchmark (decides K1's ring geometry on B200).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_ring_mb tma_ring_mb.cu
// Streams 1.34 GB fp32 through a per-CTA shared-memory ring filled by
// cp.async.bulk; consumers either just release pieces (MODE 0), sum squares
// in fp64 (MODE 1) or in fp32 (MODE 2).
#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t par) {
  uint32_t d = 0;
  while (!d) asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }" : "=r"(d) : "r"(b), "r"(par) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory"); }
__device__ __forceinline__ void tma(uint32_t dst, const void* src, uint32_t bytes, uint32_t b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(bytes), "r"(b) : "memory");
}

template <int THREADS, int MODE>
__global__ void k_ring(const float4* __restrict__ x, int64_t nv, int piece_vecs, int np, double* out) {
  extern __shared__ __align__(128) unsigned char ring[];
  const int t = threadIdx.x;
  const uint32_t rb = (uint32_t)__cvta_generic_to_shared(ring);
  const uint32_t pb = piece_vecs * 16;
  const uint32_t fb = rb + np * pb, eb = fb + 8 * np;
  constexpr int W = THREADS / 32;
  if (t == 0) {
    for (int i = 0; i < np; ++i) { mbar_init(fb + 8 * i, 1); mbar_init(eb + 8 * i, W); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t per = (nv + gridDim.x - 1) / gridDim.x;
  const int64_t v0 = min((int64_t)blockIdx.x * per, nv), v1 = min(v0 + per, nv);
  const int k = (int)((v1 - v0 + piece_vecs - 1) / piece_vecs);
  if (t >= THREADS) {
    if (t == THREADS) {
      for (int q = 0; q < k; ++q) {
        const int slot = q % np, fill = q / np;
        if (fill) mbar_wait(eb + 8 * slot, (fill - 1) & 1);
        const int64_t a = v0 + (int64_t)q * piece_vecs;
        const int n = (int)min((int64_t)piece_vecs, v1 - a);
        tma(rb + slot * pb, x + a, n * 16, fb + 8 * slot);
      }
    }
    return;
  }
  double acc = 0;
  float accf = 0;
  for (int q = 0; q < k; ++q) {
    const int slot = q % np;
    mbar_wait(fb + 8 * slot, (q / np) & 1);
    const int64_t a = v0 + (int64_t)q * piece_vecs;
    const int n = (int)min((int64_t)piece_vecs, v1 - a);
    const float4* sp = reinterpret_cast<const float4*>(ring + slot * pb);
    if (MODE == 1) {
      for (int i = t; i < n; i += THREADS) { float4 v = sp[i]; acc = fma((double)v.x, (double)v.x, acc); acc = fma((double)v.y, (double)v.y, acc); acc = fma((double)v.z, (double)v.z, acc); acc = fma((double)v.w, (double)v.w, acc); }
    } else if (MODE == 2) {
      for (int i = t; i < n; i += THREADS) { float4 v = sp[i]; accf = fmaf(v.x, v.x, accf); accf = fmaf(v.y, v.y, accf); accf = fmaf(v.z, v.z, accf); accf = fmaf(v.w, v.w, accf); }
    }
    __syncwarp();
    if ((t & 31) == 0) mbar_arrive(eb + 8 * slot);
  }
  if (acc + accf == 12345.0) out[t] = acc;
}

template <int THREADS, int MODE>
int run(float4* x, int64_t nv, double* o, int per_sm, int piece_kb, int np, int sms) {
  auto kern = k_ring<THREADS, MODE>;
  const int pv = piece_kb * 1024 / 16;
  const int smem = np * (piece_kb * 1024 + 16);
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i) kern<<<sms * per_sm, THREADS + 32, smem>>>(x, nv, pv, np, o);
  CK(cudaGetLastError());
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) kern<<<sms * per_sm, THREADS + 32, smem>>>(x, nv, pv, np, o);
  cudaEventRecord(b); CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
  printf("mode=%d threads=%d ctas/sm=%d piece=%dKB np=%d ring=%dKB: %.1f us  %.0f GB/s\n", MODE, THREADS, per_sm, piece_kb, np,
         np * piece_kb, ms * 1e3, nv * 16 / (ms * 1e-3) / 1e9);
  return 0;
}

int main() {
  const int64_t n = 335141888, nv = n / 4;
  float4* x; double* o;
  CK(cudaMalloc(&x, n * 4)); CK(cudaMalloc(&o, 8192)); CK(cudaMemset(x, 0, n * 4));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<512, 0>(x, nv, o, 1, 16, 13, sms);
  run<512, 1>(x, nv, o, 1, 16, 13, sms);
  run<512, 2>(x, nv, o, 1, 16, 13, sms);
  run<512, 1>(x, nv, o, 1, 32, 6, sms);
  run<512, 1>(x, nv, o, 1, 8, 26, sms);
  run<512, 1>(x, nv, o, 1, 4, 48, sms);
  run<256, 1>(x, nv, o, 2, 16, 6, sms);
  run<256, 1>(x, nv, o, 2, 8, 12, sms);
  run<128, 1>(x, nv, o, 4, 8, 6, sms);
  run<1024, 1>(x, nv, o, 1, 16, 13, sms);
  run<512, 0>(x, nv, o, 1, 32, 6, sms);
  run<512, 0>(x, nv, o, 1, 64, 3, sms);
  return 0;
}
