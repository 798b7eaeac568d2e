// Shared helpers for the b2ddp C-ABI library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <utility>

#include "b2ddp.h"

namespace b2 {

// thread-local last-error message returned by b2_last_error()
void set_error(const char* fmt, ...);

// Cached per-device properties (SM count, cooperative support).
struct DeviceInfo {
  int device = -1;
  int sm_count = 0;
  int coop = 0;
};
const DeviceInfo& device_info();

inline int check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
    return B2_ERR_CUDA;
  }
  return B2_OK;
}

#define B2_CHECK(expr)                                   \
  do {                                                   \
    int _rc = ::b2::check_cuda((expr), #expr);           \
    if (_rc != B2_OK) return _rc;                        \
  } while (0)

#define B2_REQUIRE(cond, code, ...)  \
  do {                               \
    if (!(cond)) {                   \
      ::b2::set_error(__VA_ARGS__);  \
      return (code);                 \
    }                                \
  } while (0)

// ---- device-side bounds checks (debug builds) -----------------------------
// Built with -DB2_DEBUG_BOUNDS (tools/ab_build.sh debug ... with B2_NVCC_EXTRA),
// every index of the hand-written shared/global protocols is checked and a
// violation traps with its file:line; release builds compile the checks out.
#ifdef B2_DEBUG_BOUNDS
#define B2_DASSERT(cond)                                                          \
  do {                                                                            \
    if (!(cond)) {                                                                \
      printf("B2_DASSERT %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,    \
             (int)blockIdx.x, (int)threadIdx.x, #cond);                           \
      __trap();                                                                   \
    }                                                                             \
  } while (0)
#else
#define B2_DASSERT(cond) \
  do {                   \
  } while (0)
#endif

// A pointer the compiler may not re-associate with later index arithmetic: keeps
// `base + (uint32_t)i` a single IMAD.WIDE.U32 instead of a 64-bit add + shifts.
template <typename T>
__device__ __forceinline__ T* opaque(T* p) {
  asm("mov.b64 %0, %0;" : "+l"(p));
  __builtin_assume(__isGlobal(p));  // still a global pointer: STG, not generic ST
  return p;
}

// ---- programmatic dependent launch ----------------------------------------
// A kernel launched with launch_pdl() may start while its predecessor in the
// stream drains; it must call pdl_wait() before touching anything the
// predecessor writes.  pdl_trigger() lets the NEXT kernel's launch begin.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---- device-side primitives -------------------------------------------

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed tree): every caller with the same inputs in
// the same thread slots gets bit-identical results.  `scratch` >= 32 doubles.
template <int THREADS>
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  constexpr int W = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();  // scratch may still be read by a previous call
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    r = lane < W ? scratch[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;  // valid in warp 0
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned atom_add_acq_rel_u32(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;"
               : "=r"(old)
               : "l"(p), "r"(v)
               : "memory");
  return old;
}

__device__ __forceinline__ void red_release_u32(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace b2
