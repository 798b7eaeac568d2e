// Shared device/host pieces of the K1 family (bucket_clip.cu, fused_allreduce.cu).
#pragma once

#include "common.cuh"

#include <cuda_bf16.h>

#include <algorithm>
#include <type_traits>

namespace b2 {
namespace clip {

constexpr int kMaxSegs = 128;   // segments per launch (kernel-parameter table)
constexpr int kMaxGrid = 2048;  // CTAs per launch the workspace is sized for

struct Seg {
  int64_t in_off, out_off, n, head;  // head: scalar elements before 16 B alignment
  int64_t nv, per;                   // body vectors; vectors per CTA (TMA kernel)
  int32_t vec;                       // 1: vector body path, 0: scalar path
  int32_t pad;
};

struct ClipParams {
  const void* in;
  void* out;
  double limit, post_scale;
  double* norms;
  double* coefs;
  int32_t* nonfinite;
  double* partials;    // [kMaxSegs][gridDim.x]
  double* coef_ws;     // [kMaxSegs]
  unsigned* counters;  // [kMaxSegs + 1]; the last one is the exit counter
  int nseg;
  int seg_vec_elems;   // elements per 16 B vector (4 for f32, 2 for f64)
  int ngroups;         // CTA groups: CTA c serves buckets s = c % ngroups (mod ngroups); 1 = whole grid
  Seg seg[kMaxSegs];
};

struct WsLayout {
  static constexpr size_t partials = 0;
  static constexpr size_t coef = partials + sizeof(double) * kMaxSegs * kMaxGrid;
  static constexpr size_t counters = coef + sizeof(double) * kMaxSegs;
  static constexpr size_t pcounters = counters + sizeof(unsigned) * (kMaxSegs + 1);  // fused allreduce
  static constexpr size_t epoch = pcounters + sizeof(unsigned) * 2 * kMaxSegs;       // fused launch count
  static constexpr size_t bytes = epoch + sizeof(unsigned) * 4;
};

template <typename T> struct VecOf;
template <> struct VecOf<float> { using V = float4; static constexpr int N = 4; };
template <> struct VecOf<double> { using V = double2; static constexpr int N = 2; };

__device__ __forceinline__ void unpack(const float4& v, double (&x)[4]) {
  x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
}
__device__ __forceinline__ void unpack(const double2& v, double (&x)[2]) {
  x[0] = v.x; x[1] = v.y;
}

template <typename Tin>
__device__ __forceinline__ double sq_of(Tin x, bool& bad) {
  double d = static_cast<double>(x);
  if constexpr (std::is_same<Tin, double>::value) bad |= !isfinite(d);
  return d * d;
}

template <typename Tout, typename Acc>
__device__ __forceinline__ void put1(Tout* o, Acc y) {
  if constexpr (std::is_same<Tout, __nv_bfloat16>::value) *o = __float2bfloat16_rn((float)y);
  else *o = static_cast<Tout>(y);
}

template <typename Tout, int N, typename Acc>
__device__ __forceinline__ void put_vec(Tout* o, const Acc (&y)[N]) {
  if constexpr (std::is_same<Tout, float>::value) {
    static_assert(N == 4, "f32 out vector is float4");
    *reinterpret_cast<float4*>(o) = make_float4((float)y[0], (float)y[1], (float)y[2], (float)y[3]);
  } else if constexpr (std::is_same<Tout, __nv_bfloat16>::value) {
    static_assert(N == 4, "bf16 out vector is 4 x bf16");
    __nv_bfloat162 a = __floats2bfloat162_rn((float)y[0], (float)y[1]);
    __nv_bfloat162 b = __floats2bfloat162_rn((float)y[2], (float)y[3]);
    uint2 w;
    w.x = *reinterpret_cast<unsigned*>(&a);
    w.y = *reinterpret_cast<unsigned*>(&b);
    *reinterpret_cast<uint2*>(o) = w;
  } else {
#pragma unroll
    for (int j = 0; j < N; j += 2)
      *reinterpret_cast<double2*>(o + j) = make_double2((double)y[j], (double)y[j + 1]);
  }
}


__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
template <typename V> __device__ __forceinline__ V ld_hint(const V* ptr, uint64_t pol);
template <> __device__ __forceinline__ float4 ld_hint(const float4* ptr, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(ptr), "l"(pol));
  return v;
}
template <> __device__ __forceinline__ double2 ld_hint(const double2* ptr, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(ptr), "l"(pol));
  return v;
}


template <int BNC> __device__ __forceinline__ float4 ld_b(const float4* ptr, uint64_t pol) {
  if constexpr (BNC) return ld_hint(ptr, pol);
  float4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(ptr), "l"(pol));
  return v;
}
template <int BNC> __device__ __forceinline__ double2 ld_b(const double2* ptr, uint64_t pol) {
  if constexpr (BNC) return ld_hint(ptr, pol);
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(ptr), "l"(pol));
  return v;
}
template <int BNC> __device__ __forceinline__ float4 ld_a(const float4* ptr, uint64_t pol) { return ld_b<BNC>(ptr, pol); }
template <int BNC> __device__ __forceinline__ double2 ld_a(const double2* ptr, uint64_t pol) { return ld_b<BNC>(ptr, pol); }


template <int NTH>
__device__ __forceinline__ void group_sync(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(NTH) : "memory");
}

template <int NTH>
__device__ __forceinline__ double group_sum(double v, double* scratch, int gt, int bar) {
  constexpr int W = NTH / 32;
  const int lane = gt & 31, w = gt >> 5;
  v = warp_sum(v);
  group_sync<NTH>(bar);
  if (lane == 0) scratch[w] = v;
  group_sync<NTH>(bar);
  double r = 0.0;
  if (w == 0) {
    r = lane < W ? scratch[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;  // valid in the group's warp 0
}

// Host: fill one launch's segment table (alignment decides the 16 B vector path).
inline int fill_params(ClipParams& p, const void* in, int in_dtype, void* out, int out_dtype,
                       const int64_t* seg_in_off, const int64_t* seg_out_off, const int64_t* seg_len, int s0,
                       int nseg, double limit, double post_scale, double* norms, double* coefs, int32_t* nonfinite,
                       void* workspace) {
  const size_t sin = in_dtype == B2_F64 ? 8 : 4;
  const size_t sout = out_dtype == B2_F64 ? 8 : (out_dtype == B2_BF16 ? 2 : 4);
  const int N = in_dtype == B2_F64 ? 2 : 4;  // elements per 16 B input vector
  char* wsb = static_cast<char*>(workspace);
  p = ClipParams{};
  p.in = in;
  p.out = out;
  p.limit = limit;
  p.post_scale = post_scale;
  p.norms = norms ? norms + s0 : nullptr;
  p.coefs = coefs ? coefs + s0 : nullptr;
  p.nonfinite = nonfinite ? nonfinite + s0 : nullptr;
  p.partials = reinterpret_cast<double*>(wsb + WsLayout::partials);
  p.coef_ws = reinterpret_cast<double*>(wsb + WsLayout::coef);
  p.counters = reinterpret_cast<unsigned*>(wsb + WsLayout::counters);
  p.nseg = std::min(kMaxSegs, nseg - s0);
  p.seg_vec_elems = N;
  p.ngroups = 1;
  for (int i = 0; i < p.nseg; ++i) {
    Seg& sg = p.seg[i];
    const int s = s0 + i;
    B2_REQUIRE(seg_len[s] >= 0 && seg_in_off[s] >= 0, B2_ERR_INVALID, "bad segment %d", s);
    sg.in_off = seg_in_off[s];
    sg.out_off = out ? seg_out_off[s] : 0;
    sg.n = seg_len[s];
    const uintptr_t ia = reinterpret_cast<uintptr_t>(in) + sg.in_off * sin;
    sg.head = 0;
    sg.vec = 0;
    if (ia % sin == 0) {
      const int64_t head = (int64_t)(((16 - ia % 16) % 16) / sin);
      bool ok = head <= sg.n;
      if (ok && out) {
        const uintptr_t oa = reinterpret_cast<uintptr_t>(out) + (sg.out_off + head) * sout;
        ok = oa % std::min<size_t>(16, N * sout) == 0;
      }
      if (ok) {
        sg.head = head;
        sg.vec = 1;
      }
    }
  }
  return B2_OK;
}

// CTA groups for small buckets: each group of ~grid/R CTAs owns every R-th
// bucket, so per-CTA chunks stay ~64-100 KB whatever the bucket size and the
// grid-wide fold shrinks to a group-wide one.  R is capped so the ~2 buckets a
// group keeps in flight (norm pass ahead of the L2 re-read) fit in L2.
inline int choose_groups(const ClipParams& p, int grid, size_t in_elem_bytes) {
  if (p.nseg <= 1) return 1;
  size_t total = 0;
  for (int s = 0; s < p.nseg; ++s) total += (size_t)p.seg[s].n * in_elem_bytes;
  const size_t avg = total / p.nseg;
  const size_t budget = 24u << 20;  // bytes of buckets in flight across groups (x2 for the lag)
  int r = (int)std::max<size_t>(1, budget / std::max<size_t>(avg, 1));
  r = std::min(r, std::max(1, grid / 4));  // >= 4 CTAs per group
  static int forced = -1;  // B2_CLIP_GROUPS: override for A/B runs
  if (forced < 0) {
    const char* e = getenv("B2_CLIP_GROUPS");
    forced = e ? atoi(e) : 0;
  }
  if (forced > 0) r = forced;
  r = std::min(r, p.nseg);
  return r;
}
__host__ __device__ __forceinline__ int group_size(int grid, int r, int gid) { return (grid - gid + r - 1) / r; }

}  // namespace clip
}  // namespace b2
