// H1 — bucket-wise gradient clipping before allreduce (sm_100a).
//
// K1  k_bucket_clip : fused per-bucket L2 norm -> clip coefficient -> scale +
//                     cast into the communication buffer.
//                     Reference: clip_by_norm (gradsync.py:106-116) applied per
//                     (worker, bucket) by sync_bucketwise (gradsync.py:148-162).
// K1b k_weighted_mean: single-process K-worker mean of clipped buckets with the
//                     reference's pairwise tree (gradsync.py:119-128).
//
// K1 design (HBM-bound, 4 B read + 2/4 B write per element):
//   * one persistent cooperative grid (ctas_per_sm x #SM CTAs, all co-resident)
//     walks a list of segments (buckets) in the order given;
//   * phase A(s): each CTA streams its contiguous chunk of segment s with
//     128-bit loads, accumulates sum(x^2) in fp64 (no fp32 overflow /
//     cancellation; 1e-5 parity needs it — SURVEY trap 4), block-reduces and
//     publishes one fp64 partial; the last CTA to arrive folds all partials in
//     a fixed order (bit-deterministic), derives norm/coef with the
//     reference's inclusive `norm >= limit` rule and releases a per-segment flag;
//   * phase B(s): once segment s's coefficient is published, each CTA re-reads
//     its chunk (an L2 hit: the chunk was read one phase earlier, a 26 MB bucket
//     is well inside the 126 MB L2) and writes g*coef*post_scale, cast;
//   * software pipeline: a CTA runs A(s+1) before waiting on s, so DRAM keeps
//     streaming while the slowest CTA's partial of s lands.  DRAM traffic is the
//     algorithmic 4 B read + out-dtype write per element; the re-read is on L2.
#include "common.cuh"

#include <cuda_bf16.h>

#include <algorithm>
#include <type_traits>

namespace b2 {
namespace {

constexpr int kMaxSegs = 128;   // segments per launch (kernel-parameter table)
constexpr int kMaxGrid = 2048;  // CTAs per launch the workspace is sized for
constexpr int kThreads = 512;
constexpr int kUnroll = 4;

struct Seg {
  int64_t in_off, out_off, n, head;  // head: scalar elements before 16 B alignment
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
  Seg seg[kMaxSegs];
};

struct WsLayout {
  static constexpr size_t partials = 0;
  static constexpr size_t coef = partials + sizeof(double) * kMaxSegs * kMaxGrid;
  static constexpr size_t counters = coef + sizeof(double) * kMaxSegs;
  static constexpr size_t bytes = counters + sizeof(unsigned) * (kMaxSegs + 1);
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

template <typename V> __device__ __forceinline__ V ld_stream_keep(const V* p);
template <> __device__ __forceinline__ float4 ld_stream_keep(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
template <> __device__ __forceinline__ double2 ld_stream_keep(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
// last use of the chunk: evict-first so it does not displace the next bucket
template <typename V> __device__ __forceinline__ V ld_last_use(const V* p) { return __ldcs(p); }

template <typename Tin>
__device__ __forceinline__ double sq_of(Tin x, bool& bad) {
  double d = static_cast<double>(x);
  if constexpr (std::is_same<Tin, double>::value) bad |= !isfinite(d);
  return d * d;
}

// Phase A: this CTA's sum of squares over its chunk of segment s.
template <typename Tin>
__device__ __forceinline__ double chunk_sumsq(const ClipParams& p, const Seg& sg, bool& bad) {
  using V = typename VecOf<Tin>::V;
  constexpr int N = VecOf<Tin>::N;
  const Tin* in = static_cast<const Tin*>(p.in) + sg.in_off;
  const int G = gridDim.x, c = blockIdx.x, t = threadIdx.x;
  double acc[N];
#pragma unroll
  for (int j = 0; j < N; ++j) acc[j] = 0.0;
  if (sg.vec) {
    const int64_t nv = (sg.n - sg.head) / N;
    const int64_t tail0 = sg.head + nv * N;
    if (c == 0 && t < sg.head) acc[0] += sq_of(in[t], bad);
    if (c == G - 1 && t < sg.n - tail0) acc[1 % N] += sq_of(in[tail0 + t], bad);
    const V* vin = reinterpret_cast<const V*>(in + sg.head);
    const int64_t per = (nv + G - 1) / G;
    const int64_t v0 = min64((int64_t)c * per, nv), v1 = min64(v0 + per, nv);
    for (int64_t v = v0 + t; v < v1; v += (int64_t)kThreads * kUnroll) {
      V x[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t vi = v + (int64_t)u * kThreads;
        if (vi < v1) x[u] = ld_stream_keep(vin + vi);
        else x[u] = V{};
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        double e[N];
        unpack(x[u], e);
#pragma unroll
        for (int j = 0; j < N; ++j) {
          if constexpr (std::is_same<Tin, double>::value) bad |= !isfinite(e[j]);
          acc[j] = fma(e[j], e[j], acc[j]);
        }
      }
    }
  } else {
    const int64_t per = (sg.n + G - 1) / G;
    const int64_t e0 = min64((int64_t)c * per, sg.n), e1 = min64(e0 + per, sg.n);
    for (int64_t e = e0 + t; e < e1; e += kThreads) acc[0] += sq_of(in[e], bad);
  }
  double r = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j) r += acc[j];
  return r;
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

// Phase B: out = cast(in * coef * post_scale) over this CTA's chunk.
template <typename Tin, typename Tout>
__device__ __forceinline__ void chunk_scale(const ClipParams& p, const Seg& sg, double coef) {
  using V = typename VecOf<Tin>::V;
  constexpr int N = VecOf<Tin>::N;
  using Acc = typename std::conditional<std::is_same<Tin, double>::value ||
                                            std::is_same<Tout, double>::value,
                                        double, float>::type;
  const Tin* in = static_cast<const Tin*>(p.in) + sg.in_off;
  Tout* out = static_cast<Tout*>(p.out) + sg.out_off;
  const Acc cf = static_cast<Acc>(coef * p.post_scale);
  const int G = gridDim.x, c = blockIdx.x, t = threadIdx.x;
  if (sg.vec) {
    const int64_t nv = (sg.n - sg.head) / N;
    const int64_t tail0 = sg.head + nv * N;
    if (c == 0 && t < sg.head) put1(out + t, static_cast<Acc>(in[t]) * cf);
    if (c == G - 1 && t < sg.n - tail0) put1(out + tail0 + t, static_cast<Acc>(in[tail0 + t]) * cf);
    const V* vin = reinterpret_cast<const V*>(in + sg.head);
    Tout* vout = out + sg.head;
    const int64_t per = (nv + G - 1) / G;
    const int64_t v0 = min64((int64_t)c * per, nv), v1 = min64(v0 + per, nv);
    for (int64_t v = v0 + t; v < v1; v += (int64_t)kThreads * kUnroll) {
      V x[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t vi = v + (int64_t)u * kThreads;
        if (vi < v1) x[u] = ld_last_use(vin + vi);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t vi = v + (int64_t)u * kThreads;
        if (vi < v1) {
          double e[N];
          unpack(x[u], e);
          Acc y[N];
#pragma unroll
          for (int j = 0; j < N; ++j) y[j] = static_cast<Acc>(e[j]) * cf;
          put_vec<Tout, N, Acc>(vout + vi * N, y);
        }
      }
    }
  } else {
    const int64_t per = (sg.n + G - 1) / G;
    const int64_t e0 = min64((int64_t)c * per, sg.n), e1 = min64(e0 + per, sg.n);
    for (int64_t e = e0 + t; e < e1; e += kThreads) put1(out + e, static_cast<Acc>(in[e]) * cf);
  }
}

template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kThreads) k_bucket_clip(const __grid_constant__ ClipParams p) {
  __shared__ double red[32];
  __shared__ double s_coef[2];  // double-buffered by segment parity
  __shared__ int s_last;
  const unsigned G = gridDim.x;
  constexpr bool kF64 = std::is_same<Tin, double>::value;

  // Phase A for segment s, then (if this CTA arrived last) publish its coef.
  auto arrive = [&](int s) {
    const Seg& sg = p.seg[s];
    bool bad = false;
    const double part = chunk_sumsq<Tin>(p, sg, bad);
    double tot = block_sum<kThreads>(part, red);
    if constexpr (kF64) {
      if (__syncthreads_or(bad)) tot = __longlong_as_double(0x7ff8000000000000ll);  // NaN marks inf/nan input
    }
    if (threadIdx.x == 0) {
      p.partials[(size_t)s * G + blockIdx.x] = tot;
      __threadfence();
      const unsigned prev = atom_add_acq_rel_u32(&p.counters[s], 1u);
      s_last = (prev == G - 1);
    }
    __syncthreads();
    if (s_last) {
      // fixed-order fold of all partials: identical bits whichever CTA is last
      double v = 0.0;
      for (unsigned j = threadIdx.x; j < G; j += kThreads) v += __ldcg(&p.partials[(size_t)s * G + j]);
      const double total = block_sum<kThreads>(v, red);
      if (threadIdx.x == 0) {
        const double norm = sqrt(total);
        const bool nf = kF64 ? isnan(total) : !isfinite(total);
        const double coef = (norm >= p.limit) ? p.limit / norm : 1.0;  // gradsync.py:114-116
        if (p.norms) p.norms[s] = norm;
        if (p.coefs) p.coefs[s] = coef;
        if (p.nonfinite) p.nonfinite[s] = nf ? 1 : 0;
        p.coef_ws[s] = coef;
        red_release_u32(&p.counters[s], 1u);  // counter -> G + 1: published
      }
    }
  };

  auto wait_coef = [&](int s) -> double {
    if (threadIdx.x == 0) {
      unsigned ns = 32;
      while (ld_acquire_u32(&p.counters[s]) < G + 1) {
        __nanosleep(ns);
        if (ns < 512) ns <<= 1;
      }
      s_coef[s & 1] = __ldcg(&p.coef_ws[s]);
    }
    __syncthreads();
    return s_coef[s & 1];
  };

  arrive(0);
  for (int s = 0; s < p.nseg; ++s) {
    if (s + 1 < p.nseg) arrive(s + 1);
    const double coef = wait_coef(s);
    if (p.out != nullptr) chunk_scale<Tin, Tout>(p, p.seg[s], coef);
  }

  // exit: the last CTA out restores the counters to zero for the next launch
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atom_add_acq_rel_u32(&p.counters[kMaxSegs], 1u);
    if (prev == G - 1) {
      for (int s = 0; s < p.nseg; ++s) p.counters[s] = 0u;
      p.counters[kMaxSegs] = 0u;
      __threadfence();
    }
  }
}

template <typename Tin, typename Tout>
int launch_clip(ClipParams& p, int ctas_per_sm, cudaStream_t stream) {
  auto kern = k_bucket_clip<Tin, Tout>;
  const DeviceInfo& di = device_info();
  B2_REQUIRE(di.coop, B2_ERR_CUDA, "device does not support cooperative launch");
  int occ = 0;
  B2_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, 0));
  B2_REQUIRE(occ >= 1, B2_ERR_CUDA, "bucket_clip kernel cannot be resident");
  int per_sm = ctas_per_sm > 0 ? std::min(ctas_per_sm, occ) : std::min(2, occ);
  int grid = std::min(per_sm * di.sm_count, kMaxGrid);
  // small problems: fewer CTAs (each still gets >= kThreads*kUnroll vectors)
  int64_t total = 0;
  for (int s = 0; s < p.nseg; ++s) total += p.seg[s].n;
  const int64_t want = (total + (int64_t)kThreads * kUnroll * 4 - 1) / ((int64_t)kThreads * kUnroll * 4);
  grid = (int)std::max<int64_t>(1, std::min<int64_t>(grid, want));
  void* args[] = {&p};
  B2_CHECK(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kThreads), args, 0, stream));
  return B2_OK;
}

// ---------------------------------------------------------------- K1b
constexpr int kMaxK = 64;
constexpr int kMeanThreads = 256;

struct MeanParams {
  const void* G;
  void* out;
  const double* coef;  // [K][B_total]
  int64_t K, ld;
  int B_total, b0, nb;  // this launch covers buckets b0 .. b0+nb-1
  int64_t bounds[kMaxSegs + 1];
};

template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kMeanThreads) k_weighted_mean(const __grid_constant__ MeanParams p) {
  __shared__ double cf[kMaxK];
  const int b = p.b0 + blockIdx.y;
  const int K = (int)p.K;
  if (threadIdx.x < K) cf[threadIdx.x] = p.coef[(int64_t)threadIdx.x * p.B_total + b];
  __syncthreads();
  const int64_t lo = p.bounds[blockIdx.y], hi = p.bounds[blockIdx.y + 1];
  const Tin* g = static_cast<const Tin*>(p.G);
  Tout* out = static_cast<Tout*>(p.out);
  for (int64_t i = lo + (int64_t)blockIdx.x * kMeanThreads + threadIdx.x; i < hi;
       i += (int64_t)gridDim.x * kMeanThreads) {
    double v[kMaxK];
    for (int k = 0; k < K; ++k) v[k] = static_cast<double>(g[(int64_t)k * p.ld + i]) * cf[k];
    int n = K;  // pairwise tree over ascending worker index (gradsync.py:123-127)
    while (n > 1) {
      int m = 0;
      for (int j = 0; j + 1 < n; j += 2) v[m++] = v[j] + v[j + 1];
      if (n & 1) v[m++] = v[n - 1];
      n = m;
    }
    out[i] = static_cast<Tout>(v[0] / (double)K);  // mean, not sum (:128)
  }
}

}  // namespace
}  // namespace b2

using namespace b2;

extern "C" size_t b2_clip_workspace_bytes(void) { return WsLayout::bytes; }

extern "C" int b2_clip_workspace_init(void* ws, size_t bytes, void* stream) {
  B2_REQUIRE(ws != nullptr && bytes >= WsLayout::bytes, B2_ERR_INVALID,
             "clip workspace needs %zu bytes", (size_t)WsLayout::bytes);
  B2_CHECK(cudaMemsetAsync(ws, 0, WsLayout::bytes, (cudaStream_t)stream));
  return B2_OK;
}

extern "C" int b2_bucket_clip_cast(const void* in, int in_dtype, void* out, int out_dtype,
                                   const int64_t* seg_in_off, const int64_t* seg_out_off,
                                   const int64_t* seg_len, int nseg, double limit,
                                   double post_scale, double* norms, double* coefs,
                                   int32_t* nonfinite, void* workspace, size_t workspace_bytes,
                                   int ctas_per_sm, void* stream) {
  B2_REQUIRE(in != nullptr, B2_ERR_INVALID, "input pointer is NULL");
  B2_REQUIRE(nseg >= 0, B2_ERR_INVALID, "nseg must be >= 0");
  B2_REQUIRE(nseg == 0 || (seg_in_off && seg_len && (out == nullptr || seg_out_off)), B2_ERR_INVALID,
             "segment arrays are NULL");
  B2_REQUIRE(limit > 0.0, B2_ERR_INVALID, "limit must be > 0, got %g", limit);
  B2_REQUIRE(workspace != nullptr && workspace_bytes >= WsLayout::bytes, B2_ERR_INVALID,
             "clip workspace needs %zu bytes", (size_t)WsLayout::bytes);
  B2_REQUIRE(in_dtype == B2_F32 || in_dtype == B2_F64, B2_ERR_INVALID, "in_dtype must be F32 or F64");
  B2_REQUIRE(out == nullptr || out_dtype == B2_F32 || out_dtype == B2_BF16 || out_dtype == B2_F64,
             B2_ERR_INVALID, "bad out_dtype %d", out_dtype);
  B2_REQUIRE(!(in_dtype == B2_F64 && out != nullptr && out_dtype != B2_F64), B2_ERR_INVALID,
             "f64 input supports f64 output only");
  if (nseg == 0) return B2_OK;
  const size_t sin = in_dtype == B2_F64 ? 8 : 4;
  const size_t sout = out_dtype == B2_F64 ? 8 : (out_dtype == B2_BF16 ? 2 : 4);
  const int N = in_dtype == B2_F64 ? 2 : 4;  // elements per 16 B input vector
  char* wsb = static_cast<char*>(workspace);

  for (int s0 = 0; s0 < nseg; s0 += kMaxSegs) {
    ClipParams p{};
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
    int rc = B2_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (in_dtype == B2_F64) rc = launch_clip<double, double>(p, ctas_per_sm, st);
    else if (out == nullptr || out_dtype == B2_F32) rc = launch_clip<float, float>(p, ctas_per_sm, st);
    else if (out_dtype == B2_BF16) rc = launch_clip<float, __nv_bfloat16>(p, ctas_per_sm, st);
    else rc = launch_clip<float, double>(p, ctas_per_sm, st);
    if (rc != B2_OK) return rc;
  }
  return B2_OK;
}

extern "C" int b2_weighted_mean(const void* G, int in_dtype, int64_t K, int64_t D, int64_t ld,
                                const double* coef, const int64_t* bounds, int B, void* out,
                                int out_dtype, void* stream) {
  B2_REQUIRE(G && coef && bounds && out, B2_ERR_INVALID, "NULL pointer argument");
  B2_REQUIRE(K >= 1 && K <= kMaxK, B2_ERR_UNSUPPORTED, "K must be in [1, %d], got %lld", kMaxK,
             (long long)K);
  B2_REQUIRE(B >= 1 && D >= 1 && ld >= D, B2_ERR_INVALID, "bad shape");
  B2_REQUIRE(bounds[0] == 0 && bounds[B] == D, B2_ERR_INVALID, "bounds must cover [0, D)");
  B2_REQUIRE(in_dtype == B2_F32 || in_dtype == B2_F64, B2_ERR_INVALID, "bad in_dtype");
  B2_REQUIRE(out_dtype == B2_F32 || out_dtype == B2_F64, B2_ERR_INVALID, "bad out_dtype");
  cudaStream_t st = (cudaStream_t)stream;
  for (int b0 = 0; b0 < B; b0 += kMaxSegs) {
    MeanParams p{};
    p.G = G;
    p.out = out;
    p.coef = coef;
    p.K = K;
    p.ld = ld;
    p.B_total = B;
    p.b0 = b0;
    p.nb = std::min(kMaxSegs, B - b0);
    int64_t maxlen = 0;
    for (int i = 0; i <= p.nb; ++i) p.bounds[i] = bounds[b0 + i];
    for (int i = 0; i < p.nb; ++i) {
      B2_REQUIRE(p.bounds[i + 1] > p.bounds[i], B2_ERR_INVALID, "bounds must be increasing");
      maxlen = std::max(maxlen, p.bounds[i + 1] - p.bounds[i]);
    }
    const int gx = (int)std::min<int64_t>((maxlen + kMeanThreads - 1) / kMeanThreads, 4096);
    dim3 grid(gx, p.nb);
    if (in_dtype == B2_F64 && out_dtype == B2_F64) k_weighted_mean<double, double><<<grid, kMeanThreads, 0, st>>>(p);
    else if (in_dtype == B2_F64) k_weighted_mean<double, float><<<grid, kMeanThreads, 0, st>>>(p);
    else if (out_dtype == B2_F64) k_weighted_mean<float, double><<<grid, kMeanThreads, 0, st>>>(p);
    else k_weighted_mean<float, float><<<grid, kMeanThreads, 0, st>>>(p);
    B2_CHECK(cudaGetLastError());
  }
  return B2_OK;
}
