// Does remote (NVLink) load traffic slow local HBM streaming on the SAME SM?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o contention_mb contention_mb.cu
//   ./contention_mb        (needs 2 visible GPUs; both run the same kernel at once)
// One kernel, 296 CTAs x 512 threads.  Work is dispensed in 64 KB chunks from
// two global counters (local: read L bytes of own HBM; remote: read R bytes
// of the peer's memory).  Role of a warp:
//   mode 0: local only (every warp)                  -> HBM baseline
//   mode 1: remote only                              -> NVLink baseline
//   mode 2: warps 0-11 local, 12-15 remote (K4-like: roles mixed inside every SM)
//   mode 3: SMs with smid < NS remote, others local  (roles separated by SM)
// Prints the completion time of each role.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int kChunk = 64 * 1024;
struct Ctl {
  unsigned long long next[2];
  unsigned long long done_ns[2];
  unsigned long long t0;
  unsigned sink;
};

__device__ __forceinline__ uint64_t gns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// kind 0: read chunk; 1: write chunk; 2: read chunk + write it back (same
// buffer, like K4's two-shot on a remote slice); 3: read chunk, write half of
// it to `out` (K1's clip: 4 B in, 2 B out)
template <int U>
__device__ void stream(uint4* base, uint4* out, int64_t bytes, Ctl* ctl, int role, int kind, int lane) {
  const int64_t nchunks = bytes / kChunk;
  uint32_t a = 0;
  while (true) {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(&ctl->next[role], 1ull);
    c = __shfl_sync(0xffffffffu, c, 0);
    if ((int64_t)c >= nchunks) break;
    uint4* p = base + c * (kChunk / 16);
    for (int i = lane; i < kChunk / 16; i += 32 * U) {
      uint4 x[U];
      if (kind != 1) {
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = __ldcg(p + i + u * 32);
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = make_uint4(i, u, 1, 2);
      }
      if (kind == 1 || kind == 2) {
#pragma unroll
        for (int u = 0; u < U; ++u) __stcg(p + i + u * 32, x[u]);
      } else if (kind == 3) {
        uint2* o = reinterpret_cast<uint2*>(out + c * (kChunk / 32));
#pragma unroll
        for (int u = 0; u < U; ++u) __stcg(o + i + u * 32, make_uint2(x[u].x ^ x[u].y, x[u].z ^ x[u].w));
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) a ^= x[u].x ^ x[u].w;
      }
    }
  }
  if (lane == 0) atomicMax(&ctl->done_ns[role], (unsigned long long)gns());
  if (a == 0x9999u) ctl->sink = a;
}

__global__ void __launch_bounds__(512, 2) k_mix(uint4* local, uint4* lout, int64_t lbytes, uint4* remote, int64_t rbytes,
                                                Ctl* ctl, int mode, int ns, int lkind, int rkind) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) atomicMin(&ctl->t0, (unsigned long long)gns());
  int role;
  if (mode == 0) role = 0;
  else if (mode == 1) role = 1;
  else if (mode == 2) role = warp >= 12 ? 1 : 0;
  else role = (int)smid() < ns ? 1 : 0;
  if (role == 0) stream<8>(local, lout, lbytes, ctl, 0, lkind, lane);
  else stream<8>(remote, nullptr, rbytes, ctl, 1, rkind, lane);
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("needs 2 GPUs\n"); return 0; }
  const int64_t L = 4ll << 30, R = 1ll << 30;
  uint4 *loc[2], *lout[2], *rbuf[2];
  Ctl* ctl[2];
  cudaStream_t st[2];
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&loc[g], L));
    CK(cudaMemset(loc[g], 1, L));
    CK(cudaMalloc(&lout[g], L / 2));
    CK(cudaMalloc(&rbuf[g], R));
    CK(cudaMemset(rbuf[g], 1, R));
    CK(cudaMalloc(&ctl[g], sizeof(Ctl)));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
  }
  const char* kinds[] = {"read", "write", "read+write", "read+write_half"};
  auto run = [&](int mode, int ns, int lkind, int rkind, const char* name) {
    for (int rep = 0; rep < 3; ++rep) {
      Ctl h{};
      h.t0 = ~0ull;
      for (int g = 0; g < 2; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaMemcpy(ctl[g], &h, sizeof(h), cudaMemcpyHostToDevice));
        CK(cudaDeviceSynchronize());
      }
      for (int g = 0; g < 2; ++g) {
        CK(cudaSetDevice(g));
        k_mix<<<296, 512, 0, st[g]>>>(loc[g], lout[g], L, rbuf[1 - g], R, ctl[g], mode, ns, lkind, rkind);
      }
      Ctl r[2];
      for (int g = 0; g < 2; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaStreamSynchronize(st[g]));
        CK(cudaMemcpy(&r[g], ctl[g], sizeof(Ctl), cudaMemcpyDeviceToHost));
      }
      if (rep == 2) {
        const double tl = r[0].done_ns[0] ? (r[0].done_ns[0] - r[0].t0) / 1e3 : 0;
        const double tr = r[0].done_ns[1] ? (r[0].done_ns[1] - r[0].t0) / 1e3 : 0;
        printf("{\"mode\": \"%s\", \"remote_sms\": %d, \"local\": \"%s\", \"remote\": \"%s\", \"local_us\": %.1f, "
               "\"local_read_gbs\": %.0f, \"remote_us\": %.1f, \"remote_gbs\": %.0f}\n",
               name, ns, kinds[lkind], kinds[rkind], tl, tl > 0 ? L / tl / 1e3 : 0, tr, tr > 0 ? R / tr / 1e3 : 0);
        fflush(stdout);
      }
    }
  };
  for (int lk : {0, 3}) {
    run(0, 0, lk, 0, "local_only");
    for (int rk : {0, 1, 2}) {
      run(1, 0, lk, rk, "remote_only");
      run(2, 0, lk, rk, "mixed_in_sm");
      run(3, 24, lk, rk, "split_by_sm");
    }
  }
  return 0;
}
