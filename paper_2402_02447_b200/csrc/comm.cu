// H1 across ranks, native: per-bucket K1 on the compute stream, ncclAllReduce
// (average) of each clipped bucket on a communication stream, event-chained
// bucket by bucket — the whole step is one C call (no per-bucket Python /
// c10d overhead) and is CUDA-graph capturable.
//
// Reference semantics: sync_bucketwise (gradsync.py:148-162) with rank r as
// worker row r: clip each worker's bucket at c/sqrt(B) (local, no norm
// collective), then the mean over workers (allreduce_mean, :119-128), buckets
// in reverse order (:157).  NCCL's reduction order differs from the
// reference's pairwise tree (within tolerance).
//
// libnccl.so.2 is dlopen'ed: the copy torch already loaded (RTLD_NOLOAD), else
// the path the caller passes (the nvidia-nccl wheel), so the library itself
// has no link-time NCCL dependency.
#include "common.cuh"

#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <vector>

namespace b2 {
namespace {

typedef struct {
  char internal[128];
} NcclUid;
typedef void* NcclCommT;
typedef int (*PGetUid)(NcclUid*);
typedef int (*PInitRank)(NcclCommT*, int, NcclUid, int);
typedef int (*PDestroy)(NcclCommT);
typedef int (*PAllReduce)(const void*, void*, size_t, int, int, NcclCommT, cudaStream_t);
typedef const char* (*PErr)(int);

constexpr int kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclBfloat16 = 9;  // nccl.h:307-309
constexpr int kNcclAvg = 4;  // ncclAvg, nccl.h:286

struct Nccl {
  void* h = nullptr;
  PGetUid get_uid = nullptr;
  PInitRank init_rank = nullptr;
  PDestroy destroy = nullptr;
  PAllReduce all_reduce = nullptr;
  PErr err = nullptr;
};

int load_nccl(const char* path, Nccl& n) {
  static std::mutex mu;
  static Nccl cached;
  std::lock_guard<std::mutex> lock(mu);
  if (!cached.h) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h && path && path[0]) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    B2_REQUIRE(h, B2_ERR_CUDA, "cannot load libnccl.so.2 (%s)", dlerror());
    cached.h = h;
    cached.get_uid = (PGetUid)dlsym(h, "ncclGetUniqueId");
    cached.init_rank = (PInitRank)dlsym(h, "ncclCommInitRank");
    cached.destroy = (PDestroy)dlsym(h, "ncclCommDestroy");
    cached.all_reduce = (PAllReduce)dlsym(h, "ncclAllReduce");
    cached.err = (PErr)dlsym(h, "ncclGetErrorString");
    B2_REQUIRE(cached.get_uid && cached.init_rank && cached.destroy && cached.all_reduce && cached.err,
               B2_ERR_CUDA, "libnccl.so.2 lacks the expected symbols");
  }
  n = cached;
  return B2_OK;
}

}  // namespace
}  // namespace b2

struct b2_comm {
  b2::Nccl nccl;
  b2::NcclCommT comm = nullptr;
  int nranks = 0, rank = 0;
  std::vector<cudaEvent_t> events;  // one per bucket slot, reused every step
};

using namespace b2;

#define B2_NCCL(n, expr)                                                  \
  do {                                                                    \
    int _r = (expr);                                                      \
    B2_REQUIRE(_r == 0, B2_ERR_CUDA, "%s: %s", #expr, (n).err(_r));       \
  } while (0)

extern "C" int b2_nccl_unique_id(void* uid128, const char* libnccl_path) {
  B2_REQUIRE(uid128, B2_ERR_INVALID, "uid buffer is NULL");
  Nccl n;
  int rc = load_nccl(libnccl_path, n);
  if (rc != B2_OK) return rc;
  B2_NCCL(n, n.get_uid(reinterpret_cast<NcclUid*>(uid128)));
  return B2_OK;
}

extern "C" int b2_comm_create(b2_comm** out, int nranks, int rank, const void* uid128,
                              const char* libnccl_path) {
  B2_REQUIRE(out && uid128, B2_ERR_INVALID, "NULL argument");
  B2_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, B2_ERR_INVALID, "bad rank %d of %d", rank, nranks);
  b2_comm* c = new b2_comm();
  int rc = load_nccl(libnccl_path, c->nccl);
  if (rc != B2_OK) {
    delete c;
    return rc;
  }
  NcclUid uid;
  memcpy(&uid, uid128, sizeof(uid));
  int r = c->nccl.init_rank(&c->comm, nranks, uid, rank);
  if (r != 0) {
    set_error("ncclCommInitRank: %s", c->nccl.err(r));
    delete c;
    return B2_ERR_CUDA;
  }
  c->nranks = nranks;
  c->rank = rank;
  *out = c;
  return B2_OK;
}

extern "C" int b2_comm_destroy(b2_comm* c) {
  if (!c) return B2_OK;
  for (cudaEvent_t e : c->events) cudaEventDestroy(e);
  int r = c->comm ? c->nccl.destroy(c->comm) : 0;
  delete c;
  B2_REQUIRE(r == 0, B2_ERR_CUDA, "ncclCommDestroy failed");
  return B2_OK;
}

extern "C" int b2_allreduce_avg(b2_comm* c, void* buf, int64_t n, int dtype, void* stream) {
  B2_REQUIRE(c && buf && n >= 0, B2_ERR_INVALID, "bad allreduce arguments");
  const int dt = dtype == B2_BF16 ? kNcclBfloat16 : dtype == B2_F64 ? kNcclFloat64 : kNcclFloat32;
  B2_NCCL(c->nccl, c->nccl.all_reduce(buf, buf, (size_t)n, dt, kNcclAvg, c->comm, (cudaStream_t)stream));
  return B2_OK;
}

extern "C" int b2_bucket_clip_allreduce(b2_comm* c, const void* in, int in_dtype, void* out, int out_dtype,
                                        const int64_t* seg_off, const int64_t* seg_len, int nseg, double limit,
                                        double* norms, int32_t* nonfinite, void* workspace,
                                        size_t workspace_bytes, void* stream, void* comm_stream) {
  B2_REQUIRE(c && out && seg_off && seg_len, B2_ERR_INVALID, "NULL argument");
  B2_REQUIRE(stream != comm_stream || stream == nullptr, B2_ERR_INVALID, "use a separate comm stream");
  while ((int)c->events.size() < nseg) {
    cudaEvent_t e;
    B2_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->events.push_back(e);
  }
  const int dt = out_dtype == B2_BF16 ? kNcclBfloat16 : out_dtype == B2_F64 ? kNcclFloat64 : kNcclFloat32;
  const size_t esz = out_dtype == B2_BF16 ? 2 : out_dtype == B2_F64 ? 8 : 4;
  for (int s = 0; s < nseg; ++s) {
    // K1 for this bucket (clip into the comm buffer at the same offset)
    int rc = b2_bucket_clip_cast(in, in_dtype, out, out_dtype, seg_off + s, seg_off + s, seg_len + s, 1, limit,
                                 1.0, norms ? norms + s : nullptr, nullptr, nonfinite ? nonfinite + s : nullptr,
                                 workspace, workspace_bytes, 0, stream);
    if (rc != B2_OK) return rc;
    B2_CHECK(cudaEventRecord(c->events[s], (cudaStream_t)stream));
    B2_CHECK(cudaStreamWaitEvent((cudaStream_t)comm_stream, c->events[s], 0));
    char* buf = static_cast<char*>(out) + seg_off[s] * esz;
    B2_NCCL(c->nccl, c->nccl.all_reduce(buf, buf, (size_t)seg_len[s], dt, kNcclAvg, c->comm,
                                        (cudaStream_t)comm_stream));
  }
  return B2_OK;
}
