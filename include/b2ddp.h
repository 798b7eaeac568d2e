/*
 * b2ddp.h — C-ABI of the B200-native hot paths of arXiv 2402.02447.
 *
 * The reference (ddpsim 0.1.0, /root/reference/pkg/src/ddpsim) is pure
 * Python; its own boundary is the Python API re-exported at
 * __init__.py:14-81.  Each entry point below replaces the inner loop of one
 * reference function; the Python package paper_2402_02447_b200 keeps the
 * reference names/signatures/errors on top of it (ctypes), and
 * INTEGRATION.md shows the binding a maintainer would add.
 *
 * Conventions (all entry points):
 *   - plain C types only; device buffers are caller-owned `void*`/typed
 *     pointers; host arrays are marked [host];
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream);
 *   - no allocation, no host synchronisation inside; kernels are enqueued
 *     on `stream` and the call returns;
 *   - return 0 (B2_OK) or a B2_ERR_* code; b2_last_error() returns a
 *     thread-local message for the last failing call on this thread.
 */
#ifndef B2DDP_H_
#define B2DDP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define B2_OK 0
#define B2_ERR_INVALID 1      /* bad argument (pointer, size, dtype)          */
#define B2_ERR_CUDA 2         /* CUDA runtime error (message has details)     */
#define B2_ERR_INDIVISIBLE 3  /* seg_len % lanes != 0 (balance.py:65-66)       */
#define B2_ERR_UNSUPPORTED 4  /* size beyond this build's limits              */

/* element types */
#define B2_F32 0
#define B2_BF16 1
#define B2_F64 2

/* scan patterns (balance.py:21-23) */
#define B2_SCAN_RASTER 0
#define B2_SCAN_SNAKE 1

const char* b2_version(void);
const char* b2_last_error(void);

/* ------------------------------------------------------------------------
 * H1 — bucket-wise clip before allreduce
 * ---------------------------------------------------------------------- */

/* Bytes of scratch one b2_bucket_clip_cast caller (one stream) needs.  The
 * buffer must be zeroed once (b2_clip_workspace_init); every launch leaves it
 * zeroed again on exit, so it is reusable without re-initialisation. */
size_t b2_clip_workspace_bytes(void);
int b2_clip_workspace_init(void* workspace, size_t workspace_bytes, void* stream);

/* K1 — fused per-bucket L2 norm + clip coefficient + scale/cast.
 *
 * Replaces clip_by_norm (gradsync.py:106-116) applied per (worker, bucket)
 * inside sync_bucketwise (gradsync.py:157-160).  For every segment s (in the
 * given order — pass buckets reversed to mirror gradsync.py:157):
 *     norm_s  = sqrt(sum in[in_off[s] .. +len[s])^2)      (fp64 accumulation)
 *     coef_s  = norm_s >= limit ? limit / norm_s : 1      (inclusive, :114)
 *     out[out_off[s] + i] = cast(in[in_off[s] + i] * coef_s * post_scale)
 * `out` may be NULL (norm/coef only).  `norms`, `coefs` (fp64) and `nonfinite`
 * (int32, 1 if the segment holds inf/nan — gradsync.py:111-112) are optional
 * device arrays of nseg entries.  in_dtype: B2_F32|B2_F64; out_dtype:
 * B2_F32|B2_BF16|B2_F64.  post_scale folds 1/K in when the following
 * collective is a plain sum.  ctas_per_sm <= 0 picks the default.
 * seg_in_off/seg_out_off/seg_len are [host] arrays of nseg int64.
 * A lone segment with an output (the DDP-hook / reducer shape) is a
 * programmatic dependent launch: it may start under the previous kernel of
 * `stream` and waits for it before reading (B2_CLIP_PDL=0: a plain
 * cooperative launch). */
int b2_bucket_clip_cast(const void* in, int in_dtype, void* out, int out_dtype,
                        const int64_t* seg_in_off, const int64_t* seg_out_off,
                        const int64_t* seg_len, int nseg, double limit, double post_scale,
                        double* norms, double* coefs, int32_t* nonfinite, void* workspace,
                        size_t workspace_bytes, int ctas_per_sm, void* stream);

/* K1b — single-process K-worker mean of clipped buckets.
 *
 * Replaces allreduce_mean (gradsync.py:119-128) over the clipped worker
 * slices of sync_bucketwise (:158-161): for element i of bucket b,
 *     out[i] = pairwise_tree_k( G[k*ld + i] * coef[k*B + b] ) / K
 * with the reference's tree (rounds merge (0,1),(2,3).., odd tail carried).
 * A coefficient of exactly 1 leaves the element untouched (clip_by_norm
 * returns g itself, :116).  `bounds` is a [host] array of B+1 bucket edges
 * (bounds[0] = 0, bounds[B] = D).  in_dtype B2_F32|B2_F64, out_dtype
 * B2_F32|B2_F64; any K >= 1. */
int b2_weighted_mean(const void* G, int in_dtype, int64_t K, int64_t D, int64_t ld,
                     const double* coef, const int64_t* bounds, int B, void* out,
                     int out_dtype, void* stream);

/* ------------------------------------------------------------------------
 * H1 across ranks (one process per GPU): NCCL, loaded at run time
 * ---------------------------------------------------------------------- */

typedef struct b2_comm b2_comm;

/* 128-byte ncclUniqueId from rank 0 (distribute it with any side channel,
 * e.g. the torch.distributed store).  libnccl_path may be NULL: the
 * libnccl.so.2 already loaded in the process (torch's) is used. */
int b2_nccl_unique_id(void* uid128, const char* libnccl_path);
int b2_comm_create(b2_comm** comm, int nranks, int rank, const void* uid128, const char* libnccl_path);
int b2_comm_destroy(b2_comm* comm);

/* In-place ncclAllReduce(avg) of n elements (B2_F32 | B2_BF16 | B2_F64). */
int b2_allreduce_avg(b2_comm* comm, void* buf, int64_t n, int dtype, void* stream);

/* One H1 step (sync_bucketwise, gradsync.py:148-162, rank r = worker row r):
 * for every bucket s in the given order (pass them reversed, :157): K1 clips
 * in[seg_off[s] .. +seg_len[s]) at `limit` into out at the same offset on
 * `stream`, an event chains `comm_stream` after it, and ncclAllReduce(avg)
 * reduces that bucket of `out` on `comm_stream` — bucket s's transfer
 * overlaps the clip of s+1.  The caller joins comm_stream before reading
 * `out`.  `norms`/`nonfinite` (device, nseg entries) are optional.  Graph
 * capturable. */
int b2_bucket_clip_allreduce(b2_comm* comm, const void* in, int in_dtype, void* out, int out_dtype,
                             const int64_t* seg_off, const int64_t* seg_len, int nseg, double limit,
                             double* norms, int32_t* nonfinite, void* workspace, size_t workspace_bytes,
                             void* stream, void* comm_stream);

/* Fused H1 step over NVLink peer memory (no NCCL), K4: ONE persistent
 * cooperative kernel per rank.  CTAs on the clip SMs compute each bucket's
 * norm and clip + cast it to bf16 into this rank's symmetric stage buffer;
 * CTAs on the comm SMs (64 at N=2, 48 at N=4, 32 with NVLS; B2_COMM_SMS
 * overrides) run a two-shot allreduce of each bucket as soon as every rank
 * has staged it (this rank reduces its 1/N slice from every stage in fixed
 * rank order and writes the mean into every stage).  Replaces, for rank r =
 * worker row r, sync_bucketwise's per-bucket clip + allreduce_mean
 * (gradsync.py:148-162, :119-128).  stages[q] / flags[q] ([host] arrays of nranks device pointers) are
 * rank q's bf16 stage (D elements, buckets at seg_off) and its flag area
 * (b2_p2p_flag_bytes(), zeroed once) as mapped in this process (b2_ipc_*).
 * On return of the launch (stream order) stages[rank] holds the averaged,
 * clipped gradient.  All ranks must issue the same calls in the same order;
 * a cross-GPU wait longer than b2_get_spin_timeout() seconds traps (default
 * 600 s; B2_SPIN_TIMEOUT_S or b2_set_spin_timeout, 0 = wait forever).  nranks <= 8, nseg <= 128, buckets
 * 8-element aligned.  The workspace (b2_clip_workspace_bytes) also carries
 * the launch epoch, so the call is CUDA-graph replayable. */
/* NVLS flavour: same contract, but the reduce of each slice is one
 * multimem.ld_reduce (fp32 accumulate in the NVSwitch) + one multimem.st
 * (broadcast) on `mc_stage`, the multicast address of the stage buffers
 * (e.g. torch symmetric memory's multicast_ptr); stages are scaled by 1/N
 * before staging so the in-switch sum is the mean. */
int b2_bucket_clip_allreduce_nvls(const void* in, void* const* stages, void* mc_stage, uint32_t* const* flags,
                                  int nranks, int rank, const int64_t* seg_off, const int64_t* seg_len, int nseg,
                                  double limit, double* norms, int32_t* nonfinite, void* workspace,
                                  size_t workspace_bytes, void* stream);
/* Bound, in seconds, on every cross-GPU wait of the fused kernels (0 = wait
 * forever).  Process-wide; read at each launch.  Default 600 s, or the
 * B2_SPIN_TIMEOUT_S environment variable. */
int b2_set_spin_timeout(double seconds);
double b2_get_spin_timeout(void);
size_t b2_p2p_flag_bytes(void);
int b2_ipc_export(const void* dev_ptr, void* handle64, int64_t* offset);
int b2_ipc_import(const void* handle64, int64_t offset, void** base, void** dev_ptr);
int b2_ipc_close(void* base);
int b2_bucket_clip_allreduce_p2p(const void* in, void* const* stages, uint32_t* const* flags, int nranks, int rank,
                                 const int64_t* seg_off, const int64_t* seg_len, int nseg, double limit,
                                 double* norms, int32_t* nonfinite, void* workspace, size_t workspace_bytes,
                                 void* stream);
/* The P2P form with a chosen stage dtype: B2_BF16 (the throughput form above)
 * or B2_F32 — the parity mode: the clipped buckets are staged and averaged
 * in fp32 (sum in fixed rank order, x 1/N), so the result meets the 1e-5
 * relative contract of sync_bucketwise across ranks (gradsync.py:148-162)
 * at twice the NVLink bytes.  stages[q] then hold D fp32 elements. */
int b2_bucket_clip_allreduce_p2p_dtype(const void* in, void* const* stages, int stage_dtype, uint32_t* const* flags,
                                       int nranks, int rank, const int64_t* seg_off, const int64_t* seg_len,
                                       int nseg, double limit, double* norms, int32_t* nonfinite, void* workspace,
                                       size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * H2 — stratified local presort
 * ---------------------------------------------------------------------- */

size_t b2_strata_workspace_bytes(int64_t n);

/* K2 — stratum histogram + stable partition.
 *
 * Replaces stratify (strata.py:61-83): stratum of sample i is
 * searchsorted(bounds, len[i], 'left') (:74); ids are emitted grouped by
 * stratum, input order kept inside each stratum (:82).  `ids` may be NULL
 * (ids = 0..n-1).  Outputs (device): ids_out[n], counts[nb] (int64), and
 * bad[1] (int64) = first index i whose length is > bounds[nb-1] or < 1, or
 * -1 (so the wrapper raises naming that sample's id, :75-80); when bad >= 0
 * ids_out and counts are unspecified (the reference raises there).  `bounds`
 * is a [host] array of nb strictly ascending values >= 1, nb <= 16.  Three
 * launches: per-tile stratum codes + counts, a per-shard scan, the scatter
 * (8.5 B/key of traffic for 8 B/key algorithmic). */
int b2_strata_partition(const int32_t* lengths, const int32_t* ids, int64_t n,
                        const int32_t* bounds, int nb, int32_t* ids_out, int64_t* counts,
                        int64_t* bad, void* workspace, size_t workspace_bytes, void* stream);

/* K2 over many rank shards in one pass (three launches in total): shard g is
 * lengths[shard_off[g] .. shard_off[g+1]) ([host] offsets, nshard <= 64) and
 * is stratified on its own, exactly like stratify() on that shard; ids_out
 * uses the same offsets, counts is [nshard][nb], bad[g] is the shard-local
 * index of its first bad sample or -1.  ids NULL -> shard-local indices.
 * Workspace: b2_strata_workspace_bytes(total samples). */
int b2_strata_partition_shards(const int32_t* lengths, const int32_t* ids, const int64_t* shard_off, int nshard,
                               const int32_t* bounds, int nb, int32_t* ids_out, int64_t* counts, int64_t* bad,
                               void* workspace, size_t workspace_bytes, void* stream);

/* Draws (host, CPU) — bit-exact native port of the reference's stratified
 * draws: numpy's SeedSequence -> PCG64 -> Generator.choice(replace=False)
 * (tail shuffle / Floyd), descending swap-pop and closest-boundary borrowing
 * of draw_batch (strata.py:113-161), and derive_seed (seeding.py:18-21).
 * A b2_draw_state owns mutable per-stratum id pools (the Strata buckets);
 * draws consume them like the reference.  Global exhaustion returns
 * B2_ERR_INVALID with the reference's stratum number / shortfall. */
typedef struct b2_draw_state b2_draw_state;
uint64_t b2_derive_seed(uint64_t seed, const uint64_t* key, int nkey);
int b2_draws_create(b2_draw_state** st, const int64_t* pool_ids, const int64_t* pool_sizes, int nstrata,
                    const int64_t* bounds);
int b2_draws_destroy(b2_draw_state* st);
int64_t b2_draws_remaining(const b2_draw_state* st, int stratum);
int b2_draw_batch(b2_draw_state* st, const int64_t* counts, uint64_t seed, int64_t* out, int* err_stratum,
                  int64_t* err_short);
/* steps t = 0..nsteps-1 with seed derive_seed(base_seed, key..., first_step + t)
 * (nkey <= 7); out is [nsteps][sum(counts)]; *done = completed steps. */
int b2_draw_epoch(b2_draw_state* st, const int64_t* counts, uint64_t base_seed, const uint64_t* key, int nkey,
                  int64_t first_step, int64_t nsteps, int64_t* out, int64_t* done, int* err_stratum,
                  int64_t* err_short);

/* K3 — per-pool stable sort by (-length, id) + raster/snake deal.
 *
 * Replaces _sorted_desc (balance.py:73-75) + _deal (:59-70) +
 * _from_per_gpu (:54-56) as applied per node by assign_local_presort
 * (:158-184) and, with one pool, by assign_global_presort (:83-88).
 * ids/lens hold nseg consecutive pools of seg_len samples (each pool is the
 * node's GPU draws concatenated in GPU order).  Outputs (device):
 *   out_ids[nseg][lanes][seg_len/lanes]   (lane g's samples in deal order)
 *   out_pos[nseg][lanes][seg_len/lanes] (may be NULL): flat input index of
 *          each dealt sample (equal keys keep input order, i.e. stable)
 *   tokens [nseg][lanes]  (int64 token sums, may be NULL)
 *   bad[1] (int64, may be NULL): first flat index with len outside
 *          [1, max_len] or id outside [0, max_id], else -1.
 * max_len/max_id bound the key width (e.g. the last stratum boundary and the
 * corpus size - 1).  seg_len % lanes != 0 -> B2_ERR_INDIVISIBLE.
 * seg_len <= 4096. */
int b2_presort_deal(const int32_t* ids, const int32_t* lens, int64_t nseg, int seg_len,
                    int lanes, int scan, int32_t max_len, int32_t max_id, int32_t* out_ids,
                    int32_t* out_pos, int64_t* tokens, int64_t* bad, void* stream);

/* K5 — the same sort + deal for pools of ANY size: a device-wide stable LSD
 * radix sort (onesweep: one upsweep histogram launch, then one
 * decoupled-look-back pass per <= 9-bit digit) over all nseg pools at once.
 * Replaces _sorted_desc + _deal + _from_per_gpu (balance.py:54-75) where a
 * pool is larger than one CTA can sort: assign_global_presort (:83-88) over a
 * whole batch, and the "stable per-rank radix sort on length keys" over a
 * whole rank shard (lanes = 1: out_ids is the shard in (-len, id) order).
 * Same arguments and outputs as b2_presort_deal; seg_len <= 4096 is passed
 * to b2_presort_deal (workspace unused).  When every pool's ids are already
 * non-decreasing (a shard in id order) the id digits are skipped on the
 * device.  `workspace` (device, b2_presort_workspace_bytes(...) bytes; no
 * initialisation needed) holds the key ping-pong buffers, histograms, the
 * first pass's per-tile digit counts and bases, and look-back words.
 * seg_len < 2^30. */
size_t b2_presort_workspace_bytes(int64_t nseg, int seg_len, int32_t max_len, int32_t max_id, int with_pos);
int b2_presort_sort_deal(const int32_t* ids, const int32_t* lens, int64_t nseg, int seg_len, int lanes, int scan,
                         int32_t max_len, int32_t max_id, int32_t* out_ids, int32_t* out_pos, int64_t* tokens,
                         int64_t* bad, void* workspace, size_t workspace_bytes, void* stream);

/* Monte-Carlo balance engine, host draws.
 *
 * Replaces the per-trial draws of mcsim (mcsim.py:146-151 _draw_uniform,
 * :166-180 _stratified_matrix) under derive_rng(seed, t) (seeding.py:8-16),
 * bit-exact with numpy 2.x.  lengths holds the strata's lengths concatenated
 * (pool_sizes[k] each; one stratum = the whole corpus for NONE /
 * GLOBAL_PRESORT).  Trial first_trial + i writes out[i][b*num_gpus], the
 * (b, G) matrix row-major, b = sum(counts).  Host memory; nthreads host
 * threads.  counts[k]*num_gpus > pool_sizes[k] -> B2_ERR_INVALID (the
 * reference's "corpus exhausted within a trial"). */
int b2_mc_draw(const int32_t* lengths, const int64_t* pool_sizes, int nstrata, const int64_t* counts,
               int num_gpus, uint64_t seed, int64_t first_trial, int64_t ntrials, int nthreads, int32_t* out);

/* Monte-Carlo trial draws ON THE DEVICE: the same bit-exact draws as
 * b2_mc_draw (derive_rng(seed, t), choice(replace=False) Floyd branch +
 * shuffle), one warp per trial.  pool_lens is device memory (strata
 * concatenated), out is device [ntrials][b*num_gpus].  A stratum in numpy's
 * tail-shuffle branch (pop > 10000 and need > pop/50) -> B2_ERR_UNSUPPORTED
 * (use b2_mc_draw).  Two launches: a compact-set kernel (16-bit Floyd set,
 * twice the trials per SM) and the 32-bit kernel for the trials it could not
 * finish exactly (marked in their first output word); B2_MC_DRAW16=0 runs
 * the 32-bit kernel alone. */
int b2_mc_draw_device(const int32_t* pool_lens, const int64_t* pool_sizes, int nstrata, const int64_t* counts,
                      int num_gpus, uint64_t seed, int64_t first_trial, int64_t ntrials, int32_t* out,
                      void* stream);

/* Monte-Carlo balance engine, device side: per-trial per-GPU token counts
 * and their min/max (mcsim._trial_token_counts :182-213, _run :284-300).
 * strategy: 0 NONE, 1 STRATIFIED (column sums), 2 LOCAL_PRESORT (per-node
 * pool sorted descending + deal; b*gpus_per_node <= 512), 3 GLOBAL_PRESORT.
 * mat [ntrials][b*num_gpus] lengths in [1, max_len] (max_len <= 4096,
 * num_gpus <= 2048); counts [ntrials][num_gpus] may be NULL; mins/maxs
 * [ntrials] int64; *bad = 1 if a length was out of range.  Device memory. */
int b2_mc_token_counts(const int32_t* mat, int64_t ntrials, int b, int num_gpus, int gpus_per_node, int strategy,
                       int scan, int32_t max_len, int64_t* counts, int64_t* mins, int64_t* maxs, int32_t* bad,
                       void* stream);

#ifdef __cplusplus
}
#endif

#endif /* B2DDP_H_ */
