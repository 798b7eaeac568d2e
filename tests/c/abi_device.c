/* A plain-C caller of the device entry points (tests/test_gpu_c_abi.py builds and runs it).
 * Reads inputs written by the test from DIR, runs K1 (b2_bucket_clip_cast), K2
 * (b2_strata_partition) and K3 (b2_presort_deal) on cudaMalloc'd buffers through
 * include/b2ddp.h only, and writes the outputs back to DIR for the oracle check.
 *   usage: abi_device DIR n_grad n_len nseg seg_len lanes */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "b2ddp.h"

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                   \
      return 2;                                                                  \
    }                                                                            \
  } while (0)
#define B2(x)                                                                    \
  do {                                                                           \
    int rc_ = (x);                                                               \
    if (rc_ != B2_OK) {                                                          \
      fprintf(stderr, "%s: rc %d: %s\n", #x, rc_, b2_last_error());              \
      return 3;                                                                  \
    }                                                                            \
  } while (0)

static void* slurp(const char* dir, const char* name, size_t bytes) {
  char path[4096];
  snprintf(path, sizeof path, "%s/%s", dir, name);
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  void* p = malloc(bytes);
  if (fread(p, 1, bytes, f) != bytes) { free(p); p = NULL; }
  fclose(f);
  return p;
}

static int spill(const char* dir, const char* name, const void* p, size_t bytes) {
  char path[4096];
  snprintf(path, sizeof path, "%s/%s", dir, name);
  FILE* f = fopen(path, "wb");
  if (!f) return 1;
  size_t w = fwrite(p, 1, bytes, f);
  fclose(f);
  return w != bytes;
}

int main(int argc, char** argv) {
  if (argc != 7) return 1;
  const char* dir = argv[1];
  const int64_t n = atoll(argv[2]), m = atoll(argv[3]), nseg = atoll(argv[4]);
  const int seg_len = atoi(argv[5]), lanes = atoi(argv[6]);
  cudaStream_t st;
  CK(cudaStreamCreate(&st));

  /* ---- K1: three buckets of a flat fp32 gradient, walked in reverse, clipped at c/sqrt(3) */
  float* hg = (float*)slurp(dir, "grad.bin", n * 4);
  if (!hg) return 4;
  float *dg, *dout;
  double* dnorm;
  CK(cudaMalloc((void**)&dg, n * 4));
  CK(cudaMalloc((void**)&dout, n * 4));
  CK(cudaMalloc((void**)&dnorm, 3 * sizeof(double)));
  CK(cudaMemcpy(dg, hg, n * 4, cudaMemcpyHostToDevice));
  const size_t wsb = b2_clip_workspace_bytes();
  void* ws;
  CK(cudaMalloc(&ws, wsb));
  B2(b2_clip_workspace_init(ws, wsb, st));
  const int64_t b1 = n / 3, b2 = 2 * (n / 3);
  const int64_t off[3] = {b2, b1, 0}, len[3] = {n - b2, b2 - b1, b1};
  B2(b2_bucket_clip_cast(dg, B2_F32, dout, B2_F32, off, off, len, 3, 1.0 / 1.7320508075688772, 1.0, dnorm, NULL,
                         NULL, ws, wsb, 0, st));
  float* hout = (float*)malloc(n * 4);
  double hnorm[3];
  CK(cudaMemcpyAsync(hout, dout, n * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hnorm, dnorm, sizeof hnorm, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (spill(dir, "clip_out.bin", hout, n * 4) || spill(dir, "clip_norms.bin", hnorm, sizeof hnorm)) return 5;

  /* ---- K2: stratify m lengths over the default boundaries */
  int32_t* hl = (int32_t*)slurp(dir, "lens.bin", m * 4);
  if (!hl) return 4;
  int32_t *dl, *dids;
  int64_t *dcnt, *dbad;
  CK(cudaMalloc((void**)&dl, m * 4));
  CK(cudaMalloc((void**)&dids, m * 4));
  CK(cudaMalloc((void**)&dcnt, 4 * 8));
  CK(cudaMalloc((void**)&dbad, 8));
  CK(cudaMemcpy(dl, hl, m * 4, cudaMemcpyHostToDevice));
  const size_t swb = b2_strata_workspace_bytes(m);
  void* sws;
  CK(cudaMalloc(&sws, swb));
  const int32_t bounds[4] = {128, 256, 384, 512};
  B2(b2_strata_partition(dl, NULL, m, bounds, 4, dids, dcnt, dbad, sws, swb, st));
  int32_t* hids = (int32_t*)malloc(m * 4);
  int64_t hcnt[5];
  CK(cudaMemcpyAsync(hids, dids, m * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hcnt, dcnt, 4 * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hcnt + 4, dbad, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (spill(dir, "strata_ids.bin", hids, m * 4) || spill(dir, "strata_counts.bin", hcnt, sizeof hcnt)) return 5;

  /* ---- K3: sort + snake deal of nseg pools of seg_len samples */
  const int64_t np = nseg * seg_len;
  int32_t* hpi = (int32_t*)slurp(dir, "pool_ids.bin", np * 4);
  int32_t* hpl = (int32_t*)slurp(dir, "pool_lens.bin", np * 4);
  if (!hpi || !hpl) return 4;
  int32_t *dpi, *dpl, *dpo;
  int64_t *dtok, *dpbad;
  CK(cudaMalloc((void**)&dpi, np * 4));
  CK(cudaMalloc((void**)&dpl, np * 4));
  CK(cudaMalloc((void**)&dpo, np * 4));
  CK(cudaMalloc((void**)&dtok, nseg * lanes * 8));
  CK(cudaMalloc((void**)&dpbad, 8));
  CK(cudaMemcpy(dpi, hpi, np * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dpl, hpl, np * 4, cudaMemcpyHostToDevice));
  B2(b2_presort_deal(dpi, dpl, nseg, seg_len, lanes, B2_SCAN_SNAKE, 512, 1 << 24, dpo, NULL, dtok, dpbad, st));
  int32_t* hpo = (int32_t*)malloc(np * 4);
  int64_t* htok = (int64_t*)malloc(nseg * lanes * 8);
  CK(cudaMemcpyAsync(hpo, dpo, np * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(htok, dtok, nseg * lanes * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (spill(dir, "deal_ids.bin", hpo, np * 4) || spill(dir, "deal_tokens.bin", htok, nseg * lanes * 8)) return 5;
  printf("ok %s\n", b2_version());
  return 0;
}
