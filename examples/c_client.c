/* examples/c_client.c -- a plain C program linked against libhs.so through
 * include/hs.h only (no Python, no torch): the C-ABI is usable on its own.
 *
 *   gcc -std=c11 -I include -I /usr/local/cuda/include examples/c_client.c \
 *       -L paper_2505_12566_b200 -lhs -Wl,-rpath,$PWD/paper_2505_12566_b200 \
 *       -L /usr/local/cuda/lib64 -lcudart -lm -o /tmp/hs_c_client && /tmp/hs_c_client [--gpu]
 *
 * Without --gpu it exercises the host-only calls (workspace queries, grid and
 * skip-edge helpers, status strings) and the synchronous argument checks, which
 * return before any CUDA call.  With --gpu (a B200 present) it also routes one
 * tiny 3-stage cascade through hs_cascade_step with device buffers from the
 * CUDA runtime and checks the lists against a hand-worked answer. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "hs.h"

#define CHECK(c, msg) do { if (!(c)) { fprintf(stderr, "FAIL: %s\n", msg); return 1; } } while (0)

static int host_only(void) {
  CHECK(strcmp(hs_status_string(HS_ERR_NCCL), "HS_ERR_NCCL") == 0, "status string");
  CHECK(strncmp(hs_build_info(), "libhs: sm_100a", 14) == 0, "build info");
  CHECK(hs_route_compact_workspace(1000) > 0, "route workspace");
  CHECK(hs_calibrate_workspace(5, 12) > 0 && hs_calibrate_workspace(5, 15) == 0, "calibration workspace");
  CHECK(hs_peer_region_bytes(8, 1024, 0, 12) > 0 && hs_peer_region_bytes(9, 1024, 0, 12) == 0, "peer region");
  CHECK(hs_grid_size(3, 1) == 16, "grid size (B+2)^(K-1)");
  int32_t b[2];
  CHECK(hs_grid_vector(5, 3, 1, b) == HS_OK && b[0] == 1 && b[1] == 1, "grid vector");
  float e[2];
  CHECK(hs_skip_edges(0.9f, 3, 0, e) == HS_OK && fabsf(e[0] - 0.6f) < 1e-6f && fabsf(e[1] - 0.3f) < 1e-6f,
        "uniform skip edges");
  /* argument errors are reported before any launch */
  float conf[4];
  CHECK(hs_confidence(NULL, HS_BF16, 4, 1, 1, 8, NULL, NULL, 1.0f, HS_CONF_MAXPROB, HS_SEQ_NONE, conf, NULL,
                      NULL, NULL, NULL, 0, NULL, 0) == HS_ERR_INVALID_ARGUMENT, "C < 2 rejected");
  CHECK(strstr(hs_last_error(), "n_classes") != NULL, "error detail");
  CHECK(hs_confidence(NULL, HS_BF16, 4, 1, 8, 8, NULL, NULL, -1.0f, HS_CONF_MAXPROB, HS_SEQ_NONE, conf,
                      NULL, NULL, NULL, NULL, 0, NULL, 0) == HS_ERR_INVALID_ARGUMENT, "T <= 0 rejected");
  int64_t counts[2];
  CHECK(hs_route_compact(conf, 4, NULL, 1.5f, NULL, 0, NULL, NULL, 1, NULL, NULL, NULL, NULL, NULL, NULL, 0,
                         NULL, counts, NULL, 0, 0) == HS_ERR_INVALID_ARGUMENT, "threshold outside [0,1]");
  return 0;
}

/* 6 requests, 3 stages, 2-class fp32 logits chosen so that the confidences are
 * c_1 = (.9, .2, .75, .5, .7, .69) etc. are easy to reason about: here each
 * stage's row r is (x, 0) with p_max = sigmoid(|x|); thresholds t = (0.7, 0.6). */
static int gpu_cascade(void) {
  const int n = 6, K = 3;
  /* logit gaps: stage 1 accepts rows 0, 2, 4 (sigmoid(gap) >= 0.7) */
  const float gap[3][6] = {{3.0f, 0.1f, 1.5f, 0.2f, 1.0f, 0.3f},
                           {0.f, 0.1f, 0.f, 2.0f, 0.f, 1.0f},
                           {0.f, 0.0f, 0.f, 0.0f, 0.f, 0.0f}};
  const float thr[3] = {0.7f, 0.6f, 0.0f};
  float host[6 * 4];
  void *logits, *ws, *ids_in, *acc, *nxt, *cnt;
  int64_t acc_h[6], cnt_h[2], batch_h[6];
  int64_t m = n;
  size_t wsb = hs_cascade_step_workspace(n, 1);
  if (cudaMalloc(&logits, sizeof host) || cudaMalloc(&ws, wsb) || cudaMalloc(&acc, 8 * n) ||
      cudaMalloc(&nxt, 8 * n) || cudaMalloc(&cnt, 16) || cudaMalloc(&ids_in, 8 * n)) {
    fprintf(stderr, "no GPU\n");
    return 1;
  }
  cudaMemset(ws, 0, wsb);
  for (int i = 0; i < n; ++i) batch_h[i] = i;
  const int want_stage[6] = {0, 2, 0, 1, 0, 1};
  for (int k = 0; k < K; ++k) {
    for (int i = 0; i < m; ++i) {   /* row i of this stage's dense batch: request batch_h[i] */
      host[4 * i + 0] = gap[k][batch_h[i]];
      host[4 * i + 1] = 0.f;
      host[4 * i + 2] = -INFINITY;  /* padding to a 16-byte row, masked classes */
      host[4 * i + 3] = -INFINITY;
    }
    cudaMemcpy(logits, host, sizeof host, cudaMemcpyHostToDevice);
    cudaMemcpy(ids_in, batch_h, 8 * m, cudaMemcpyHostToDevice);
    hs_status_t st = hs_cascade_step(k, K, logits, HS_F32, m, 1, 4, 4, NULL, NULL, 1.0f, HS_CONF_MAXPROB,
                                     HS_SEQ_NONE, thr[k], NULL, ids_in, NULL, 0, acc, NULL, NULL, nxt, NULL,
                                     cnt, ws, wsb, NULL, 0);
    CHECK(st == HS_OK, hs_last_error());
    cudaDeviceSynchronize();
    cudaMemcpy(cnt_h, cnt, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(acc_h, acc, 8 * cnt_h[0], cudaMemcpyDeviceToHost);
    for (int j = 0; j < cnt_h[0]; ++j) CHECK(want_stage[acc_h[j]] == k, "request answered by the wrong model");
    for (int j = 1; j < cnt_h[0]; ++j) CHECK(acc_h[j] > acc_h[j - 1], "accepted list not stable");
    m = cnt_h[1];
    cudaMemcpy(batch_h, nxt, 8 * m, cudaMemcpyDeviceToHost);
  }
  CHECK(m == 0, "the last model answers everything");
  cudaFree(logits); cudaFree(ws); cudaFree(acc); cudaFree(nxt); cudaFree(cnt); cudaFree(ids_in);
  return 0;
}

int main(int argc, char** argv) {
  if (host_only()) return 1;
  if (argc > 1 && strcmp(argv[1], "--gpu") == 0 && gpu_cascade()) return 1;
  printf("c client ok\n");
  return 0;
}
