/*
 * c_abi_demo.c — the LARS library driven from plain C through include/lars.h (no Python, no torch).
 *
 *   gcc -O2 -I include examples/c_abi_demo.c -L paper_1903_12650_b200 -llars_b200 \
 *       -Wl,-rpath,$PWD/paper_1903_12650_b200 -o build/c_abi_demo            (host-only: plan + schedule)
 *   add -DWITH_CUDA -I /usr/local/cuda/include -L /usr/local/cuda/lib64 -lcudart to also run one step
 *
 * Host-only mode plans the `tiny` layout (BASELINE.json configs[0]), prints the schedule of PAPER.md:210-211
 * (16 updates/epoch, 1,440 updates, 80 warm-up iterations) and checks the error codes of the boundary.
 * With WITH_CUDA and argv[1] = "gpu" it also runs one lars_step at t = 80 on inputs given by closed-form
 * formulas (so tests/test_c_abi.py can recompute them with the oracle) and prints w, m and the norms.
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "lars.h"

#ifdef WITH_CUDA
#include <cuda_runtime.h>
#endif

#define CHECK(expr)                                                                   \
  do {                                                                                \
    lars_status_t st_ = (expr);                                                       \
    if (st_ != LARS_OK) {                                                             \
      fprintf(stderr, "%s failed: %s (%d)\n", #expr, lars_strerror(st_), (int)st_);  \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

#ifdef WITH_CUDA
/* Deterministic, exactly representable inputs (element i of tensor l: small integers times powers of two),
 * recomputed bit for bit by tests/test_c_abi.py. */
static float w_of(int l, long i) { return (float)(((i * 37 + l * 11) % 2001) - 1000) * 0x1p-16f + (l == 2 ? 1.0f : 0.0f); }
static float g_of(int l, long i) { return (float)(((i * 53 + l * 7) % 1999) - 999) * 0x1p-20f; }
static float m_of(int l, long i) { return (float)(((i * 29 + l * 3) % 997) - 498) * 0x1p-24f; }
#endif

int main(int argc, char** argv) {
  const lars_tensor_t tiny[3] = {{9408, LARS_KIND_WEIGHT, 147}, {999, LARS_KIND_WEIGHT, 999}, {64, LARS_KIND_BN_GAMMA, 64}};
  lars_hparams_t hp;
  lars_hparams_default(&hp);
  hp.base_lr = 32.0;
  hp.grad_dtype = LARS_F32;
  printf("version %s\n", lars_version());

  /* boundary errors are returned synchronously */
  lars_handle_t bad = NULL;
  lars_tensor_t zero = {0, LARS_KIND_WEIGHT, 0};
  printf("err_layout %d\n", (int)lars_init(&zero, 1, &hp, -1, &bad));
  lars_hparams_t nolr = hp;
  nolr.base_lr = 0.0;
  printf("err_no_base_lr %d\n", (int)lars_init(tiny, 3, &nolr, -1, &bad));

  int gpu = argc > 1 && strcmp(argv[1], "gpu") == 0;
  lars_handle_t h = NULL;
  CHECK(lars_init(tiny, 3, &hp, gpu ? 0 : -1, &h));
  int64_t ipe, T, W, offs[3], padded;
  CHECK(lars_schedule(h, &ipe, &T, &W));
  CHECK(lars_layout(h, offs, &padded));
  printf("schedule ipe=%lld T=%lld W=%lld\n", (long long)ipe, (long long)T, (long long)W);
  printf("layout %lld %lld %lld padded=%lld\n", (long long)offs[0], (long long)offs[1], (long long)offs[2],
         (long long)padded);
  const int64_t its[5] = {0, 79, 80, 719, 1439};
  for (int k = 0; k < 5; ++k) {
    double lr;
    CHECK(lars_lr_at(h, its[k], &lr));
    printf("lr %lld %.17g\n", (long long)its[k], lr);
  }
  double lr;
  printf("err_iter_range %d\n", (int)lars_lr_at(h, T, &lr));

#ifdef WITH_CUDA
  if (gpu) {
    const size_t n = (size_t)padded;
    float *hw = calloc(n, 4), *hg = calloc(n, 4), *hm = calloc(n, 4);
    for (int l = 0; l < 3; ++l)
      for (long i = 0; i < tiny[l].numel; ++i) {
        hw[offs[l] + i] = w_of(l, i);
        hg[offs[l] + i] = g_of(l, i);
        hm[offs[l] + i] = m_of(l, i);
      }
    float *dw, *dg, *dm;
    if (cudaMalloc((void**)&dw, n * 4) || cudaMalloc((void**)&dg, n * 4) || cudaMalloc((void**)&dm, n * 4)) return 2;
    cudaMemcpy(dw, hw, n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dg, hg, n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dm, hm, n * 4, cudaMemcpyHostToDevice);
    CHECK(lars_step(h, dw, dg, dm, 80, NULL));
    int32_t skipped = -1;
    CHECK(lars_last_step_skipped(h, &skipped));
    double wn[3], gn[3], lam[3], coef[3];
    CHECK(lars_last_norms(h, wn, gn, lam, coef));
    cudaMemcpy(hw, dw, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hm, dm, n * 4, cudaMemcpyDeviceToHost);
    printf("skipped %d\n", (int)skipped);
    for (int l = 0; l < 3; ++l) printf("norms %d %.17g %.17g %.17g %.9g\n", l, wn[l], gn[l], lam[l], coef[l]);
    for (int l = 0; l < 3; ++l)
      for (long i = 0; i < tiny[l].numel; i += 97)
        printf("wm %d %ld %.9g %.9g\n", l, i, (double)hw[offs[l] + i], (double)hm[offs[l] + i]);
    cudaFree(dw);
    cudaFree(dg);
    cudaFree(dm);
    free(hw);
    free(hg);
    free(hm);
  }
#endif
  CHECK(lars_destroy(h));
  printf("done\n");
  return 0;
}
