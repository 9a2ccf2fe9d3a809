/*
 * Minimal C client of the C ABI (include/kx.h), no Python: integrates the 2-D Schnakenberg
 * system of PAPER.md §3.1 with exprk3ds_real (Algorithm 1, Table 1) on the GPU and
 * prints the range of u every `report` steps.  Fixed pseudo-random initial data (an LCG here,
 * not the tests' SplitMix64 recipe).
 *
 *   build:  gcc -O2 -o build/schnakenberg_2d examples/schnakenberg_2d.c -Iinclude \
 *               -Lpaper_2310_07551_b200 -lkx -I/usr/local/cuda/include -L/usr/local/cuda/lib64 \
 *               -lcudart -Wl,-rpath,$PWD/paper_2310_07551_b200
 *   run:    build/schnakenberg_2d [n=256] [steps=6000] [T=2]
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "kx.h"

#define CHECK(x)                                                                 \
  do {                                                                           \
    kx_status s_ = (x);                                                          \
    if (s_ != KX_OK) {                                                           \
      fprintf(stderr, "%s failed (%d): %s\n", #x, (int)s_, kx_last_error(ctx)); \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

/* (delta/h^2) * FD Laplacian with ghost-point Neumann rows, column-major (R5) */
static void laplacian(double* A, int n, double L, double delta) {
  const double h = L / (n - 1), c = delta / (h * h);
  for (int i = 0; i < n * n; ++i) A[i] = 0.0;
  for (int i = 0; i < n; ++i) {
    A[i + i * n] = -2.0 * c;
    if (i == 0) A[0 + 1 * n] = 2.0 * c;
    else if (i == n - 1) A[i + (i - 1) * n] = 2.0 * c;
    else {
      A[i + (i - 1) * n] = c;
      A[i + (i + 1) * n] = c;
    }
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 256;
  const int steps = argc > 2 ? atoi(argv[2]) : 6000;
  const double T = argc > 3 ? atof(argv[3]) : 2.0;
  const long long N = (long long)n * n;
  const double params[5] = {1.0, 10.0, 1000.0, 0.1, 0.9}; /* du, dv, rho, au, av */
  kx_ctx* ctx = NULL;
  if (kx_create(&ctx, 0, NULL) != KX_OK) {
    fprintf(stderr, "kx_create: %s\n", kx_create_error());
    return 1;
  }
  const long long ext[2] = {n, n};
  CHECK(kx_set_grid(ctx, 2, ext, 2));
  double* A = (double*)malloc(sizeof(double) * n * n);
  for (int c = 0; c < 2; ++c) {
    laplacian(A, n, 1.0, params[c]);
    CHECK(kx_set_direction_matrix(ctx, c, 1, A));
    CHECK(kx_set_direction_matrix(ctx, c, 2, A));
  }
  CHECK(kx_set_model(ctx, KX_MODEL_SCHNAKENBERG, params, 5));
  CHECK(kx_set_tau(ctx, T / steps, KX_ETD3RKDS_REAL));
  /* u0 = u_e + 1e-5 U(0,1), v0 = v_e + 1e-5 U(0,1) */
  double* h[2];
  double* d[2];
  unsigned long long st = 12345;
  for (int c = 0; c < 2; ++c) {
    h[c] = (double*)malloc(sizeof(double) * N);
    for (long long i = 0; i < N; ++i) {
      st = st * 6364136223846793005ULL + 1442695040888963407ULL;
      h[c][i] = (c == 0 ? 1.0 : 0.9) + 1e-5 * (double)(st >> 11) / 9007199254740992.0;
    }
    cudaMalloc((void**)&d[c], sizeof(double) * N);
    cudaMemcpy(d[c], h[c], sizeof(double) * N, cudaMemcpyHostToDevice);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, 0);
  const int report = steps / 4 > 0 ? steps / 4 : 1;
  for (int k = 1; k <= steps; ++k) {
    CHECK(kx_step(ctx, (k - 1) * (T / steps), d));
    if (k % report == 0 || k == steps) {
      CHECK(kx_sync(ctx));
      cudaMemcpy(h[0], d[0], sizeof(double) * N, cudaMemcpyDeviceToHost);
      double lo = h[0][0], hi = h[0][0];
      for (long long i = 1; i < N; ++i) {
        lo = h[0][i] < lo ? h[0][i] : lo;
        hi = h[0][i] > hi ? h[0][i] : hi;
      }
      printf("t = %.4f  u in [%.6f, %.6f]\n", k * (T / steps), lo, hi);
    }
  }
  cudaEventRecord(e1, 0);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  kx_counters cnt;
  kx_get_counters(ctx, &cnt);
  printf("%d steps of %dx%d in %.1f ms (%.1f steps/s incl. reporting); %lld Tucker operators\n", steps, n, n,
         ms, steps / (ms / 1e3), cnt.tucker_ops);
  kx_destroy(ctx);
  return 0;
}
