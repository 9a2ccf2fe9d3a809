// K*6 roofline microbenchmarks (SURVEY.md §2.3 K★6, §8.d "Rooflines"):
//   fp64 DMMA (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4) throughput + latency,
//   fp64 DFMA throughput, HBM copy bandwidth.
// Standalone executable; prints one JSON object. Not part of the product path.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int CHAINS>
__global__ void dmma_loop(double* out, long iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c0[CHAINS], c1[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; i++) { c0[i] = 0.0; c1[i] = 0.0; }
  for (long it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CHAINS; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0[i]), "+d"(c1[i]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; i++) s += c0[i] + c1[i];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, long iters, double seed) {
  double x[CHAINS];
  double a = seed + threadIdx.x * 1e-9, b = 0.999999;
#pragma unroll
  for (int i = 0; i < CHAINS; i++) x[i] = i;
  for (long it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CHAINS; i++) x[i] = fma(x[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; i++) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, long n) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x, st = (long)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}

static float time_ms(cudaEvent_t e0, cudaEvent_t e1) { float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); return ms; }

int main() {
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  double* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  printf("{\"gpu\": \"%s\", \"sms\": %d", p.name, nsm);
  // DMMA latency: one warp, one chain
  {
    long it = 100000;
    dmma_loop<1><<<1, 32>>>(out, 1000, 1.0); CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0)); dmma_loop<1><<<1, 32>>>(out, it, 1.0); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    double ms = time_ms(e0, e1);
    int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    printf(", \"dmma_latency_ns\": %.3f", ms * 1e6 / it);
  }
  // DMMA throughput sweep: warps per SM x chains; ~1 s sustained at the best config
  double best = 0; int bw = 0;
  for (int warps : {4, 8, 16, 32}) {
    long it = 20000;
    dim3 grid(nsm * 2), block(warps * 16);
    dmma_loop<8><<<grid, block>>>(out, 100, 1.0); CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0)); dmma_loop<8><<<grid, block>>>(out, it, 1.0); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    double ms = time_ms(e0, e1);
    double fl = 2.0 * 8 * 8 * 4 * 8.0 * it * (double)grid.x * (block.x / 32);
    double tf = fl / ms / 1e9;
    printf(", \"dmma_tflops_w%d\": %.3f", warps, tf);
    if (tf > best) { best = tf; bw = warps; }
  }
  {
    // sustained ~1.5 s
    long it = 20000; dim3 grid(nsm * 2), block(bw * 16);
    double tot = 0, totms = 0;
    for (int r = 0; r < 200 && totms < 1500; r++) {
      CK(cudaEventRecord(e0)); dmma_loop<8><<<grid, block>>>(out, it, 1.0); CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      totms += time_ms(e0, e1); tot += 2.0 * 8 * 8 * 4 * 8.0 * it * (double)grid.x * (block.x / 32);
    }
    printf(", \"dmma_tflops_best\": %.3f, \"dmma_tflops_sustained\": %.3f, \"dmma_sustained_ms\": %.1f", best, tot / totms / 1e9, totms);
  }
  // DFMA throughput
  {
    long it = 20000; dim3 grid(nsm * 4), block(256);
    dfma_loop<8><<<grid, block>>>(out, 100, 1.0); CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0)); dfma_loop<8><<<grid, block>>>(out, it, 1.0); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    double ms = time_ms(e0, e1);
    double fl = 2.0 * 8 * it * (double)grid.x * block.x;
    printf(", \"dfma_tflops\": %.3f", fl / ms / 1e9);
  }
  // HBM copy (read + write bytes), 2 GiB each way
  {
    long n = (2L << 30) / 16;
    double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
    CK(cudaMemset(a, 0, n * 16));
    double best_gbs = 0;
    for (int r = 0; r < 10; r++) {
      CK(cudaEventRecord(e0)); copy_k<<<nsm * 8, 512>>>(a, b, n); CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      best_gbs = std::max(best_gbs, 2.0 * n * 16 / time_ms(e0, e1) / 1e6);
    }
    printf(", \"hbm_copy_gbs\": %.1f", best_gbs);
    CK(cudaFree(a)); CK(cudaFree(b));
  }
  printf("}\n");
  return 0;
}
