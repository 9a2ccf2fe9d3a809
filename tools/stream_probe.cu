// Achievable time of a pure streaming kernel with the fused first phase's traffic shape at C2 /
// C3 sizes (read R fields, write W fields of N doubles, 16-B accesses), buffers rotated over
// more than L2 so no launch reuses the previous one's lines.  Build / run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_probe tools/stream_probe.cu && /tmp/stream_probe
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

template <int R, int W>
__global__ void __launch_bounds__(256) stream_kernel(const double2* const* __restrict__ in, double2* const* __restrict__ out,
                                                     long long n2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) {
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = in[r][i];
    double2 s = v[0];
#pragma unroll
    for (int r = 1; r < R; ++r) s.x += v[r].x, s.y += v[r].y;
#pragma unroll
    for (int w = 0; w < W; ++w) out[w][i] = make_double2(s.x + w, s.y);
  }
}

template <int R, int W>
void run(long long N, int occ_mult) {
  const int sets = 6;
  std::vector<double*> bufs;
  double2** din;
  double2** dout;
  cudaMalloc(&din, sets * R * sizeof(void*));
  cudaMalloc(&dout, sets * W * sizeof(void*));
  std::vector<double2*> hin(sets * R), hout(sets * W);
  for (auto& p : hin) cudaMalloc(&p, N * 8), cudaMemset(p, 0, N * 8);
  for (auto& p : hout) cudaMalloc(&p, N * 8);
  cudaMemcpy(din, hin.data(), hin.size() * sizeof(void*), cudaMemcpyHostToDevice);
  cudaMemcpy(dout, hout.data(), hout.size() * sizeof(void*), cudaMemcpyHostToDevice);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const long long n2 = N / 2;
  long long blocks = (n2 + 255) / 256;
  if (occ_mult > 0 && blocks > (long long)nsm * occ_mult) blocks = (long long)nsm * occ_mult;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int k = 0; k < 12; ++k) stream_kernel<R, W><<<blocks, 256>>>(din + (k % sets) * R, dout + (k % sets) * W, n2);
  const int reps = 60;
  cudaEventRecord(a);
  for (int k = 0; k < reps; ++k) stream_kernel<R, W><<<blocks, 256>>>(din + (k % sets) * R, dout + (k % sets) * W, n2);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double us = 1e3 * ms / reps, bytes = 8.0 * N * (R + W);
  printf("N=%lld R=%d W=%d grid=%lld: %.2f us/launch, %.0f GB/s\n", N, R, W, blocks, us, bytes / us / 1e3);
  for (auto& p : hin) cudaFree(p);
  for (auto& p : hout) cudaFree(p);
  cudaFree(din);
  cudaFree(dout);
}

int main() {
  for (long long N : {1LL << 20, 1LL << 21, 1LL << 24}) {
    for (int occ : {0, 8, 16}) {
      run<2, 4>(N, occ);
      run<4, 2>(N, occ);
      run<2, 2>(N, occ);
    }
  }
  return 0;
}
