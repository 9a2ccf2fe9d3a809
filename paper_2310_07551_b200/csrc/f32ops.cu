// fp32 precision variant: the pointwise kernels of the fp32 path.
//
// The static operand of the tcgen05 mode-product GEMM (tf32gemm.cu: the phi-matrices / L) is
// stored as two tf32-valued planes hi = rna_tf32(x), lo = rna_tf32(x - hi), K-major.  These
// kernels produce such planes from fp32 or fp64 data (transposing column-major matrices), and run
// the fp32 first phase / nonlinearity of a step:
//   G = g(U), F = K U + G        (tridiagonal A_mu: the (2d+1)-point stencil, eq:kronsumv P:636-640)
//   D = g(U_s) - G
// with the Schnakenberg / FitzHugh-Nagumo reaction terms evaluated in
// fp32.
#include "kx_internal.h"

namespace kx {
namespace {

__device__ __forceinline__ float rna(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void split(float x, float& h, float& l) {
  h = rna(x);
  l = rna(x - h);
}

int grid_of(long long work) {
  static int nsm[32] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 32) dev = 0;
  if (nsm[dev] == 0 && (cudaDeviceGetAttribute(&nsm[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
                        nsm[dev] <= 0))
    nsm[dev] = 148;
  long long b = (work + 255) / 256;
  const long long cap = (long long)nsm[dev] * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

__global__ void split_f32_kernel(const float* __restrict__ x, float* __restrict__ h, float* __restrict__ l,
                                 long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    split(x[i], h[i], l[i]);
}

// fp32 -> planes of rows x cols blocks; transpose as split_f64_kernel
__global__ void split_f32_2d_kernel(const float* __restrict__ x, float* __restrict__ h, float* __restrict__ l,
                                    long long rows, long long cols, long long total) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long nn = rows * cols, b = i / nn, r = (i - b * nn) / cols, c = i - b * nn - r * cols;
    split(x[b * nn + c * rows + r], h[i], l[i]);
  }
}

// fp64 -> (hi, lo) fp32 planes of rows x cols blocks; transpose: out[b][r][c] = x[b][c][r]
// (x column-major: element (r, c) at c * rows + r; out row-major)
__global__ void split_f64_kernel(const double* __restrict__ x, float* __restrict__ h, float* __restrict__ l,
                                 long long rows, long long cols, long long total, int transpose, double scale) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    long long src = i;
    if (transpose) {
      const long long nn = rows * cols, b = i / nn, r = (i - b * nn) / cols, c = i - b * nn - r * cols;
      src = b * nn + c * rows + r;
    }
    const double v = scale * x[src];
    const float hh = rna((float)v);
    h[i] = hh;
    l[i] = rna((float)(v - (double)hh));
  }
}

__global__ void f64_to_f32_kernel(const double* __restrict__ x, float* __restrict__ y, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = (float)x[i];
}

__device__ __forceinline__ void g32(int model, const float* p, float u, float v, float& g1, float& g2) {
  if (model == MODEL_SCHNAKENBERG) {
    const float u2v = u * u * v;
    g1 = p[2] * (p[3] - u + u2v);
    g2 = p[2] * (p[4] - u2v);
  } else if (model == MODEL_FHN) {
    g1 = p[2] * (-u * (u * u - 1.0f) - v);
    g2 = p[2] * p[3] * (u - p[4] * v);
  } else {
    g1 = 0.0f;
    g2 = 0.0f;
  }
}

// first phase: G = g(U), F = K U + G (fp32), tridiagonal A_mu, 2 species
template <int D>
__global__ void __launch_bounds__(256) first_phase_f32_kernel(const F32PhaseArgs a) {
  const long long N = a.N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    float uu[2] = {a.U[0][i], a.U[1][i]};
    float g[2];
    g32(a.model, a.p, uu[0], uu[1], g[0], g[1]);
    long long idx[D], str[D];
    long long rem = i, st = 1;
#pragma unroll
    for (int mu = 0; mu < D; ++mu) {
      idx[mu] = rem % a.n[mu];
      rem /= a.n[mu];
      str[mu] = st;
      st *= a.n[mu];
    }
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      float f = g[s];
      const float* X = a.U[s];
#pragma unroll
      for (int mu = D - 1; mu >= 0; --mu) {   // descending mu, as the fp64 stencil
        const long long k = idx[mu];
        const float* lo = a.tri[s][mu];
        const float* di = lo + a.n[mu];
        const float* up = di + a.n[mu];
        float acc = di[k] * uu[s];
        if (k > 0) acc += lo[k] * X[i - str[mu]];
        if (k + 1 < a.n[mu]) acc += up[k] * X[i + str[mu]];
        f += acc;
      }
      a.G[s][i] = g[s];
      a.F[s][i] = f;
    }
  }
}

// D = g(U_s) - G, 2 species
__global__ void __launch_bounds__(256) nonlin_f32_kernel(const F32PhaseArgs a) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.N; i += (long long)gridDim.x * blockDim.x) {
    float g[2];
    g32(a.model, a.p, a.U[0][i], a.U[1][i], g[0], g[1]);
#pragma unroll
    for (int s = 0; s < 2; ++s) a.F[s][i] = g[s] - a.G[s][i];
  }
}

}  // namespace

cudaError_t launch_split_f32(const float* x, float* hi, float* lo, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  split_f32_kernel<<<grid_of(n), 256, 0, s>>>(x, hi, lo, n);
  return cudaGetLastError();
}

cudaError_t launch_split_f32_2d(const float* x, float* hi, float* lo, long long rows, long long cols, int nbatch,
                                bool transpose, cudaStream_t s) {
  const long long total = rows * cols * nbatch;
  if (total <= 0) return cudaSuccess;
  if (!transpose) return launch_split_f32(x, hi, lo, total, s);
  split_f32_2d_kernel<<<grid_of(total), 256, 0, s>>>(x, hi, lo, rows, cols, total);
  return cudaGetLastError();
}

cudaError_t launch_split_f64(const double* x, float* hi, float* lo, long long rows, long long cols, int nbatch,
                             bool transpose, double scale, cudaStream_t s) {
  const long long total = rows * cols * nbatch;
  if (total <= 0) return cudaSuccess;
  split_f64_kernel<<<grid_of(total), 256, 0, s>>>(x, hi, lo, rows, cols, total, transpose ? 1 : 0, scale);
  return cudaGetLastError();
}

cudaError_t launch_f64_to_f32(const double* x, float* y, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  f64_to_f32_kernel<<<grid_of(n), 256, 0, s>>>(x, y, n);
  return cudaGetLastError();
}

cudaError_t launch_first_phase_f32(const F32PhaseArgs& a, cudaStream_t s) {
  if (a.N <= 0) return cudaSuccess;
  if (a.d == 2) first_phase_f32_kernel<2><<<grid_of(a.N), 256, 0, s>>>(a);
  else if (a.d == 3) first_phase_f32_kernel<3><<<grid_of(a.N), 256, 0, s>>>(a);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_nonlin_f32(const F32PhaseArgs& a, cudaStream_t s) {
  if (a.N <= 0) return cudaSuccess;
  nonlin_f32_kernel<<<grid_of(a.N), 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace kx
