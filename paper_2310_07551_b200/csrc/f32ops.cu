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

// The same first phase, 4 consecutive points per thread (n_1 % 4 == 0, 16-B aligned fields):
// float4 loads / stores, 32-bit indices, the i_1 neighbours from the adjacent lanes by warp
// shuffles (lane 0 / 31 read theirs), the i_2 / i_3 neighbour lines as float4 loads that hit L2.
// Arithmetic as first_phase_f32_kernel, point by point.
template <int D>
__global__ void __launch_bounds__(256, D == 3 ? 3 : 4) first_phase_f32_vec_kernel(const F32PhaseArgs a) {
  const int n1 = (int)a.n[0], n2 = (int)a.n[1], n3 = D == 3 ? (int)a.n[2] : 1;
  const int q4 = (int)(a.N / 4), l4 = n1 / 4, p4 = l4 * n2;   // quads: field, line, plane
  const int lane = threadIdx.x & 31;
  for (int base = blockIdx.x * blockDim.x; base < q4; base += gridDim.x * blockDim.x) {
    const int q = min(base + (int)threadIdx.x, q4 - 1);
    const bool live = base + (int)threadIdx.x < q4;
    const int line = q / l4, c = q - line * l4, i1 = 4 * c;
    const int i2 = line % n2, i3 = D == 3 ? line / n2 : 0;
    const bool l2 = i2 > 0, u2 = i2 + 1 < n2, l3 = D == 3 && i3 > 0, u3 = D == 3 && i3 + 1 < n3;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 x[2], ym2[2], yp2[2], ym3[2], yp3[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const float4* U = reinterpret_cast<const float4*>(a.U[s]);
      x[s] = U[q];
      ym2[s] = l2 ? U[q - l4] : z4;
      yp2[s] = u2 ? U[q + l4] : z4;
      ym3[s] = l3 ? U[q - p4] : z4;
      yp3[s] = u3 ? U[q + p4] : z4;
    }
    float4 g[2];
    g32(a.model, a.p, x[0].x, x[1].x, g[0].x, g[1].x);
    g32(a.model, a.p, x[0].y, x[1].y, g[0].y, g[1].y);
    g32(a.model, a.p, x[0].z, x[1].z, g[0].z, g[1].z);
    g32(a.model, a.p, x[0].w, x[1].w, g[0].w, g[1].w);
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      float xm = __shfl_up_sync(0xffffffffu, x[s].w, 1);    // point i1 - 1
      float xp = __shfl_down_sync(0xffffffffu, x[s].x, 1);  // point i1 + 4
      if (lane == 0 && i1 > 0) xm = a.U[s][4 * (long long)q - 1];
      if (lane == 31 && i1 + 4 < n1) xp = a.U[s][4 * (long long)q + 4];
      const float xs[6] = {xm, x[s].x, x[s].y, x[s].z, x[s].w, xp};
      const float m2[4] = {ym2[s].x, ym2[s].y, ym2[s].z, ym2[s].w}, p2[4] = {yp2[s].x, yp2[s].y, yp2[s].z, yp2[s].w};
      const float m3[4] = {ym3[s].x, ym3[s].y, ym3[s].z, ym3[s].w}, p3[4] = {yp3[s].x, yp3[s].y, yp3[s].z, yp3[s].w};
      const float gs[4] = {g[s].x, g[s].y, g[s].z, g[s].w};
      const float* t1 = a.tri[s][0];
      const float4 lo1 = *reinterpret_cast<const float4*>(t1 + i1);
      const float4 di1 = *reinterpret_cast<const float4*>(t1 + n1 + i1);
      const float4 up1 = *reinterpret_cast<const float4*>(t1 + 2 * n1 + i1);
      const float clo1[4] = {lo1.x, lo1.y, lo1.z, lo1.w}, cdi1[4] = {di1.x, di1.y, di1.z, di1.w};
      const float cup1[4] = {up1.x, up1.y, up1.z, up1.w};
      const float* t2 = a.tri[s][1];
      const float clo2 = t2[i2], cdi2 = t2[n2 + i2], cup2 = t2[2 * n2 + i2];
      float clo3 = 0.f, cdi3 = 0.f, cup3 = 0.f;
      if (D == 3) {
        const float* t3 = a.tri[s][2];
        clo3 = t3[i3], cdi3 = t3[n3 + i3], cup3 = t3[2 * n3 + i3];
      }
      float f[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float u = xs[j + 1];
        float fj = gs[j];
        if (D == 3) {   // descending mu, as first_phase_f32_kernel
          float acc = cdi3 * u;
          if (l3) acc += clo3 * m3[j];
          if (u3) acc += cup3 * p3[j];
          fj += acc;
        }
        {
          float acc = cdi2 * u;
          if (l2) acc += clo2 * m2[j];
          if (u2) acc += cup2 * p2[j];
          fj += acc;
        }
        {
          const int k = i1 + j;
          float acc = cdi1[j] * u;
          if (k > 0) acc += clo1[j] * xs[j];
          if (k + 1 < n1) acc += cup1[j] * xs[j + 2];
          fj += acc;
        }
        f[j] = fj;
      }
      if (live) {
        reinterpret_cast<float4*>(a.G[s])[q] = g[s];
        reinterpret_cast<float4*>(a.F[s])[q] = make_float4(f[0], f[1], f[2], f[3]);
        if (a.Ucopy[s]) reinterpret_cast<float4*>(a.Ucopy[s])[q] = x[s];
      }
    }
  }
}

// D = g(U_s) - G, 2 species, 4 points per thread (16-B aligned, N % 4 == 0)
__global__ void __launch_bounds__(256) nonlin_f32_vec_kernel(const F32PhaseArgs a) {
  const int q4 = (int)(a.N / 4);
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < q4; q += gridDim.x * blockDim.x) {
    const float4 u = reinterpret_cast<const float4*>(a.U[0])[q], v = reinterpret_cast<const float4*>(a.U[1])[q];
    const float4 G0 = reinterpret_cast<const float4*>(a.G[0])[q], G1 = reinterpret_cast<const float4*>(a.G[1])[q];
    float4 d0, d1;
    g32(a.model, a.p, u.x, v.x, d0.x, d1.x);
    g32(a.model, a.p, u.y, v.y, d0.y, d1.y);
    g32(a.model, a.p, u.z, v.z, d0.z, d1.z);
    g32(a.model, a.p, u.w, v.w, d0.w, d1.w);
    d0.x -= G0.x, d0.y -= G0.y, d0.z -= G0.z, d0.w -= G0.w;
    d1.x -= G1.x, d1.y -= G1.y, d1.z -= G1.z, d1.w -= G1.w;
    reinterpret_cast<float4*>(a.F[0])[q] = d0;
    reinterpret_cast<float4*>(a.F[1])[q] = d1;
    if (a.Ucopy[0]) {
      reinterpret_cast<float4*>(a.Ucopy[0])[q] = reinterpret_cast<const float4*>(a.Usrc[0])[q];
      reinterpret_cast<float4*>(a.Ucopy[1])[q] = reinterpret_cast<const float4*>(a.Usrc[1])[q];
    }
  }
}

bool al16f(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

bool vec_ok(const F32PhaseArgs& a, bool first) {
  if (a.N % 4 || a.N >= (1LL << 31) || a.n[0] % 4) return false;
  for (int s = 0; s < 2; ++s) {
    if (!al16f(a.U[s]) || !al16f(a.G[s]) || !al16f(a.F[s])) return false;
    if (first && !al16f(a.tri[s][0])) return false;
    if (!al16f(a.Ucopy[s]) || !al16f(a.Usrc[s])) return false;
  }
  return true;
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

bool f32_phase_vec_ok(const F32PhaseArgs& a, bool first) { return vec_ok(a, first); }

cudaError_t launch_first_phase_f32(const F32PhaseArgs& a, cudaStream_t s) {
  if (a.N <= 0) return cudaSuccess;
  if (vec_ok(a, true) && (a.d == 2 || a.d == 3)) {
    const long long q4 = a.N / 4;
    if (a.d == 2) first_phase_f32_vec_kernel<2><<<grid_of(q4), 256, 0, s>>>(a);
    else first_phase_f32_vec_kernel<3><<<grid_of(q4), 256, 0, s>>>(a);
    return cudaGetLastError();
  }
  if (a.Ucopy[0]) return cudaErrorInvalidValue;   // the copy is a vectorised-path feature
  if (a.d == 2) first_phase_f32_kernel<2><<<grid_of(a.N), 256, 0, s>>>(a);
  else if (a.d == 3) first_phase_f32_kernel<3><<<grid_of(a.N), 256, 0, s>>>(a);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_nonlin_f32(const F32PhaseArgs& a, cudaStream_t s) {
  if (a.N <= 0) return cudaSuccess;
  if (vec_ok(a, false)) {
    nonlin_f32_vec_kernel<<<grid_of(a.N / 4), 256, 0, s>>>(a);
    return cudaGetLastError();
  }
  if (a.Ucopy[0]) return cudaErrorInvalidValue;
  nonlin_f32_kernel<<<grid_of(a.N), 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace kx
