// Kernel K*3 (nonlinearity) and small pointwise helpers.
//
// g is pointwise over the grid and couples the components only at a point
// (eq:twocompdisc), so one thread handles both species at 2 consecutive points
// with 16-B (double2) loads/stores: HBM-bound, 32 B/point for G = g(U) and 48 B/point for
// D = g(U_s) - G.  Grid-stride over a grid sized in multiples of the SM count.
//   Schnakenberg: g1 = rho (a_u - u + u^2 v),  g2 = rho (a_v - u^2 v)
//   FitzHugh-Nagumo: g1 = rho (-u (u^2 - 1) - v),  g2 = rho a1 (u - a2 v)
#include "kx_internal.h"

#include <algorithm>
#include "kx_model.cuh"

namespace kx {
namespace {

__device__ __forceinline__ long long out_index(const PointwiseArgs& a, long long p) {
  if (a.pack_n1l == 0) return p;
  const long long row = p / a.pack_n1, i1 = p - row * a.pack_n1;
  const long long q = i1 / a.pack_n1l;
  return q * (a.N / a.pack_n1 * a.pack_n1l) + row * a.pack_n1l + (i1 - q * a.pack_n1l);
}

// Contiguous, equal chunk of [0, n) for this CTA (the grid is a whole number of resident waves,
// so every SM streams the same number of bytes: no partial last wave on these short kernels)
__device__ __forceinline__ void cta_chunk(long long n, long long align, long long& b0, long long& b1) {
  long long per = (n + gridDim.x - 1) / gridDim.x;
  per = (per + align - 1) / align * align;
  b0 = min(n, (long long)blockIdx.x * per);
  b1 = min(n, b0 + per);
}

template <int MODE>
__global__ void __launch_bounds__(256) nonlin2_kernel(const PointwiseArgs a) {
  // two components, vectorised by 2 points (N even); two pairs per thread per iteration, every
  // load of both issued before any arithmetic (bytes in flight)
  const long long n2 = a.N / 2;
  const double2* __restrict__ u = reinterpret_cast<const double2*>(a.u[0]);
  const double2* __restrict__ v = reinterpret_cast<const double2*>(a.u[1]);
  double2* __restrict__ o1 = reinterpret_cast<double2*>(a.out[0]);
  double2* __restrict__ o2 = reinterpret_cast<double2*>(a.out[1]);
  const double2* __restrict__ G1 = reinterpret_cast<const double2*>(a.G[0]);
  const double2* __restrict__ G2 = reinterpret_cast<const double2*>(a.G[1]);
  long long b0, b1;
  cta_chunk(n2, 1, b0, b1);
  const int B = blockDim.x;
  for (long long i0 = b0 + threadIdx.x; i0 < b1; i0 += 2 * B) {
    double2 uu[2], vv[2], h1[2], h2[2];
    bool ok[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const long long i = i0 + k * B;
      ok[k] = i < b1;
      const long long j = ok[k] ? i : i0;
      uu[k] = u[j];
      vv[k] = v[j];
      if (MODE == 1) {
        h1[k] = G1[j];
        h2[k] = G2[j];
      }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (!ok[k]) continue;
      const long long i = i0 + k * B;
      double2 r1, r2;
      g_point(a.model, a.p, uu[k].x, vv[k].x, r1.x, r2.x);
      g_point(a.model, a.p, uu[k].y, vv[k].y, r1.y, r2.y);
      if (MODE == 1) {
        r1.x -= h1[k].x;
        r1.y -= h1[k].y;
        r2.x -= h2[k].x;
        r2.y -= h2[k].y;
      }
      const long long oi = out_index(a, 2 * i) / 2;   // pairs never straddle a peer block
      *reinterpret_cast<double2*>(peer_redirect(a.peer, 0, reinterpret_cast<double*>(o1 + oi))) = r1;
      *reinterpret_cast<double2*>(peer_redirect(a.peer, 1, reinterpret_cast<double*>(o2 + oi))) = r2;
    }
  }
  if (a.peer.P) __threadfence_system();
}

template <int MODE>
__global__ void __launch_bounds__(256) nonlin_scalar_kernel(const PointwiseArgs a) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.N;
       i += (long long)gridDim.x * blockDim.x) {
    if (a.ncomp == 2) {
      double r1, r2;
      g_point(a.model, a.p, a.u[0][i], a.u[1][i], r1, r2);
      if (MODE == 1) {
        r1 -= a.G[0][i];
        r2 -= a.G[1][i];
      }
      const long long oi = out_index(a, i);
      *peer_redirect(a.peer, 0, a.out[0] + oi) = r1;
      *peer_redirect(a.peer, 1, a.out[1] + oi) = r2;
    } else {
      const long long oi = out_index(a, i);
      for (int c = 0; c < a.ncomp; ++c)   // g = 0 (KX_MODEL_NONE)
        *peer_redirect(a.peer, c, a.out[c] + oi) = MODE == 1 ? -a.G[c][i] : 0.0;
    }
  }
  if (a.peer.P) __threadfence_system();   // peer stores performed before the kernel completes
}

__global__ void scale_kernel(double* __restrict__ y, const double* __restrict__ x, double alpha,
                             long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = alpha * x[i];
}

__global__ void axpby_kernel(double* __restrict__ y, double a, const double* __restrict__ x1, double b,
                             const double* __restrict__ x2, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = a * x1[i] + b * x2[i];
}

__global__ void copy2d_kernel(double* __restrict__ y, long long ldy, long long sy,
                              const double* __restrict__ x, long long ldx, long long sx,
                              long long rows, long long cols, double alpha, double beta) {
  const int bz = blockIdx.y;
  const long long total = rows * cols;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / cols, c = i % cols;
    double* yp = y + bz * sy + r * ldy + c;
    const double v = alpha * x[bz * sx + r * ldx + c];
    *yp = beta != 0.0 ? v + beta * *yp : v;
  }
}

__global__ void set_identity_kernel(double* __restrict__ y, long long n, double v) {
  const long long total = n * n;
  double* yb = y + blockIdx.y * total;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x)
    yb[i] = (i / n == i % n) ? v : 0.0;
}

__global__ void check_finite_kernel(const double* __restrict__ x, long long n, int* flag) {
  int bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// Tridiagonal Kronecker-sum action.  One CTA row-loop over "lines" (fixed i_2..i_d),
// threads along the contiguous i_1: every load is coalesced along i_1 and the i_mu +- 1
// neighbours (mu >= 2) are other lines read by neighbouring CTAs, so each X element is fetched
// from HBM about once.  HBM-bound: 8 B (X) + 8 B (Dd) + 8 B (Y) per point.
template <int D, typename I>
__device__ __forceinline__ double tridiag_point(const StencilArgs& a, int s, const double* __restrict__ X,
                                                I p) {
  // multi-index of point p (32-bit arithmetic when the tensor fits)
  const I n1 = (I)a.n[0];
  I rem = p / n1;
  const I i1 = p - rem * n1;
  I idx[D > 1 ? D : 2], str[D > 1 ? D : 2];
  I stride = n1;
#pragma unroll
  for (int mu = 1; mu < D; ++mu) {
    const I nm = (I)a.n[mu];
    const I q = rem / nm;
    idx[mu] = rem - q * nm;
    rem = q;
    str[mu] = stride;
    stride *= nm;
  }
  const double xp = X[p];
  double acc = a.Dd[s] ? a.beta * a.Dd[s][p] : 0.0;
  // mu = d .. 2 (descending, as the dense path)
#pragma unroll
  for (int mu = D - 1; mu >= 1; --mu) {
    const I i = idx[mu], st = str[mu];
    const bool sh = (mu == D - 1) && a.n_glob_d != 0;
    const long long ig = sh ? (long long)i + a.d_off : (long long)i;
    const long long ng = sh ? a.n_glob_d : a.n[mu];
    double t = a.di[s][mu][ig] * xp;
    if (sh) {
      // sharded last direction: neighbour planes from the halos
      const I pp = p - i * st;   // offset inside the plane
      if (ig > 0) t = fma(a.lo[s][mu][ig], i > 0 ? X[p - st] : a.halo_lo[s][pp], t);
      if (ig + 1 < ng) t = fma(a.up[s][mu][ig], i + 1 < (I)a.n[mu] ? X[p + st] : a.halo_hi[s][pp], t);
    } else {
      if (i > 0) t = fma(a.lo[s][mu][i], X[p - st], t);
      if (i + 1 < (I)ng) t = fma(a.up[s][mu][i], X[p + st], t);
    }
    acc += t;
  }
  double t = a.di[s][0][i1] * xp;
  if (i1 > 0) t = fma(a.lo[s][0][i1], X[p - 1], t);
  if (i1 + 1 < n1) t = fma(a.up[s][0][i1], X[p + 1], t);
  return acc + t;
}

// Grid-stride over points, U points per thread in flight (their loads are independent, so
// U x ~10 loads are outstanding per thread: the kernel is bound by bytes in flight).
template <int D, typename I, int U>
__global__ void __launch_bounds__(256) kronsum_tridiag_kernel(const StencilArgs a) {
  const int s = blockIdx.y;
  const double* __restrict__ X = a.X[s];
  double* __restrict__ Y = a.Y[s];
  const I N = (I)a.N;
  const I step = (I)gridDim.x * blockDim.x;
  for (I p0 = (I)blockIdx.x * blockDim.x + threadIdx.x; p0 < N; p0 += U * step) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const I p = p0 + u * step;
      v[u] = p < N ? tridiag_point<D, I>(a, s, X, p) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const I p = p0 + u * step;
      if (p < N) {
        I o = p;
        if (a.pack_n1l) {   // peer-packed output (distributed contexts)
          const I n1 = (I)a.n[0], n1l = (I)a.pack_n1l;
          const I line = p / n1, i1 = p - line * n1;
          const I q = i1 / n1l;
          o = q * (N / n1 * n1l) + line * n1l + (i1 - q * n1l);
        }
        *peer_redirect(a.peer, s, Y + o) = v[u];
      }
    }
  }
  if (a.peer.P) __threadfence_system();
}

// Fused first phase of a step (K*3 + K*2'): G = g(U) and F = K U + G for both species in one
// pass over U.  Two consecutive points per thread with 16-B loads/stores; the i_1 neighbours
// come from the adjacent lanes by warp shuffles, the i_2 / i_3 neighbour lines by 16-B loads
// that hit L2 (the neighbouring lines are being read by the neighbouring warps).  HBM traffic:
// U read once, G and F written once (48 B per point pair of species vs 80 B for the two
// separate kernels).  Arithmetic identical to nonlin2_kernel + kronsum_tridiag_kernel.
template <int D>
__global__ void __launch_bounds__(256) g_kronsum_kernel(const GKronArgs a) {
  const int n1 = a.n[0], n2 = a.n[1], n3 = D == 3 ? a.n[2] : 1;
  const int npairs = a.N / 2;
  const int lane = threadIdx.x & 31;
  const double2* __restrict__ U0 = reinterpret_cast<const double2*>(a.U[0]);
  const double2* __restrict__ U1 = reinterpret_cast<const double2*>(a.U[1]);
  double2* __restrict__ G0 = reinterpret_cast<double2*>(a.G[0]);
  double2* __restrict__ G1 = reinterpret_cast<double2*>(a.G[1]);
  double2* __restrict__ F0 = reinterpret_cast<double2*>(a.F[0]);
  double2* __restrict__ F1 = reinterpret_cast<double2*>(a.F[1]);
  const int st3 = n1 * n2;
  for (int base = blockIdx.x * blockDim.x; base < npairs; base += gridDim.x * blockDim.x) {
    const int q = base + threadIdx.x;
    const bool live = q < npairs;
    const int h = live ? q : npairs - 1;   // pair index (points 2h, 2h+1)
    const int p = 2 * h;
    const int line = p / n1, i1 = p - line * n1;
    const int i2 = line % n2, i3 = D == 3 ? line / n2 : 0;
    const bool l2 = i2 > 0, u2 = i2 + 1 < n2, l3 = D == 3 && i3 > 0, u3 = D == 3 && i3 + 1 < n3;
    // every load of the pair first (no store in between: all loads in flight together)
    const double2 zero = make_double2(0.0, 0.0);
    double2 x[2], ym2[2], yp2[2], ym3[2], yp3[2];
    x[0] = U0[h];
    x[1] = U1[h];
    ym2[0] = l2 ? U0[h - n1 / 2] : zero;
    ym2[1] = l2 ? U1[h - n1 / 2] : zero;
    yp2[0] = u2 ? U0[h + n1 / 2] : zero;
    yp2[1] = u2 ? U1[h + n1 / 2] : zero;
    if (D == 3) {
      ym3[0] = l3 ? U0[h - st3 / 2] : zero;
      ym3[1] = l3 ? U1[h - st3 / 2] : zero;
      yp3[0] = u3 ? U0[h + st3 / 2] : zero;
      yp3[1] = u3 ? U1[h + st3 / 2] : zero;
    }
    double xm[2], xp[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      // i_1 neighbours: x[p-1] is the previous lane's .y, x[p+2] the next lane's .x
      xm[s] = __shfl_up_sync(0xffffffffu, x[s].y, 1);
      xp[s] = __shfl_down_sync(0xffffffffu, x[s].x, 1);
      if (lane == 0 && i1 > 0) xm[s] = a.U[s][p - 1];
      if (lane == 31 && i1 + 2 < n1) xp[s] = a.U[s][p + 2];
    }
    double2 gv[2];
    g_point(a.model, a.p, x[0].x, x[1].x, gv[0].x, gv[1].x);
    g_point(a.model, a.p, x[0].y, x[1].y, gv[0].y, gv[1].y);
    double2 f[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      double acc0 = 1.0 * gv[s].x, acc1 = 1.0 * gv[s].y;
      // directions mu = d .. 2 (descending, as the dense path)
      if (D == 3) {
        const double* __restrict__ t = a.tri[s][2];
        const double c_di = t[n3 + i3];
        double v0 = c_di * x[s].x, v1 = c_di * x[s].y;
        if (l3) {
          const double c = t[i3];
          v0 = fma(c, ym3[s].x, v0);
          v1 = fma(c, ym3[s].y, v1);
        }
        if (u3) {
          const double c = t[2 * n3 + i3];
          v0 = fma(c, yp3[s].x, v0);
          v1 = fma(c, yp3[s].y, v1);
        }
        acc0 += v0;
        acc1 += v1;
      }
      {
        const double* __restrict__ t = a.tri[s][1];
        const double c_di = t[n2 + i2];
        double v0 = c_di * x[s].x, v1 = c_di * x[s].y;
        if (l2) {
          const double c = t[i2];
          v0 = fma(c, ym2[s].x, v0);
          v1 = fma(c, ym2[s].y, v1);
        }
        if (u2) {
          const double c = t[2 * n2 + i2];
          v0 = fma(c, yp2[s].x, v0);
          v1 = fma(c, yp2[s].y, v1);
        }
        acc0 += v0;
        acc1 += v1;
      }
      {
        const double* __restrict__ t = a.tri[s][0];
        double v0 = t[n1 + i1] * x[s].x;
        if (i1 > 0) v0 = fma(t[i1], xm[s], v0);
        v0 = fma(t[2 * n1 + i1], x[s].y, v0);   // i1 + 1 < n1 always (n1 even)
        double v1 = t[n1 + i1 + 1] * x[s].y;
        v1 = fma(t[i1 + 1], x[s].x, v1);
        if (i1 + 2 < n1) v1 = fma(t[2 * n1 + i1 + 1], xp[s], v1);
        acc0 += v0;
        acc1 += v1;
      }
      f[s] = make_double2(acc0, acc1);
    }
    if (live) {
      G0[h] = gv[0];
      G1[h] = gv[1];
      F0[h] = f[0];
      F1[h] = f[1];
    }
  }
}

// d = 3 variant: one species at a time (fewer live registers: 64, no spills at full
// occupancy; the all-loads-first form of g_kronsum_kernel needs 80)
template <int D>
__global__ void __launch_bounds__(256) g_kronsum_seq_kernel(const GKronArgs a) {
  const int n1 = a.n[0], n2 = a.n[1], n3 = D == 3 ? a.n[2] : 1;
  const int npairs = a.N / 2;
  const int lane = threadIdx.x & 31;
  const double2* __restrict__ U2[2] = {reinterpret_cast<const double2*>(a.U[0]),
                                       reinterpret_cast<const double2*>(a.U[1])};
  for (int base = blockIdx.x * blockDim.x; base < npairs; base += gridDim.x * blockDim.x) {
    const int q = base + threadIdx.x;
    const bool live = q < npairs;
    const int p = 2 * (live ? q : npairs - 1);
    const int line = p / n1, i1 = p - line * n1;
    const int i2 = D >= 2 ? line % n2 : 0, i3 = D == 3 ? line / n2 : 0;
    double2 x[2];
    x[0] = U2[0][p / 2];
    x[1] = U2[1][p / 2];
    double2 gv[2];
    g_point(a.model, a.p, x[0].x, x[1].x, gv[0].x, gv[1].x);
    g_point(a.model, a.p, x[0].y, x[1].y, gv[0].y, gv[1].y);
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      // i_1 neighbours: x[p-1] is the previous lane's .y, x[p+2] the next lane's .x
      double xm = __shfl_up_sync(0xffffffffu, x[s].y, 1);
      double xp = __shfl_down_sync(0xffffffffu, x[s].x, 1);
      if (lane == 0 && i1 > 0) xm = a.U[s][p - 1];
      if (lane == 31 && i1 + 2 < n1) xp = a.U[s][p + 2];
      double acc0 = 1.0 * gv[s].x, acc1 = 1.0 * gv[s].y;
      // directions mu = d .. 2 (descending, as the dense path)
      if (D == 3) {
        const double* t = a.tri[s][2];
        const double c_lo = t[i3], c_di = t[n3 + i3], c_up = t[2 * n3 + i3];
        const int st = n1 * n2;
        double v0 = c_di * x[s].x, v1 = c_di * x[s].y;
        if (i3 > 0) {
          const double2 y = U2[s][(p - st) / 2];
          v0 = fma(c_lo, y.x, v0);
          v1 = fma(c_lo, y.y, v1);
        }
        if (i3 + 1 < n3) {
          const double2 y = U2[s][(p + st) / 2];
          v0 = fma(c_up, y.x, v0);
          v1 = fma(c_up, y.y, v1);
        }
        acc0 += v0;
        acc1 += v1;
      }
      {
        const double* t = a.tri[s][1];
        const double c_lo = t[i2], c_di = t[n2 + i2], c_up = t[2 * n2 + i2];
        double v0 = c_di * x[s].x, v1 = c_di * x[s].y;
        if (i2 > 0) {
          const double2 y = U2[s][(p - n1) / 2];
          v0 = fma(c_lo, y.x, v0);
          v1 = fma(c_lo, y.y, v1);
        }
        if (i2 + 1 < n2) {
          const double2 y = U2[s][(p + n1) / 2];
          v0 = fma(c_up, y.x, v0);
          v1 = fma(c_up, y.y, v1);
        }
        acc0 += v0;
        acc1 += v1;
      }
      {
        const double* t = a.tri[s][0];
        double v0 = t[n1 + i1] * x[s].x;
        if (i1 > 0) v0 = fma(t[i1], xm, v0);
        v0 = fma(t[2 * n1 + i1], x[s].y, v0);   // i1 + 1 < n1 always (n1 even)
        double v1 = t[n1 + i1 + 1] * x[s].y;
        v1 = fma(t[i1 + 1], x[s].x, v1);
        if (i1 + 2 < n1) v1 = fma(t[2 * n1 + i1 + 1], xp, v1);
        acc0 += v0;
        acc1 += v1;
      }
      if (live) {
        reinterpret_cast<double2*>(a.G[s])[p / 2] = gv[s];
        reinterpret_cast<double2*>(a.F[s])[p / 2] = make_double2(acc0, acc1);
      }
    }
  }
}

// NaN/Inf watchdog (SURVEY §5 failure detection): mon = {steps completed, first bad step (-1)}
__global__ void watch_finite_kernel(const double* __restrict__ x, long long n, int* mon) {
  int bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicCAS(mon + 1, -1, mon[0]);
}
__global__ void watch_tick_kernel(int* mon) { mon[0] += 1; }

int grid_for(long long work, int block) {
  static int nsm_of[32] = {};   // per device
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 32) dev = 0;
  if (nsm_of[dev] == 0 && (cudaDeviceGetAttribute(&nsm_of[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
                           nsm_of[dev] <= 0))
    nsm_of[dev] = 148;
  const int nsm = nsm_of[dev];
  long long blocks = (work + block - 1) / block;
  const long long cap = (long long)nsm * 16;   // 2 waves of 8 resident 256-thread CTAs per SM
  if (blocks > cap) blocks = cap;
  return (int)(blocks < 1 ? 1 : blocks);
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// One whole wave of resident CTAs (occupancy API, per device and kernel), at most enough CTAs
// for `work` threads: with cta_chunk every SM then streams the same share of the field.
template <class K>
int resident_grid(K kernel, long long work, int block) {
  static int occ_of[32] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 32) dev = 0;
  if (occ_of[dev] == 0) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, block, 0) != cudaSuccess || occ < 1) occ = 4;
    occ_of[dev] = occ;
  }
  const long long wave = (long long)(grid_for(1LL << 40, block) / 16) * occ_of[dev];   // SMs x resident
  const long long need = (work + block - 1) / block;
  return (int)std::max<long long>(1, std::min(wave, need));
}

}  // namespace

cudaError_t launch_nonlinearity(const PointwiseArgs& a, int mode, cudaStream_t stream) {
  if (a.N <= 0) return cudaSuccess;
  bool vec = a.ncomp == 2 && a.N % 2 == 0 && al16(a.u[0]) && al16(a.u[1]) && al16(a.out[0]) &&
             al16(a.out[1]) && (a.pack_n1l == 0 || a.pack_n1l % 2 == 0);
  if (mode == 1) vec = vec && al16(a.G[0]) && al16(a.G[1]);
  if (vec) {
    if (mode == 0) nonlin2_kernel<0><<<resident_grid(nonlin2_kernel<0>, a.N / 4, 256), 256, 0, stream>>>(a);
    else nonlin2_kernel<1><<<resident_grid(nonlin2_kernel<1>, a.N / 4, 256), 256, 0, stream>>>(a);
  } else {
    const int grid = grid_for(a.N, 256);
    if (mode == 0) nonlin_scalar_kernel<0><<<grid, 256, 0, stream>>>(a);
    else nonlin_scalar_kernel<1><<<grid, 256, 0, stream>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_g_kronsum(const GKronArgs& a, cudaStream_t stream) {
  if (a.N <= 0) return cudaSuccess;
  // one whole wave of resident CTAs, each streaming a contiguous chunk (its neighbour lines are
  // mostly its own: L2 hits)
  // one wave of 8 CTAs per SM (its neighbour loads hit L2 better than two waves; measured: a
  // contiguous chunk per CTA and an all-loads-first d = 3 form were no faster)
  const int grid = (int)std::min<long long>(grid_for(a.N / 2, 256), 8LL * (grid_for(1LL << 40, 256) / 16));
  if (a.d == 2) g_kronsum_kernel<2><<<grid, 256, 0, stream>>>(a);
  else if (a.d == 3) g_kronsum_seq_kernel<3><<<grid, 256, 0, stream>>>(a);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_kronsum_tridiag(const StencilArgs& a, cudaStream_t stream) {
  if (a.N <= 0) return cudaSuccess;
  // U = 4 points per thread in flight on large grids; small grids spread one point per
  // thread over more CTAs (latency-bound there)
  constexpr int block = 256;
  const bool wide = a.N >= 148LL * block * 4 * 2;
  const dim3 grid((unsigned)grid_for(wide ? (a.N + 3) / 4 : a.N, block), a.ns);
  const bool small = a.N < (1LL << 30);   // 32-bit point indices (p + st stays < 2^31)
#define KX_TRIDIAG(DD)                                                                    \
  case DD:                                                                                \
    if (!small) kronsum_tridiag_kernel<DD, long long, 4><<<grid, block, 0, stream>>>(a);  \
    else if (wide) kronsum_tridiag_kernel<DD, int, 4><<<grid, block, 0, stream>>>(a);     \
    else kronsum_tridiag_kernel<DD, int, 1><<<grid, block, 0, stream>>>(a);               \
    break;
  switch (a.d) {
    KX_TRIDIAG(1)
    KX_TRIDIAG(2)
    KX_TRIDIAG(3)
    KX_TRIDIAG(4)
    KX_TRIDIAG(5)
    KX_TRIDIAG(6)
    default: return cudaErrorInvalidValue;
  }
#undef KX_TRIDIAG
  return cudaGetLastError();
}

cudaError_t launch_scale(double* Y, const double* X, double alpha, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  scale_kernel<<<grid_for(n, 256), 256, 0, s>>>(Y, X, alpha, n);
  return cudaGetLastError();
}

cudaError_t launch_axpby(double* Y, double a, const double* X1, double b, const double* X2, long long n,
                         cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  axpby_kernel<<<grid_for(n, 256), 256, 0, s>>>(Y, a, X1, b, X2, n);
  return cudaGetLastError();
}

cudaError_t launch_copy2d(double* Y, long long ldy, long long sy, const double* X, long long ldx,
                          long long sx, long long rows, long long cols, int nbatch, double alpha,
                          cudaStream_t s) {
  if (rows <= 0 || cols <= 0 || nbatch <= 0) return cudaSuccess;
  dim3 grid(grid_for(rows * cols, 256), nbatch);
  copy2d_kernel<<<grid, 256, 0, s>>>(Y, ldy, sy, X, ldx, sx, rows, cols, alpha, 0.0);
  return cudaGetLastError();
}

cudaError_t launch_copy2d_axpby(double* Y, long long ldy, long long sy, const double* X, long long ldx,
                                long long sx, long long rows, long long cols, int nbatch, double alpha,
                                double beta, cudaStream_t s) {
  if (rows <= 0 || cols <= 0 || nbatch <= 0) return cudaSuccess;
  dim3 grid(grid_for(rows * cols, 256), nbatch);
  copy2d_kernel<<<grid, 256, 0, s>>>(Y, ldy, sy, X, ldx, sx, rows, cols, alpha, beta);
  return cudaGetLastError();
}

cudaError_t launch_set_identity(double* Y, long long n, int nbatch, double v, cudaStream_t s) {
  if (n <= 0 || nbatch <= 0) return cudaSuccess;
  dim3 grid(grid_for(n * n, 256), nbatch);
  set_identity_kernel<<<grid, 256, 0, s>>>(Y, n, v);
  return cudaGetLastError();
}

cudaError_t launch_watch_finite(const double* X, long long n, int* mon, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  watch_finite_kernel<<<grid_for(n, 256), 256, 0, s>>>(X, n, mon);
  return cudaGetLastError();
}

cudaError_t launch_watch_tick(int* mon, cudaStream_t s) {
  watch_tick_kernel<<<1, 1, 0, s>>>(mon);
  return cudaGetLastError();
}

cudaError_t launch_check_finite(const double* X, long long n, int* flag, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  check_finite_kernel<<<grid_for(n, 256), 256, 0, s>>>(X, n, flag);
  return cudaGetLastError();
}

}  // namespace kx
