// Kernel K*5: whole time steps of ETD2RKDS / exprk3ds_real on a small 2-D grid
// (8 <= n_2 <= 64, n_1 <= 64) in ONE thread-block cluster (SURVEY.md §2 K*5, §8(a) a2:
// "for d = 2 and n <= 128 a single CTA holds the slab and does L_2 X L_1^T", the shape of
// eq:exp2d).
//
// At these sizes a step of the general path is a chain of ~7-11 latency-bound launches
// (~5 us each) moving kilobytes.  Here 8 CTAs of one cluster split the rows i_2 of the grid
// (<= 8 rows each, one DMMA m8 fragment) and keep the whole state in shared memory across
// any number of steps; the only inter-CTA traffic is distributed shared memory:
//   * the Kronecker-sum stencil reads the neighbouring rows (halo) from the peer CTAs;
//   * the input of every split phi-action (F, then D) is broadcast row-block by row-block
//     into a full copy in every CTA (the mode-2 product L_2[I,:] X needs all of X), then
//   * each CTA forms its rows of the stage combination as
//       out_I = base_I + sum_seg ( P2_seg[I,:] * X_seg ) * B_seg
//     i.e. the fused mode-2 / mode-1 products of every term with the stage scalars folded
//     into B_seg (the same banks the general path's concat-K GEMM uses), the intermediate
//     row block never leaving shared memory.
// Cluster barriers: 3 per ETD2RKDS step, 5 per exprk3ds step.  The two species run on two
// warp groups (warps 0-3, 4-7) in the phi-action phases.
#include <cooperative_groups.h>

#include "kx_internal.h"
#include "kx_model.cuh"

namespace cg = cooperative_groups;

namespace kx {
namespace {

constexpr int CL = kFusedCluster;   // CTAs per cluster (portable maximum)
constexpr int NMAX = kFusedNMax;
constexpr int SS = NMAX + 4;        // smem row stride in doubles (= 4 mod 16: conflict-free)
constexpr int RMAX = (NMAX + CL - 1) / CL;
constexpr int NT = 256;

struct Smem {
  double Ffull[2][NMAX][SS];   // full copies of the phi-action inputs (per species)
  double Dfull[2][NMAX][SS];
  double Ul[2][RMAX][SS];      // this CTA's rows of U, the stage value and G
  double Us[2][RMAX][SS];
  double Gl[2][RMAX][SS];
  double Zs[2][RMAX][SS];      // intermediate P2[I,:] X (per species)
  double tri[2][2][3][NMAX];   // [species][direction]: lo, di, up of the tridiagonal A_mu
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void group_bar(int id) {
  asm volatile("bar.sync %0, 128;\n" ::"r"(id) : "memory");
}

__device__ __forceinline__ int row0(int c, int n2) { return c * n2 / CL; }

__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NT, 1)
    fused2d_kernel(const Fused2dArgs a) {
  extern __shared__ __align__(16) double smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const int c = (int)cluster.block_rank();
  const int n1 = a.n1, n2 = a.n2, ns = a.ncomp;
  const int r0 = row0(c, n2), r = row0(c + 1, n2) - r0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;

  // the padding rows (>= n2) and columns (>= n1) of the full copies feed the DMMAs as exact
  // zeros; everything else is written before it is read
  for (int s = 0; s < 2; ++s)
    for (int i = tid; i < NMAX * SS; i += NT) {
      const int row = i / SS, col = i - row * SS;
      if (row >= n2 || col >= n1) {
        S.Ffull[s][row][col] = 0.0;
        S.Dfull[s][row][col] = 0.0;
      }
    }
  for (int s = 0; s < ns; ++s)
    for (int p = tid; p < r * n1; p += NT) {
      const int i = p / n1, j = p - i * n1;
      S.Ul[s][i][j] = a.U[s][(long long)(r0 + i) * n1 + j];
    }
  for (int s = 0; s < ns; ++s)
    for (int mu = 0; mu < 2; ++mu) {
      const int n = mu == 0 ? n1 : n2;
      for (int i = tid; i < 3 * n; i += NT) S.tri[s][mu][i / n][i % n] = a.tri[s][mu][i];
    }
  Smem* peer[CL];
#pragma unroll
  for (int q = 0; q < CL; ++q) peer[q] = cluster.map_shared_rank(&S, q);
  // halo owners: the row above r0 lives in CTA c-1, the row below r0+r-1 in CTA c+1
  const int lo_rank = c > 0 ? c - 1 : 0, hi_rank = c + 1 < CL ? c + 1 : CL - 1;
  const int lo_row = r0 - 1 - row0(lo_rank, n2), hi_row = 0;

  // U row i2 of species s, own or halo
  auto u_at = [&](int s, int i2, int j) -> double {
    if (i2 < r0) return peer[lo_rank]->Ul[s][lo_row][j];
    if (i2 >= r0 + r) return peer[hi_rank]->Ul[s][hi_row][j];
    return S.Ul[s][i2 - r0][j];
  };

  // D = g(Us) - G on the own rows, broadcast into every CTA's Dfull
  auto nonlin_d = [&]() {
    for (int p = tid; p < r * n1; p += NT) {
      const int i = p / n1, j = p - i * n1;
      double d[2];
      g_point(a.model, a.p, S.Us[0][i][j], ns > 1 ? S.Us[1][i][j] : 0.0, d[0], d[1]);
      for (int s = 0; s < ns; ++s) {
        const double v = d[s] - S.Gl[s][i][j];
#pragma unroll
        for (int q = 0; q < CL; ++q) peer[q]->Dfull[s][r0 + i][j] = v;
      }
    }
  };

  // out_I = base_I + sum_seg (P2_seg[I,:] X_seg) B_seg, species s on warps 4s..4s+3.  All
  // global operand loads of a product are issued before its DMMA chain (one L2 round trip per
  // product instead of one per k-step).
  constexpr int KS = NMAX / 4;
  auto stage = [&](int k) {
    const int s = warp >> 2, w4 = warp & 3;
    if (s < ns) {
      double acc[2][2][2] = {};   // [fragment][k parity][element]
      for (int sg = 0; sg < a.nseg[k]; ++sg) {
        const double* __restrict__ P2 = a.P2[k][sg][s];
        const long long ld = a.ld2[k][sg];
        const double(*X)[SS] = a.seg_in[k][sg] ? S.Dfull[s] : S.Ffull[s];
        const double* __restrict__ B = a.B[k][sg][s];
        double av[KS], bv[KS][2];
#pragma unroll
        for (int q = 0; q < KS; ++q) {
          const int kr = 4 * q + t4;
          av[q] = (g < r && kr < n2) ? __ldg(P2 + (long long)kr * ld + r0 + g) : 0.0;
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const int col = (w4 * 2 + jj) * 8 + g;
            bv[q][jj] = (kr < n1 && col < n1) ? __ldg(B + (long long)kr * n1 + col) : 0.0;
          }
        }
        // two accumulators per fragment (even / odd k-step): independent DMMA chains
        double z[2][2][2] = {};
#pragma unroll
        for (int q = 0; q < KS; ++q) {
          const int kr = 4 * q + t4;
#pragma unroll
          for (int jj = 0; jj < 2; ++jj)
            dmma(z[jj][q & 1][0], z[jj][q & 1][1], av[q], X[kr][(w4 * 2 + jj) * 8 + g]);
        }
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          S.Zs[s][g][(w4 * 2 + jj) * 8 + 2 * t4] = z[jj][0][0] + z[jj][1][0];
          S.Zs[s][g][(w4 * 2 + jj) * 8 + 2 * t4 + 1] = z[jj][0][1] + z[jj][1][1];
        }
        group_bar(1 + s);
#pragma unroll
        for (int q = 0; q < KS; ++q) {
          const double zv = S.Zs[s][g][4 * q + t4];
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) dmma(acc[jj][q & 1][0], acc[jj][q & 1][1], zv, bv[q][jj]);
        }
        group_bar(1 + s);
      }
      double(*base)[SS] = a.base[k] ? S.Us[s] : S.Ul[s];
      double(*out)[SS] = k == a.nstages - 1 ? S.Ul[s] : S.Us[s];
      if (g < r) {
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = (w4 * 2 + jj) * 8 + 2 * t4 + e;
            if (col < n1) out[g][col] = base[g][col] + (acc[jj][0][e] + acc[jj][1][e]);
          }
      }
    }
    __syncthreads();
  };

  int tp = 0;   // diagnostics: phase timestamps of CTA 0's thread 0 (a.prof, normally null)
  auto stamp = [&]() {
    if (a.prof && tid == 0 && c == 0 && tp < 64) a.prof[tp++] = clock64();
  };
  for (int step = 0; step < a.nsteps; ++step) {
    stamp();
    cluster.sync();   // peers' U rows are current; nobody reads Ffull/Dfull any more
    stamp();
    // G = g(U); F = K U + G (tridiagonal stencil, the order of kronsum_tridiag_kernel), broadcast
    for (int p = tid; p < r * n1; p += NT) {
      const int i = p / n1, j = p - i * n1, i2 = r0 + i;
      double gv[2];
      g_point(a.model, a.p, S.Ul[0][i][j], ns > 1 ? S.Ul[1][i][j] : 0.0, gv[0], gv[1]);
      for (int s = 0; s < ns; ++s) {
        S.Gl[s][i][j] = gv[s];
        const double x = S.Ul[s][i][j];
        double acc = 1.0 * gv[s];
        {
          const double(*t)[NMAX] = S.tri[s][1];   // direction 2: lo, di, up
          double v = t[1][i2] * x;
          if (i2 > 0) v = fma(t[0][i2], u_at(s, i2 - 1, j), v);
          if (i2 + 1 < n2) v = fma(t[2][i2], u_at(s, i2 + 1, j), v);
          acc += v;
        }
        {
          const double(*t)[NMAX] = S.tri[s][0];   // direction 1
          double v = t[1][j] * x;
          if (j > 0) v = fma(t[0][j], S.Ul[s][i][j - 1], v);
          if (j + 1 < n1) v = fma(t[2][j], S.Ul[s][i][j + 1], v);
          acc += v;
        }
#pragma unroll
        for (int q = 0; q < CL; ++q) peer[q]->Ffull[s][i2][j] = acc;
      }
    }
    stamp();
    cluster.sync();
    stamp();
    stage(0);          // ETD2: u2 = U + tau S[F];  exprk3ds: U2 = U + tau/3 S_1[F]
    stamp();
    nonlin_d();        // D (ETD2) / D2 (exprk3ds)
    stamp();
    cluster.sync();
    stamp();
    stage(1);          // ETD2: U = u2 + 2 tau S_2[D];  exprk3ds: U3 = U + ... [F] + ... [D2]
    stamp();
    if (a.nstages == 3) {
      cluster.sync();  // every CTA is done reading D2
      stamp();
      nonlin_d();      // D3
      stamp();
      cluster.sync();
      stamp();
      stage(2);        // U+ = U + tau S_1[F] + 3tau/2 S_2[D3]
      stamp();
    }
  }
  cluster.sync();      // no CTA leaves while a peer may still address its shared memory
  for (int s = 0; s < ns; ++s)
    for (int p = tid; p < r * n1; p += NT) {
      const int i = p / n1, j = p - i * n1;
      a.U[s][(long long)(r0 + i) * n1 + j] = S.Ul[s][i][j];
    }
}

}  // namespace

size_t fused2d_smem_bytes() { return sizeof(Smem); }

cudaError_t launch_fused2d(const Fused2dArgs& a, cudaStream_t stream) {
  static bool attr[32] = {};   // per-device function attribute
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 32) dev = 0;
  if (!attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(fused2d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(Smem));
    if (e != cudaSuccess) return e;
    attr[dev] = true;
  }
  fused2d_kernel<<<CL, NT, sizeof(Smem), stream>>>(a);
  return cudaGetLastError();
}

}  // namespace kx

// ---------------------------------------------------------------------------------------
// A single small 2-D Tucker operator in one launch ("1 fused for d=2 small
// n", eq:exp2d P:240-250):  Y = alpha L_2 X L_1^T + beta Y  for n_1, n_2 <= 128.  CTA c forms
// rows I = [8c, 8c+8) of Y: it stages the whole X (<= 128 x 128) in shared memory, computes
// Z_I = L_2[I,:] X (one m8 fragment row block, kept in shared memory) and then Y_I = Z_I L_1^T;
// the operands of L are read from L2 once per product.  The intermediate never reaches HBM and
// the two mode products are one launch of ceil(n_2/8) CTAs.
namespace kx {
namespace {
constexpr int TS_NMAX = 128;
constexpr int TS_SS = TS_NMAX + 4;   // = 4 mod 16 doubles
constexpr int TS_NT = 256;

__global__ void __launch_bounds__(TS_NT) tucker2d_small_kernel(const double* __restrict__ X, double* Y,
                                                               const double* __restrict__ L1,
                                                               const double* __restrict__ L2, int n1, int n2,
                                                               double alpha, double beta) {
  extern __shared__ __align__(16) double ts_smem[];
  double(*Xs)[TS_SS] = reinterpret_cast<double(*)[TS_SS]>(ts_smem);   // X, then L1^T
  double(*Zs)[TS_SS] = reinterpret_cast<double(*)[TS_SS]>(ts_smem + TS_NMAX * TS_SS);
  double(*As)[TS_SS] = reinterpret_cast<double(*)[TS_SS]>(ts_smem + (TS_NMAX + 8) * TS_SS);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int r0 = blockIdx.x * 8, r = min(8, n2 - r0);
  const int n1p = (n1 + 7) & ~7, n2p = (n2 + 3) & ~3, n1q = (n1 + 3) & ~3;
  // stage X (rows < n2p, columns < n1p, zero padded) and the rows I of L2 in shared memory
  // a row-major n_rows x n1 matrix into the padded tile, 16-B loads when n1 is even
  auto stage = [&](const double* __restrict__ src, int rows, int rows_p) {
    if ((n1 & 1) == 0) {
      const int h = n1p / 2;
#pragma unroll 4
      for (int i = tid; i < rows_p * h; i += TS_NT) {
        const int row = i / h, col = 2 * (i - row * h);
        const double2 v = (row < rows && col < n1)
                              ? __ldg(reinterpret_cast<const double2*>(src + (long long)row * n1 + col))
                              : make_double2(0.0, 0.0);
        *reinterpret_cast<double2*>(&Xs[row][col]) = v;
      }
    } else {
#pragma unroll 4
      for (int i = tid; i < rows_p * n1p; i += TS_NT) {
        const int row = i / n1p, col = i - row * n1p;
        Xs[row][col] = (row < rows && col < n1) ? __ldg(src + (long long)row * n1 + col) : 0.0;
      }
    }
  };
  stage(X, n2, n2p);
  for (int i = tid; i < 8 * n2p; i += TS_NT) {
    const int k = i / 8, m = i - k * 8;   // column-major L2: consecutive threads, consecutive rows
    As[m][k] = (m < r && k < n2) ? L2[(long long)k * n2 + r0 + m] : 0.0;
  }
  __syncthreads();
  const int nf = n1p / 8;   // n-fragments of 8 columns: warp w takes w, w+8
  double z[2][2] = {};
  for (int kk = 0; kk < n2p; kk += 4) {
    const double av = As[g][kk + t4];
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const int j = warp + 8 * f;
      if (j < nf) dmma(z[f][0], z[f][1], av, Xs[kk + t4][j * 8 + g]);
    }
  }
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    const int j = warp + 8 * f;
    if (j < nf) {
      Zs[g][j * 8 + 2 * t4] = z[f][0];
      Zs[g][j * 8 + 2 * t4 + 1] = z[f][1];
    }
  }
  __syncthreads();
  // stage L1^T (L1's column-major buffer read row-major) over X
  stage(L1, n1, n1q);
  __syncthreads();
  double y[2][2] = {};
  for (int kk = 0; kk < n1q; kk += 4) {
    const double zv = Zs[g][kk + t4];
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const int j = warp + 8 * f;
      if (j < nf) dmma(y[f][0], y[f][1], zv, Xs[kk + t4][j * 8 + g]);
    }
  }
  if (g < r) {
    double* yr = Y + (long long)(r0 + g) * n1;
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const int c0 = (warp + 8 * f) * 8 + 2 * t4;
      if (c0 < n1) yr[c0] = alpha * y[f][0] + (beta != 0.0 ? beta * yr[c0] : 0.0);
      if (c0 + 1 < n1) yr[c0 + 1] = alpha * y[f][1] + (beta != 0.0 ? beta * yr[c0 + 1] : 0.0);
    }
  }
}
}  // namespace

bool tucker2d_small_fits(long long n1, long long n2) {
  return n1 >= 1 && n2 >= 1 && n1 <= TS_NMAX && n2 <= TS_NMAX;
}

cudaError_t launch_tucker2d_small(const double* X, double* Y, const double* L1, const double* L2, int n1,
                                  int n2, double alpha, double beta, cudaStream_t stream) {
  const size_t smem = (size_t)(TS_NMAX + 16) * TS_SS * sizeof(double);
  static bool attr[32] = {};   // per-device function attribute
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 32) dev = 0;
  if (!attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(tucker2d_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr[dev] = true;
  }
  tucker2d_small_kernel<<<(n2 + 7) / 8, TS_NT, smem, stream>>>(X, Y, L1, L2, n1, n2, alpha, beta);
  return cudaGetLastError();
}

}  // namespace kx
