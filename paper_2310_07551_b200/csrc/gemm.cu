// Kernel K*1: the mu-mode product as an fp64 tensor-core GEMM on sm_100a.
//
// PAPER.md P:196-206 defines S = T x_mu L elementwise; "a single (full) matrix-
// matrix product ... a single GEMM call", d of them per Tucker operator.  In vec order
// (first index fastest) no permute is needed:
//   mu = 1 :  Y_r = X_r * L^T      (A = X_r, k-contiguous  -> layout ROW; B = L^T row-major
//                                    = L's column-major buffer)
//   mu >= 2:  Y_b = L * X_b        (A = L column-major -> layout COL; B = X_b row-major
//                                    n_mu x prod_{nu<mu} n_nu; batched over prod_{nu>mu} n_nu)
// The split phi-actions use the same kernel with concatenated M (first mode: stacked
// [L^1; ...; L^T] reading X once) and concatenated K (last mode: sum over terms folded into
// the K loop, with the stage combination "+U" in the epilogue).
//
// fp64 tensor cores on sm_100a are reached only through the warp-level mma.sync.m8n8k4.f64
// (SASS DMMA.8x8x4); tcgen05/UMMA has no f64 kind.  Measured on the
// pool's B200 (profiles/peaks_r01.json): DMMA 37.1 TFLOP/s sustained, latency ~26 cycles.
// Design: cp.async multi-stage smem pipeline (16-B chunks, zero-filled edges), padded smem rows
// (stride = 4 mod 16 doubles -> conflict-free fragment loads for both layouts), each warp owns
// a WM x WN accumulator block (up to 64 x 32 = 32 DMMA per k-step from 12 fragment loads),
// epilogue C = alpha*acc + beta*D + gamma*E + diag*I with 16-B stores.
#include "kx_internal.h"

#include <algorithm>
#include <cmath>
#include <cstdio>

namespace kx {
namespace {


__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// D(8x8) += A(8x4, row) * B(4x8, col); fragments: a = A[g][t], b = B[t][g],
// c = {C[g][2t], C[g][2t+1]} with g = lane/4, t = lane%4.
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

template <int BM, int BN, int BK, int WM, int WN, bool AROW, int VEC, int STAGES>
struct Cfg {
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int NT = WARPS_M * WARPS_N * 32;
  static constexpr int SA = AROW ? (BK + 4) : (BM + 4);   // smem row stride (doubles)
  static constexpr int A_ST = AROW ? BM * SA : BK * SA;
  static constexpr int SB = BN + 4;
  static constexpr int B_ST = BK * SB;
  static constexpr int SMEM = STAGES * (A_ST + B_ST) * 8;
  // loader geometry: chunks of VEC doubles, each thread owns IA (A) and IB (B) chunks
  static constexpr int CPR_A = AROW ? BK / VEC : BM / VEC;   // chunks per smem row of A
  static constexpr int IA = BM * BK / VEC / NT;
  static constexpr int CPR_B = BN / VEC;
  static constexpr int IB = BK * BN / VEC / NT;
  static_assert(SA % 16 == 4 && SB % 16 == 4, "conflict-free fragment loads");
  static_assert((BM * BK / VEC) % NT == 0 && (BK * BN / VEC) % NT == 0, "loader divisibility");
  static_assert(IA <= 32 && IB <= 32, "validity masks are 32-bit");
};

// Launch schedule.  persistent = 0: one output tile per CTA (grid.x = tiles, grid.y = z).
// persistent = 1 (hybrid data-parallel + stream-K): grid.x = G co-resident CTAs; tiles
// [0, dp_tiles) are processed whole, round-robin; the remaining tiles' k-iterations are split
// into G_sk contiguous ranges.  A CTA whose range starts inside a tile stores its partial
// accumulators to its workspace slot and raises its flag; the CTA that owns the tile's first
// k-range adds the later partials in increasing-k order (deterministic), then runs the
// epilogue.  Waits only go to higher CTA indices, whose partial comes first in their range.
struct Sched {
  int tiles_m = 1, tiles_n = 1, m_fastest = 0, z0 = 0;
  int persistent = 0, G = 0, G_sk = 0, ktiles = 0;
  long long dp_tiles = 0, sk_units = 0;
};

template <int BM, int BN, int BK, int WM, int WN, bool AROW, int VEC, int STAGES>
struct GemmTile {
  using C_ = Cfg<BM, BN, BK, WM, WN, AROW, VEC, STAGES>;
  static constexpr int NT = C_::NT, SA = C_::SA, SB = C_::SB, A_ST = C_::A_ST, B_ST = C_::B_ST;
  static constexpr int IA = C_::IA, IB = C_::IB, CPR_A = C_::CPR_A, CPR_B = C_::CPR_B;
  static constexpr int FM = WM / 8, FN = WN / 8;

  struct Coord {
    int m0, n0, s, t, b;
  };

  __device__ __forceinline__ static Coord coords(const GemmArgs& p, const Sched& sc, long long tl) {
    const long long tmn = (long long)sc.tiles_m * sc.tiles_n;
    const int z = sc.z0 + (int)(tl / tmn);
    const int r = (int)(tl - (tl / tmn) * tmn);
    int tm, tn;
    if (sc.m_fastest) {
      tm = r % sc.tiles_m;
      tn = r / sc.tiles_m;
    } else {
      tn = r % sc.tiles_n;
      tm = r / sc.tiles_n;
    }
    Coord c;
    c.m0 = tm * BM;
    c.n0 = tn * BN;
    c.b = z % p.nb;
    const int zt = z / p.nb;
    c.t = zt % p.nt;
    c.s = zt / p.nt;
    return c;
  }

  // acc += sum over k-tiles [kb, ke) of the (m0, n0) tile.
  __device__ __forceinline__ static void mainloop(const GemmArgs& p, double* smem, const Coord& cd,
                                                  int kb, int ke, double (&acc)[FM][FN][2]) {
    double* As = smem;
    double* Bs = smem + STAGES * A_ST;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int wm0 = (warp / C_::WARPS_N) * WM, wn0 = (warp % C_::WARPS_N) * WN;
    const int m0 = cd.m0, n0 = cd.n0;
    const double* __restrict__ A = p.A[cd.s] + cd.t * p.sA_t + cd.b * p.sA_b;
    const double* __restrict__ B = p.B[cd.s] + cd.t * p.sB_t + cd.b * p.sB_b;
    const int M = p.M, N = p.N, kseg = p.kseg;
    const int lda = (int)p.lda, ldb = (int)p.ldb;
    const int kps = (kseg + BK - 1) / BK;

    // per-thread loader state: 32-bit offsets inside the operand + validity masks; per k-tile
    // only a pointer add and a predicate remain
    int offA[IA], krA[IA], offB[IB], krB[IB], smA[IA], smB[IB];
    unsigned okA = 0, okB = 0;
#pragma unroll
    for (int it = 0; it < IA; ++it) {
      const int c = tid + it * NT;
      if constexpr (AROW) {
        const int r = c / CPR_A, kc = (c % CPR_A) * VEC;
        const bool v = m0 + r < M;
        offA[it] = (v ? (m0 + r) : 0) * lda + kc;
        krA[it] = kc;
        okA |= (unsigned)v << it;
      } else {
        const int kr = c / CPR_A, mc = (c % CPR_A) * VEC;
        const bool v = m0 + mc < M;
        offA[it] = kr * lda + (v ? m0 + mc : 0);
        krA[it] = kr;
        okA |= (unsigned)v << it;
      }
      smA[it] = (c / CPR_A) * SA + (c % CPR_A) * VEC;
    }
#pragma unroll
    for (int it = 0; it < IB; ++it) {
      const int c = tid + it * NT;
      const int kr = c / CPR_B, nc = (c % CPR_B) * VEC;
      const bool v = n0 + nc < N;
      offB[it] = kr * ldb + (v ? n0 + nc : 0);
      krB[it] = kr;
      okB |= (unsigned)v << it;
      smB[it] = (c / CPR_B) * SB + (c % CPR_B) * VEC;
    }

    int lseg = kb / kps, lk0 = (kb - (kb / kps) * kps) * BK;   // load cursor
    auto issue_loads = [&](int stage) {
      double* as = As + stage * A_ST;
      double* bs = Bs + stage * B_ST;
      const double* Ab = A + p.seg_off[lseg] + (AROW ? (long long)lk0 : (long long)lk0 * lda);
      const double* Bb = B + ((long long)lseg * kseg + lk0) * ldb;
#pragma unroll
      for (int it = 0; it < IA; ++it) {
        const bool v = ((okA >> it) & 1u) && (lk0 + krA[it] < kseg);
        const double* src = v ? Ab + offA[it] : A;
        if constexpr (VEC == 2) cp_async16(as + smA[it], src, v);
        else cp_async8(as + smA[it], src, v);
      }
#pragma unroll
      for (int it = 0; it < IB; ++it) {
        const bool v = ((okB >> it) & 1u) && (lk0 + krB[it] < kseg);
        const double* src = v ? Bb + offB[it] : B;
        if constexpr (VEC == 2) cp_async16(bs + smB[it], src, v);
        else cp_async8(bs + smB[it], src, v);
      }
      lk0 += BK;
      if (lk0 >= kseg) {
        lk0 = 0;
        ++lseg;
      }
    };

    const int n = ke - kb;
    __syncthreads();   // the previous tile's readers are done with every stage
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
      if (st < n) issue_loads(st);
      cp_async_commit();
    }
    for (int kt = 0; kt < n; ++kt) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      const double* as = As + (kt % STAGES) * A_ST;
      const double* bs = Bs + (kt % STAGES) * B_ST;
      const int nk = kt + STAGES - 1;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double af[FM], bf[FN];
#pragma unroll
        for (int i = 0; i < FM; ++i) {
          if constexpr (AROW) af[i] = as[(wm0 + i * 8 + g) * SA + kk + t4];
          else af[i] = as[(kk + t4) * SA + wm0 + i * 8 + g];
        }
#pragma unroll
        for (int j = 0; j < FN; ++j) bf[j] = bs[(kk + t4) * SB + wn0 + j * 8 + g];
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        if (kk == 0) {
          // prefetch tile kt+STAGES-1 into the stage freed by iteration kt-1, interleaved
          // with the DMMAs already queued for this k-step
          if (nk < n) issue_loads(nk % STAGES);
          cp_async_commit();
        }
      }
    }
    cp_async_wait<0>();
  }

  // C = alpha*acc + beta*D + gamma*E + diag*[m==n]
  __device__ __forceinline__ static void epilogue(const GemmArgs& p, const Coord& cd,
                                                  const double (&acc)[FM][FN][2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int wm0 = (warp / C_::WARPS_N) * WM, wn0 = (warp % C_::WARPS_N) * WN;
    const int M = p.M, N = p.N;
    double* __restrict__ C = p.C[cd.s] + cd.t * p.sC_t + cd.b * p.sC_b;
    const double* D = p.D[cd.s] ? p.D[cd.s] + cd.t * p.sD_t + cd.b * p.sD_b : nullptr;
    const double* E = p.E[cd.s] ? p.E[cd.s] + cd.t * p.sE_t + cd.b * p.sE_b : nullptr;
    const double alpha = p.alpha, beta = p.beta, gamma = p.gamma, diag = p.diag;
#pragma unroll
    for (int i = 0; i < FM; ++i) {
      const int m = cd.m0 + wm0 + i * 8 + g;
      if (m >= M) continue;
#pragma unroll
      for (int j = 0; j < FN; ++j) {
        const int n = cd.n0 + wn0 + j * 8 + 2 * t4;
        if (n >= N) continue;
        double v0 = alpha * acc[i][j][0], v1 = alpha * acc[i][j][1];
        if constexpr (VEC == 2) {
          if (D) {
            const double2 d2 = *reinterpret_cast<const double2*>(D + (long long)m * p.ldd + n);
            v0 += beta * d2.x;
            v1 += beta * d2.y;
          }
          if (E) {
            const double2 e2 = *reinterpret_cast<const double2*>(E + (long long)m * p.lde + n);
            v0 += gamma * e2.x;
            v1 += gamma * e2.y;
          }
          if (m == n) v0 += diag;
          if (m == n + 1) v1 += diag;
          *reinterpret_cast<double2*>(C + (long long)m * p.ldc + n) = make_double2(v0, v1);
        } else {
          if (D) v0 += beta * D[(long long)m * p.ldd + n];
          if (E) v0 += gamma * E[(long long)m * p.lde + n];
          if (m == n) v0 += diag;
          C[(long long)m * p.ldc + n] = v0;
          if (n + 1 < N) {
            if (D) v1 += beta * D[(long long)m * p.ldd + n + 1];
            if (E) v1 += gamma * E[(long long)m * p.lde + n + 1];
            if (m == n + 1) v1 += diag;
            C[(long long)m * p.ldc + n + 1] = v1;
          }
        }
      }
    }
  }

  __device__ __forceinline__ static void zero(double (&acc)[FM][FN][2]) {
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  }
};

template <int BM, int BN, int BK, int WM, int WN, bool AROW, int VEC, int STAGES, bool SKP>
__global__ void __launch_bounds__(Cfg<BM, BN, BK, WM, WN, AROW, VEC, STAGES>::NT)
    gemm_kernel(const GemmArgs p, const Sched sc) {
  using T_ = GemmTile<BM, BN, BK, WM, WN, AROW, VEC, STAGES>;
  constexpr int NT = T_::NT, FM = T_::FM, FN = T_::FN;
  extern __shared__ __align__(16) double smem[];
  double acc[FM][FN][2];
  const int ktiles = sc.ktiles;
  if constexpr (!SKP) {
    const long long tl = (long long)blockIdx.y * sc.tiles_m * sc.tiles_n + blockIdx.x;
    const typename T_::Coord cd = T_::coords(p, sc, tl);
    T_::zero(acc);
    T_::mainloop(p, smem, cd, 0, ktiles, acc);
    T_::epilogue(p, cd, acc);
    return;
  } else {
  const int i = blockIdx.x, G = sc.G;
  for (long long tl = i; tl < sc.dp_tiles; tl += G) {
    const typename T_::Coord cd = T_::coords(p, sc, tl);
    T_::zero(acc);
    T_::mainloop(p, smem, cd, 0, ktiles, acc);
    T_::epilogue(p, cd, acc);
  }
  const int Gs = sc.G_sk;
  if (i >= Gs || sc.sk_units == 0) return;
  const long long u0 = (long long)i * sc.sk_units / Gs, u1 = (long long)(i + 1) * sc.sk_units / Gs;
  double* ws_me = p.sk_ws + (size_t)i * (FM * FN * 2 * NT);
  for (long long u = u0; u < u1;) {
    const long long tr = u / ktiles;
    const int kb = (int)(u - tr * ktiles);
    const int ke = (int)((long long)kb + (u1 - u) < ktiles ? kb + (u1 - u) : ktiles);
    const typename T_::Coord cd = T_::coords(p, sc, sc.dp_tiles + tr);
    T_::zero(acc);
    T_::mainloop(p, smem, cd, kb, ke, acc);
    if (kb > 0) {
      // contributor: publish the partial (thread-fragment order, coalesced) and signal
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int c = 0; c < FN; ++c)
#pragma unroll
          for (int e = 0; e < 2; ++e) __stcg(ws_me + ((a * FN + c) * 2 + e) * NT + threadIdx.x, acc[a][c][e]);
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) atomicExch(p.sk_flags + i, 1);
    } else {
      if (ke < ktiles) {
        // owner of a split tile: add the later k-ranges' partials in increasing k
        for (int j = i + 1; j < Gs; ++j) {
          const long long bj = (long long)j * sc.sk_units / Gs;
          if (bj >= (tr + 1) * ktiles) break;
          if (threadIdx.x == 0) {
            volatile int* f = p.sk_flags + j;
            while (*f == 0) __nanosleep(64);
            __threadfence();
            *f = 0;
          }
          __syncthreads();
          const double* wj = p.sk_ws + (size_t)j * (FM * FN * 2 * NT);
#pragma unroll
          for (int a = 0; a < FM; ++a)
#pragma unroll
            for (int c = 0; c < FN; ++c)
#pragma unroll
              for (int e = 0; e < 2; ++e) acc[a][c][e] += __ldcg(wj + ((a * FN + c) * 2 + e) * NT + threadIdx.x);
        }
      }
      T_::epilogue(p, cd, acc);
    }
    u += ke - kb;
  }
  }
}

struct TileChoice {
  int bm, bn, occ;
  double eff;
};
// Resident CTAs per SM (register/smem-limited) and relative per-SM efficiency of each config.
constexpr TileChoice kTiles[3] = {{128, 128, 1, 1.00}, {128, 64, 2, 0.97}, {64, 64, 3, 0.90}};

template <int BM, int BN, int BK, int WM, int WN, bool AROW, int VEC, int STAGES>
cudaError_t prepare_cfg() {
  using C_ = Cfg<BM, BN, BK, WM, WN, AROW, VEC, STAGES>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel<BM, BN, BK, WM, WN, AROW, VEC, STAGES, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM);
    if (e != cudaSuccess) return e;
    if constexpr (BM == 128 && BN == 128) {
      e = cudaFuncSetAttribute(gemm_kernel<BM, BN, BK, WM, WN, AROW, VEC, STAGES, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM);
      if (e != cudaSuccess) return e;
    }
    attr_done = true;
  }
  return cudaSuccess;
}

int num_sms();

template <int BM, int BN, int BK, int WM, int WN, bool AROW, int VEC, int STAGES>
cudaError_t launch_cfg(const GemmArgs& g, int nz, bool allow_sk, cudaStream_t stream) {
  using C_ = Cfg<BM, BN, BK, WM, WN, AROW, VEC, STAGES>;
  auto kern = gemm_kernel<BM, BN, BK, WM, WN, AROW, VEC, STAGES, false>;
  cudaError_t e = prepare_cfg<BM, BN, BK, WM, WN, AROW, VEC, STAGES>();
  if (e != cudaSuccess) return e;
  Sched sc;
  sc.tiles_m = (g.M + BM - 1) / BM;
  sc.tiles_n = (g.N + BN - 1) / BN;
  sc.m_fastest = AROW ? 0 : 1;
  sc.ktiles = ((g.kseg + BK - 1) / BK) * g.nseg;
  const long long tmn = (long long)sc.tiles_m * sc.tiles_n;
  const long long T = tmn * nz;
  const int G = num_sms();   // 1 CTA/SM for the configs that allow stream-K
  if (allow_sk && g.sk_ws && g.sk_flags && G <= kSkSlots && T % G != 0 && sc.ktiles >= 8) {
    const double waves = (double)T / G;
    const double quant = std::ceil(waves) / waves;   // classic-schedule slowdown
    if (quant > 1.06) {
      long long dp = (T / G) * G;
      if (dp >= G && (T - dp) * 2 < G) dp -= G;      // short tail: spread one more wave
      sc.persistent = 1;
      sc.G = G;
      sc.dp_tiles = dp;
      sc.sk_units = (T - dp) * sc.ktiles;
      sc.G_sk = (int)std::min<long long>(G, sc.sk_units / 4);
      if constexpr (BM == 128 && BN == 128)
        gemm_kernel<BM, BN, BK, WM, WN, AROW, VEC, STAGES, true><<<dim3(G, 1), C_::NT, C_::SMEM, stream>>>(g, sc);
      return cudaGetLastError();
    }
  }
  for (int z0 = 0; z0 < nz; z0 += 65535) {
    sc.z0 = z0;
    dim3 grid((unsigned)tmn, (unsigned)std::min(65535, nz - z0));
    kern<<<grid, C_::NT, C_::SMEM, stream>>>(g, sc);
  }
  return cudaGetLastError();
}

template <bool AROW, int VEC>
cudaError_t launch_layout(const GemmArgs& g, int nz, int which, cudaStream_t stream) {
  switch (which) {
    case 0: return launch_cfg<128, 128, 32, 64, 32, AROW, VEC, 3>(g, nz, true, stream);
    case 1: return launch_cfg<128, 64, 16, 64, 32, AROW, VEC, 3>(g, nz, false, stream);
    default: return launch_cfg<64, 64, 16, 32, 32, AROW, VEC, 3>(g, nz, false, stream);
  }
}

template <bool AROW, int VEC>
void prepare_layout() {
  prepare_cfg<128, 128, 32, 64, 32, AROW, VEC, 3>();
  prepare_cfg<128, 64, 16, 64, 32, AROW, VEC, 3>();
  prepare_cfg<64, 64, 16, 32, 32, AROW, VEC, 3>();
}

int num_sms() {
  static int nsm = 0;   // defined once; declared above for launch_cfg
  if (nsm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) nsm = 148;
  }
  return nsm;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

// Set the dynamic-smem attribute of every instantiation up front (kx_create), so that no
// attribute call happens while a step is being captured into a CUDA graph.
void gemm_prepare_all() {
  prepare_layout<true, 2>();
  prepare_layout<true, 1>();
  prepare_layout<false, 2>();
  prepare_layout<false, 1>();
  num_sms();
}

double gemm_flops(const GemmArgs& g) {
  return 2.0 * g.M * (double)g.N * (double)g.kseg * g.nseg * g.ns * g.nt * g.nb;
}

cudaError_t launch_gemm(const GemmArgs& g, cudaStream_t stream) {
  const int nz = g.ns * g.nt * g.nb;
  if (g.M <= 0 || g.N <= 0 || nz <= 0) return cudaSuccess;
  if (g.kseg <= 0) return cudaErrorInvalidValue;
  // Vector (16-B) path: every contiguous extent, leading dimension, batch stride, segment
  // offset and base pointer must keep 2-double chunks 16-B aligned.
  bool vec = (g.N % 2 == 0) && (g.ldb % 2 == 0) && (g.ldc % 2 == 0) && (g.ldd % 2 == 0) &&
             (g.lde % 2 == 0) && (g.lda % 2 == 0);
  vec = vec && (g.arow ? (g.kseg % 2 == 0) : (g.M % 2 == 0));
  const long long strides[] = {g.sA_t, g.sA_b, g.sB_t, g.sB_b, g.sC_t, g.sC_b,
                               g.sD_t, g.sD_b, g.sE_t, g.sE_b};
  for (long long st : strides) vec = vec && (st % 2 == 0);
  for (int i = 0; i < g.nseg && i < MAXSEG; ++i) vec = vec && (g.seg_off[i] % 2 == 0);
  for (int s = 0; s < g.ns; ++s) {
    vec = vec && aligned16(g.A[s]) && aligned16(g.B[s]) && aligned16(g.C[s]);
    if (g.D[s]) vec = vec && aligned16(g.D[s]);
    if (g.E[s]) vec = vec && aligned16(g.E[s]);
  }
  // Tile choice: minimise (waves x per-wave work) / efficiency on 148 SMs.
  const int nsm = num_sms();
  int best = 0;
  double best_cost = 1e300;
  for (int i = 0; i < 3; ++i) {
    const TileChoice& c = kTiles[i];
    const double tiles = (double)((g.M + c.bm - 1) / c.bm) * ((g.N + c.bn - 1) / c.bn) * nz;
    double waves = std::ceil(tiles / ((double)nsm * c.occ));
    const int kt = (g.kseg + 31) / 32 * g.nseg;
    if (i == 0 && g.sk_ws && kt >= 8 && waves / (tiles / nsm) > 1.06)
      waves = 1.03 * tiles / nsm;   // stream-K tail: ~3% fix-up overhead
    const double cost = waves * c.occ * c.bm * c.bn / c.eff;
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = i;
    }
  }
  if (g.arow) return vec ? launch_layout<true, 2>(g, nz, best, stream) : launch_layout<true, 1>(g, nz, best, stream);
  return vec ? launch_layout<false, 2>(g, nz, best, stream) : launch_layout<false, 1>(g, nz, best, stream);
}

}  // namespace kx
