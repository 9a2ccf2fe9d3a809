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

#include <cuda.h>
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

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
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(bar))
               : "memory");
}
// arrives on `bar` once all of this thread's prior cp.async operations have completed
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// VEC == 3: the operand tiles arrive by TMA (cp.async.bulk.tensor) in FRAGMENT ORDER: the 4-D
// boxes are chosen so that the 32 doubles one m8n8k4 fragment load of a warp reads are one
// contiguous 256-B block of shared memory whose two 128-B halves are lanes 0-15 and 16-31 (a
// 64-bit shared load is served per half-warp): 2 wavefronts, no bank conflicts, no swizzle:
//   B and COL A (k rows, n / m contiguous): box {4 n, 4 k, n/4, k/4} -> [k/4][n/4][k%4][n%4];
//   ROW A (m rows, k contiguous): box {4 k, 8 m, k/4, m/8} -> [m/8][k/4][m%8][k%4].
// (Tried first: a 64-B-swizzled [chunk][row][8] layout — rows k and k+2 share banks — and
// [k/4][n/8][k%4][n%8] — lanes 0-15 then span all 256 B: 2-way conflicts either way.)
constexpr int kTmaMaxA = 16;   // A maps: species x concatenated-K segments
struct TmaMaps {
  CUtensorMap A[kTmaMaxA];
  CUtensorMap B[MAXS];
  int nsegmaps = 1;            // A map of (species s, segment j) = A[s * nsegmaps + j]
};
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load5(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                          int c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
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
  // resident CTAs per SM the register budget must allow (512 threads: 1 at <= 128 registers;
  // 256: 2 at <= 128; 128: 3 at <= 170)
  static constexpr int MINB = NT >= 512 ? 1 : (NT >= 256 ? 2 : 3);
  static constexpr bool TMA = VEC == 3;                     // TMA loads, swizzled unpadded tiles
  static constexpr int LV = TMA ? 2 : VEC;                   // cp.async chunk (doubles)
  static constexpr int SA = TMA ? 0 : (AROW ? (BK + 4) : (BM + 4));   // smem row stride (doubles)
  static constexpr int A_ST = TMA ? BM * BK : (AROW ? BM * SA : BK * SA);
  static constexpr int SB = TMA ? 0 : BN + 4;
  static constexpr int B_ST = TMA ? BK * BN : BK * SB;
  static constexpr int ALIGN = TMA ? 1024 : 0;               // swizzle atoms 512-B aligned
  static constexpr int SMEM = STAGES * (A_ST + B_ST) * 8 + 2 * STAGES * 8 + ALIGN + (TMA ? 512 : 0);   // + mbarriers (+ TMA producer state)
  // loader geometry: chunks of LV doubles, each thread owns IA (A) and IB (B) chunks
  static constexpr int CPR_A = AROW ? BK / LV : BM / LV;   // chunks per smem row of A
  static constexpr int IA = BM * BK / LV / NT;
  static constexpr int CPR_B = BN / LV;
  static constexpr int IB = BK * BN / LV / NT;
  static_assert(TMA || (SA % 16 == 4 && SB % 16 == 4), "conflict-free fragment loads");
  static_assert(!TMA || (BK % 8 == 0 && BM % 8 == 0 && BN % 8 == 0 && BM <= 256 && BN / 8 <= 256),
                "TMA boxes");
  static_assert((BM * BK / LV) % NT == 0 && (BK * BN / LV) % NT == 0, "loader divisibility");
  static_assert(IA <= 32 && IB <= 32, "validity masks are 32-bit");
};

// Persistent, cross-tile pipelined schedule.  grid.x = G co-resident CTAs.  CTA i walks
// a work list: data-parallel tiles i, i+G, ... < dp_tiles (whole k range), then its share of
// the stream-K region (tiles [dp_tiles, T) with their k-iterations split into G_sk contiguous
// ranges).  The cp.async producer runs STAGES-1 k-tiles ahead of the DMMA consumer ACROSS
// tile boundaries, so the next tile's first stages load while this tile's epilogue runs.
// Stream-K fix-up: every CTA holding a k-range of a split tile stores its partial accumulators
// to a workspace slot and counts itself in on the tile's counter; the contributors for which
// the tile is the last item of their work list wait until all are in, then each sums a share
// of the tile's fragments over the partials in increasing-k order (deterministic, independent
// of which CTA sums) and stores it.  Waits happen only at the end of a CTA's list and only on
// partials that are the first or last item of another CTA's list, so every wait ends (all
// CTAs are co-resident: cooperative launch).
struct Sched {
  int tiles_m = 1, tiles_n = 1, m_fastest = 0, ktiles = 0;
  // > 1: cluster split-K — the CTAs of one thread-block cluster (csplit of them) each take an
  // equal k-range of the same tile and reduce their partials through distributed shared memory
  int csplit = 0;
  int G = 1, G_sk = 0;
  long long dp_tiles = 0, sk_units = 0;
};

struct Seg {
  long long tl;
  int kb, ke;
};

struct WorkIter {
  long long next_dp, dp_tiles, u, u1;
  int G, ktiles;
  __device__ __forceinline__ void init(const Sched& sc, int i) {
    next_dp = i;
    dp_tiles = sc.dp_tiles;
    G = sc.G;
    ktiles = sc.ktiles;
    if (i < sc.G_sk) {
      u = (long long)i * sc.sk_units / sc.G_sk;
      u1 = (long long)(i + 1) * sc.sk_units / sc.G_sk;
    } else {
      u = u1 = 0;
    }
  }
  __device__ __forceinline__ bool next(Seg& s) {
    if (next_dp < dp_tiles) {
      s.tl = next_dp;
      s.kb = 0;
      s.ke = ktiles;
      next_dp += G;
      return true;
    }
    if (u < u1) {
      const long long tr = u / ktiles;
      s.kb = (int)(u - tr * ktiles);
      s.ke = (int)((long long)s.kb + (u1 - u) < ktiles ? s.kb + (u1 - u) : ktiles);
      s.tl = dp_tiles + tr;
      u += s.ke - s.kb;
      return true;
    }
    return false;
  }
};

// first stream-K unit of CTA i (i = G_sk: the end)
__device__ __forceinline__ long long sk_begin(const Sched& sc, int i) {
  return (long long)i * sc.sk_units / sc.G_sk;
}
// workspace slot of CTA i's partial of the split tile starting at unit t0u: a CTA holds at
// most two split segments (the tail of the tile its range starts in, the head of the tile it
// ends in), so slot 2i serves the first and 2i+1 the second and neither is overwritten while
// the other tile's contributors may still read it
__device__ __forceinline__ int sk_slot(const Sched& sc, int i, long long t0u) {
  return 2 * i + (sk_begin(sc, i) >= t0u ? 0 : 1);
}

template <int BM, int BN, int BK, int WM, int WN, bool AROW, int VEC, int STAGES, bool PEER = false>
struct GemmTile {
  using C_ = Cfg<BM, BN, BK, WM, WN, AROW, VEC, STAGES>;
  static constexpr int NT = C_::NT, SA = C_::SA, SB = C_::SB, A_ST = C_::A_ST, B_ST = C_::B_ST;
  static constexpr int IA = C_::IA, IB = C_::IB, CPR_A = C_::CPR_A, CPR_B = C_::CPR_B, LV = C_::LV;
  static constexpr int FM = WM / 8, FN = WN / 8;
  static constexpr bool TMA = C_::TMA;

  struct Coord {
    int m0, n0, s, t, b;
  };

  __device__ __forceinline__ static Coord coords(const GemmArgs& p, const Sched& sc, long long tl) {
    // 32-bit arithmetic: tile counts stay far below 2^31
    const unsigned tmn = (unsigned)sc.tiles_m * (unsigned)sc.tiles_n;
    const unsigned zq = (unsigned)tl / tmn;
    const int z = (int)zq;
    const int r = (int)((unsigned)tl - zq * tmn);
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

  // cp.async producer state for one tile: 32-bit offsets inside the operands + validity
  // masks; per k-tile only a pointer add and a predicate remain.
  struct Loader {
    const double* A;
    const double* B;
    int offA[TMA ? 1 : IA], offB[TMA ? 1 : IB];
    unsigned okA, okB;
    int lseg, lk0;
    Coord tc;   // TMA: the tile's coordinates

    __device__ __forceinline__ void setup(const GemmArgs& p, const Coord& cd, int kb) {
      const int tid = threadIdx.x;
      if constexpr (TMA) {
        tc = cd;
        const int kps = (p.kseg + BK - 1) / BK;
        lseg = kb / kps;
        lk0 = (kb - lseg * kps) * BK;
        return;
      }
      A = p.A[cd.s] + cd.t * p.sA_t + cd.b * p.sA_b;
      B = p.B[cd.s] + cd.t * p.sB_t + cd.b * p.sB_b;
      const int lda = (int)p.lda, ldb = (int)p.ldb;
      okA = okB = 0;
#pragma unroll
      for (int it = 0; it < IA; ++it) {
        const int c = tid + it * NT;
        if constexpr (AROW) {
          const int r = c / CPR_A, kc = (c % CPR_A) * LV;
          const bool v = cd.m0 + r < p.M;
          offA[it] = (v ? (cd.m0 + r) : 0) * lda + kc;
          okA |= (unsigned)v << it;
        } else {
          const int kr = c / CPR_A, mc = (c % CPR_A) * LV;
          const bool v = cd.m0 + mc < p.M;
          offA[it] = kr * lda + (v ? cd.m0 + mc : 0);
          okA |= (unsigned)v << it;
        }
      }
#pragma unroll
      for (int it = 0; it < IB; ++it) {
        const int c = tid + it * NT;
        const int kr = c / CPR_B, nc = (c % CPR_B) * LV;
        const int np = cd.n0 + nc;
        const bool v = np < p.N;
        if (p.nflat) {   // flattened batches: column np is batch np / nflat
          const int b = v ? np / p.nflat : 0;
          offB[it] = v ? b * (int)p.sB_b + kr * ldb + (np - b * p.nflat) : kr * ldb;
        } else {
          offB[it] = kr * ldb + (v ? np : 0);
        }
        okB |= (unsigned)v << it;
      }
      const int kps = (p.kseg + BK - 1) / BK;
      lseg = kb / kps;
      lk0 = (kb - lseg * kps) * BK;
    }

    // TMA (one thread): the A and B boxes of the next k-tile, completion counted on `bar`
    __device__ __forceinline__ void issue_tma(const GemmArgs& p, const TmaMaps& tm, double* as, double* bs,
                                              uint64_t* bar) {
      mbar_expect_tx(bar, (BM * BK + BK * BN) * 8);
      const CUtensorMap* mA = &tm.A[tc.s * tm.nsegmaps + (AROW ? lseg : 0)];
      if constexpr (AROW) tma_load5(as, mA, 0, 0, lk0 / 4, tc.m0 / 8, tc.t, bar);   // [m/8][k/4][8][4]
      else tma_load5(as, mA, 0, 0, tc.m0 / 4, lk0 / 4, tc.t, bar);                 // [k/4][m/4][4][4]
      tma_load5(bs, &tm.B[tc.s], 0, 0, tc.n0 / 4, (lseg * p.kseg + lk0) / 4, tc.t, bar);   // [k/4][n/4][4][4]
      lk0 += BK;
      if (lk0 >= p.kseg) {
        lk0 = 0;
        ++lseg;
      }
    }

    __device__ __forceinline__ void issue(const GemmArgs& p, double* as, double* bs) {
      const int tid = threadIdx.x;
      if (p.diag_noload) {   // diagnostics: the pipeline without its copies
        lk0 += BK;
        if (lk0 >= p.kseg) {
          lk0 = 0;
          ++lseg;
        }
        return;
      }
      const int kseg = p.kseg;
      const double* Ab = A + p.seg_off[lseg] + (AROW ? (long long)lk0 : (long long)lk0 * p.lda);
      const double* Bb = B + ((long long)lseg * kseg + lk0) * p.ldb;
#pragma unroll
      for (int it = 0; it < IA; ++it) {
        const int c = tid + it * NT;
        const int kr = AROW ? (c % CPR_A) * VEC : c / CPR_A;
        const bool v = ((okA >> it) & 1u) && (lk0 + kr < kseg);
        const double* src = v ? Ab + offA[it] : A;
        double* dst = as + (c / CPR_A) * SA + (c % CPR_A) * LV;
        if constexpr (LV == 2) cp_async16(dst, src, v);
        else cp_async8(dst, src, v);
      }
#pragma unroll
      for (int it = 0; it < IB; ++it) {
        const int c = tid + it * NT;
        const int kr = c / CPR_B;
        const bool v = ((okB >> it) & 1u) && (lk0 + kr < kseg);
        const double* src = v ? Bb + offB[it] : B;
        double* dst = bs + kr * SB + (c % CPR_B) * LV;
        if constexpr (LV == 2) cp_async16(dst, src, v);
        else cp_async8(dst, src, v);
      }
      lk0 += BK;
      if (lk0 >= kseg) {
        lk0 = 0;
        ++lseg;
      }
    }
  };

  __device__ __forceinline__ static double* out_ptr(const GemmArgs& p, int s, double* q) {
    if constexpr (PEER) return peer_redirect(p.peer, s, q);
    else return q;
  }

  // C = alpha*acc + beta*D + gamma*E + diag*[m==n]
  __device__ __forceinline__ static void epilogue(const GemmArgs& p, const Coord& cd,
                                                  const double (&acc)[FM][FN][2], unsigned mask) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int wm0 = (warp / C_::WARPS_N) * WM, wn0 = (warp % C_::WARPS_N) * WN;
    const int M = p.M, N = p.N;
    double* __restrict__ C = p.C[cd.s] + cd.t * p.sC_t + cd.b * p.sC_b;
    const double* D = p.D[cd.s] ? p.D[cd.s] + cd.t * p.sD_t + cd.b * p.sD_b : nullptr;
    const double* E = p.E[cd.s] ? p.E[cd.s] + cd.t * p.sE_t + cd.b * p.sE_b : nullptr;
    const double alpha = p.alpha, beta = p.beta, gamma = p.gamma, diag = p.diag;
    if constexpr (VEC >= 2) {
      // fast paths for whole interior tiles (every launch of the large configs): no bounds
      // checks, row pointers hoisted, the D loads issued before the stores
      const bool plain = !PEER && !p.nflat && mask == ~0u && !E && diag == 0.0 && cd.m0 + BM <= M &&
                         cd.n0 + BN <= N;
      if (plain) {
        const long long ls = 8 * p.ldc;
        double* Cw = C + (long long)(cd.m0 + wm0 + g) * p.ldc + cd.n0 + wn0 + 2 * t4;
        if (!D) {
#pragma unroll
          for (int i = 0; i < FM; ++i)
#pragma unroll
            for (int j = 0; j < FN; ++j)
              *reinterpret_cast<double2*>(Cw + i * ls + j * 8) =
                  make_double2(alpha * acc[i][j][0], alpha * acc[i][j][1]);
          return;
        }
        const long long ld = 8 * p.ldd;
        const double* Dw = D + (long long)(cd.m0 + wm0 + g) * p.ldd + cd.n0 + wn0 + 2 * t4;
#pragma unroll
        for (int i = 0; i < FM; ++i) {
          double2 dv[FN];   // one fragment row of D in flight at a time (register budget)
#pragma unroll
          for (int j = 0; j < FN; ++j) dv[j] = *reinterpret_cast<const double2*>(Dw + i * ld + j * 8);
#pragma unroll
          for (int j = 0; j < FN; ++j)
            *reinterpret_cast<double2*>(Cw + i * ls + j * 8) =
                make_double2(alpha * acc[i][j][0] + beta * dv[j].x, alpha * acc[i][j][1] + beta * dv[j].y);
        }
        return;
      }
    }
#pragma unroll
    for (int i = 0; i < FM; ++i) {
      const int m = cd.m0 + wm0 + i * 8 + g;
      if (m >= M) continue;
#pragma unroll
      for (int j = 0; j < FN; ++j) {
        const int n = cd.n0 + wn0 + j * 8 + 2 * t4;
        if (n >= N || !((mask >> (i * FN + j)) & 1u)) continue;
        double v0 = alpha * acc[i][j][0], v1 = alpha * acc[i][j][1];
        // element offsets of (m, n) in C / D / E (flattened batches: n is batch n / nflat)
        long long oc = (long long)m * p.ldc + n, od = (long long)m * p.ldd + n, oe = (long long)m * p.lde + n;
        if (p.nflat) {
          const int b = n / p.nflat, nn = n - b * p.nflat;
          oc = b * p.sC_b + (long long)m * p.ldc + nn;
          od = b * p.sD_b + (long long)m * p.ldd + nn;
          oe = b * p.sE_b + (long long)m * p.lde + nn;
        }
        if constexpr (VEC >= 2) {
          if (D) {
            const double2 d2 = *reinterpret_cast<const double2*>(D + od);
            v0 += beta * d2.x;
            v1 += beta * d2.y;
          }
          if (E) {
            const double2 e2 = *reinterpret_cast<const double2*>(E + oe);
            v0 += gamma * e2.x;
            v1 += gamma * e2.y;
          }
          if (m == n) v0 += diag;
          if (m == n + 1) v1 += diag;
          *reinterpret_cast<double2*>(out_ptr(p, cd.s, C + oc)) = make_double2(v0, v1);
        } else {
          if (D) v0 += beta * D[od];
          if (E) v0 += gamma * E[oe];
          if (m == n) v0 += diag;
          *out_ptr(p, cd.s, C + oc) = v0;
          if (n + 1 < N) {
            if (D) v1 += beta * D[od + 1];
            if (E) v1 += gamma * E[oe + 1];
            if (m == n + 1) v1 += diag;
            *out_ptr(p, cd.s, C + oc + 1) = v1;
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

template <int BM, int BN, int BK, int WM, int WN, bool AROW, int VEC, int STAGES, bool PEER = false>
__global__ void __launch_bounds__(Cfg<BM, BN, BK, WM, WN, AROW, VEC, STAGES>::NT,
                                  Cfg<BM, BN, BK, WM, WN, AROW, VEC, STAGES>::MINB)
    gemm_kernel(const GemmArgs p, const Sched sc, const __grid_constant__ TmaMaps tm) {
  using T_ = GemmTile<BM, BN, BK, WM, WN, AROW, VEC, STAGES, PEER>;
  using Coord = typename T_::Coord;
  constexpr int NT = T_::NT, FM = T_::FM, FN = T_::FN, SA = T_::SA, SB = T_::SB;
  constexpr int A_ST = T_::A_ST, B_ST = T_::B_ST;
  constexpr bool TMA = T_::TMA;
  extern __shared__ __align__(16) double smem_dyn[];
  double* smem = TMA ? reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023))
                     : smem_dyn;
  double* As = smem;
  double* Bs = smem + STAGES * A_ST;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm0 = (warp / T_::C_::WARPS_N) * WM, wn0 = (warp % T_::C_::WARPS_N) * WN;
  const int cta = blockIdx.x;

  // Pipeline synchronisation with mbarriers instead of a CTA barrier per k-tile:
  //   full[s]  — every thread's cp.async into stage s has landed (cp.async.mbarrier.arrive)
  //   empty[s] — every thread has finished reading stage s
  // so a warp may run ahead into the next k-tile as soon as its data is there.
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + STAGES * B_ST);
  uint64_t* empty = full + STAGES;
  if (tid == 0) {
    for (int st = 0; st < STAGES; ++st) {
      mbar_init(full + st, TMA ? 1 : NT);   // TMA: the issuing thread's expect-tx arrival
      mbar_init(empty + st, NT);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // Programmatic dependent launch: this CTA may have started while the previous kernel of the
  // stream was still draining (its SM freed early); wait for that grid's completion and memory
  // flush before the first global access, and let the next kernel's CTAs be scheduled as SMs
  // free up.  Both are no-ops for a launch without the attribute.
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");

  // ---- producer
  WorkIter pit;
  pit.init(sc, cta);
  Seg ps;
  bool p_ok = pit.next(ps);
  int pk = 0;
  int pkt = 0;   // k-tiles issued so far (stage = pkt % STAGES, fill = pkt / STAGES)
  typename T_::Loader ld;
  if (TMA) p_ok = false;   // TMA: the releasing warps issue (below), produce() is unused
  if (p_ok) {
    pk = ps.kb;
    ld.setup(p, T_::coords(p, sc, ps.tl), ps.kb);
  }
  auto produce = [&]() {
    if (!p_ok) return;
    const int stage = pkt % STAGES, fill = pkt / STAGES;
    if (fill > 0) mbar_wait(empty + stage, (fill - 1) & 1);
    if constexpr (TMA) {
      ld.issue_tma(p, tm, As + stage * A_ST, Bs + stage * B_ST, full + stage);
    } else {
      ld.issue(p, As + stage * A_ST, Bs + stage * B_ST);
      cp_async_mbar_arrive(full + stage);
    }
    ++pkt;
    if (++pk == ps.ke) {
      p_ok = pit.next(ps);
      if (p_ok) {
        pk = ps.kb;
        ld.setup(p, T_::coords(p, sc, ps.tl), ps.kb);
      }
    }
  };
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) produce();

  // TMA: the lookahead over the k-tile sequence lives in shared memory, and the warp that
  // releases a stage LAST issues that stage's refill (the k-tile STAGES ahead) at once — no
  // thread ever waits for a stage to drain (a per-stage release counter replaces the empty
  // mbarrier).  Refills are issued in k-tile order: the last release of k-tile i+1 happens after
  // the issuing warp of i released i+1 itself.
  struct ProdSt {
    WorkIter it;
    Seg seg;
    int pk, ok;
    typename T_::Loader ld;
  };
  unsigned* relc = reinterpret_cast<unsigned*>(empty + STAGES);
  ProdSt* sprod = reinterpret_cast<ProdSt*>(reinterpret_cast<uintptr_t>(relc + 8 + STAGES) & ~uintptr_t(15));
  auto tma_issue_next = [&](int stage) {   // one thread
    ProdSt S = *sprod;
    if (!S.ok) return;
    S.ld.issue_tma(p, tm, As + stage * A_ST, Bs + stage * B_ST, full + stage);
    if (++S.pk == S.seg.ke) {
      S.ok = S.it.next(S.seg);
      if (S.ok) {
        S.pk = S.seg.kb;
        S.ld.setup(p, T_::coords(p, sc, S.seg.tl), S.seg.kb);
      }
    }
    *sprod = S;
  };
  if constexpr (TMA) {
    static_assert(sizeof(ProdSt) + 8 * 4 + 64 <= 512, "TMA producer state fits");
    if (tid == 0) {
      for (int st = 0; st < STAGES; ++st) relc[st] = 0;
      ProdSt S;
      S.it.init(sc, cta);
      S.ok = S.it.next(S.seg);
      S.pk = S.seg.kb;
      if (S.ok) S.ld.setup(p, T_::coords(p, sc, S.seg.tl), S.seg.kb);
      *sprod = S;
      for (int st = 0; st < STAGES; ++st) tma_issue_next(st);   // fill every stage
    }
  }

  // ---- consumer
  WorkIter cit;
  cit.init(sc, cta);
  Seg cs;
  bool c_ok = cit.next(cs);
  if (!c_ok) {
    cp_async_wait<0>();
    return;
  }
  int ck = cs.kb;
  int ckt = 0;   // k-tiles consumed so far
  Coord cd = T_::coords(p, sc, cs.tl);
  double acc[FM][FN][2];
  T_::zero(acc);
  // the prefetch of k-tile t+STAGES-1 is issued behind the DMMAs of this tile's last k-step:
  // its empty-wait then targets a stage every warp left a whole k-tile ago (measured best of
  // k-step 0 / 4 / 12 / 28: +0.7% at C2)
  // with 2 stages the refill of the other stage must start at the first k-step (one k-tile
  // of latency hiding); with 3 it is issued behind the last k-step
  constexpr int PRODUCE_KK = STAGES == 2 ? 0 : BK - 4;
  // ragged K (kseg not a multiple of BK, e.g. the paper's n = 100, 150, 200): the last k-tile
  // of every segment runs only its valid k-steps (the zero-filled rows would add exact zeros)
  const int kps = (p.kseg + BK - 1) / BK;
  const int ktail = p.kseg - (kps - 1) * BK;   // valid k of a segment's last k-tile
  int cks = ck % kps;                          // k-tile position inside its segment
  // TMA (fragment-ordered) layout: this thread's byte offset inside the 256-B block of a fragment
  int tma_a = 0, tma_b = 0;
  if constexpr (TMA) {
    if constexpr (AROW) tma_a = (wm0 >> 3) * (BK / 4) * 256 + g * 32 + t4 * 8;
    else tma_a = ((wm0 >> 2) * 16 + (g >> 2) * 16 + t4 * 4 + (g & 3)) * 8;
    tma_b = ((wn0 >> 2) * 16 + (g >> 2) * 16 + t4 * 4 + (g & 3)) * 8;
  }
  auto kstep = [&](const double* as, const double* bs, int kk) {
    double af[FM], bf[FN];
    if constexpr (TMA) {
      // one contiguous 256-B block per fragment; block index from (k/4, chunk) as immediates
      const char* a8 = reinterpret_cast<const char*>(as);
      const char* b8 = reinterpret_cast<const char*>(bs);
#pragma unroll
      for (int i = 0; i < FM; ++i) {
        if constexpr (AROW) af[i] = *reinterpret_cast<const double*>(a8 + (i * (BK / 4) + (kk >> 2)) * 256 + tma_a);
        else af[i] = *reinterpret_cast<const double*>(a8 + (kk >> 2) * (BM * 32) + i * 256 + tma_a);
      }
#pragma unroll
      for (int j = 0; j < FN; ++j)
        bf[j] = *reinterpret_cast<const double*>(b8 + (kk >> 2) * (BN * 32) + j * 256 + tma_b);
    } else {
#pragma unroll
      for (int i = 0; i < FM; ++i) {
        if constexpr (AROW) af[i] = as[(wm0 + i * 8 + g) * SA + kk + t4];
        else af[i] = as[(kk + t4) * SA + wm0 + i * 8 + g];
      }
#pragma unroll
      for (int j = 0; j < FN; ++j) bf[j] = bs[(kk + t4) * SB + wn0 + j * 8 + g];
    }
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  };
  while (true) {
    const int stage_c = ckt % STAGES;
    mbar_wait(full + stage_c, (ckt / STAGES) & 1);
    const double* as = As + stage_c * A_ST;
    const double* bs = Bs + stage_c * B_ST;
    if (ktail == BK || cks != kps - 1) {
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        kstep(as, bs, kk);
        if (kk == PRODUCE_KK) produce();
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        if (kk < ktail) kstep(as, bs, kk);
        if (kk == PRODUCE_KK) produce();
      }
    }
    if constexpr (TMA) {
      __syncwarp();   // every lane's fragment loads of this stage have been consumed
      if (lane == 0) {
        __threadfence_block();
        if (atomicAdd(relc + stage_c, 1u) == (unsigned)(NT / 32 - 1)) {   // the last warp out
          relc[stage_c] = 0;
          __threadfence_block();
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          tma_issue_next(stage_c);
        }
      }
    } else {
      mbar_arrive(empty + stage_c);
    }
    ++ckt;
    if (++cks == kps) cks = 0;
    if (++ck < cs.ke) continue;

    // ---- segment finished
    if (sc.csplit > 1) {
      // cluster split-K: publish the partial in this CTA's (now idle) pipeline shared memory,
      // then every CTA sums its share of the fragments over the cluster's partials in
      // cluster-rank (= k) order, read through DSMEM, and stores that share
      namespace cg = cooperative_groups;
      cg::cluster_group cl = cg::this_cluster();
      cp_async_wait<0>();
      __syncthreads();
      double* part = smem;
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int c = 0; c < FN; ++c)
#pragma unroll
          for (int e = 0; e < 2; ++e) part[((a * FN + c) * 2 + e) * NT + tid] = acc[a][c][e];
      cl.sync();
      const int q = (int)cl.block_rank(), S = sc.csplit;
      unsigned mask = 0;
#pragma unroll
      for (int f = 0; f < FM * FN; ++f)
        if (f % S == q) mask |= 1u << f;
      T_::zero(acc);
      for (int j = 0; j < S; ++j) {
        const double* pj = cl.map_shared_rank(part, j);
#pragma unroll
        for (int a = 0; a < FM; ++a)
#pragma unroll
          for (int c = 0; c < FN; ++c)
            if ((mask >> (a * FN + c)) & 1u) {
#pragma unroll
              for (int e = 0; e < 2; ++e) acc[a][c][e] += pj[((a * FN + c) * 2 + e) * NT + tid];
            }
      }
      T_::epilogue(p, cd, acc, mask);
      cl.sync();   // no CTA leaves while its partial may still be read
      break;       // exactly one segment per CTA in this mode
    } else if (cs.kb == 0 && cs.ke == sc.ktiles) {
      T_::epilogue(p, cd, acc, ~0u);
    } else {
      // split tile (stream-K): every contributor publishes its partial and counts itself in.
      // The contributors whose work list ENDS in this tile (all but a tail CTA that continues
      // into the next tile) then wait for the rest and each sums a 1/nr share of the
      // fragments over all partials in increasing-k order (contributor order: the result does
      // not depend on who sums) and stores it.  Only a CTA's last segment ever waits, so no
      // CTA's own work queues behind a wait.
      const long long tr = cs.tl - sc.dp_tiles;
      const long long t0u = tr * sc.ktiles, t1u = t0u + sc.ktiles;
      int i0 = cta, i1 = cta;
      while (i0 > 0 && sk_begin(sc, i0) > t0u) --i0;
      while (i1 + 1 < sc.G_sk && sk_begin(sc, i1 + 1) < t1u) ++i1;
      const int nc = i1 - i0 + 1;
      const int nr = sk_begin(sc, i1 + 1) <= t1u ? nc : nc - 1;   // reducers: i0 .. i0+nr-1
      int* arrive = p.sk_flags + 2 * tr;
      const int q = cta - i0;
      const bool solo = nr == 1 && q == 0;   // the only reducer keeps its own partial in registers
      if (!solo) {
        double* ws_me = p.sk_ws + (size_t)sk_slot(sc, cta, t0u) * (FM * FN * 2 * NT);
#pragma unroll
        for (int a = 0; a < FM; ++a)
#pragma unroll
          for (int c = 0; c < FN; ++c)
#pragma unroll
            for (int e = 0; e < 2; ++e) __stcg(ws_me + ((a * FN + c) * 2 + e) * NT + tid, acc[a][c][e]);
        __threadfence();
        __syncthreads();
      }
      if (solo) {
        if (tid == 0) {
          while (*reinterpret_cast<volatile int*>(arrive) < nc - 1) __nanosleep(32);
          __threadfence();
        }
        __syncthreads();
        for (int j = i0 + 1; j <= i1; ++j) {
          const double* wj = p.sk_ws + (size_t)sk_slot(sc, j, t0u) * (FM * FN * 2 * NT);
#pragma unroll
          for (int a = 0; a < FM; ++a)
#pragma unroll
            for (int c = 0; c < FN; ++c)
#pragma unroll
              for (int e = 0; e < 2; ++e) acc[a][c][e] += __ldcg(wj + ((a * FN + c) * 2 + e) * NT + tid);
        }
        T_::epilogue(p, cd, acc, ~0u);
        if (tid == 0) arrive[0] = 0;
      } else if (q < nr) {
        if (tid == 0) {
          atomicAdd(arrive, 1);
          while (*reinterpret_cast<volatile int*>(arrive) < nc) __nanosleep(32);
          __threadfence();
        }
        __syncthreads();
        unsigned mask = 0;
#pragma unroll
        for (int f = 0; f < FM * FN; ++f)
          if (f % nr == q) mask |= 1u << f;
        T_::zero(acc);
        for (int j = i0; j <= i1; ++j) {
          const double* wj = p.sk_ws + (size_t)sk_slot(sc, j, t0u) * (FM * FN * 2 * NT);
#pragma unroll
          for (int a = 0; a < FM; ++a)
#pragma unroll
            for (int c = 0; c < FN; ++c)
              if ((mask >> (a * FN + c)) & 1u) {
#pragma unroll
                for (int e = 0; e < 2; ++e) acc[a][c][e] += __ldcg(wj + ((a * FN + c) * 2 + e) * NT + tid);
              }
        }
        T_::epilogue(p, cd, acc, mask);
        __syncthreads();
        if (tid == 0 && atomicAdd(arrive + 1, 1) == nr - 1) {   // last reducer out resets
          arrive[0] = 0;
          arrive[1] = 0;
          __threadfence();
        }
      } else if (tid == 0) {
        atomicAdd(arrive, 1);   // a tail contributor that continues into the next tile
      }
    }
    if (!cit.next(cs)) break;
    ck = cs.kb;
    cks = ck % kps;
    cd = T_::coords(p, sc, cs.tl);
    T_::zero(acc);
  }
  cp_async_wait<0>();
  if constexpr (PEER) __threadfence_system();   // peer stores performed before the kernel completes
}

struct TileChoice {
  int bm, bn, bk, occ;
  double eff;
};
// Resident CTAs per SM (register/smem-limited) and relative per-SM efficiency of each config.
constexpr TileChoice kTiles[3] = {{128, 128, 32, 1, 1.00}, {128, 64, 16, 2, 0.85}, {64, 64, 16, 3, 0.80}};

// Per-device state: the dynamic-smem opt-in is a per-device function attribute, and occupancy /
// cluster residency are queried per device (contexts on several devices in one process).
constexpr int kMaxDev = 32;
int cur_dev() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) dev = 0;
  return dev;
}

template <int BM, int BN, int BK, int WM, int WN, bool AROW, int VEC, int STAGES, bool PEER = false>
struct Prepared {
  static inline bool done[kMaxDev] = {};
  static inline int occ[kMaxDev] = {};   // resident CTAs per SM (occupancy API)
};

template <int BM, int BN, int BK, int WM, int WN, bool AROW, int VEC, int STAGES, bool PEER = false>
cudaError_t prepare_cfg() {
  using C_ = Cfg<BM, BN, BK, WM, WN, AROW, VEC, STAGES>;
  using P_ = Prepared<BM, BN, BK, WM, WN, AROW, VEC, STAGES, PEER>;
  const int dev = cur_dev();
  if (!P_::done[dev]) {
    auto kern = gemm_kernel<BM, BN, BK, WM, WN, AROW, VEC, STAGES, PEER>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C_::NT, C_::SMEM);
    if (e != cudaSuccess) return e;
    P_::occ[dev] = occ < 1 ? 1 : occ;
    P_::done[dev] = true;
  }
  return cudaSuccess;
}

template <int BM, int BN, int BK, int WM, int WN, bool AROW, int VEC, int STAGES, bool PEER = false>
int occ_of() {
  return Prepared<BM, BN, BK, WM, WN, AROW, VEC, STAGES, PEER>::occ[cur_dev()];
}

int num_sms();
template <int BM, int WM>
constexpr int FM_OF() { return WM / 8; }
template <int BN, int WN>
constexpr int FN_OF() { return WN / 8; }

// clusters of S CTAs of this configuration that can be resident at once (GPC packing), cached
template <int BM, int BN, int BK, int WM, int WN, bool AROW, int VEC, int STAGES, bool PEER>
int max_clusters(int S) {
  static int cache_all[kMaxDev][9];
  static bool init[kMaxDev] = {};
  if (S < 1 || S > 8) return 0;
  const int dev = cur_dev();
  int* cache = cache_all[dev];
  if (!init[dev]) {
    for (int i = 0; i < 9; ++i) cache[i] = -1;
    init[dev] = true;
  }
  if (cache[S] < 0) {
    using C_ = Cfg<BM, BN, BK, WM, WN, AROW, VEC, STAGES>;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(S * 64);
    cfg.blockDim = dim3(C_::NT);
    cfg.dynamicSmemBytes = C_::SMEM;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, gemm_kernel<BM, BN, BK, WM, WN, AROW, VEC, STAGES, PEER>, &cfg) !=
        cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    cache[S] = n;
  }
  return cache[S];
}

// Schedule of one launch for one tile configuration (data-parallel waves, a stream-K tail or a
// whole-launch split, or a cluster split-K) and its estimated time in microseconds: per SM,
// the k-tiles it computes times the SM-alone k-tile time (4.2 us for 128x128x32 at full DMMA
// rate, scaled by tile volume and the configuration's measured efficiency), plus ~3 us for a
// global stream-K fix-up or ~0.5 us for a DSMEM one.
template <int BM, int BN, int BK, int WM, int WN, bool AROW, int VEC, int STAGES, bool PEER>
double plan_cfg(const GemmArgs& g, int nz, double eff, Sched& sc) {
  using C_ = Cfg<BM, BN, BK, WM, WN, AROW, VEC, STAGES>;
  prepare_cfg<BM, BN, BK, WM, WN, AROW, VEC, STAGES, PEER>();
  sc = Sched{};
  sc.tiles_m = (g.M + BM - 1) / BM;
  sc.tiles_n = (g.N + BN - 1) / BN;
  sc.m_fastest = AROW ? 0 : 1;
  sc.ktiles = ((g.kseg + BK - 1) / BK) * g.nseg;
  const int nsm = num_sms();
  const long long T = (long long)sc.tiles_m * sc.tiles_n * nz;
  const long long Gmax = (long long)nsm * occ_of<BM, BN, BK, WM, WN, AROW, VEC, STAGES, PEER>();
  const double kt_us = 4.2 * (BM * BN * BK) / (128.0 * 128 * 32) / eff;
  static const double* fix = [] {   // KX_GEMM_FIX="sk_us,cluster_us": tuning experiments only
    static double f[2] = {6.0, 0.5};   // tuned on the size sweep, the Tucker sweep and C2/C3
    if (const char* e = getenv("KX_GEMM_FIX")) sscanf(e, "%lf,%lf", &f[0], &f[1]);
    return f;
  }();
  const long long kt = sc.ktiles;
  auto per_sm = [&](long long ctas, long long units_per_cta) {   // SM-alone k-tile units
    return (double)((ctas + nsm - 1) / nsm) * (double)units_per_cta;
  };
  sc.G = (int)std::min<long long>(T, Gmax);
  sc.dp_tiles = T;
  double best = per_sm(T, kt) * kt_us;   // data-parallel
  // cluster split-K (few tiles): every tile over the S CTAs of a cluster, DSMEM reduction
  static const int cs_env = [] {   // KX_GEMM_CSPLIT=0: tuning experiments only
    const char* e = getenv("KX_GEMM_CSPLIT");
    return e ? atoi(e) : 1;
  }();
  const int partial = FM_OF<BM, WM>() * FN_OF<BN, WN>() * 2 * C_::NT;   // doubles per partial
  for (int S = 8; cs_env && S >= 2 && T * 2 <= Gmax; S /= 2) {
    if (T * S <= Gmax && kt >= S && (long long)g.kseg * g.nseg >= 128 && partial * 8 <= STAGES * (C_::A_ST + C_::B_ST) * 8 &&
        max_clusters<BM, BN, BK, WM, WN, AROW, VEC, STAGES, PEER>(S) >= T) {
      const double t = per_sm(T * S, (kt + S - 1) / S) * kt_us + fix[1];
      if (t < best) {
        best = t;
        sc.csplit = S;
        sc.G = (int)(T * S);
        sc.dp_tiles = 0;
        sc.sk_units = T * kt;
        sc.G_sk = (int)(T * S);
      }
    }
  }
  // stream-K (needs two workspace slots per CTA and a counter pair per split tile)
  const bool sk_ok = g.sk_ws && g.sk_flags && 2 * Gmax * BM * BN <= (long long)kSkSlots * 128 * 128 &&
                     kt >= 2 && T % Gmax != 0;
  if (sk_ok) {
    long long dp = (T / Gmax) * Gmax;
    if (dp >= Gmax && (T - dp) * 2 < Gmax) dp -= Gmax;   // short tail: spread one more wave
    // >= 4 k-tiles per CTA behind a data-parallel part, >= 2 when the whole launch is split
    const long long units = (T - dp) * kt;
    const int G_sk = (int)std::min<long long>(Gmax, units / (dp > 0 ? 4 : 2));
    const bool worth = dp > 0 || (long long)g.kseg * g.nseg >= 128;   // tiny K: latency-bound
    if (worth && G_sk >= 1 && 2 * (T - dp) <= kSkFlags) {
      const double t = (per_sm(dp, kt) + per_sm(G_sk, (units + G_sk - 1) / G_sk)) * kt_us + fix[0];
      if (t < 0.97 * best) {
        best = t;
        sc.csplit = 0;
        sc.G = dp > 0 ? (int)Gmax : G_sk;
        sc.dp_tiles = dp;
        sc.sk_units = units;
        sc.G_sk = G_sk;
      }
    }
  }
  return best;
}

// Programmatic dependent launch of the GEMMs: opt-in (KX_PDL=1).  Measured slower in the step
// graphs (C2 2.644 vs 2.623, C3 1.720 vs 1.712 ms/step): the next GEMM's early CTAs gain no
// prologue work worth the SMs they hold while the previous grid's stream-K reducers finish.
bool pdl_on() {
  static const bool on = [] {
    const char* e = getenv("KX_PDL");
    return e && e[0] == '1';
  }();
  return on;
}

const TmaMaps& no_maps() {
  static const TmaMaps m = {};
  return m;
}

template <int BM, int BN, int BK, int WM, int WN, bool AROW, int VEC, int STAGES, bool PEER = false>
cudaError_t launch_cfg(const GemmArgs& g, int nz, double eff, cudaStream_t stream, const TmaMaps& tm = no_maps()) {
  using C_ = Cfg<BM, BN, BK, WM, WN, AROW, VEC, STAGES>;
  cudaError_t e = prepare_cfg<BM, BN, BK, WM, WN, AROW, VEC, STAGES, PEER>();
  if (e != cudaSuccess) return e;
  Sched sc;
  plan_cfg<BM, BN, BK, WM, WN, AROW, VEC, STAGES, PEER>(g, nz, eff, sc);
  const long long T = (long long)sc.tiles_m * sc.tiles_n * nz;
  const long long Gmax = (long long)num_sms() * occ_of<BM, BN, BK, WM, WN, AROW, VEC, STAGES, PEER>();
  static const bool trace = getenv("KX_TRACE") != nullptr;   // diagnostics only
  if (trace)
    fprintf(stderr, "kx-gemm %s M=%d N=%d K=%dx%d nz=%d cfg=%dx%dx%d tiles=%lld kt=%d G=%d dp=%lld sk_units=%lld G_sk=%d csplit=%d (max clusters of 8/4/2: %d/%d/%d) flops=%.4g\n",
            AROW ? (VEC == 3 ? "row/tma" : "row") : (VEC == 3 ? "col/tma" : "col"), g.M, g.N, g.kseg, g.nseg, nz, BM, BN, BK, T, sc.ktiles, sc.G,
            sc.dp_tiles, sc.sk_units, sc.G_sk, sc.csplit, max_clusters<BM, BN, BK, WM, WN, AROW, VEC, STAGES, PEER>(8),
            max_clusters<BM, BN, BK, WM, WN, AROW, VEC, STAGES, PEER>(4), max_clusters<BM, BN, BK, WM, WN, AROW, VEC, STAGES, PEER>(2),
            2.0 * g.M * g.N * (double)g.kseg * g.nseg * nz);
  if (sc.csplit > 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sc.G);
    cfg.blockDim = dim3(C_::NT);
    cfg.dynamicSmemBytes = C_::SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = sc.csplit;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_on() ? 2 : 1;
    const cudaError_t ce = cudaLaunchKernelEx(&cfg, gemm_kernel<BM, BN, BK, WM, WN, AROW, VEC, STAGES, PEER>, g, sc, tm);
    if (ce == cudaSuccess) return ce;
    // the cluster launch was refused (e.g. SMs taken by concurrent work): plain data-parallel
    cudaGetLastError();
    sc.csplit = 0;
    sc.G = (int)std::min<long long>(T, Gmax);
    sc.dp_tiles = T;
    sc.sk_units = 0;
    sc.G_sk = 0;
  }
  if (sc.sk_units > 0) {
    // stream-K CTAs wait on each other: a cooperative launch guarantees that the whole grid is
    // co-resident even when other kernels share the GPU (otherwise the driver refuses it)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sc.G);
    cfg.blockDim = dim3(C_::NT);
    cfg.dynamicSmemBytes = C_::SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_on() ? 2 : 1;
    const cudaError_t ce = cudaLaunchKernelEx(&cfg, gemm_kernel<BM, BN, BK, WM, WN, AROW, VEC, STAGES, PEER>, g, sc, tm);
    if (ce != cudaErrorCooperativeLaunchTooLarge) return ce;
    // not all CTAs can be co-resident right now: the data-parallel schedule needs no waits
    cudaGetLastError();
    sc.G = (int)std::min<long long>(T, Gmax);
    sc.dp_tiles = T;
    sc.sk_units = 0;
    sc.G_sk = 0;
  }
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sc.G);
    cfg.blockDim = dim3(C_::NT);
    cfg.dynamicSmemBytes = C_::SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_on() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, gemm_kernel<BM, BN, BK, WM, WN, AROW, VEC, STAGES, PEER>, g, sc, tm);
  }
}

// ---------------------------------------------------------------- TMA tensor maps (VEC == 3)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn tma_encoder() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      f = nullptr;
    }
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// 5-D fp64 view (element extents / strides, stride[0] = 1) with the given box, no swizzle;
// extent-1 dims get a packed stride; false if TMA cannot express the view.
bool make_map64(CUtensorMap* map, const double* base, const long long* ext, const long long* str,
                const int* boxd) {
  EncodeTiledFn enc = tma_encoder();
  if (!enc || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < 5; ++i) box[i] = (cuuint32_t)boxd[i];
  long long prev = 1;
  for (int i = 0; i < 5; ++i) {
    if (ext[i] < 1 || ext[i] > (1LL << 32)) return false;
    dims[i] = (cuuint64_t)ext[i];
  }
  for (int i = 1; i < 5; ++i) {
    long long st = str[i];
    if (ext[i] == 1) st = prev * ext[i - 1];
    if (st <= 0 || (st * 8) % 16 || st * 8 >= (1LL << 40)) return false;
    strides[i - 1] = (cuuint64_t)(st * 8);
    prev = st;
  }
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Maps of the 128 x 128 x 32 configuration: A per (species, K segment), B per species.  Needs
// k chunks of 8 doubles that never straddle a segment (kseg % 8), 8-wide n / m chunks, no
// flattened batches and no zero batch strides.
bool build_tma(const GemmArgs& g, TmaMaps& tm) {
  // Where the TMA-fed variant runs (KX_GEMM_TMA=0: never, =1: wherever eligible; default: the
  // long-K launches, >= 32 k-tiles per tile).  Measured per launch (ncu, one step, conflict-free
  // fragment-ordered boxes): C2 DMMA active 92.4 -> 93.4% (first mode, K = 1024), 88.7 -> 89.2%
  // (D2 / D3 first modes), 91.7 -> 93.5% (stage GEMMs, K = 2048 / 4096); C2 2.618 -> 2.579
  // ms/step.  Below 32 k-tiles per tile it does not pay in the live step graphs: the C3 short-K
  // COL launches (4 k-tiles) lose up to 5% and, with the ROW stage GEMMs (12 / 24 k-tiles) on
  // TMA too, a C3 step is 1.715 vs 1.710 ms.
  static const int mode = [] {
    const char* e = getenv("KX_GEMM_TMA");
    return e ? atoi(e) : -1;
  }();
  if (mode == 0) return false;
  const int ktiles_tile = (g.kseg + 31) / 32 * g.nseg;
  if (mode < 0 && ktiles_tile < 32) return false;
  if (g.nflat || g.peer.P || g.kseg % 8 || g.N % 8 || (!g.arow && g.M % 8)) return false;
  if (g.ns * (g.arow ? g.nseg : 1) > kTmaMaxA || (!g.arow && g.nseg != 1)) return false;
  // the fragment-ordered boxes use 4 of the 5 dims; the fifth carries the t batch (nb == 1)
  if (g.nb > 1 || (g.nt > 1 && (g.sA_t == 0 || g.sB_t == 0)) || g.M % 8) return false;
  tm.nsegmaps = g.arow ? g.nseg : 1;
  for (int s = 0; s < g.ns; ++s) {
    for (int j = 0; j < tm.nsegmaps; ++j) {
      // ROW A (m rows, k contiguous): (4 k, 8 m, k/4, m/8, t);  COL A (k rows, m contiguous): (4 m, 4 k, m/4, k/4, t)
      const long long ext_r[5] = {4, 8, g.kseg / 4, g.M / 8, g.nt};
      const long long str_r[5] = {1, g.lda, 4, 8 * g.lda, g.sA_t};
      const int box_r[5] = {4, 8, 32 / 4, 128 / 8, 1};
      const long long ext_c[5] = {4, 4, g.M / 4, g.kseg / 4, g.nt};
      const long long str_c[5] = {1, g.lda, 4, 4 * g.lda, g.sA_t};
      const int box_c[5] = {4, 4, 128 / 4, 32 / 4, 1};
      const double* base = g.A[s] + (g.arow ? g.seg_off[j] : 0);
      if (!make_map64(&tm.A[s * tm.nsegmaps + j], base, g.arow ? ext_r : ext_c, g.arow ? str_r : str_c,
                      g.arow ? box_r : box_c))
        return false;
    }
    // B (k rows, n contiguous): (4 n, 4 k, n/4, k/4, t)
    const long long ext_b[5] = {4, 4, g.N / 4, (long long)g.nseg * g.kseg / 4, g.nt};
    const long long str_b[5] = {1, g.ldb, 4, 4 * g.ldb, g.sB_t};
    const int box_b[5] = {4, 4, 128 / 4, 32 / 4, 1};
    if (!make_map64(&tm.B[s], g.B[s], ext_b, str_b, box_b)) return false;
  }
  return true;
}

// Pick the tile configuration with the smallest planned time (unless forced) and launch it.
// The 128 x 128 x 32 configuration runs its TMA-fed variant (VEC = 3) whenever the launch allows.
template <bool AROW, int VEC, bool PEER>
cudaError_t launch_layout_p(const GemmArgs& g, int nz, int forced, const double* eff, cudaStream_t stream) {
  Sched sc;
  TmaMaps tm;
  bool tma = false;
  if constexpr (VEC == 2 && !PEER) tma = build_tma(g, tm);
  double t0;
  if constexpr (VEC == 2 && !PEER)
    t0 = tma ? plan_cfg<128, 128, 32, 32, 32, AROW, 3, 3, PEER>(g, nz, eff[0], sc)
             : plan_cfg<128, 128, 32, 32, 32, AROW, VEC, 3, PEER>(g, nz, eff[0], sc);
  else
    t0 = plan_cfg<128, 128, 32, 32, 32, AROW, VEC, 3, PEER>(g, nz, eff[0], sc);
  const double t1 = plan_cfg<128, 64, 16, 32, 32, AROW, VEC, 3, PEER>(g, nz, eff[1], sc);
  const double t2 = plan_cfg<64, 64, 16, 32, 32, AROW, VEC, 3, PEER>(g, nz, eff[2], sc);
  int which = 0;
  if (t1 < t0 * 0.999 && t1 <= t2) which = 1;
  else if (t2 < t0 * 0.999 && t2 < t1) which = 2;
  if (forced >= 0 && forced < 3) which = forced;
  switch (which) {
    case 0:
      if constexpr (VEC == 2 && !PEER)
        if (tma) return launch_cfg<128, 128, 32, 32, 32, AROW, 3, 3, PEER>(g, nz, eff[0], stream, tm);
      return launch_cfg<128, 128, 32, 32, 32, AROW, VEC, 3, PEER>(g, nz, eff[0], stream);
    case 1: return launch_cfg<128, 64, 16, 32, 32, AROW, VEC, 3, PEER>(g, nz, eff[1], stream);
    default: return launch_cfg<64, 64, 16, 32, 32, AROW, VEC, 3, PEER>(g, nz, eff[2], stream);
  }
}

template <bool AROW, int VEC>
cudaError_t launch_layout(const GemmArgs& g, int nz, int forced, const double* eff, cudaStream_t stream) {
  // direct peer stores (sharded steps): separate instantiations so the redirect arithmetic
  // costs the plain kernels no registers
  if (g.peer.P) return launch_layout_p<AROW, VEC, true>(g, nz, forced, eff, stream);
  return launch_layout_p<AROW, VEC, false>(g, nz, forced, eff, stream);
}

template <bool AROW, int VEC>
void prepare_layout() {
  prepare_cfg<128, 128, 32, 32, 32, AROW, VEC, 3>();
  if constexpr (VEC == 2) {
    prepare_cfg<128, 128, 32, 32, 32, AROW, 3, 3>();
    for (int S = 2; S <= 8; S *= 2) max_clusters<128, 128, 32, 32, 32, AROW, 3, 3, false>(S);
  }
  prepare_cfg<128, 128, 32, 32, 32, AROW, VEC, 3, true>();
  prepare_cfg<128, 64, 16, 32, 32, AROW, VEC, 3, true>();
  prepare_cfg<64, 64, 16, 32, 32, AROW, VEC, 3, true>();
  prepare_cfg<128, 64, 16, 32, 32, AROW, VEC, 3>();
  prepare_cfg<64, 64, 16, 32, 32, AROW, VEC, 3>();
  // cluster residency queries outside any graph capture, after the smem attributes are set
  for (int S = 2; S <= 8; S *= 2) {
    max_clusters<128, 128, 32, 32, 32, AROW, VEC, 3, false>(S);
    max_clusters<128, 64, 16, 32, 32, AROW, VEC, 3, false>(S);
    max_clusters<64, 64, 16, 32, 32, AROW, VEC, 3, false>(S);
  }
}

int num_sms() {
  static int nsm_of[kMaxDev] = {};   // per device; declared above for launch_cfg
  const int dev = cur_dev();
  if (nsm_of[dev] == 0) {
    int nsm = 0;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || nsm <= 0) nsm = 148;
    nsm_of[dev] = nsm;
  }
  return nsm_of[dev];
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

cudaError_t launch_gemm(const GemmArgs& g_in, cudaStream_t stream) {
  GemmArgs g = g_in;
  static const int noload = getenv("KX_GEMM_NOLOAD") ? 1 : 0;   // diagnostics only
  g.diag_noload = noload;
  // batched COL-layout launches (middle modes) with ragged N: one launch over nb * N columns
  // instead of nb launches' worth of padded tiles (the paper's n = 100, 150, 200)
  g.nflat = 0;
  if (!g.arow && g.nb > 1 && g.N % 64 != 0 && g.N % 2 == 0 && !g.peer.P &&
      (long long)g.N * g.nb < (1LL << 30) && g.sB_b * (long long)g.nb < (1LL << 31)) {
    g.nflat = g.N;
    g.N *= g.nb;
    g.nb = 1;
  }
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
  // Tile choice: the configuration whose planned schedule (plan_cfg) is fastest.
  static const TileChoice* tiles = [] {   // KX_GEMM_EFF="e0,e1,e2": tuning experiments only
    static TileChoice t[3] = {kTiles[0], kTiles[1], kTiles[2]};
    if (const char* e = getenv("KX_GEMM_EFF")) sscanf(e, "%lf,%lf,%lf", &t[0].eff, &t[1].eff, &t[2].eff);
    return t;
  }();
  const double eff[3] = {tiles[0].eff, tiles[1].eff, tiles[2].eff};
  static int forced = [] {
    const char* e = getenv("KX_GEMM_CFG");   // tuning experiments only: 0, 1, 2
    return e ? atoi(e) : -1;
  }();
  if (g.arow) return vec ? launch_layout<true, 2>(g, nz, forced, eff, stream) : launch_layout<true, 1>(g, nz, forced, eff, stream);
  return vec ? launch_layout<false, 2>(g, nz, forced, eff, stream) : launch_layout<false, 1>(g, nz, forced, eff, stream);
}

}  // namespace kx
