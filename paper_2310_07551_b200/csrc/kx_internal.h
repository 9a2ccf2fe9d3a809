// Internal declarations shared by the library's translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace kx {

constexpr int MAXS = 4;        // components (species) batched in one launch
constexpr int MAXSEG = 64;     // K segments of a concatenated-K last-mode product (terms x ranks)

// One launch of the mode-product GEMM (kernel K*1):
//   for z in [0, nz):  s = z / (nt*nb), t = (z / nb) % nt, b = z % nb
//   C_z(m, n) = alpha * sum_k A_z(m, k) B_z(k, n) + beta * D_z(m, n) + gamma * E_z(m, n)
//              + diag * [m == n]
// A layout ROW ("k contiguous"): A_z(m, k) = A[seg_off[k / kseg] + m*lda + k % kseg]
//          (K = nseg * kseg; concatenated-K over term tensors; reading 2 of §8(a) a3)
// A layout COL ("m contiguous"): A_z(m, k) = A[k*lda + m]
// B_z(k, n) = B[k*ldb + n];  C/D/E row-major with ldc/ldd/lde.
// X_z = X_s[s] + t*sX_t + b*sX_b for X in {A, B, C, D, E}.
// Direct peer stores (the all-to-all of the slab decomposition fused into the producing
// kernel): a kernel whose output is a peer-packed send buffer (P blocks of
// `chunk` doubles per `span`-long slot) instead stores block q straight into peer q's receive
// buffer at block `rank` — the receive layout the all-to-all would have produced.  peer_base
// are device pointers valid in this process (same-device buffers of an in-process group, or
// CUDA IPC mappings of the peers' buffers).
constexpr int kMaxPeers = 8;
struct PeerMap {
  int P = 0;                       // 0: plain local stores
  int rank = 0;
  long long chunk = 0, span = 0;
  const double* local_base[MAXS] = {};
  double* peer_base[MAXS][kMaxPeers] = {};
};
// 32-bit arithmetic: the host enables peer stores only when a buffer holds < 2^31 doubles
__device__ __forceinline__ double* peer_redirect(const PeerMap& pm, int s, double* ptr) {
  if (pm.P == 0) return ptr;
  const unsigned off = (unsigned)(ptr - pm.local_base[s]);
  const unsigned span = (unsigned)pm.span, chunk = (unsigned)pm.chunk;
  const unsigned slot = off / span, within = off - slot * span;
  const unsigned q = within / chunk;
  return pm.peer_base[s][q] + (size_t)slot * span + (size_t)pm.rank * chunk + (within - q * chunk);
}

struct GemmArgs {
  int M = 0, N = 0, kseg = 0, nseg = 1;
  bool arow = true;
  const double* A[MAXS] = {};
  const double* B[MAXS] = {};
  double* C[MAXS] = {};
  const double* D[MAXS] = {};
  const double* E[MAXS] = {};
  long long lda = 0, ldb = 0, ldc = 0, ldd = 0, lde = 0;
  long long seg_off[MAXSEG] = {};
  long long sA_t = 0, sA_b = 0, sB_t = 0, sB_b = 0, sC_t = 0, sC_b = 0, sD_t = 0, sD_b = 0,
            sE_t = 0, sE_b = 0;
  int ns = 1, nt = 1, nb = 1;
  double alpha = 1.0, beta = 0.0, gamma = 0.0, diag = 0.0;
  // stream-K scratch (library-owned, per context): kSkSlots x 128 x 128 doubles + flags
  double* sk_ws = nullptr;
  int* sk_flags = nullptr;
  PeerMap peer;                    // epilogue stores redirected to peers (P > 0)
  // set by launch_gemm (not by callers): batched COL-layout launches whose N is not a multiple
  // of the tile width are run as one launch over N' = nb N columns; column n' is batch
  // n' / nflat, column n' % nflat (the B/C/D/E batch strides apply per column)
  int nflat = 0;
  int diag_noload = 0;   // diagnostics only (KX_GEMM_NOLOAD=1): skip the operand copies (wrong results)
};
constexpr int kSkSlots = 304;    // partial-tile slots of 128x128 doubles (>= 2 x SM count)
constexpr int kSkFlags = 2048;   // counters: a pair per split tile

// Launch on `stream`; returns cudaSuccess or the launch error.  Chooses tile config.
cudaError_t launch_gemm(const GemmArgs& g, cudaStream_t stream);
// Algorithmic flops of a launch: 2 * M * N * K * nz.
double gemm_flops(const GemmArgs& g);

// fp32 mode-product GEMM on tcgen05 (kind::tf32, three-pass hi/lo split; tf32gemm.cu).
// kind::tf32 reads K-major operands only, so the two operands take different routes:
//   S, the "static" operand (phi-matrix / L): two tf32-valued planes hi, lo, K-major, prepared
//      by the caller (launch_split_f64 / launch_split_f32_2d with transpose);
//   T, the "tensor" operand: plain fp32 (T.hi; T.lo unused), split by the kernel's converter
//      warps (and transposed for TF32_COL).
// Operands are 5-D views (element extents / strides, stride[0] = 1) read through TMA maps:
//   TF32_COL (mu >= 2, and the concatenated-M first mode):  C = S T
//       S (K-major phi-matrix stack): dims (k, m, t, s, 1);   T (MN-major tensor): (n, k, b, t, s)
//   TF32_ROW (mu = 1, concatenated K over nseg segments of kseg; segment j = (j % slo, j / slo),
//       so two arithmetic progressions of workspace slots form one concatenated K):  C = T S^T
//       T (K-major tensor rows): dims (k, m, j % slo, j / slo, s);  S (K-major stack): (k, n, j, s, 1)
//   z = (s * nt + t) * nb + b;  C_z(m, n) = alpha sum_k A B + beta D_z(m, n), with
//   C_z = C[s] + t sC_t + b sC_b + m ldc + n (same for D), fp32.
// Requirements: every row stride a multiple of 4 floats, 16-B aligned bases (KX_ERR_UNSUPPORTED
// otherwise, checked by the caller).
enum { TF32_COL = 0, TF32_ROW = 1 };
struct Tf32Dim {
  const float* hi = nullptr;
  const float* lo = nullptr;
  long long ext[5] = {1, 1, 1, 1, 1};
  long long stride[5] = {1, 0, 0, 0, 0};
};
struct Tf32Gemm {
  int kind = TF32_COL;
  int M = 0, N = 0, kseg = 0, nseg = 1, slo = 1, ns = 1, nt = 1, nb = 1;
  Tf32Dim S, T;
  float* C[MAXS] = {};
  const float* D[MAXS] = {};
  long long ldc = 0, ldd = 0, sC_t = 0, sC_b = 0, sD_t = 0, sD_b = 0;
  float alpha = 1.0f, beta = 0.0f;
};
cudaError_t launch_tf32_gemm(const Tf32Gemm& g, cudaStream_t stream);
double tf32_gemm_flops(const Tf32Gemm& g);
cudaError_t tf32_prepare();

// fp32 pointwise kernels (f32ops.cu).  Static-operand planes: hi = rna_tf32(x), lo = rna_tf32(x - hi).
struct F32PhaseArgs {
  int d = 0, model = 0;
  long long n[3] = {1, 1, 1};
  long long N = 0;
  float p[8] = {};
  const float* U[2] = {};
  float* G[2] = {};          // first phase: written; nonlinearity: read
  float* F[2] = {};          // first phase: F = K U + G; nonlinearity: D = g(U) - G
  const float* tri[2][3] = {};   // [species][mu-1]: lo | di | up (3 n_mu floats)
  // optional (vectorised kernels): also write Ucopy = Usrc (the state the next stage GEMM adds
  // its split action to, in place by TMA reduce-add); the nonlinearity may overwrite its own
  // input U this way (each element is read before it is written)
  const float* Usrc[2] = {};
  float* Ucopy[2] = {};
};
bool f32_phase_vec_ok(const F32PhaseArgs& a, bool first);
cudaError_t launch_split_f32(const float* x, float* hi, float* lo, long long n, cudaStream_t s);
// fp32 rows x cols blocks (nbatch, contiguous) -> planes; transpose as launch_split_f64
cudaError_t launch_split_f32_2d(const float* x, float* hi, float* lo, long long rows, long long cols, int nbatch,
                                bool transpose, cudaStream_t s);
// rows x cols blocks (nbatch of them, contiguous): out = planes of scale * x, transposed
// (out[b][r][c] = x[b][c][r], x column-major rows x cols) when `transpose`
cudaError_t launch_split_f64(const double* x, float* hi, float* lo, long long rows, long long cols, int nbatch,
                             bool transpose, double scale, cudaStream_t s);
cudaError_t launch_f64_to_f32(const double* x, float* y, long long n, cudaStream_t s);
cudaError_t launch_first_phase_f32(const F32PhaseArgs& a, cudaStream_t s);
cudaError_t launch_nonlin_f32(const F32PhaseArgs& a, cudaStream_t s);

// Nonlinearity (kernel K*3): for each point i (N per component, ns <= MAXS components):
//   mode 0:  out_c = g_c(u_1..u_ncomp)
//   mode 1:  out_c = g_c(u) - G_c
enum ModelId { MODEL_NONE = 0, MODEL_SCHNAKENBERG = 1, MODEL_FHN = 2 };
struct PointwiseArgs {
  int model = 0;
  int ncomp = 2;
  long long N = 0;
  const double* u[MAXS] = {};
  const double* G[MAXS] = {};
  double* out[MAXS] = {};
  double p[8] = {};
  // optional peer-packed output (distributed contexts): point (row, i1) of a row-major
  // (N/n1) x n1 slab goes to out[q*(N/P) + row*n1l + i1 - q*n1l], q = i1 / n1l, n1l = n1/P
  long long pack_n1 = 0, pack_n1l = 0;
  PeerMap peer;                    // packed output stored straight into the peers (P > 0)
};
cudaError_t launch_nonlinearity(const PointwiseArgs& a, int mode, cudaStream_t stream);

// Kronecker-sum action with TRIDIAGONAL A_mu: for each component s,
//   Y_s = beta * Dd_s + sum_{mu=d..1} (lo_mu[i] X[.., i-1, ..] + di_mu[i] X[.., i, ..]
//                                     + up_mu[i] X[.., i+1, ..])
// the same sum as eq:kronsumv with the exact zeros of a tridiagonal A_mu skipped.
// lo/di/up: device arrays of n_mu doubles (lo[0] and up[n-1] unused).
struct StencilArgs {
  int d = 0, ns = 1;
  long long n[6] = {1, 1, 1, 1, 1, 1};
  long long N = 0;
  const double* X[MAXS] = {};
  double* Y[MAXS] = {};
  const double* Dd[MAXS] = {};
  const double* lo[MAXS][6] = {};
  const double* di[MAXS][6] = {};
  const double* up[MAXS][6] = {};
  double beta = 0.0;
  // distributed slab (layout A): the local i_d range starts at global index d_off of n_glob_d;
  // halo_lo/halo_hi hold the neighbouring ranks' boundary planes (null at the global ends)
  long long d_off = 0, n_glob_d = 0;
  const double* halo_lo[MAXS] = {};
  const double* halo_hi[MAXS] = {};
  // optional peer-packed output, as PointwiseArgs::pack_*
  long long pack_n1 = 0, pack_n1l = 0;
  PeerMap peer;
};
cudaError_t launch_kronsum_tridiag(const StencilArgs& a, cudaStream_t stream);

// Fused G = g(U), F = K U + G for two species, d in {2, 3}, tridiagonal A_mu, n_1 even,
// N < 2^30, 16-B aligned tensors (one GPU).
struct GKronArgs {
  int d = 0, model = 0;
  int n[3] = {1, 1, 1};
  int N = 0;
  double p[8] = {};
  const double* U[2] = {};
  double* G[2] = {};
  double* F[2] = {};
  const double* tri[2][3] = {};   // [species][mu-1]: lo | di | up (3 n_mu doubles)
};
cudaError_t launch_g_kronsum(const GKronArgs& a, cudaStream_t stream);

// Kernel K*5 (fused2d.cu): nsteps whole ETD2RKDS / exprk3ds_real steps of a small 2-D grid
// (8 <= n2 <= kFusedNMax, n1 <= kFusedNMax, tridiagonal A_mu) in one 8-CTA cluster.
constexpr int kFusedCluster = 8;
constexpr int kFusedNMax = 64;
constexpr int kFusedMaxSeg = 6;
struct Fused2dArgs {
  int n1 = 0, n2 = 0, ncomp = 2, model = 0, nsteps = 1, nstages = 2;
  double p[8] = {};
  double* U[2] = {};
  const double* tri[2][2] = {};            // [species][mu-1]: lo | di | up (3 n_mu doubles)
  int nseg[3] = {}, base[3] = {};          // base: 0 = U, 1 = the previous stage value
  int seg_in[3][kFusedMaxSeg] = {};        // 0 = F, 1 = D
  const double* P2[3][kFusedMaxSeg][2] = {};   // mode-2 matrix, column-major, leading dim ld2
  long long ld2[3][kFusedMaxSeg] = {};
  const double* B[3][kFusedMaxSeg][2] = {};    // scaled mode-1 block, row-major n1 x n1
  long long* prof = nullptr;                   // diagnostics: clock64 phase stamps (<= 64)
};
cudaError_t launch_fused2d(const Fused2dArgs& a, cudaStream_t stream);
// One d = 2 Tucker operator Y = alpha L2 X L1^T + beta Y in one launch (n_1, n_2 <= 128).
bool tucker2d_small_fits(long long n1, long long n2);
cudaError_t launch_tucker2d_small(const double* X, double* Y, const double* L1, const double* L2, int n1,
                                  int n2, double alpha, double beta, cudaStream_t stream);
size_t fused2d_smem_bytes();

// Y = alpha * X (elementwise, n doubles); used for bank assembly.
cudaError_t launch_scale(double* Y, const double* X, double alpha, long long n, cudaStream_t s);
// Y = a X1 + b X2 (elementwise, n doubles); complex bank blocks.
cudaError_t launch_axpby(double* Y, double a, const double* X1, double b, const double* X2, long long n,
                         cudaStream_t s);
// Strided matrix copy with scale: Y[r*ldy + c] = alpha * X[r*ldx + c], rows x cols, batched
// over nbatch with strides sy / sx.
cudaError_t launch_copy2d(double* Y, long long ldy, long long sy, const double* X, long long ldx,
                          long long sx, long long rows, long long cols, int nbatch, double alpha,
                          cudaStream_t s);
// Same with Y = alpha X + beta Y (beta != 0 reads Y): the peer-chunk pack / unpack of the
// distributed operators.
cudaError_t launch_copy2d_axpby(double* Y, long long ldy, long long sy, const double* X, long long ldx,
                                long long sx, long long rows, long long cols, int nbatch, double alpha,
                                double beta, cudaStream_t s);
// Set n x n identity * v into each of nbatch matrices (stride n*n).
cudaError_t launch_set_identity(double* Y, long long n, int nbatch, double v, cudaStream_t s);
// flag[0] |= any(!isfinite(X[0..n)))
cudaError_t launch_check_finite(const double* X, long long n, int* flag, cudaStream_t s);
// watchdog: mon[1] = mon[0] (steps completed) if X holds a non-finite value and mon[1] == -1;
// tick: mon[0] += 1
cudaError_t launch_watch_finite(const double* X, long long n, int* mon, cudaStream_t s);
cudaError_t launch_watch_tick(int* mon, cudaStream_t s);

// Split coefficient tables (host).  Returns number of terms (0 if unsupported).
int scheme_terms(int scheme, int ell, int d, double* eta, int* inner, double* alpha);
int scheme_terms_cplx(int ell, int d, double* eta_re, double* eta_im, int* inner, double* alpha_re,
                      double* alpha_im);

}  // namespace kx
