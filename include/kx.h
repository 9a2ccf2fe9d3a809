/*
 * kx.h — C ABI of the B200-native Tucker-operator / ETD3RKDS library (arXiv 2310.07551).
 *
 * Citations: "P:n" = line n of the paper's LaTeX source; equation labels as in
 * the source (eq:kronsum, eq:krontomu, eq:kronsumv, ...).
 *
 * Problem (eq:ODE, eq:kronsum; eq:twocompdisc):
 *     u_c'(t) = K_c u_c(t) + g_c(t, u_1, ..., u_ncomp),   K_c = A^c_d (+) ... (+) A^c_1,
 * with A^c_mu dense n_mu x n_mu.  The library integrates it with the directionally split
 * exponential integrators ETD2RKDS (eq:ETD2RK + eq:phisplit) and exprk3ds_real
 * (eq:exprk3; Algorithm 1 for d = 2 with Table 1, Algorithm 2 for d > 2 with
 * Table 3), whose hot path is the Tucker operator.
 *
 * CONVENTIONS (all entry points)
 *  - Tensors are fp64 DEVICE buffers of N = n_1*...*n_d doubles in vec order: the first index
 *    is fastest, vec(T)[i_1 + n_1*(i_2 + n_2*(...))] = t_{i_1...i_d} ("stacks by columns",
 *    P:187-189).  Equivalently a C-contiguous array of shape (n_d, ..., n_1).  Buffers must
 *    be 8-byte aligned; 16-byte alignment enables the vectorised load path.
 *  - Matrices (A_mu, L_mu) are n_mu x n_mu, column-major: L[i + j*n_mu] = l_{ij}.
 *  - Ownership: the caller owns every tensor and matrix it passes (e.g. torch allocations
 *    passed by data_ptr); the library never frees them and keeps no reference beyond the call,
 *    except that kx_step caches a CUDA graph keyed on the U pointers it was given.
 *    The library owns its context, the phi-matrix bank, its workspaces (sized by kx_set_grid /
 *    kx_set_tau) and its internal streams/graphs.
 *  - Streams: every compute call is enqueued asynchronously on the stream given to
 *    kx_create (NULL = the legacy default stream) and returns immediately; use kx_sync (or
 *    synchronise that stream) before reading results on the host.  kx_set_tau is synchronous.
 *  - Errors: argument validation is synchronous — an invalid call returns KX_ERR_INVALID,
 *    enqueues nothing and records a message (kx_last_error) that names mu and both extents on
 *    shape mismatches.  Asynchronous CUDA failures surface at kx_sync or at the next call
 *    (KX_ERR_CUDA).  A context is single-stream and not thread-safe; distinct contexts are
 *    independent.
 *  - Aliasing: input tensors must not alias output tensors unless stated.
 *  - Devices: every call that takes a context runs on that context's device and restores the
 *    caller's current CUDA device before returning; contexts on different devices in one process
 *    are independent (per-device kernel attributes and occupancy data are kept per device).
 */
#ifndef KX_H
#define KX_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  KX_OK = 0,
  KX_ERR_INVALID = 2,      /* bad argument / call order; nothing enqueued            */
  KX_ERR_NUMERIC = 3,      /* non-finite state detected by kx_check_finite            */
  KX_ERR_IO = 4,
  KX_ERR_CUDA = 5,         /* CUDA runtime error (no device, launch failure, ...)     */
  KX_ERR_NCCL = 6,         /* NCCL error (multi-GPU contexts)                         */
  KX_ERR_UNSUPPORTED = 7,  /* valid request this build does not implement             */
  KX_ERR_NOMEM = 8         /* device allocation failed                                */
} kx_status;

typedef enum {
  KX_ETD2RKDS = 1,         /* second-order split ETD2RK, any d >= 1            */
  KX_ETD3RKDS_REAL = 2,    /* exprk3ds_real: Table 1 (d = 2) / Table 3 (d >= 3)          */
  KX_ETD3RKDS_CPLX = 3     /* exprk3ds_cplx: Algorithm 1 with Table 2 (complex, any d >= 2);
                              the real part is kept after each stage combination (R19)     */
} kx_scheme;

typedef enum {
  KX_MODEL_NONE = 0,          /* g = 0 (linear problem; ncomp any)                         */
  KX_MODEL_SCHNAKENBERG = 1,  /* params {delta_u, delta_v, rho, a_u, a_v}     */
  KX_MODEL_FHN = 2            /* params {delta_u, delta_v, rho, a1_v, a2_v}  */
} kx_model;

typedef struct kx_ctx kx_ctx;

typedef struct {
  long long steps;            /* kx_step calls                                           */
  long long tucker_ops;       /* Tucker operators applied (per component)      */
  long long mode_products;    /* mu-mode products executed (dense, per component)         */
  long long kronsum_actions;  /* Kronecker-sum actions (per component)                    */
  long long phi_builds;       /* small phi-matrices formed by kx_set_tau                  */
  long long gemm_launches;    /* mode-product kernel launches                             */
  long long other_launches;   /* elementwise / bank-assembly kernel launches              */
  double    mode_product_flops; /* algorithmic flops of all mode products, 2*N*n_mu each */
} kx_counters;

/* ---------------------------------------------------------------- context ---------- */
/* Create a context on CUDA device `device`, enqueueing on `cuda_stream` (a cudaStream_t,
 * NULL = legacy default stream).  Returns KX_ERR_CUDA if the device is unavailable. */
kx_status kx_create(kx_ctx **ctx, int device, void *cuda_stream);
/* Free the context and everything it owns.  NULL is a no-op. */
void kx_destroy(kx_ctx *ctx);
/* Last error message of this context ("" if none).  Pointer valid until the next call. */
const char *kx_last_error(const kx_ctx *ctx);
/* Message of the last failed kx_create on this thread. */
const char *kx_create_error(void);

/* Grid: d in 1..6 directions with extents n[0..d-1] = n_1..n_d (each >= 1), ncomp in 1..4
 * components (species).  Resets matrices, model, tau and counters. */
kx_status kx_set_grid(kx_ctx *ctx, int d, const long long *n, int ncomp);
/* Direction matrix A^comp_mu (mu = 1..d, comp = 0..ncomp-1), HOST column-major n_mu x n_mu,
 * copied (host and device copies kept).  Invalidates the phi bank. */
kx_status kx_set_direction_matrix(kx_ctx *ctx, int comp, int mu, const double *A_host);
/* Nonlinearity g (pointwise over the components; ncomp must be 2 for the two models). */
kx_status kx_set_model(kx_ctx *ctx, kx_model model, const double *params, int nparams);
/* Step size tau > 0 and scheme: forms every small phi-matrix the scheme needs on the device
 * ("Needed phi-functions" loop, P:2212-2228 / P:2285-2301) with a Taylor base approximant and
 * the modified squaring identities of [SW09], then lays out the bank.
 * Synchronous.  Requires all direction matrices. */
kx_status kx_set_tau(kx_ctx *ctx, double tau, kx_scheme scheme);

/* ---------------------------------------------------------------- operators -------- */
/* mu-mode product: Y = alpha * (X x_mu L) + beta * Y, L a DEVICE column-major
 * n_mu x n_mu matrix.  X and Y distinct; beta == 0 ignores Y's contents. */
kx_status kx_mode_product(kx_ctx *ctx, const double *X, double *Y, int mu, const double *L,
                          double alpha, double beta);
/* Tucker operator: Y = alpha * (X x_1 L[0] x_2 ... x_d L[d-1]) + beta * Y.
 * L is a HOST array of d DEVICE matrix pointers.  Modes are applied d, d-1, ..., 1
 * (reading R2).  X and Y distinct. */
kx_status kx_tucker(kx_ctx *ctx, const double *X, double *Y, const double *const *L,
                    double alpha, double beta);
/* Batched Tucker operator: nbatch independent tensors sharing the matrices {L_mu},
 *   Y_b = alpha * (X_b x_1 L[0] ... x_d L[d-1]) + beta * Y_b,   b = 0 .. nbatch-1,
 * with X_b = X + b*N and Y_b = Y + b*N (nbatch tensors of N doubles back to back, DEVICE).
 * One GEMM launch per mode for the whole batch (modes d..1): the tensors' outer slabs are one
 * strided batch for mu >= 2 and one tall matrix of nbatch*N/n_1 rows for mu = 1, so small
 * grids (n_mu = 256, 512) fill the GPU that a single Tucker cannot (every mode is a
 * single GEMM).  Library-owned intermediates of nbatch*N doubles are grown on demand (the first
 * call with a larger batch synchronises the stream).  nbatch*N must stay below 2^31; X, Y
 * distinct. */
kx_status kx_tucker_batched(kx_ctx *ctx, int nbatch, const double *X, double *Y,
                            const double *const *L, double alpha, double beta);
/* Kronecker-sum action (eq:kronsumv): Y = K_comp X + beta * Y with the context's
 * direction matrices of component comp.  X and Y distinct. */
kx_status kx_kronsum(kx_ctx *ctx, int comp, const double *X, double *Y, double beta);
/* How the Kronecker-sum action (kx_kronsum and the F = K U + G of kx_step) is executed:
 * mode 0 (default) uses a fused stencil kernel when every A^c_mu is tridiagonal (as for the FD
 * Laplacians of Sec. 3) — the dense mode products would only add exact zeros —
 * and d dense mode products otherwise; mode 1 always uses the dense mode products. */
kx_status kx_set_kronsum_mode(kx_ctx *ctx, int mode);
/* Split phi-action from the current bank: Y = alpha * S[X] + beta * Y (for KX_ETD3RKDS_CPLX
 * the real part of S[X]) where
 *   S[X] = sum_i eta_i T(X, {phi_{l_i}(c tau alpha_{i,mu} A^comp_mu)}_mu)
 * (eq:split2d / eq:splitnd3 via eq:krontomu).  ETD3RKDS bank: ell in {1,2},
 * stage 0: c = 1/3 (ell = 1 only), stage 1: c = 2/3, stage 2: c = 1.
 * ETD2RKDS bank: stage must be 2 (c = 1), ell in {1,2}, second-order split (eq:secondord). */
kx_status kx_phi_apply(kx_ctx *ctx, int comp, int ell, int stage, const double *X, double *Y,
                       double alpha, double beta);
/* One time step of the scheme set by kx_set_tau, in place on the ncomp DEVICE tensors U[c]
 * (HOST array of device pointers).  t is the time at the start of the step (the built-in
 * models are autonomous).  Replays a cached CUDA graph when the U pointers repeat. */
kx_status kx_step(kx_ctx *ctx, double t, double *const *U);
/* nsteps (>= 0) consecutive kx_step calls from time t0.  On a small 2-D grid (see
 * kx_set_fused_small) all nsteps run inside ONE kernel launch; otherwise the step graph is
 * replayed nsteps times.  With the NaN watchdog on, steps are launched one by one. */
kx_status kx_step_n(kx_ctx *ctx, double t0, int nsteps, double *const *U);
/* Same as kx_step but U are HOST buffers (N doubles each): copies them to the device,
 * steps `nsteps` times (as kx_step_n), copies back, synchronises (end-to-end entry point).
 * With page-locked buffers (cudaHostAlloc / cudaHostRegister / torch pin_memory) the last
 * step's final stage GEMM runs in 4 row chunks (KX_TAIL_CHUNKS=1..8) and each chunk's rows are
 * copied back while the next chunk computes.  The result then equals kx_step_n up to the
 * rounding of that GEMM's split K sums (~1e-16 relative).  It stays deterministic run to run.
 * Pageable buffers are copied after the last step, bitwise as kx_step_n. */
kx_status kx_integrate_host(kx_ctx *ctx, double t0, int nsteps, double *const *U_host);
/* Small 2-D grids (d = 2, 8 <= n_2 <= 64, n_1 <= 64, tridiagonal A_mu, real scheme, one GPU):
 * on = 1 (default) executes each step as ONE kernel on an 8-CTA thread-block cluster that
 * keeps the state in shared memory and fuses the mode-2 and mode-1 products of every term
 * (the shape of eq:exp2d; SURVEY §2 K*5); and kx_tucker on a 2-D grid with
 * n_1, n_2 <= 128 runs both mode products in one launch (intermediate in shared memory).
 * on = 0 forces the general path for both. */
kx_status kx_set_fused_small(kx_ctx *ctx, int on);

/* ---------------------------------------------------------------- multi-GPU -------- */
/* Slab decomposition along i_d over P ranks (one process per GPU); see DESIGN.md §8.
 * Every rank calls kx_set_grid with the GLOBAL extents (n_1 and n_d divisible by P, d >= 2),
 * the same direction matrices, model and tau; its tensors U[c] hold the local slab
 * i_d in [rank n_d/P, (rank+1) n_d/P) in vec order (N/P doubles).  kx_step then performs the
 * sharded step with NCCL all-to-all exchanges (ncclSend/ncclRecv groups, fp64) enqueued on the
 * context stream.
 * The operators kx_tucker, kx_mode_product, kx_phi_apply and kx_kronsum (dense A_mu: the mode-d
 * term through the exchange) also work on NCCL ranks, on the
 * rank's layout-A slab X, Y (N/P doubles each; the matrices / bank are global): modes 1..d-1
 * are local; an operator that contracts mode d runs [A] pack by i_1 block -> all-to-all ->
 * [B] modes d..2 on full fibres -> all-to-all -> [A] mode 1 as one concatenated-K GEMM over the
 * source ranks' chunks (alpha, beta in its epilogue), so it matches one GPU up to rounding
 * (BASELINE.json configs[4] at 2-8 GPUs).  Collective: every rank calls it with the
 * same arguments apart from X, Y.  kx_tucker_batched and kx_integrate_host return
 * KX_ERR_UNSUPPORTED on distributed contexts. */
/* 128-byte ncclUniqueId (NCCL from the process, dlopen'ed); create on rank 0, broadcast. */
kx_status kx_nccl_unique_id(void *out128);
kx_status kx_create_dist(kx_ctx **ctx, int device, void *cuda_stream, const void *nccl_unique_id,
                         int rank, int nranks);
/* In-process loopback group: nranks contexts on ONE device sharing one stream; the exchanges are
 * device copies issued between phases by kx_step_group (no kernel ever waits on another rank).
 * Used to test the sharded schedule on a single GPU.  U holds nranks*ncomp device pointers,
 * rank-major (U[r*ncomp + c]). */
kx_status kx_create_group(kx_ctx **ctxs, int nranks, int device, void *cuda_stream);
/* NCCL ranks (default: on when nranks > 1): the 3T + T + T term slots of each step are sent to the peers term
 * by term on an internal communication stream while the next term's mode products run
 * (SURVEY §8(f) f2); off = one exchange per phase on the context stream. */
kx_status kx_set_dist_overlap(kx_ctx *ctx, int on);
kx_status kx_step_group(kx_ctx *const *ctxs, int nranks, double t, double *const *U);
/* The distributed operators on a loopback group: X[r], Y[r] are rank r's layout-A slabs
 * (device, N/P doubles); L / the bank as for the one-context calls. */
kx_status kx_tucker_group(kx_ctx *const *ctxs, int nranks, const double *const *X, double *const *Y,
                          const double *const *L, double alpha, double beta);
kx_status kx_mode_product_group(kx_ctx *const *ctxs, int nranks, const double *const *X,
                                double *const *Y, int mu, const double *L, double alpha, double beta);
kx_status kx_kronsum_group(kx_ctx *const *ctxs, int nranks, int comp, const double *const *X,
                           double *const *Y, double beta);
kx_status kx_phi_apply_group(kx_ctx *const *ctxs, int nranks, int comp, int ell, int stage,
                             const double *const *X, double *const *Y, double alpha, double beta);
/* Direct peer stores: the kernel producing each exchanged tensor (stencil F,
 * nonlinearity D, the last mode product of every term group) stores block q of its
 * peer-packed output straight into rank q's receive buffer, so the all-to-all becomes a barrier
 * (stream order in a loopback group; a 1-double NCCL all-reduce across processes).  Real
 * schemes with tridiagonal A_mu; other cases keep the exchanges.  Loopback group: enable after
 * every member's kx_set_tau (which disables it again). */
kx_status kx_group_set_p2p(kx_ctx *const *ctxs, int nranks, int on);
/* NCCL ranks (one process per GPU): export this rank's receive buffers as CUDA IPC handles
 * (blob == NULL: *len = size needed), all-gather the blobs (e.g. torch.distributed), then
 * import all nranks blobs (rank order, len_each bytes each) on every rank.  After kx_set_tau,
 * which disables it; every rank must import before the next kx_step. */
kx_status kx_dist_ipc_export(kx_ctx *ctx, void *blob, size_t cap, size_t *len);
kx_status kx_dist_ipc_import(kx_ctx *ctx, const void *blobs, size_t len_each);

/* ---------------------------------------------------------------- utilities -------- */
kx_status kx_get_counters(const kx_ctx *ctx, kx_counters *out);
kx_status kx_reset_counters(kx_ctx *ctx);
/* Synchronise the context stream; returns KX_ERR_CUDA with a message on async failure, and
 * KX_ERR_NUMERIC if the NaN watchdog (kx_set_nan_check) has fired. */
kx_status kx_sync(kx_ctx *ctx);
/* Per-step NaN/Inf watchdog (off by default): when on, every kx_step / kx_step_group also checks
 * the updated U on the device; kx_sync then returns KX_ERR_NUMERIC naming the first step (counted
 * from this call) whose result was non-finite.  Resets the step count and the flag. */
kx_status kx_set_nan_check(kx_ctx *ctx, int on);
/* KX_ERR_NUMERIC if any entry of the device tensor X (N doubles) is NaN/Inf (synchronous). */
kx_status kx_check_finite(kx_ctx *ctx, const double *X);
/* Per-launch CUDA-event timing of kx_step's kernels (disables graph replay while on).
 * kx_get_profile fills gemm_ms / other_ms (summed device time) and gemm_launches /
 * other_launches counted since profiling was enabled, and gemm_flops (algorithmic). */
kx_status kx_set_profiling(kx_ctx *ctx, int on);
kx_status kx_get_profile(kx_ctx *ctx, double *gemm_ms, double *other_ms, long long *gemm_launches,
                         long long *other_launches, double *gemm_flops);
/* Algorithmic HBM bytes (reads + writes of whole fields) of the non-GEMM kernels timed since
 * profiling was enabled (nonlinearity, stencil, fused G/F pass, watchdog): divided by
 * other_ms of kx_get_profile it is their achieved bandwidth. */
kx_status kx_get_profile_hbm(kx_ctx *ctx, double *other_bytes);
/* Copy one phi-matrix of the current bank to the host (column-major n_mu x n_mu, unscaled):
 * phi_{l_term}(c tau alpha_{term,mu} A^comp_mu) for (ell, stage) as in kx_phi_apply.  For
 * KX_ETD3RKDS_CPLX, `term` indexes real planes: 2i = Re, 2i+1 = Im of term i. */
kx_status kx_get_phi_matrix(kx_ctx *ctx, int comp, int ell, int stage, int term, int mu,
                            double *out_host);

/* Replace one phi-matrix of the current bank by a caller-supplied HOST matrix (column-major
 * n_mu x n_mu), the inverse of kx_get_phi_matrix with the same (comp, ell, stage, term, mu)
 * indexing: P_term{mu} = phi_{l_term}(c tau alpha_{term,mu} A^comp_mu) of eq:split2d /
 * eq:splitnd3 as listed by Algorithms 1-2's "Needed phi-functions"
 * (P:2212-2228).  Every scaled block derived from it (the eta- and stage-scaled mu = 1 blocks
 * of eq:exprk3) is re-formed on the device.  Lets the hot path run on an externally
 * formed bank — e.g. the CPU oracle's — so that its parity is checked independently of the phi
 * algorithm (SURVEY §8(c) ledger row 8, "shared bank").  Synchronous; drops the cached step
 * graph; the next kx_set_tau rebuilds the library's own bank.  KX_ERR_INVALID on a bad index
 * or non-finite entries (nothing changed). */
kx_status kx_set_phi_matrix(kx_ctx *ctx, int comp, int ell, int stage, int term, int mu,
                            const double *in_host);

/* ---------------------------------------------------------------- fp32 variant ----- */
/* The paper's single-precision runs ("CUDA single" columns of Table 5, and
 * Table 7; the laptop single-precision timings).
 * Same operators and step schedule as the fp64 calls, on fp32 DEVICE tensors / matrices (same
 * vec order and column-major conventions), with every mode product on the tcgen05 tensor cores
 * (kind::tf32) in a three-pass split x = hi + lo of both operands (hi, lo tf32-valued;
 * AB ~ A_hi B_hi + A_hi B_lo + A_lo B_hi, fp32 accumulation), which keeps fp32 accuracy.
 * Requirements: one GPU, every n_mu a multiple of 4, 16-byte aligned buffers; otherwise
 * KX_ERR_UNSUPPORTED / KX_ERR_INVALID with nothing enqueued.  Library-owned fp32 scratch is
 * grown on demand (the first larger call synchronises the stream).
 *
 * mu-mode product: Y = alpha (X x_mu L) + beta Y; X, Y, L fp32, X and Y distinct. */
kx_status kx_mode_product_f32(kx_ctx *ctx, const float *X, float *Y, int mu, const float *L,
                              float alpha, float beta);
/* Tucker operator: Y = alpha (X x_1 L[0] ... x_d L[d-1]) + beta Y, modes applied
 * d, ..., 1; L a HOST array of d fp32 DEVICE matrices. */
kx_status kx_tucker_f32(kx_ctx *ctx, const float *X, float *Y, const float *const *L,
                        float alpha, float beta);
/* nsteps (>= 0) steps of the scheme set by kx_set_tau (KX_ETD2RKDS or KX_ETD3RKDS_REAL), in place
 * on the 2 fp32 DEVICE tensors U[c], d in {2, 3}, tridiagonal A_mu (the stencil Kronecker sum),
 * a built-in model; the phi-matrices are the fp64 bank of kx_set_tau rounded once.  Replays a
 * cached CUDA graph per step when the U pointers repeat. */
kx_status kx_step_f32(kx_ctx *ctx, double t0, int nsteps, float *const *U);

/* Host-only (no device needed): the split coefficients the library uses.
 * scheme KX_ETD2RKDS -> second-order single term; KX_ETD3RKDS_REAL -> Table 1 (d = 2) or
 * Table 3 (d >= 3), "+" branch.  Writes *nterms, eta[i], inner_ell[i] and
 * alpha[i*d + mu-1]; arrays must hold 3 terms (3*d alphas). */
kx_status kx_scheme_coefficients(kx_scheme scheme, int ell, int d, int *nterms, double *eta,
                                 int *inner_ell, double *alpha);
/* Host-only: Table 2 coefficients (complex), "+ in alpha_{1,mu}" branch; arrays hold 2 terms. */
kx_status kx_scheme_coefficients_cplx(int ell, int d, int *nterms, double *eta_re, double *eta_im,
                                      int *inner_ell, double *alpha_re, double *alpha_im);
/* Library version string. */
const char *kx_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KX_H */
