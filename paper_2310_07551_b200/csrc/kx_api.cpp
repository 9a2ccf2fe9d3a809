// C ABI (include/kx.h): argument validation and dispatch to the internals.
#include <dlfcn.h>

#include "kx_ctx.h"

using namespace kx::detail;

namespace {
thread_local std::string g_create_error;
}  // namespace

namespace kx {
void gemm_prepare_all();
}

// ============================================================================ C ABI ======
extern "C" {

const char* kx_version(void) { return "kx 0.2 (sm_100a, fp64 DMMA mode products; fp32 on tcgen05 kind::tf32 x3)"; }

const char* kx_create_error(void) { return g_create_error.c_str(); }

kx_status kx_create(kx_ctx** out, int device, void* cuda_stream) {
  if (!out) return KX_ERR_INVALID;
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    g_create_error = std::string("no CUDA device: ") + cudaGetErrorString(e);
    return KX_ERR_CUDA;
  }
  if (device < 0 || device >= ndev) {
    g_create_error = "device index out of range";
    return KX_ERR_INVALID;
  }
  DevGuard dg_(device);   // the caller's current device is restored on return
  int now = -1;
  e = cudaGetDevice(&now);
  if (e == cudaSuccess && now != device) e = cudaErrorInvalidDevice;
  if (e != cudaSuccess) {
    g_create_error = std::string("cudaSetDevice: ") + cudaGetErrorString(e);
    return KX_ERR_CUDA;
  }
  kx_ctx* c = new kx_ctx();
  c->device = device;
  c->stream = static_cast<cudaStream_t>(cuda_stream);
  c->cur = c->stream;
  e = cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&c->flag), sizeof(int));
  if (e == cudaSuccess)
    e = cudaMalloc(reinterpret_cast<void**>(&c->sk_ws), sizeof(double) * kx::kSkSlots * 128 * 128);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&c->sk_flags), sizeof(int) * kx::kSkFlags);
  if (e == cudaSuccess) e = cudaMemset(c->sk_flags, 0, sizeof(int) * kx::kSkFlags);
  if (e != cudaSuccess) {
    g_create_error = std::string("context setup: ") + cudaGetErrorString(e);
    delete c;
    return KX_ERR_CUDA;
  }
  kx::gemm_prepare_all();
  *out = c;
  return KX_OK;
}

void kx_destroy(kx_ctx* c) {
  DevGuard dg_(c);
  if (!c) return;
  cudaStreamSynchronize(c->stream);
  drop_bank(c);
  f32_free(c);
  dop_free(c);
  for (auto& v : c->A_dev)
    for (double* p : v) cudaFree(p);
  for (auto& v : c->A_tri)
    for (double* p : v) cudaFree(p);
  if (c->tmp1) cudaFree(c->tmp1);
  if (c->tmp2) cudaFree(c->tmp2);
  for (double* p : c->btmp)
    if (p) cudaFree(p);
  for (int s = 0; s < MAXS; ++s)
    if (c->hostU[s]) cudaFree(c->hostU[s]);
  if (c->flag) cudaFree(c->flag);
#ifdef KX_HAVE_NCCL
  if (c->nccl_comm && nccl().ok) nccl().CommDestroy(static_cast<ncclComm_t>(c->nccl_comm));
#endif
  if (c->comm) cudaStreamDestroy(c->comm);
  if (c->copy) cudaStreamDestroy(c->copy);
  for (auto e : c->ev_tail)
    if (e) cudaEventDestroy(e);
  for (auto e : c->ev_term)
    if (e) cudaEventDestroy(e);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->watch) cudaFree(c->watch);
  if (c->bar_buf) cudaFree(c->bar_buf);
  if (c->sk_ws) cudaFree(c->sk_ws);
  if (c->sk_flags) cudaFree(c->sk_flags);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->cap) cudaStreamDestroy(c->cap);
  delete c;
}

const char* kx_last_error(const kx_ctx* c) { return c ? c->err.c_str() : "null context"; }

kx_status kx_set_grid(kx_ctx* c, int d, const long long* n, int ncomp) {
  DevGuard dg_(c);
  if (!c) return KX_ERR_INVALID;
  if (d < 1 || d > KX_MAXD) return fail(c, KX_ERR_INVALID, "d must be in 1..6");
  if (ncomp < 1 || ncomp > MAXS) return fail(c, KX_ERR_INVALID, "ncomp must be in 1..4");
  if (!n) return fail(c, KX_ERR_INVALID, "n is NULL");
  long long N = 1;
  for (int mu = 0; mu < d; ++mu) {
    if (n[mu] < 1 || n[mu] > (1LL << 20))
      return fail(c, KX_ERR_INVALID, "extent n_" + std::to_string(mu + 1) + " out of range");
    N *= n[mu];
    if (N > (1LL << 31) - 1) return fail(c, KX_ERR_INVALID, "N = prod n_mu exceeds 2^31-1");
  }
  cudaStreamSynchronize(c->stream);
  drop_bank(c);
  dop_free(c);
  for (auto& v : c->A_dev)
    for (double* p : v) cudaFree(p);
  for (auto& v : c->A_tri)
    for (double* p : v) cudaFree(p);
  c->A_dev.clear();
  c->A_tri.clear();
  c->A_host.clear();
  if (c->tmp1) cudaFree(c->tmp1);
  if (c->tmp2) cudaFree(c->tmp2);
  c->tmp1 = c->tmp2 = nullptr;
  for (double*& p : c->btmp) {
    if (p) cudaFree(p);
    p = nullptr;
  }
  c->btmp_cap = 0;
  for (int s = 0; s < MAXS; ++s) {
    if (c->hostU[s]) cudaFree(c->hostU[s]);
    c->hostU[s] = nullptr;
  }
  c->d = d;
  c->ncomp = ncomp;
  for (int mu = 0; mu < KX_MAXD; ++mu) c->n[mu] = mu < d ? n[mu] : 1;
  c->N = N;
  for (int mu = 0; mu < KX_MAXD; ++mu) c->tn[mu] = c->n[mu];
  c->tN = N;
  if (c->dist) {
    const int P = c->nranks;
    if (d < 2 || n[0] % P != 0 || n[d - 1] % P != 0)
      return fail(c, KX_ERR_INVALID, "distributed grids need d >= 2 and n_1, n_d divisible by the rank count");
    for (int mu = 0; mu < KX_MAXD; ++mu) c->nA[mu] = c->nB[mu] = c->n[mu];
    c->nA[d - 1] = n[d - 1] / P;
    c->nB[0] = n[0] / P;
    c->Nloc = N / P;
    for (int mu = 0; mu < KX_MAXD; ++mu) c->tn[mu] = c->nA[mu];
    c->tN = c->Nloc;
  }
  c->A_host.assign(ncomp, std::vector<std::vector<double>>(d));
  c->A_dev.assign(ncomp, std::vector<double*>(d, nullptr));
  c->A_tri.assign(ncomp, std::vector<double*>(d, nullptr));
  c->model = 0;
  c->cnt = kx_counters{};
  std::vector<double*> keep;
  KX_TRY(dalloc(c, &c->tmp1, (size_t)N, keep));
  KX_TRY(dalloc(c, &c->tmp2, (size_t)N, keep));
  return KX_OK;
}

kx_status kx_set_direction_matrix(kx_ctx* c, int comp, int mu, const double* A_host) {
  DevGuard dg_(c);
  KX_TRY(need_grid(c));
  if (comp < 0 || comp >= c->ncomp) return fail(c, KX_ERR_INVALID, "comp out of range");
  if (mu < 1 || mu > c->d) return fail(c, KX_ERR_INVALID, "mu out of range 1..d");
  if (!A_host) return fail(c, KX_ERR_INVALID, "A_host is NULL");
  const long long n = c->n[mu - 1];
  for (long long i = 0; i < n * n; ++i)
    if (!std::isfinite(A_host[i])) return fail(c, KX_ERR_INVALID, "A has non-finite entries");
  cudaStreamSynchronize(c->stream);
  drop_bank(c);
  c->A_host[comp][mu - 1].assign(A_host, A_host + n * n);
  if (!c->A_dev[comp][mu - 1]) {
    std::vector<double*> keep;
    KX_TRY(dalloc(c, &c->A_dev[comp][mu - 1], (size_t)(n * n), keep));
  }
  KX_CUDA(c, cudaMemcpy(c->A_dev[comp][mu - 1], A_host, n * n * 8, cudaMemcpyHostToDevice));
  // tridiagonal? keep lo | di | up for the stencil form of the Kronecker-sum action
  bool tri = true;
  for (long long j = 0; j < n && tri; ++j)
    for (long long i = 0; i < n; ++i)
      if ((i - j > 1 || j - i > 1) && A_host[i + j * n] != 0.0) {
        tri = false;
        break;
      }
  if (c->A_tri[comp][mu - 1]) {
    cudaFree(c->A_tri[comp][mu - 1]);
    c->A_tri[comp][mu - 1] = nullptr;
  }
  if (tri) {
    std::vector<double> t(3 * n, 0.0);
    for (long long i = 0; i < n; ++i) {
      if (i > 0) t[i] = A_host[i + (i - 1) * n];
      t[n + i] = A_host[i + i * n];
      if (i + 1 < n) t[2 * n + i] = A_host[i + (i + 1) * n];
    }
    std::vector<double*> keep;
    KX_TRY(dalloc(c, &c->A_tri[comp][mu - 1], (size_t)(3 * n), keep));
    KX_CUDA(c, cudaMemcpy(c->A_tri[comp][mu - 1], t.data(), 3 * n * 8, cudaMemcpyHostToDevice));
  }
  return KX_OK;
}

kx_status kx_set_model(kx_ctx* c, kx_model model, const double* params, int nparams) {
  DevGuard dg_(c);
  KX_TRY(need_grid(c));
  if (model == KX_MODEL_NONE) {
    c->model = 0;
    return KX_OK;
  }
  if (model != KX_MODEL_SCHNAKENBERG && model != KX_MODEL_FHN)
    return fail(c, KX_ERR_INVALID, "unknown model");
  if (c->ncomp != 2) return fail(c, KX_ERR_INVALID, "the built-in models need ncomp == 2");
  if (!params || nparams != 5) return fail(c, KX_ERR_INVALID, "models take 5 parameters");
  for (int i = 0; i < 5; ++i) {
    if (!std::isfinite(params[i])) return fail(c, KX_ERR_INVALID, "non-finite model parameter");
    c->params[i] = params[i];
  }
  c->model = model;
  drop_graph(c);
  return KX_OK;
}

kx_status kx_set_tau(kx_ctx* c, double tau, kx_scheme scheme) {
  DevGuard dg_(c);
  KX_TRY(need_grid(c));
  if (!(tau > 0.0) || !std::isfinite(tau)) return fail(c, KX_ERR_INVALID, "tau must be > 0");
  if (scheme != KX_ETD2RKDS && scheme != KX_ETD3RKDS_REAL && scheme != KX_ETD3RKDS_CPLX)
    return fail(c, KX_ERR_INVALID, "unknown scheme");
  if (scheme != KX_ETD2RKDS && c->d < 2)
    return fail(c, KX_ERR_UNSUPPORTED, "exprk3ds needs d >= 2 (Tables 1-3)");
  for (int comp = 0; comp < c->ncomp; ++comp)
    for (int mu = 1; mu <= c->d; ++mu)
      if (c->A_host[comp][mu - 1].empty())
        return fail(c, KX_ERR_INVALID, "direction matrix (comp " + std::to_string(comp) +
                                           ", mu " + std::to_string(mu) + ") not set");
  KX_CUDA(c, cudaStreamSynchronize(c->stream));
  c->cur = c->stream;
  kx_status s = set_tau_impl(c, tau, scheme);
  if (s != KX_OK) drop_bank(c);
  return s;
}

kx_status kx_mode_product(kx_ctx* c, const double* X, double* Y, int mu, const double* L,
                          double alpha, double beta) {
  DevGuard dg_(c);
  KX_TRY(need_grid(c));
  if (c->dist == 2) return fail(c, KX_ERR_INVALID, "loopback group members use kx_mode_product_group");
  if (mu < 1 || mu > c->d)
    return fail(c, KX_ERR_INVALID, "mode " + std::to_string(mu) + " outside 1.." + std::to_string(c->d));
  KX_TRY(check_ptr(c, X, "X"));
  KX_TRY(check_ptr(c, Y, "Y"));
  KX_TRY(check_ptr(c, L, "L"));
  if (X == Y) return fail(c, KX_ERR_INVALID, "X and Y must be distinct");
  c->cur = c->stream;
  if (c->dist == 1 && mu == c->d) {   // the sharded direction: two all-to-alls (kx_dist_ops.cpp)
    DistOp op;
    op.kind = 2;
    op.X = X;
    op.Y = Y;
    op.L[mu - 1] = L;
    op.alpha = alpha;
    op.beta = beta;
    return dist_op_nccl(c, op);
  }
  if (c->dist) set_layout(c, false);   // modes 1..d-1 are local to the slab
  const double* Xs[1] = {X};
  double* Ys[1] = {Y};
  const double* Ls[1] = {L};
  const double* Ds[1] = {Y};
  return mode_product_multi(c, 1, Xs, Ys, mu, Ls, alpha, beta, Ds);
}

kx_status kx_tucker(kx_ctx* c, const double* X, double* Y, const double* const* L, double alpha,
                    double beta) {
  DevGuard dg_(c);
  KX_TRY(need_grid(c));
  if (c->dist == 2) return fail(c, KX_ERR_INVALID, "loopback group members use kx_tucker_group");
  KX_TRY(check_ptr(c, X, "X"));
  KX_TRY(check_ptr(c, Y, "Y"));
  if (!L) return fail(c, KX_ERR_INVALID, "L is NULL");
  for (int mu = 0; mu < c->d; ++mu) KX_TRY(check_ptr(c, L[mu], "L[mu]"));
  if (X == Y) return fail(c, KX_ERR_INVALID, "X and Y must be distinct");
  c->cur = c->stream;
  const int d = c->d;
  if (c->dist == 1) {   // slab-sharded: [A] pack -> [B] modes d..2 -> [A] concat-K mode 1
    DistOp op;
    op.X = X;
    op.Y = Y;
    for (int mu = 0; mu < d; ++mu) op.L[mu] = L[mu];
    op.alpha = alpha;
    op.beta = beta;
    KX_TRY(dist_op_nccl(c, op));
    c->cnt.tucker_ops += 1;
    return KX_OK;
  }
  if (d == 2 && c->fused_small && kx::tucker2d_small_fits(c->tn[0], c->tn[1])) {
    // small 2-D grid: both mode products in one launch, the intermediate in shared memory
    const double fl = 2.0 * (double)c->tN * (double)(c->tn[0] + c->tn[1]);
    int e0 = -1;
    if (c->profiling) {
      e0 = c->ev_used;
      c->ev_used += 2;
      KX_CUDA(c, record(c, pool_event(c, e0)));
    }
    KX_CUDA(c, kx::launch_tucker2d_small(X, Y, L[0], L[1], (int)c->tn[0], (int)c->tn[1], alpha, beta, c->cur));
    if (c->profiling) {
      KX_CUDA(c, record(c, pool_event(c, e0 + 1)));
      c->recs.push_back({0, e0, e0 + 1, fl});
    }
    c->cnt.gemm_launches += 1;
    c->cnt.mode_products += 2;
    c->cnt.mode_product_flops += fl;
    c->cnt.tucker_ops += 1;
    return KX_OK;
  }
  const double* src = X;
  double* bufs[2] = {c->tmp1, c->tmp2};
  int w = 0;
  for (int mu = d; mu >= 2; --mu) {
    const double* Xs[1] = {src};
    double* Ys[1] = {bufs[w]};
    const double* Ls[1] = {L[mu - 1]};
    KX_TRY(mode_product_multi(c, 1, Xs, Ys, mu, Ls, 1.0, 0.0, nullptr));
    src = bufs[w];
    w ^= 1;
  }
  const double* Xs[1] = {src};
  double* Ys[1] = {Y};
  const double* Ls[1] = {L[0]};
  const double* Ds[1] = {Y};
  KX_TRY(mode_product_multi(c, 1, Xs, Ys, 1, Ls, alpha, beta, Ds));
  c->cnt.tucker_ops += 1;
  return KX_OK;
}

kx_status kx_tucker_batched(kx_ctx* c, int nbatch, const double* X, double* Y, const double* const* L,
                            double alpha, double beta) {
  DevGuard dg_(c);
  KX_TRY(need_grid(c));
  if (c->dist) return fail(c, KX_ERR_UNSUPPORTED, "single-GPU operator on a distributed context");
  if (nbatch < 0) return fail(c, KX_ERR_INVALID, "nbatch must be >= 0");
  if (nbatch == 0) return KX_OK;
  KX_TRY(check_ptr(c, X, "X"));
  KX_TRY(check_ptr(c, Y, "Y"));
  if (!L) return fail(c, KX_ERR_INVALID, "L is NULL");
  for (int mu = 0; mu < c->d; ++mu) KX_TRY(check_ptr(c, L[mu], "L[mu]"));
  if (X == Y) return fail(c, KX_ERR_INVALID, "X and Y must be distinct");
  const int d = c->d;
  const long long N = c->tN;
  if ((double)nbatch * (double)N > 2147483647.0)
    return fail(c, KX_ERR_INVALID, "nbatch * N exceeds 2^31-1");
  c->cur = c->stream;
  const size_t need = d >= 2 ? (size_t)nbatch * (size_t)N : 0;
  if (need > c->btmp_cap) {
    KX_CUDA(c, cudaStreamSynchronize(c->stream));
    for (double*& p : c->btmp) {
      if (p) cudaFree(p);
      p = nullptr;
    }
    c->btmp_cap = 0;
    std::vector<double*> keep;
    KX_TRY(dalloc(c, &c->btmp[0], need, keep));
    if (d >= 3) KX_TRY(dalloc(c, &c->btmp[1], need, keep));
    c->btmp_cap = need;
  }
  // modes d..2: Y_b = L X_b over every (tensor, outer slab) pair — the tensors are contiguous,
  // so the batch of nbatch x prod_{nu>mu} n_nu slabs has one stride (n_mu prod_{nu<mu} n_nu)
  const double* src = X;
  int w = 0;
  for (int mu = d; mu >= 2; --mu) {
    const long long nm = c->tn[mu - 1];
    const long long R = prod_range(c, 1, mu - 1);
    const long long Bt = prod_range(c, mu + 1, d);
    GemmArgs g;
    g.arow = false;
    g.M = (int)nm;
    g.N = (int)R;
    g.kseg = (int)nm;
    g.lda = nm;
    g.ldb = R;
    g.ldc = R;
    g.nb = (int)(Bt * nbatch);
    g.sB_b = g.sC_b = nm * R;
    g.A[0] = L[mu - 1];
    g.B[0] = src;
    g.C[0] = c->btmp[w];
    KX_TRY(run_gemm(c, g));
    src = c->btmp[w];
    w ^= 1;
  }
  // mode 1: Y_r = X_r L_1^T over all nbatch * N / n_1 rows
  const long long n1 = c->tn[0];
  GemmArgs g;
  g.arow = true;
  g.M = (int)((long long)nbatch * N / n1);
  g.N = (int)n1;
  g.kseg = (int)n1;
  g.lda = g.ldb = g.ldc = g.ldd = n1;
  g.alpha = alpha;
  g.beta = beta;
  g.A[0] = src;
  g.B[0] = L[0];
  g.C[0] = Y;
  g.D[0] = beta != 0.0 ? Y : nullptr;
  KX_TRY(run_gemm(c, g));
  c->cnt.mode_products += (long long)nbatch * d;
  c->cnt.tucker_ops += nbatch;
  return KX_OK;
}

kx_status kx_kronsum(kx_ctx* c, int comp, const double* X, double* Y, double beta) {
  DevGuard dg_(c);
  KX_TRY(need_grid(c));
  if (c->dist == 2) return fail(c, KX_ERR_INVALID, "loopback group members use kx_kronsum_group");
  if (comp < 0 || comp >= c->ncomp) return fail(c, KX_ERR_INVALID, "comp out of range");
  for (int mu = 1; mu <= c->d; ++mu)
    if (!c->A_dev[comp][mu - 1])
      return fail(c, KX_ERR_INVALID, "direction matrix mu=" + std::to_string(mu) + " not set");
  KX_TRY(check_ptr(c, X, "X"));
  KX_TRY(check_ptr(c, Y, "Y"));
  if (X == Y) return fail(c, KX_ERR_INVALID, "X and Y must be distinct");
  c->cur = c->stream;
  if (c->dist == 1) {   // slab-sharded: modes 1..d-1 local, mode d through the exchange
    DistOp op;
    op.kind = 3;
    op.X = X;
    op.Y = Y;
    op.beta = beta;
    op.comp = comp;
    return dist_op_nccl(c, op);
  }
  const double* Xs[1] = {X};
  double* Ys[1] = {Y};
  const double* Ds[1] = {Y};
  return kronsum_multi(c, comp, 1, Xs, Ys, beta, Ds);
}

kx_status kx_set_dist_overlap(kx_ctx* c, int on) {
  DevGuard dg_(c);
  if (!c) return KX_ERR_INVALID;
  c->overlap = on != 0;
  return KX_OK;
}

kx_status kx_set_kronsum_mode(kx_ctx* c, int mode) {
  DevGuard dg_(c);
  if (!c) return KX_ERR_INVALID;
  if (mode != 0 && mode != 1) return fail(c, KX_ERR_INVALID, "kronsum mode must be 0 or 1");
  if (c->kronsum_mode != mode) drop_graph(c);
  c->kronsum_mode = mode;
  return KX_OK;
}

kx_status kx_phi_apply(kx_ctx* c, int comp, int ell, int stage, const double* X, double* Y,
                       double alpha, double beta) {
  DevGuard dg_(c);
  KX_TRY(need_grid(c));
  if (c->dist == 2) return fail(c, KX_ERR_INVALID, "loopback group members use kx_phi_apply_group");
  if (!c->bank_ready) return fail(c, KX_ERR_INVALID, "kx_set_tau has not been called");
  if (comp < 0 || comp >= c->ncomp) return fail(c, KX_ERR_INVALID, "comp out of range");
  auto it = c->phi.find({ell, stage});
  if (it == c->phi.end())
    return fail(c, KX_ERR_INVALID, "(ell, stage) not in this scheme's bank");
  KX_TRY(check_ptr(c, X, "X"));
  KX_TRY(check_ptr(c, Y, "Y"));
  if (X == Y) return fail(c, KX_ERR_INVALID, "X and Y must be distinct");
  c->cur = c->stream;
  const PhiStack& ps = it->second;
  if (c->dist == 1) {   // slab-sharded (kx_dist_ops.cpp)
    DistOp op;
    op.kind = 1;
    op.X = X;
    op.Y = Y;
    op.alpha = alpha;
    op.beta = beta;
    op.comp = comp;
    op.ps = &ps;
    KX_TRY(dist_op_nccl(c, op));
    c->cnt.tucker_ops += ps.nterms;
    return KX_OK;
  }
  const Group& G = c->groups[ps.group];
  // run on component `comp` only: temporarily view the context as 1 component
  const int saved_nc = c->ncomp;
  double* savedW1[MAXS];
  double* savedW2[MAXS];
  for (int s = 0; s < MAXS; ++s) {
    savedW1[s] = c->W1[s];
    savedW2[s] = c->W2[s];
  }
  Group Gc;
  Gc.nterms = G.nterms;
  Gc.first[0] = G.first[comp];
  for (int mu = 0; mu < KX_MAXD; ++mu) Gc.mid[0][mu] = G.mid[comp][mu];
  c->ncomp = 1;
  c->W1[0] = savedW1[comp];
  c->W2[0] = savedW2[comp];
  const double* Xs[1] = {X};
  double* const* ws = nullptr;
  kx_status s = group_modes(c, Gc, ps.t0, ps.nterms, Xs, 0, &ws);
  int slots[MAXSEG];
  for (int k = 0; k < ps.nterms; ++k) slots[k] = k;
  double* Bs[1] = {ps.B[comp]};
  double* Ys[1] = {Y};
  const double* Ds[1] = {Y};
  if (s == KX_OK) s = last_mode_concat(c, ws, Xs, ps.nterms, slots, Bs, Ys, alpha, beta, Ds);
  c->ncomp = saved_nc;
  for (int k = 0; k < MAXS; ++k) {
    c->W1[k] = savedW1[k];
    c->W2[k] = savedW2[k];
  }
  if (s == KX_OK) c->cnt.tucker_ops += ps.nterms;
  return s;
}

kx_status kx_step(kx_ctx* c, double t, double* const* U) {
  DevGuard dg_(c);
  (void)t;   // both models are autonomous (reading R7)
  KX_TRY(need_grid(c));
  if (!c->bank_ready) return fail(c, KX_ERR_INVALID, "kx_set_tau has not been called");
  if (!U) return fail(c, KX_ERR_INVALID, "U is NULL");
  if (c->model != 0 && c->ncomp != 2) return fail(c, KX_ERR_INVALID, "model needs 2 components");
  for (int s = 0; s < c->ncomp; ++s) {
    KX_TRY(check_ptr(c, U[s], "U[c]"));
    for (int r = 0; r < s; ++r)
      if (U[r] == U[s]) return fail(c, KX_ERR_INVALID, "U components must be distinct");
  }
  if (c->dist == 2) return fail(c, KX_ERR_INVALID, "loopback group members step through kx_step_group");
  if (c->dist == 1) return dist_step_nccl(c, U);
  return step_impl(c, U);
}

kx_status kx_set_fused_small(kx_ctx* c, int on) {
  DevGuard dg_(c);
  if (!c) return KX_ERR_INVALID;
  if ((c->fused_small != 0) != (on != 0)) drop_graph(c);
  c->fused_small = on != 0;
  return KX_OK;
}

namespace {
// nsteps steps on device tensors that passed kx_step's checks (one GPU)
kx_status steps_impl(kx_ctx* c, double* const* U, int nsteps) {
  if (nsteps > 0 && !c->nan_check && !c->profiling && fused_eligible(c)) {
    c->cur = c->stream;
    KX_TRY(enqueue_fused(c, U, nsteps));
    c->cnt.steps += nsteps;
    return KX_OK;
  }
  for (int k = 0; k < nsteps; ++k) KX_TRY(step_impl(c, U));
  return KX_OK;
}
}  // namespace

kx_status kx_step_n(kx_ctx* c, double t0, int nsteps, double* const* U) {
  DevGuard dg_(c);
  (void)t0;
  KX_TRY(need_grid(c));
  if (!c->bank_ready) return fail(c, KX_ERR_INVALID, "kx_set_tau has not been called");
  if (!U || nsteps < 0) return fail(c, KX_ERR_INVALID, "bad arguments");
  if (c->model != 0 && c->ncomp != 2) return fail(c, KX_ERR_INVALID, "model needs 2 components");
  for (int s = 0; s < c->ncomp; ++s) {
    KX_TRY(check_ptr(c, U[s], "U[c]"));
    for (int r = 0; r < s; ++r)
      if (U[r] == U[s]) return fail(c, KX_ERR_INVALID, "U components must be distinct");
  }
  if (c->dist == 2) return fail(c, KX_ERR_INVALID, "loopback group members step through kx_step_group");
  if (c->dist == 1) {
    for (int k = 0; k < nsteps; ++k) KX_TRY(dist_step_nccl(c, U));
    return KX_OK;
  }
  return steps_impl(c, U, nsteps);
}

kx_status kx_integrate_host(kx_ctx* c, double t0, int nsteps, double* const* U_host) {
  DevGuard dg_(c);
  KX_TRY(need_grid(c));
  if (c->dist) return fail(c, KX_ERR_UNSUPPORTED, "single-GPU operator on a distributed context");
  if (!c->bank_ready) return fail(c, KX_ERR_INVALID, "kx_set_tau has not been called");
  if (!U_host || nsteps < 0) return fail(c, KX_ERR_INVALID, "bad arguments");
  const size_t bytes = (size_t)c->tN * 8;
  for (int s = 0; s < c->ncomp; ++s) {
    if (!U_host[s]) return fail(c, KX_ERR_INVALID, "U_host[c] is NULL");
    if (!c->hostU[s]) {
      std::vector<double*> keep;
      KX_TRY(dalloc(c, &c->hostU[s], (size_t)c->tN, keep));
    }
    KX_CUDA(c, cudaMemcpyAsync(c->hostU[s], U_host[s], bytes, cudaMemcpyHostToDevice, c->stream));
  }
  (void)t0;
  // the last step's final stage GEMM in row chunks, each chunk's rows copied back while the
  // next one computes (final_concat); KX_TAIL_CHUNKS=1 / profiling: copy after the last step
  static const int chunks = [] {
    const char* e = getenv("KX_TAIL_CHUNKS");
    return e ? std::max(1, std::min(atoi(e), kTailMaxChunks)) : 4;
  }();
  c->tail_chunks = chunks;
  bool pinned = true;   // graph-captured copies need page-locked host buffers
  for (int s = 0; s < c->ncomp && pinned; ++s) {
    cudaPointerAttributes at{};
    pinned = cudaPointerGetAttributes(&at, U_host[s]) == cudaSuccess && at.type == cudaMemoryTypeHost;
  }
  cudaGetLastError();
  if (nsteps >= 1 && chunks > 1 && !c->profiling && pinned) {
    KX_TRY(steps_impl(c, c->hostU, nsteps - 1));
    KX_TRY(tail_step_impl(c, c->hostU, U_host));
  } else {
    KX_TRY(steps_impl(c, c->hostU, nsteps));
    for (int s = 0; s < c->ncomp; ++s)
      KX_CUDA(c, cudaMemcpyAsync(U_host[s], c->hostU[s], bytes, cudaMemcpyDeviceToHost, c->stream));
  }
  KX_CUDA(c, cudaStreamSynchronize(c->stream));
  return KX_OK;
}

kx_status kx_get_counters(const kx_ctx* c, kx_counters* out) {
  DevGuard dg_(c);
  if (!c || !out) return KX_ERR_INVALID;
  *out = c->cnt;
  return KX_OK;
}

kx_status kx_reset_counters(kx_ctx* c) {
  DevGuard dg_(c);
  if (!c) return KX_ERR_INVALID;
  c->cnt = kx_counters{};
  return KX_OK;
}

kx_status kx_sync(kx_ctx* c) {
  DevGuard dg_(c);
  if (!c) return KX_ERR_INVALID;
  KX_CUDA(c, cudaStreamSynchronize(c->stream));
  KX_CUDA(c, cudaGetLastError());
  if (c->nan_check && c->watch) {
    int mon[2];
    KX_CUDA(c, cudaMemcpy(mon, c->watch, sizeof(mon), cudaMemcpyDeviceToHost));
    if (mon[1] >= 0)
      return fail(c, KX_ERR_NUMERIC, "non-finite state after step " + std::to_string(mon[1] + 1) +
                                         " (counting since kx_set_nan_check)");
  }
  return KX_OK;
}

kx_status kx_set_nan_check(kx_ctx* c, int on) {
  DevGuard dg_(c);
  if (!c) return KX_ERR_INVALID;
  if (!c->watch) KX_CUDA(c, cudaMalloc(reinterpret_cast<void**>(&c->watch), 2 * sizeof(int)));
  const int init[2] = {0, -1};
  KX_CUDA(c, cudaMemcpy(c->watch, init, sizeof(init), cudaMemcpyHostToDevice));
  if ((c->nan_check != 0) != (on != 0)) drop_graph(c);
  c->nan_check = on != 0;
  return KX_OK;
}

kx_status kx_check_finite(kx_ctx* c, const double* X) {
  DevGuard dg_(c);
  KX_TRY(need_grid(c));
  KX_TRY(check_ptr(c, X, "X"));
  int h = 0;
  KX_CUDA(c, cudaMemsetAsync(c->flag, 0, sizeof(int), c->stream));
  KX_CUDA(c, kx::launch_check_finite(X, c->tN, c->flag, c->stream));
  KX_CUDA(c, cudaMemcpyAsync(&h, c->flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  KX_CUDA(c, cudaStreamSynchronize(c->stream));
  if (h) return fail(c, KX_ERR_NUMERIC, "non-finite values in tensor");
  return KX_OK;
}

kx_status kx_set_profiling(kx_ctx* c, int on) {
  DevGuard dg_(c);
  if (!c) return KX_ERR_INVALID;
  KX_TRY(collect_profile(c));
  c->profiling = on != 0;
  c->prof_ms[0] = c->prof_ms[1] = 0;
  c->prof_launches[0] = c->prof_launches[1] = 0;
  c->prof_flops = 0;
  c->prof_bytes = 0;
  return KX_OK;
}

kx_status kx_get_profile(kx_ctx* c, double* gemm_ms, double* other_ms, long long* gemm_launches,
                         long long* other_launches, double* gemm_flops) {
  DevGuard dg_(c);
  if (!c) return KX_ERR_INVALID;
  KX_TRY(collect_profile(c));
  if (gemm_ms) *gemm_ms = c->prof_ms[0];
  if (other_ms) *other_ms = c->prof_ms[1];
  if (gemm_launches) *gemm_launches = c->prof_launches[0];
  if (other_launches) *other_launches = c->prof_launches[1];
  if (gemm_flops) *gemm_flops = c->prof_flops;
  return KX_OK;
}

kx_status kx_get_profile_hbm(kx_ctx* c, double* other_bytes) {
  DevGuard dg_(c);
  if (!c) return KX_ERR_INVALID;
  KX_TRY(collect_profile(c));
  if (other_bytes) *other_bytes = c->prof_bytes;
  return KX_OK;
}

kx_status kx_get_phi_matrix(kx_ctx* c, int comp, int ell, int stage, int term, int mu,
                            double* out_host) {
  DevGuard dg_(c);
  KX_TRY(need_grid(c));
  if (!c->bank_ready) return fail(c, KX_ERR_INVALID, "kx_set_tau has not been called");
  if (comp < 0 || comp >= c->ncomp || mu < 1 || mu > c->d || !out_host)
    return fail(c, KX_ERR_INVALID, "bad arguments");
  auto it = c->phi.find({ell, stage});
  if (it == c->phi.end()) return fail(c, KX_ERR_INVALID, "(ell, stage) not in this bank");
  const PhiStack& ps = it->second;
  if (term < 0 || term >= ps.nterms) return fail(c, KX_ERR_INVALID, "term out of range");
  const Group& G = c->groups[ps.group];
  const int t = ps.t0 + term;
  const long long nm = c->n[mu - 1];
  KX_CUDA(c, cudaStreamSynchronize(c->stream));
  if (mu == 1) {
    KX_CUDA(c, cudaMemcpy(out_host, G.last[comp] + t * nm * nm, nm * nm * 8, cudaMemcpyDeviceToHost));
  } else if (mu == c->d) {
    KX_CUDA(c, cudaMemcpy2D(out_host, nm * 8, G.first[comp] + t * nm, (size_t)G.nterms * nm * 8,
                            nm * 8, nm, cudaMemcpyDeviceToHost));
  } else {
    KX_CUDA(c, cudaMemcpy(out_host, G.mid[comp][mu - 1] + t * nm * nm, nm * nm * 8,
                          cudaMemcpyDeviceToHost));
  }
  return KX_OK;
}

kx_status kx_set_phi_matrix(kx_ctx* c, int comp, int ell, int stage, int term, int mu,
                            const double* in_host) {
  DevGuard dg_(c);
  KX_TRY(need_grid(c));
  if (!c->bank_ready) return fail(c, KX_ERR_INVALID, "kx_set_tau has not been called");
  if (comp < 0 || comp >= c->ncomp || mu < 1 || mu > c->d || !in_host)
    return fail(c, KX_ERR_INVALID, "bad arguments");
  auto it = c->phi.find({ell, stage});
  if (it == c->phi.end()) return fail(c, KX_ERR_INVALID, "(ell, stage) not in this bank");
  const PhiStack& ps = it->second;
  if (term < 0 || term >= ps.nterms) return fail(c, KX_ERR_INVALID, "term out of range");
  const long long nm = c->n[mu - 1];
  for (long long i = 0; i < nm * nm; ++i)
    if (!std::isfinite(in_host[i])) return fail(c, KX_ERR_INVALID, "phi-matrix has non-finite entries");
  const Group& G = c->groups[ps.group];
  const int t = ps.t0 + term;   // plane index inside the group
  KX_CUDA(c, cudaStreamSynchronize(c->stream));
  drop_graph(c);
  f32_drop(c);   // the fp32 planes are re-derived from the changed bank at the next kx_step_f32
  c->cur = c->stream;
  if (mu == 1) {
    KX_CUDA(c, cudaMemcpy(G.last[comp] + t * nm * nm, in_host, nm * nm * 8, cudaMemcpyHostToDevice));
    // re-form every scaled block derived from this plane (phi stacks and stage stacks)
    const int pl = c->cplx ? 2 : 1;
    for (const BlockRecipe& r : c->recipes)
      if (r.gi == ps.group && r.comp == comp && r.t == t / pl) KX_TRY(form_block(c, c->groups, r));
  } else if (mu == c->d) {
    KX_CUDA(c, cudaMemcpy2D(G.first[comp] + t * nm, (size_t)G.nterms * nm * 8, in_host, nm * 8, nm * 8, nm,
                            cudaMemcpyHostToDevice));
  } else {
    KX_CUDA(c, cudaMemcpy(G.mid[comp][mu - 1] + t * nm * nm, in_host, nm * nm * 8, cudaMemcpyHostToDevice));
  }
  KX_CUDA(c, cudaStreamSynchronize(c->stream));
  return KX_OK;
}

kx_status kx_nccl_unique_id(void* out) {
  if (!out) return KX_ERR_INVALID;
#ifdef KX_HAVE_NCCL
  NcclApi& api = nccl();
  if (!api.ok) {
    g_create_error = api.why;
    return KX_ERR_NCCL;
  }
  ncclUniqueId id;
  if (api.GetUniqueId(&id) != ncclSuccess) return KX_ERR_NCCL;
  std::memcpy(out, &id, sizeof(id));
  return KX_OK;
#else
  g_create_error = "built without NCCL";
  return KX_ERR_UNSUPPORTED;
#endif
}

kx_status kx_create_dist(kx_ctx** out, int device, void* cuda_stream, const void* nccl_unique_id,
                         int rank, int nranks) {
  if (!out || !nccl_unique_id || nranks < 1 || rank < 0 || rank >= nranks) return KX_ERR_INVALID;
  KX_TRY(kx_create(out, device, cuda_stream));
  kx_ctx* c = *out;
#ifdef KX_HAVE_NCCL
  NcclApi& api = nccl();
  if (!api.ok) {
    g_create_error = api.why;
    kx_destroy(c);
    *out = nullptr;
    return KX_ERR_NCCL;
  }
  ncclUniqueId id;
  std::memcpy(&id, nccl_unique_id, sizeof(id));
  ncclComm_t comm = nullptr;
  ncclResult_t r = api.CommInitRank(&comm, nranks, id, rank);
  if (r != ncclSuccess) {
    g_create_error = std::string("ncclCommInitRank: ") + api.GetErrorString(r);
    kx_destroy(c);
    *out = nullptr;
    return KX_ERR_NCCL;
  }
  c->nccl_comm = comm;
  c->dist = 1;
  c->overlap = nranks > 1;   // with one rank there is nothing to hide (self-copies only)
  if (cudaStreamCreateWithFlags(&c->comm, cudaStreamNonBlocking) != cudaSuccess) c->comm = nullptr;
  for (auto& e : c->ev_term) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
  c->rank = rank;
  c->nranks = nranks;
  return KX_OK;
#else
  (void)rank;
  (void)nranks;
  kx_destroy(c);
  *out = nullptr;
  g_create_error = "built without NCCL";
  return KX_ERR_UNSUPPORTED;
#endif
}

kx_status kx_create_group(kx_ctx** ctxs, int nranks, int device, void* cuda_stream) {
  if (!ctxs || nranks < 1) return KX_ERR_INVALID;
  for (int r = 0; r < nranks; ++r) ctxs[r] = nullptr;
  for (int r = 0; r < nranks; ++r) {
    kx_status st = kx_create(&ctxs[r], device, cuda_stream);
    if (st != KX_OK) {
      for (int q = 0; q < r; ++q) kx_destroy(ctxs[q]);
      return st;
    }
    ctxs[r]->dist = 2;
    ctxs[r]->rank = r;
    ctxs[r]->nranks = nranks;
  }
  return KX_OK;
}

kx_status kx_step_group(kx_ctx* const* ctxs, int nranks, double t, double* const* U) {
  DevGuard dg_(ctxs && nranks > 0 ? ctxs[0] : nullptr);
  (void)t;
  if (!ctxs || !U || nranks < 1) return KX_ERR_INVALID;
  for (int r = 0; r < nranks; ++r) {
    kx_ctx* c = ctxs[r];
    if (!c || c->dist != 2 || c->rank != r || c->nranks != nranks) return KX_ERR_INVALID;
    KX_TRY(need_grid(c));
    if (!c->bank_ready) return fail(c, KX_ERR_INVALID, "kx_set_tau has not been called");
    if (c->scheme != ctxs[0]->scheme || c->N != ctxs[0]->N || c->ncomp != ctxs[0]->ncomp ||
        c->stream != ctxs[0]->stream)
      return fail(c, KX_ERR_INVALID, "group members differ in scheme, grid or stream");
    c->cur = c->stream;
  }
  const int nc = ctxs[0]->ncomp;
  for (int r = 0; r < nranks; ++r)
    if (ctxs[r]->p2p != ctxs[0]->p2p)
      return fail(ctxs[0], KX_ERR_INVALID, "direct peer stores are on for some members only: call kx_group_set_p2p after kx_set_tau");
  std::vector<Exchange> xs(nranks);
  for (int ph = 0; ph < dist_phases(ctxs[0]); ++ph) {
    for (int r = 0; r < nranks; ++r) KX_TRY(dist_phase(ctxs[r], U + (size_t)r * nc, ph, xs[r]));
    // loopback exchanges: device copies on the shared stream, after every rank's phase
    KX_TRY(loopback_exchange(ctxs, nranks, xs));
  }
  for (int r = 0; r < nranks; ++r) {
    KX_TRY(enqueue_watch(ctxs[r], U + (size_t)r * nc));
    ctxs[r]->cnt.steps += 1;
  }
  return KX_OK;
}

namespace {
// Checks shared by the loopback-group operators; every member must be a group rank in order
// with the same grid and stream.
kx_status group_members(kx_ctx* const* ctxs, int nranks) {
  if (!ctxs || nranks < 1) return KX_ERR_INVALID;
  for (int r = 0; r < nranks; ++r) {
    kx_ctx* c = ctxs[r];
    if (!c || c->dist != 2 || c->rank != r || c->nranks != nranks) return KX_ERR_INVALID;
    KX_TRY(need_grid(c));
    if (c->N != ctxs[0]->N || c->d != ctxs[0]->d || c->stream != ctxs[0]->stream)
      return fail(c, KX_ERR_INVALID, "group members differ in grid or stream");
    c->cur = c->stream;
  }
  return KX_OK;
}

kx_status group_op(kx_ctx* const* ctxs, int nranks, const std::vector<DistOp>& ops) {
  std::vector<Exchange> xs(nranks);
  for (int ph = 0; ph < kDistOpPhases; ++ph) {
    for (int r = 0; r < nranks; ++r) KX_TRY(dist_op_phase(ctxs[r], ops[r], ph, xs[r]));
    KX_TRY(loopback_exchange(ctxs, nranks, xs));
  }
  return KX_OK;
}
}  // namespace

kx_status kx_tucker_group(kx_ctx* const* ctxs, int nranks, const double* const* X, double* const* Y,
                          const double* const* L, double alpha, double beta) {
  DevGuard dg_(ctxs && nranks > 0 ? ctxs[0] : nullptr);
  KX_TRY(group_members(ctxs, nranks));
  if (!X || !Y || !L) return fail(ctxs[0], KX_ERR_INVALID, "X, Y or L is NULL");
  std::vector<DistOp> ops(nranks);
  for (int r = 0; r < nranks; ++r) {
    KX_TRY(check_ptr(ctxs[r], X[r], "X[r]"));
    KX_TRY(check_ptr(ctxs[r], Y[r], "Y[r]"));
    if (X[r] == Y[r]) return fail(ctxs[r], KX_ERR_INVALID, "X and Y must be distinct");
    for (int mu = 0; mu < ctxs[0]->d; ++mu) {
      KX_TRY(check_ptr(ctxs[r], L[mu], "L[mu]"));
      ops[r].L[mu] = L[mu];
    }
    ops[r].X = X[r];
    ops[r].Y = Y[r];
    ops[r].alpha = alpha;
    ops[r].beta = beta;
  }
  KX_TRY(group_op(ctxs, nranks, ops));
  for (int r = 0; r < nranks; ++r) ctxs[r]->cnt.tucker_ops += 1;
  return KX_OK;
}

kx_status kx_mode_product_group(kx_ctx* const* ctxs, int nranks, const double* const* X, double* const* Y,
                                int mu, const double* L, double alpha, double beta) {
  DevGuard dg_(ctxs && nranks > 0 ? ctxs[0] : nullptr);
  KX_TRY(group_members(ctxs, nranks));
  if (!X || !Y) return fail(ctxs[0], KX_ERR_INVALID, "X or Y is NULL");
  if (mu < 1 || mu > ctxs[0]->d) return fail(ctxs[0], KX_ERR_INVALID, "mode out of range");
  KX_TRY(check_ptr(ctxs[0], L, "L"));
  std::vector<DistOp> ops(nranks);
  for (int r = 0; r < nranks; ++r) {
    KX_TRY(check_ptr(ctxs[r], X[r], "X[r]"));
    KX_TRY(check_ptr(ctxs[r], Y[r], "Y[r]"));
    if (X[r] == Y[r]) return fail(ctxs[r], KX_ERR_INVALID, "X and Y must be distinct");
    if (mu < ctxs[r]->d) {   // local to every slab
      kx_ctx* c = ctxs[r];
      set_layout(c, false);
      const double* Xs[1] = {X[r]};
      double* Ys[1] = {Y[r]};
      const double* Ls[1] = {L};
      const double* Ds[1] = {Y[r]};
      KX_TRY(mode_product_multi(c, 1, Xs, Ys, mu, Ls, alpha, beta, Ds));
      continue;
    }
    ops[r].kind = 2;
    ops[r].X = X[r];
    ops[r].Y = Y[r];
    ops[r].L[mu - 1] = L;
    ops[r].alpha = alpha;
    ops[r].beta = beta;
  }
  if (mu < ctxs[0]->d) return KX_OK;
  return group_op(ctxs, nranks, ops);
}

kx_status kx_kronsum_group(kx_ctx* const* ctxs, int nranks, int comp, const double* const* X, double* const* Y,
                           double beta) {
  DevGuard dg_(ctxs && nranks > 0 ? ctxs[0] : nullptr);
  KX_TRY(group_members(ctxs, nranks));
  if (!X || !Y) return fail(ctxs[0], KX_ERR_INVALID, "X or Y is NULL");
  std::vector<DistOp> ops(nranks);
  for (int r = 0; r < nranks; ++r) {
    kx_ctx* c = ctxs[r];
    if (comp < 0 || comp >= c->ncomp) return fail(c, KX_ERR_INVALID, "comp out of range");
    for (int mu = 1; mu <= c->d; ++mu)
      if (!c->A_dev[comp][mu - 1])
        return fail(c, KX_ERR_INVALID, "direction matrix mu=" + std::to_string(mu) + " not set");
    KX_TRY(check_ptr(c, X[r], "X[r]"));
    KX_TRY(check_ptr(c, Y[r], "Y[r]"));
    if (X[r] == Y[r]) return fail(c, KX_ERR_INVALID, "X and Y must be distinct");
    ops[r].kind = 3;
    ops[r].X = X[r];
    ops[r].Y = Y[r];
    ops[r].beta = beta;
    ops[r].comp = comp;
  }
  return group_op(ctxs, nranks, ops);
}

kx_status kx_phi_apply_group(kx_ctx* const* ctxs, int nranks, int comp, int ell, int stage,
                             const double* const* X, double* const* Y, double alpha, double beta) {
  DevGuard dg_(ctxs && nranks > 0 ? ctxs[0] : nullptr);
  KX_TRY(group_members(ctxs, nranks));
  if (!X || !Y) return fail(ctxs[0], KX_ERR_INVALID, "X or Y is NULL");
  std::vector<DistOp> ops(nranks);
  for (int r = 0; r < nranks; ++r) {
    kx_ctx* c = ctxs[r];
    if (!c->bank_ready) return fail(c, KX_ERR_INVALID, "kx_set_tau has not been called");
    if (comp < 0 || comp >= c->ncomp) return fail(c, KX_ERR_INVALID, "comp out of range");
    auto it = c->phi.find({ell, stage});
    if (it == c->phi.end()) return fail(c, KX_ERR_INVALID, "(ell, stage) not in this scheme's bank");
    KX_TRY(check_ptr(c, X[r], "X[r]"));
    KX_TRY(check_ptr(c, Y[r], "Y[r]"));
    if (X[r] == Y[r]) return fail(c, KX_ERR_INVALID, "X and Y must be distinct");
    ops[r].kind = 1;
    ops[r].X = X[r];
    ops[r].Y = Y[r];
    ops[r].alpha = alpha;
    ops[r].beta = beta;
    ops[r].comp = comp;
    ops[r].ps = &it->second;
  }
  KX_TRY(group_op(ctxs, nranks, ops));
  for (int r = 0; r < nranks; ++r) ctxs[r]->cnt.tucker_ops += ops[r].ps->nterms;
  return KX_OK;
}

kx_status kx_group_set_p2p(kx_ctx* const* ctxs, int nranks, int on) {
  DevGuard dg_(ctxs && nranks > 0 ? ctxs[0] : nullptr);
  if (!ctxs || nranks < 1 || nranks > kx::kMaxPeers) return KX_ERR_INVALID;
  for (int r = 0; r < nranks; ++r) {
    kx_ctx* c = ctxs[r];
    if (!c || c->dist != 2 || c->rank != r || c->nranks != nranks) return KX_ERR_INVALID;
    if (on && !c->bank_ready) return fail(c, KX_ERR_INVALID, "kx_set_tau has not been called");
  }
  for (int r = 0; r < nranks; ++r) {
    kx_ctx* c = ctxs[r];
    p2p_close(c);
    if (!on) continue;
    for (int q = 0; q < nranks; ++q)
      for (int s = 0; s < c->ncomp; ++s) {
        c->peerRA[q][s] = ctxs[q]->RA[s];
        c->peerFB[q][s] = ctxs[q]->F_B[s];
        c->peerDB[q][s] = ctxs[q]->D_B[s];
        c->peerHlo[q][s] = ctxs[q]->halo_lo[s];
        c->peerHhi[q][s] = ctxs[q]->halo_hi[s];
      }
    c->p2p = 1;
  }
  return KX_OK;
}

// Receive buffers of this rank as CUDA IPC handles, in the fixed order (RA, F_B, D_B,
// halo_lo, halo_hi) x component.
static const int kIpcBufs = 5;
static double** ipc_slot(kx_ctx* c, int k, int s) {
  switch (k) {
    case 0: return &c->RA[s];
    case 1: return &c->F_B[s];
    case 2: return &c->D_B[s];
    case 3: return &c->halo_lo[s];
    default: return &c->halo_hi[s];
  }
}

kx_status kx_dist_ipc_export(kx_ctx* c, void* blob, size_t cap, size_t* len) {
  DevGuard dg_(c);
  if (!c || !len) return KX_ERR_INVALID;
  if (c->dist != 1) return fail(c, KX_ERR_INVALID, "not an NCCL-distributed context");
  if (!c->bank_ready) return fail(c, KX_ERR_INVALID, "kx_set_tau has not been called");
  const size_t need = (size_t)kIpcBufs * c->ncomp * sizeof(cudaIpcMemHandle_t);
  *len = need;
  if (!blob) return KX_OK;
  if (cap < need) return fail(c, KX_ERR_INVALID, "blob too small");
  auto* h = static_cast<cudaIpcMemHandle_t*>(blob);
  for (int k = 0; k < kIpcBufs; ++k)
    for (int s = 0; s < c->ncomp; ++s)
      KX_CUDA(c, cudaIpcGetMemHandle(&h[k * c->ncomp + s], *ipc_slot(c, k, s)));
  return KX_OK;
}

kx_status kx_dist_ipc_import(kx_ctx* c, const void* blobs, size_t len_each) {
  DevGuard dg_(c);
  if (!c || !blobs) return KX_ERR_INVALID;
  if (c->dist != 1) return fail(c, KX_ERR_INVALID, "not an NCCL-distributed context");
  if (c->nranks > kx::kMaxPeers) return fail(c, KX_ERR_UNSUPPORTED, "more ranks than kMaxPeers");
  if (!c->bank_ready) return fail(c, KX_ERR_INVALID, "kx_set_tau has not been called");
  const size_t need = (size_t)kIpcBufs * c->ncomp * sizeof(cudaIpcMemHandle_t);
  if (len_each != need) return fail(c, KX_ERR_INVALID, "blob size mismatch");
  p2p_close(c);
  for (int q = 0; q < c->nranks; ++q) {
    const auto* h = reinterpret_cast<const cudaIpcMemHandle_t*>(static_cast<const char*>(blobs) + q * need);
    for (int k = 0; k < kIpcBufs; ++k)
      for (int s = 0; s < c->ncomp; ++s) {
        double* p = nullptr;
        if (q == c->rank) {
          p = *ipc_slot(c, k, s);
        } else {
          void* m = nullptr;
          cudaError_t e = cudaIpcOpenMemHandle(&m, h[k * c->ncomp + s], cudaIpcMemLazyEnablePeerAccess);
          if (e != cudaSuccess) {
            cudaGetLastError();
            p2p_close(c);
            return fail(c, KX_ERR_CUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
          }
          c->ipc_open.push_back(m);
          p = static_cast<double*>(m);
        }
        double* (*dst)[MAXS] = k == 0 ? c->peerRA : k == 1 ? c->peerFB : k == 2 ? c->peerDB
                             : k == 3 ? c->peerHlo : c->peerHhi;
        dst[q][s] = p;
      }
  }
  c->p2p = 1;
  return KX_OK;
}

kx_status kx_scheme_coefficients_cplx(int ell, int d, int* nterms, double* eta_re, double* eta_im,
                                      int* inner_ell, double* alpha_re, double* alpha_im) {
  if (!nterms || !eta_re || !eta_im || !inner_ell || !alpha_re || !alpha_im) return KX_ERR_INVALID;
  if (d < 1 || d > KX_MAXD) return KX_ERR_INVALID;
  const int t = kx::scheme_terms_cplx(ell, d, eta_re, eta_im, inner_ell, alpha_re, alpha_im);
  *nterms = t;
  return t ? KX_OK : KX_ERR_UNSUPPORTED;
}

kx_status kx_scheme_coefficients(kx_scheme scheme, int ell, int d, int* nterms, double* eta,
                                 int* inner_ell, double* alpha) {
  if (!nterms || !eta || !inner_ell || !alpha) return KX_ERR_INVALID;
  if (d < 1 || d > KX_MAXD) return KX_ERR_INVALID;
  const int t = kx::scheme_terms(scheme, ell, d, eta, inner_ell, alpha);
  *nterms = t;
  return t ? KX_OK : KX_ERR_UNSUPPORTED;
}

}  // extern "C"

