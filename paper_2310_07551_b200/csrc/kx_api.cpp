// C ABI (include/kx.h): context, validation, phi-bank formation on the device, the ETD
// schedules, CUDA-graph capture, counters and profiling.  All arithmetic runs in the CUDA
// kernels of gemm.cu / pointwise.cu; this file only plans and enqueues launches.
#include "kx.h"

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "kx_internal.h"
#ifdef KX_HAVE_NCCL
#include <nccl.h>
#endif

using kx::GemmArgs;
using kx::MAXS;
using kx::MAXSEG;

namespace {

thread_local std::string g_create_error;

constexpr int KX_MAXD = 6;
constexpr int TAYLOR_K = 18;       // Horner degree of the phi_2 Taylor base (theta = 1)
constexpr double THETA = 1.0;      // ||X||_1 bound after scaling (reading R8)

// ------------------------------------------------------------------------------------------
// Bank layout (per component c):
//   group g (an input tensor: F, D2, D3 for exprk3ds; F, D for ETD2RKDS) with TG terms:
//     first[c]   : stacked [P_1{d}; ...; P_TG{d}]  column-major (TG*n_d) x n_d (d >= 2)
//     mid[c][mu] : TG column-major n_mu x n_mu matrices, 1 < mu < d
//     last[c]    : TG column-major n_1 x n_1 matrices (unscaled)
//   phi stacks (ell, stage): row-major (T*n_1) x n_1, block t = eta_t * P_t{1} (col-major buf)
//   stage stacks (U2, U3, U+): row-major (nseg*n_1) x n_1, block k = scale_k * P{1}
// ------------------------------------------------------------------------------------------
struct Group {
  int nterms = 0;
  int slot0 = 0;                        // first workspace slot of its intermediates
  std::vector<int> chain;               // chain id per (term, mu): chain[t*d + mu-1]
  std::vector<int> level;               // 0: 1/3, 1: 2/3, 2: 1 (ETD3) / 2 (ETD2)
  std::vector<int> inner;               // l_t
  double* first[MAXS] = {};
  double* mid[MAXS][KX_MAXD] = {};
  double* last[MAXS] = {};
};

struct PhiStack {            // for kx_phi_apply
  int group = -1, t0 = 0, nterms = 0;
  double* B[MAXS] = {};
};

struct Stage {               // last-mode concatenated-K stage combination
  int nseg = 0;
  int slot[MAXSEG] = {};
  double* B[MAXS] = {};
};

struct Chain {               // one phi-matrix family phi_{0,1,2}(sigma * A^c_mu)
  int c = 0, mu = 0;
  double sigma = 0.0;          // real part of the scale
  double sigma_im = 0.0;       // imaginary part (complex schemes: built on the real 2n x 2n
  int q = 0;                   //  embedding [[Re, -Im], [Im, Re]] of sigma A)
};

}  // namespace

struct kx_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;      // user stream
  cudaStream_t cap = nullptr;         // internal capture stream
  cudaStream_t cur = nullptr;         // stream launches go to
  std::string err;

  int d = 0, ncomp = 0;
  long long n[KX_MAXD] = {};     // global extents (matrix sizes)
  long long N = 0;
  long long tn[KX_MAXD] = {};    // extents of the local tensors the current launches act on
  long long tN = 0;              // (= n, N on one GPU; a slab layout on a distributed context)
  std::vector<std::vector<std::vector<double>>> A_host;   // [c][mu]
  std::vector<std::vector<double*>> A_dev;                 // [c][mu]
  std::vector<std::vector<double*>> A_tri;                 // [c][mu]: lo|di|up (3 n) or null
  int kronsum_mode = 0;   // 0 auto (tridiagonal stencil when every A is tridiagonal), 1 dense

  int model = 0;
  double params[8] = {};

  // bank
  int scheme = 0;
  double tau = 0.0;
  bool bank_ready = false;
  long long bank_version = 0;
  int T = 0;                      // terms of the split scheme
  bool cplx = false;              // complex split (Table 2): terms stored as (Re, Im) planes
  std::vector<Group> groups;
  std::map<std::pair<int, int>, PhiStack> phi;   // (ell, stage)
  Stage stages[3];
  int nstages = 0;
  std::vector<double*> bank_allocs;
  int nslots = 0;

  // workspaces
  double* tmp1 = nullptr;
  double* tmp2 = nullptr;
  double* G[MAXS] = {};
  double* F[MAXS] = {};
  double* D[MAXS] = {};
  double* Us[MAXS] = {};
  double* W1[MAXS] = {};
  double* W2[MAXS] = {};
  std::vector<double*> ws_allocs;
  double* hostU[MAXS] = {};
  int* flag = nullptr;
  double* sk_ws = nullptr;      // stream-K partial tiles (kx::kSkSlots x 128 x 128)
  int* sk_flags = nullptr;      // stream-K flags (zero between launches)

  kx_counters cnt{};

  // CUDA graph of one step
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  double* graph_U[MAXS] = {};
  long long graph_version = -1;
  bool graph_prof = false;
  kx_counters step_delta{};

  // profiling
  // distributed slab decomposition along i_d: dist = 1 NCCL rank,
  // dist = 2 member of an in-process loopback group (exchanges are device copies)
  int dist = 0, rank = 0, nranks = 1;
  void* nccl_comm = nullptr;
  // f2: term-by-term exchange overlapped with the remaining terms' mode products (NCCL ranks)
  int overlap = 1;
  cudaStream_t comm = nullptr;
  cudaEvent_t ev_term[64] = {};
  cudaEvent_t ev_join = nullptr;
  long long nA[KX_MAXD] = {};    // local extents, layout A: i_d sharded (n_d / P)
  long long nB[KX_MAXD] = {};    // local extents, layout B: i_1 sharded (n_1 / P)
  long long Nloc = 0;
  double* RA[MAXS] = {};         // received term slots, peer-major layout A (nslots x Nloc)
  double* T1G_pack[MAXS] = {};   // (U x_1 A_1 + G), peer-packed
  double* U_pack[MAXS] = {};
  double* T1G_B[MAXS] = {};
  double* U_B[MAXS] = {};
  double* F_B[MAXS] = {};
  double* D_pack[MAXS] = {};
  double* D_B[MAXS] = {};

  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  struct Rec { int cls; int e0, e1; double flops; };
  std::vector<Rec> recs;        // eager launches awaiting collection
  std::vector<Rec> graph_recs;  // event pairs captured inside the step graph
  int graph_ev_end = 0;         // pool indices [0, graph_ev_end) belong to the graph
  int ev_used = 0;
  double prof_ms[2] = {0, 0};
  long long prof_launches[2] = {0, 0};
  double prof_flops = 0;
};

namespace {

kx_status fail(kx_ctx* c, kx_status s, const std::string& m) {
  if (c) c->err = m;
  return s;
}

#define KX_CUDA(ctx, expr)                                                                \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(ctx, KX_ERR_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                        " at " #expr);                                    \
  } while (0)

#define KX_TRY(expr)               \
  do {                             \
    kx_status s_ = (expr);         \
    if (s_ != KX_OK) return s_;    \
  } while (0)

// ---------------------------------------------------------------- launch wrappers ---------
// Record an event on the current launch stream; while capturing a graph the record becomes an
// event-record node (cudaEventRecordExternal) so that it fires on every replay.
cudaError_t record(kx_ctx* c, cudaEvent_t e) {
  return c->cur == c->cap ? cudaEventRecordWithFlags(e, c->cur, cudaEventRecordExternal)
                          : cudaEventRecord(e, c->cur);
}

cudaEvent_t pool_event(kx_ctx* c, int idx) {
  while ((int)c->ev_pool.size() <= idx) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[idx];
}

kx_status collect_profile(kx_ctx* c);

kx_status run_gemm(kx_ctx* c, const GemmArgs& g_in) {
  GemmArgs g = g_in;
  g.sk_ws = c->sk_ws;
  g.sk_flags = c->sk_flags;
  const double fl = kx::gemm_flops(g);
  if (c->profiling && c->cur == c->stream && c->ev_used > 20000) KX_TRY(collect_profile(c));
  int e0 = -1;
  if (c->profiling) {
    e0 = c->ev_used;
    c->ev_used += 2;
    KX_CUDA(c, record(c, pool_event(c, e0)));
  }
  KX_CUDA(c, kx::launch_gemm(g, c->cur));
  if (c->profiling) {
    KX_CUDA(c, record(c, pool_event(c, e0 + 1)));
    c->recs.push_back({0, e0, e0 + 1, fl});
  }
  c->cnt.gemm_launches += 1;
  c->cnt.mode_product_flops += fl;
  return KX_OK;
}

template <class F>
kx_status run_other(kx_ctx* c, F&& launch) {
  int e0 = -1;
  if (c->profiling) {
    e0 = c->ev_used;
    c->ev_used += 2;
    KX_CUDA(c, record(c, pool_event(c, e0)));
  }
  KX_CUDA(c, launch());
  if (c->profiling) {
    KX_CUDA(c, record(c, pool_event(c, e0 + 1)));
    c->recs.push_back({1, e0, e0 + 1, 0.0});
  }
  c->cnt.other_launches += 1;
  return KX_OK;
}

kx_status dalloc(kx_ctx* c, double** p, size_t count, std::vector<double*>& owner) {
  *p = nullptr;
  if (count == 0) return KX_OK;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(double));
  if (e != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    return fail(c, KX_ERR_NOMEM, "device allocation of " + std::to_string(count * 8) +
                                     " bytes failed: " + cudaGetErrorString(e));
  }
  owner.push_back(*p);
  return KX_OK;
}

void free_list(std::vector<double*>& v) {
  for (double* p : v) cudaFree(p);
  v.clear();
}

void drop_graph(kx_ctx* c) {
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->graph) cudaGraphDestroy(c->graph);
  c->gexec = nullptr;
  c->graph = nullptr;
  c->graph_version = -1;
  c->graph_recs.clear();
  c->graph_ev_end = 0;
}

void drop_bank(kx_ctx* c) {
  drop_graph(c);
  free_list(c->bank_allocs);
  free_list(c->ws_allocs);
  c->groups.clear();
  c->phi.clear();
  for (auto& s : c->stages) s = Stage{};
  c->nstages = 0;
  c->bank_ready = false;
  for (int s = 0; s < MAXS; ++s) {
    c->G[s] = c->F[s] = c->D[s] = c->Us[s] = c->W1[s] = c->W2[s] = nullptr;
    c->RA[s] = c->T1G_pack[s] = c->U_pack[s] = c->T1G_B[s] = c->U_B[s] = c->F_B[s] = nullptr;
    c->D_pack[s] = c->D_B[s] = nullptr;
  }
}

long long prod_range(const kx_ctx* c, int lo, int hi) {   // prod_{lo <= mu <= hi} n_mu (1-based)
  long long p = 1;
  for (int mu = lo; mu <= hi; ++mu) p *= c->tn[mu - 1];
  return p;
}

kx_status need_grid(kx_ctx* c) {
  if (!c) return KX_ERR_INVALID;
  if (c->d == 0) return fail(c, KX_ERR_INVALID, "kx_set_grid has not been called");
  return KX_OK;
}

// ---------------------------------------------------------------- mode products -----------
// One mu-mode product for ns components: Y_s = alpha * (X_s x_mu L_s) + beta * Dd_s.
kx_status mode_product_multi(kx_ctx* c, int ns, const double* const* X, double* const* Y,
                             int mu, const double* const* L, double alpha, double beta,
                             const double* const* Dd) {
  GemmArgs g;
  const long long nm = c->tn[mu - 1];
  const long long R = prod_range(c, 1, mu - 1);     // prod_{nu<mu}
  const long long Bt = prod_range(c, mu + 1, c->d); // prod_{nu>mu}
  g.ns = ns;
  g.alpha = alpha;
  g.beta = beta;
  if (mu == 1) {
    // Y_r = X_r * L^T : A = X (ROW, k contiguous), B = L column-major buffer (row-major L^T)
    g.arow = true;
    g.M = (int)(c->tN / nm);
    g.N = (int)nm;
    g.kseg = (int)nm;
    g.nseg = 1;
    g.lda = nm;
    g.ldb = nm;
    g.ldc = nm;
    g.ldd = nm;
    for (int s = 0; s < ns; ++s) {
      g.A[s] = X[s];
      g.B[s] = L[s];
      g.C[s] = Y[s];
      g.D[s] = (Dd && beta != 0.0) ? Dd[s] : nullptr;
    }
  } else {
    // Y_b = L * X_b for b < prod_{nu>mu}: A = L (COL), B = X_b row-major nm x R
    g.arow = false;
    g.M = (int)nm;
    g.N = (int)R;
    g.kseg = (int)nm;
    g.nseg = 1;
    g.lda = nm;
    g.ldb = R;
    g.ldc = R;
    g.ldd = R;
    g.nb = (int)Bt;
    g.sB_b = g.sC_b = g.sD_b = nm * R;
    for (int s = 0; s < ns; ++s) {
      g.A[s] = L[s];
      g.B[s] = X[s];
      g.C[s] = Y[s];
      g.D[s] = (Dd && beta != 0.0) ? Dd[s] : nullptr;
    }
  }
  KX_TRY(run_gemm(c, g));
  c->cnt.mode_products += ns;
  return KX_OK;
}

// ---------------------------------------------------------------- Kronecker sum ------------
// Y_s = K_{comp0+s} X_s + beta * Dd_s  for s < ns   (eq:kronsumv: sum_mu X x_mu A_mu)
bool all_tridiag(const kx_ctx* c, int comp0, int ns) {
  if (c->kronsum_mode != 0) return false;
  for (int s = 0; s < ns; ++s)
    for (int mu = 0; mu < c->d; ++mu)
      if (!c->A_tri[comp0 + s][mu]) return false;
  return true;
}

kx_status kronsum_multi(kx_ctx* c, int comp0, int ns, const double* const* X, double* const* Y,
                        double beta, const double* const* Dd) {
  if (all_tridiag(c, comp0, ns)) {
    // every A_mu is tridiagonal: the dense mode products would only add exact zeros
    kx::StencilArgs a;
    a.d = c->d;
    a.ns = ns;
    a.N = c->tN;
    a.beta = beta;
    for (int mu = 0; mu < c->d; ++mu) a.n[mu] = c->tn[mu];
    for (int s = 0; s < ns; ++s) {
      a.X[s] = X[s];
      a.Y[s] = Y[s];
      a.Dd[s] = (Dd && beta != 0.0) ? Dd[s] : nullptr;
      for (int mu = 0; mu < c->d; ++mu) {
        const double* t = c->A_tri[comp0 + s][mu];
        const long long n = c->tn[mu];
        a.lo[s][mu] = t;
        a.di[s][mu] = t + n;
        a.up[s][mu] = t + 2 * n;
      }
    }
    KX_TRY(run_other(c, [&] { return kx::launch_kronsum_tridiag(a, c->cur); }));
    c->cnt.mode_products += (long long)ns * c->d;
    c->cnt.kronsum_actions += ns;
    return KX_OK;
  }
  const double* L[MAXS];
  for (int mu = c->d; mu >= 1; --mu) {
    for (int s = 0; s < ns; ++s) L[s] = c->A_dev[comp0 + s][mu - 1];
    if (mu == c->d) {
      KX_TRY(mode_product_multi(c, ns, X, Y, mu, L, 1.0, beta, Dd));
    } else {
      const double* Yc[MAXS];
      for (int s = 0; s < ns; ++s) Yc[s] = Y[s];
      KX_TRY(mode_product_multi(c, ns, X, Y, mu, L, 1.0, 1.0, Yc));
    }
  }
  c->cnt.kronsum_actions += ns;
  return KX_OK;
}

// ---------------------------------------------------------------- split application -------
// First (mu = d, concatenated M) and middle (1 < mu < d, batched over terms) modes of terms
// [t0, t0+nt) of group gi applied to inputs X[s]; results land in slots [slot, slot+nt) of
// the returned workspace (W1 or W2).
kx_status group_modes(kx_ctx* c, const Group& G, int t0, int nt, const double* const* X,
                      int slot, double* const** out_ws) {
  const int d = c->d;
  const long long N = c->tN;
  const int ns = c->ncomp;
  *out_ws = nullptr;
  if (d == 1) return KX_OK;
  {
    const long long nd = c->tn[d - 1];
    const long long R = N / nd;
    GemmArgs g;
    g.arow = false;
    g.M = (int)(nt * nd);
    g.N = (int)R;
    g.kseg = (int)nd;
    g.lda = (long long)G.nterms * nd;
    g.ldb = R;
    g.ldc = R;
    g.ns = ns;
    for (int s = 0; s < ns; ++s) {
      g.A[s] = G.first[s] + t0 * nd;
      g.B[s] = X[s];
      g.C[s] = c->W1[s] + (long long)slot * N;
    }
    KX_TRY(run_gemm(c, g));
  }
  double** cur = c->W1;
  double** nxt = c->W2;
  for (int mu = d - 1; mu >= 2 && c->cplx; --mu) {
    // complex terms (Re, Im planes): W' = P W  ->  Re = P_re W_re - P_im W_im,
    // Im = P_re W_im + P_im W_re; four launches batched over terms, slabs and components
    const long long nm = c->tn[mu - 1];
    const long long R = prod_range(c, 1, mu - 1);
    const long long Bt = prod_range(c, mu + 1, d);
    const int pa[4] = {0, 1, 0, 1};   // plane of P
    const int pw[4] = {0, 1, 1, 0};   // plane of W read
    const int po[4] = {0, 0, 1, 1};   // plane of W' written
    const double al[4] = {1.0, -1.0, 1.0, 1.0};
    for (int k = 0; k < 4; ++k) {
      GemmArgs g;
      g.arow = false;
      g.M = (int)nm;
      g.N = (int)R;
      g.kseg = (int)nm;
      g.lda = nm;
      g.ldb = R;
      g.ldc = R;
      g.ldd = R;
      g.ns = ns;
      g.nt = nt / 2;
      g.nb = (int)Bt;
      g.sA_t = 2 * nm * nm;
      g.sB_t = g.sC_t = g.sD_t = 2 * N;
      g.sB_b = g.sC_b = g.sD_b = nm * R;
      g.alpha = al[k];
      g.beta = (k == 1 || k == 3) ? 1.0 : 0.0;
      for (int s = 0; s < ns; ++s) {
        g.A[s] = G.mid[s][mu - 1] + (t0 + pa[k]) * nm * nm;
        g.B[s] = cur[s] + (long long)(slot + pw[k]) * N;
        g.C[s] = nxt[s] + (long long)(slot + po[k]) * N;
        g.D[s] = g.beta != 0.0 ? g.C[s] : nullptr;
      }
      KX_TRY(run_gemm(c, g));
    }
    std::swap(cur, nxt);
  }
  for (int mu = d - 1; mu >= 2 && !c->cplx; --mu) {
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
    g.ns = ns;
    g.nt = nt;
    g.nb = (int)Bt;
    g.sA_t = nm * nm;
    g.sB_t = g.sC_t = N;
    g.sB_b = g.sC_b = nm * R;
    for (int s = 0; s < ns; ++s) {
      g.A[s] = G.mid[s][mu - 1] + t0 * nm * nm;
      g.B[s] = cur[s] + (long long)slot * N;
      g.C[s] = nxt[s] + (long long)slot * N;
    }
    KX_TRY(run_gemm(c, g));
    std::swap(cur, nxt);
  }
  c->cnt.mode_products += (long long)ns * nt * (d - 1);
  *out_ws = cur;
  return KX_OK;
}

// Last mode (mu = 1) with concatenated K over `nseg` slots of ws (or over the single input
// tensor src when d == 1):  Y_s = alpha * sum_k Wslot_k x_1 Bblock_k + beta * Dd_s.
kx_status last_mode_concat(kx_ctx* c, double* const* ws, const double* const* src, int nseg,
                           const int* slots, double* const* B, double* const* Y, double alpha,
                           double beta, const double* const* Dd) {
  const long long n1 = c->tn[0];
  GemmArgs g;
  g.arow = true;
  g.M = (int)(c->tN / n1);
  g.N = (int)n1;
  g.kseg = (int)n1;
  g.nseg = nseg;
  g.lda = n1;
  g.ldb = n1;
  g.ldc = n1;
  g.ldd = n1;
  g.ns = c->ncomp;
  g.alpha = alpha;
  g.beta = beta;
  for (int k = 0; k < nseg; ++k) g.seg_off[k] = ws ? (long long)slots[k] * c->tN : 0;
  for (int s = 0; s < c->ncomp; ++s) {
    g.A[s] = ws ? ws[s] : src[s];
    g.B[s] = B[s];
    g.C[s] = Y[s];
    g.D[s] = (Dd && beta != 0.0) ? Dd[s] : nullptr;
  }
  KX_TRY(run_gemm(c, g));
  c->cnt.mode_products += (long long)c->ncomp * nseg;
  return KX_OK;
}

kx_status nonlin(kx_ctx* c, int mode, const double* const* u, double* const* out) {
  kx::PointwiseArgs a;
  a.model = c->model;
  a.ncomp = c->ncomp;
  a.N = c->tN;
  for (int s = 0; s < c->ncomp; ++s) {
    a.u[s] = u[s];
    a.out[s] = out[s];
    a.G[s] = c->G[s];
  }
  for (int i = 0; i < 8; ++i) a.p[i] = c->params[i];
  return run_other(c, [&] { return kx::launch_nonlinearity(a, mode, c->cur); });
}

// ---------------------------------------------------------------- time steps --------------
// exprk3ds_real, Algorithm 1 (d = 2) / Algorithm 2 (d > 2), P:2229-2264 / P:2302-2342,
// fused schedule of SURVEY.md §3 CS2.  Groups: 0 = F (3T terms), 1 = D2 (T), 2 = D3 (T).
kx_status enqueue_step_etd3(kx_ctx* c, double* const* U) {
  const int ns = c->ncomp;
  // G = g(t, U); F = K(U, A) + G
  KX_TRY(nonlin(c, 0, U, c->G));
  KX_TRY(kronsum_multi(c, 0, ns, U, c->F, 1.0, c->G));
  // all 3T first/middle modes on F at once
  double* const* ws = nullptr;
  KX_TRY(group_modes(c, c->groups[0], 0, c->groups[0].nterms, c->F, c->groups[0].slot0, &ws));
  // U2 = U + tau/3 S_1^{tau/3}[F]
  KX_TRY(last_mode_concat(c, ws, c->F, c->stages[0].nseg, c->stages[0].slot, c->stages[0].B,
                          c->Us, 1.0, 1.0, U));
  // D2 = g(U2) - G; U3 = U + 2tau/3 S_1^{2tau/3}[F] + 4tau/3 S_2^{2tau/3}[D2]
  KX_TRY(nonlin(c, 1, c->Us, c->D));
  KX_TRY(group_modes(c, c->groups[1], 0, c->groups[1].nterms, c->D, c->groups[1].slot0, &ws));
  KX_TRY(last_mode_concat(c, ws, nullptr, c->stages[1].nseg, c->stages[1].slot, c->stages[1].B,
                          c->Us, 1.0, 1.0, U));
  // D3 = g(U3) - G; U+ = U + tau S_1^tau[F] + 3tau/2 S_2^tau[D3]
  KX_TRY(nonlin(c, 1, c->Us, c->D));
  KX_TRY(group_modes(c, c->groups[2], 0, c->groups[2].nterms, c->D, c->groups[2].slot0, &ws));
  KX_TRY(last_mode_concat(c, ws, nullptr, c->stages[2].nseg, c->stages[2].slot, c->stages[2].B,
                          U, 1.0, 1.0, U));
  c->cnt.tucker_ops += (long long)ns * 5 * c->T;   // 3T on F, T on D2, T on D3
  return KX_OK;
}

// ETD2RKDS (eq:ETD2RK with eq:phisplit).  Groups: 0 = F (phi_1), 1 = D (phi_2).
kx_status enqueue_step_etd2(kx_ctx* c, double* const* U) {
  const int ns = c->ncomp;
  KX_TRY(nonlin(c, 0, U, c->G));
  KX_TRY(kronsum_multi(c, 0, ns, U, c->F, 1.0, c->G));
  double* const* ws = nullptr;
  KX_TRY(group_modes(c, c->groups[0], 0, 1, c->F, c->groups[0].slot0, &ws));
  KX_TRY(last_mode_concat(c, ws, c->F, 1, c->stages[0].slot, c->stages[0].B, c->Us, 1.0, 1.0, U));
  KX_TRY(nonlin(c, 1, c->Us, c->D));
  KX_TRY(group_modes(c, c->groups[1], 0, 1, c->D, c->groups[1].slot0, &ws));
  KX_TRY(last_mode_concat(c, ws, c->D, 1, c->stages[1].slot, c->stages[1].B, U, 1.0, 1.0, c->Us));
  c->cnt.tucker_ops += (long long)ns * 2;
  return KX_OK;
}

kx_status enqueue_step(kx_ctx* c, double* const* U) {
  if (c->scheme == KX_ETD3RKDS_REAL || c->scheme == KX_ETD3RKDS_CPLX) return enqueue_step_etd3(c, U);
  return enqueue_step_etd2(c, U);
}

// ---------------------------------------------------------------- phi bank ----------------
double norm_bound(const std::vector<double>& A, long long n) {
  double n1 = 0, ninf = 0;
  for (long long j = 0; j < n; ++j) {
    double s = 0;
    for (long long i = 0; i < n; ++i) s += std::fabs(A[i + j * n]);
    n1 = std::max(n1, s);
  }
  for (long long i = 0; i < n; ++i) {
    double s = 0;
    for (long long j = 0; j < n; ++j) s += std::fabs(A[i + j * n]);
    ninf = std::max(ninf, s);
  }
  return std::max(n1, ninf);
}

// Batched row-major GEMM over `cnt` chains (stride n^2): C = alpha A B + beta D + gamma E + diag I
kx_status chain_gemm(kx_ctx* c, long long n, int cnt, const double* A, const double* B, double* C,
                     double alpha, const double* D, double beta, const double* E, double gamma,
                     double diag) {
  if (cnt <= 0) return KX_OK;
  GemmArgs g;
  g.arow = true;
  g.M = (int)n;
  g.N = (int)n;
  g.kseg = (int)n;
  g.lda = g.ldb = g.ldc = g.ldd = g.lde = n;
  g.nb = cnt;
  g.sA_b = g.sB_b = g.sC_b = g.sD_b = g.sE_b = n * n;
  g.A[0] = A;
  g.B[0] = B;
  g.C[0] = C;
  g.D[0] = D;
  g.E[0] = E;
  g.alpha = alpha;
  g.beta = beta;
  g.gamma = gamma;
  g.diag = diag;
  return run_gemm(c, g);
}

// Forms phi_0..2 of sigma_k * M_k for chains sharing extent n, all on the device.  M_k is the
// column-major A^c_mu buffer read row-major (= A^T): every product below is a function of the
// same matrix, so phi(sigma A^T) computed row-major IS phi(sigma A) column-major.
// Taylor base (Horner, degree TAYLOR_K) at X = sigma 2^{-q} M with ||X|| <= THETA, then q
// doublings  E' = E E,  P1' = (P1 E + P1)/2,  P2' = (E P2 + P2 + P1)/4  (SW09 modified
// squaring; derived from e^{2Y} = e^Y e^Y).  For ETD3 banks one more doubling gives the 2/3
// level and the addition formula (a = 2/3, b = 1/3 of the step)
//   P1(1) = 2/3 P1(2/3) E(1/3) + 1/3 P1(1/3)
//   P2(1) = 1/9 E(2/3) P2(1/3) + 4/9 P2(2/3) + 2/9 P1(2/3)
// gives level 1.  Outputs: out[k][level][l-1] device pointers (level 0..2), l in {1,2}.
struct ChainOut {
  double* p[3][2] = {};
};

kx_status build_chains(kx_ctx* c, long long n_a, bool emb, std::vector<Chain>& ch, bool thirds,
                       std::vector<ChainOut>& out, std::vector<double*>& scratch) {
  const int C = (int)ch.size();
  if (C == 0) return KX_OK;
  const long long n = emb ? 2 * n_a : n_a;   // matrix size of the chain arithmetic
  const long long n2 = n * n;
  // sort by q descending (active chains in a doubling round form a prefix)
  std::vector<int> order(C);
  for (int i = 0; i < C; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return ch[a].q > ch[b].q; });
  auto alloc = [&](double** p) { return dalloc(c, p, (size_t)C * n2, scratch); };
  double *X, *H0, *H1, *SE, *SP1, *SP2, *TE, *TP1, *TP2, *O1 = nullptr, *O2 = nullptr;
  KX_TRY(alloc(&X));
  KX_TRY(alloc(&H0));
  KX_TRY(alloc(&H1));
  KX_TRY(alloc(&SE));
  KX_TRY(alloc(&SP1));
  KX_TRY(alloc(&SP2));
  KX_TRY(alloc(&TE));
  KX_TRY(alloc(&TP1));
  KX_TRY(alloc(&TP2));
  if (thirds) {
    KX_TRY(alloc(&O1));
    KX_TRY(alloc(&O2));
  }
  // X_k = sigma_k 2^{-q_k} A  (position k in sorted order)
  for (int k = 0; k < C; ++k) {
    const Chain& h = ch[order[k]];
    const double sre = std::ldexp(h.sigma, -h.q), sim = std::ldexp(h.sigma_im, -h.q);
    const double* Ad = c->A_dev[h.c][h.mu - 1];
    double* Xk = X + k * n2;
    if (!emb) {
      KX_TRY(run_other(c, [&] { return kx::launch_scale(Xk, Ad, sre, n2, c->cur); }));
    } else {
      // row-major [[sre A^T, -sim A^T], [sim A^T, sre A^T]]  (A's column-major buffer = A^T)
      const long long m = n_a;
      KX_TRY(run_other(c, [&] { return kx::launch_copy2d(Xk, n, 0, Ad, m, 0, m, m, 1, sre, c->cur); }));
      KX_TRY(run_other(c, [&] { return kx::launch_copy2d(Xk + m, n, 0, Ad, m, 0, m, m, 1, -sim, c->cur); }));
      KX_TRY(run_other(c, [&] { return kx::launch_copy2d(Xk + m * n, n, 0, Ad, m, 0, m, m, 1, sim, c->cur); }));
      KX_TRY(run_other(c, [&] { return kx::launch_copy2d(Xk + m * n + m, n, 0, Ad, m, 0, m, m, 1, sre, c->cur); }));
    }
  }
  // Horner for phi_2: H = I/(K+2)!; H = X H + I/(k+2)!, k = K-1..0
  double fact[TAYLOR_K + 3];
  fact[0] = 1.0;
  for (int i = 1; i < TAYLOR_K + 3; ++i) fact[i] = fact[i - 1] * i;
  KX_TRY(run_other(c, [&] { return kx::launch_set_identity(H0, n, C, 1.0 / fact[TAYLOR_K + 2], c->cur); }));
  double* h = H0;
  double* hn = H1;
  for (int k = TAYLOR_K - 1; k >= 0; --k) {
    KX_TRY(chain_gemm(c, n, C, X, h, hn, 1.0, nullptr, 0, nullptr, 0, 1.0 / fact[k + 2]));
    std::swap(h, hn);
  }
  KX_CUDA(c, cudaMemcpyAsync(SP2, h, (size_t)C * n2 * 8, cudaMemcpyDeviceToDevice, c->cur));
  KX_TRY(chain_gemm(c, n, C, X, SP2, SP1, 1.0, nullptr, 0, nullptr, 0, 1.0));   // P1 = X P2 + I
  KX_TRY(chain_gemm(c, n, C, X, SP1, SE, 1.0, nullptr, 0, nullptr, 0, 1.0));    // E = X P1 + I
  // doublings
  const int qmax = ch[order[0]].q;
  for (int r = 1; r <= qmax; ++r) {
    int act = 0;
    while (act < C && ch[order[act]].q >= r) ++act;
    KX_TRY(chain_gemm(c, n, act, SE, SE, TE, 1.0, nullptr, 0, nullptr, 0, 0));
    KX_TRY(chain_gemm(c, n, act, SP1, SE, TP1, 0.5, SP1, 0.5, nullptr, 0, 0));
    KX_TRY(chain_gemm(c, n, act, SE, SP2, TP2, 0.25, SP2, 0.25, SP1, 0.25, 0));
    KX_CUDA(c, cudaMemcpyAsync(SE, TE, (size_t)act * n2 * 8, cudaMemcpyDeviceToDevice, c->cur));
    KX_CUDA(c, cudaMemcpyAsync(SP1, TP1, (size_t)act * n2 * 8, cudaMemcpyDeviceToDevice, c->cur));
    KX_CUDA(c, cudaMemcpyAsync(SP2, TP2, (size_t)act * n2 * 8, cudaMemcpyDeviceToDevice, c->cur));
  }
  out.assign(C, ChainOut{});
  if (thirds) {
    // 2/3 level into T
    KX_TRY(chain_gemm(c, n, C, SE, SE, TE, 1.0, nullptr, 0, nullptr, 0, 0));
    KX_TRY(chain_gemm(c, n, C, SP1, SE, TP1, 0.5, SP1, 0.5, nullptr, 0, 0));
    KX_TRY(chain_gemm(c, n, C, SE, SP2, TP2, 0.25, SP2, 0.25, SP1, 0.25, 0));
    // level 1 by the addition formula
    KX_TRY(chain_gemm(c, n, C, TP1, SE, O1, 2.0 / 3.0, SP1, 1.0 / 3.0, nullptr, 0, 0));
    KX_TRY(chain_gemm(c, n, C, TE, SP2, O2, 1.0 / 9.0, TP2, 4.0 / 9.0, TP1, 2.0 / 9.0, 0));
    for (int k = 0; k < C; ++k) {
      ChainOut& o = out[order[k]];
      o.p[0][0] = SP1 + k * n2;
      o.p[0][1] = SP2 + k * n2;
      o.p[1][0] = TP1 + k * n2;
      o.p[1][1] = TP2 + k * n2;
      o.p[2][0] = O1 + k * n2;
      o.p[2][1] = O2 + k * n2;
    }
  } else {
    for (int k = 0; k < C; ++k) {
      ChainOut& o = out[order[k]];
      o.p[2][0] = SP1 + k * n2;
      o.p[2][1] = SP2 + k * n2;
    }
  }
  c->cnt.phi_builds += C;
  return KX_OK;
}

kx_status set_tau_impl(kx_ctx* c, double tau, kx_scheme scheme) {
  const int d = c->d, nc = c->ncomp;
  drop_bank(c);
  c->scheme = scheme;
  c->tau = tau;
  const bool cplx = scheme == KX_ETD3RKDS_CPLX;
  const bool etd3 = scheme == KX_ETD3RKDS_REAL || cplx;
  const int pl = cplx ? 2 : 1;   // real planes per term (Re, Im for the complex split)
  c->cplx = cplx;
  // --- coefficients (imaginary parts zero for the real schemes)
  double eta[2][3] = {}, eta_im[2][3] = {}, alpha[2][3 * KX_MAXD] = {}, alpha_im[2][3 * KX_MAXD] = {};
  int inner[2][3];
  int T = 0;
  for (int ell = 1; ell <= 2; ++ell) {
    const int t = cplx ? kx::scheme_terms_cplx(ell, d, eta[ell - 1], eta_im[ell - 1], inner[ell - 1],
                                               alpha[ell - 1], alpha_im[ell - 1])
                       : kx::scheme_terms(scheme, ell, d, eta[ell - 1], inner[ell - 1], alpha[ell - 1]);
    if (t == 0) return fail(c, KX_ERR_UNSUPPORTED, "scheme not available for this d");
    T = t;
  }
  c->T = T;
  // --- groups (input tensors) of terms; every term occupies `pl` real planes / slots
  std::vector<Group> groups;
  if (etd3) {
    groups.resize(3);
    groups[0].nterms = 3 * T * pl;  // F: (stage 1/3, l=1) (2/3, l=1) (1, l=1)
    groups[1].nterms = T * pl;      // D2: (2/3, l=2)
    groups[2].nterms = T * pl;      // D3: (1, l=2)
    groups[0].slot0 = 0;
    groups[1].slot0 = 3 * T * pl;
    groups[2].slot0 = 3 * T * pl;
    c->nslots = 4 * T * pl;
  } else {
    groups.resize(2);
    groups[0].nterms = 1;
    groups[1].nterms = 1;
    groups[0].slot0 = 0;
    groups[1].slot0 = 1;
    c->nslots = 2;
  }
  // --- unique chains (dedupe identical (A, sigma)), bucketed by matrix extent
  std::vector<std::vector<Chain>> chains_by_n;
  std::vector<long long> ext;
  struct ChainRef { int bucket, idx; };
  auto find_or_add = [&](int comp, int mu, double sre, double sim) -> ChainRef {
    const long long n = c->n[mu - 1];
    int bkt = -1;
    for (size_t i = 0; i < ext.size(); ++i)
      if (ext[i] == n) bkt = (int)i;
    if (bkt < 0) {
      ext.push_back(n);
      chains_by_n.emplace_back();
      bkt = (int)ext.size() - 1;
    }
    auto& v = chains_by_n[bkt];
    for (size_t i = 0; i < v.size(); ++i) {
      if (v[i].sigma == sre && v[i].sigma_im == sim &&
          c->A_host[v[i].c][v[i].mu - 1] == c->A_host[comp][mu - 1])
        return {bkt, (int)i};
    }
    Chain h;
    h.c = comp;
    h.mu = mu;
    h.sigma = sre;
    h.sigma_im = sim;
    const double nrm = (std::fabs(sre) + std::fabs(sim)) * norm_bound(c->A_host[comp][mu - 1], n);
    h.q = nrm > THETA ? (int)std::ceil(std::log2(nrm / THETA)) : 0;
    v.push_back(h);
    return {bkt, (int)v.size() - 1};
  };
  // refs[g][comp][term][mu-1] -> (chain, level, l); term indexes complex terms
  struct Ref { ChainRef ch; int level; int l; };
  std::vector<std::vector<std::vector<std::vector<Ref>>>> refs(groups.size());
  for (size_t gi = 0; gi < groups.size(); ++gi)
    refs[gi].assign(nc, std::vector<std::vector<Ref>>(groups[gi].nterms / pl, std::vector<Ref>(d)));
  for (int comp = 0; comp < nc; ++comp) {
    for (int mu = 1; mu <= d; ++mu) {
      if (etd3) {
        for (int ellt = 1; ellt <= 2; ++ellt) {
          for (int i = 0; i < T; ++i) {
            const double sre = tau / 3.0 * alpha[ellt - 1][i * d + mu - 1];
            const double sim = tau / 3.0 * alpha_im[ellt - 1][i * d + mu - 1];
            ChainRef r = find_or_add(comp, mu, sre, sim);
            const int l = inner[ellt - 1][i];
            if (ellt == 1) {
              for (int lev = 0; lev < 3; ++lev) refs[0][comp][lev * T + i][mu - 1] = {r, lev, l};
            } else {
              refs[1][comp][i][mu - 1] = {r, 1, l};
              refs[2][comp][i][mu - 1] = {r, 2, l};
            }
          }
        }
      } else {
        ChainRef r = find_or_add(comp, mu, tau, 0.0);
        refs[0][comp][0][mu - 1] = {r, 2, 1};
        refs[1][comp][0][mu - 1] = {r, 2, 2};
      }
    }
  }
  // --- build chains on the device (scratch freed on every exit path)
  struct Scratch {
    std::vector<double*> v;
    ~Scratch() { free_list(v); }
  } scratch_guard;
  std::vector<double*>& scratch = scratch_guard.v;
  std::vector<std::vector<ChainOut>> outs(chains_by_n.size());
  for (size_t b = 0; b < chains_by_n.size(); ++b)
    KX_TRY(build_chains(c, ext[b], cplx, chains_by_n[b], etd3, outs[b], scratch));
  // plane `part` (0 = Re, 1 = Im) of a referenced phi-matrix, column-major with leading dim ld
  auto plane_src = [&](const Ref& r, int part, long long n, long long* ld) -> const double* {
    const double* p = outs[r.ch.bucket][r.ch.idx].p[r.level][r.l - 1];
    if (!cplx) {
      *ld = n;
      return p;
    }
    *ld = 2 * n;
    return part == 0 ? p : p + n * 2 * n;
  };
  // --- lay out the bank (planes of term t: t*pl + part)
  const long long n1 = c->n[0], nd = c->n[d - 1];
  auto bal = [&](double** p, size_t cnt) { return dalloc(c, p, cnt, c->bank_allocs); };
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    Group& G = groups[gi];
    const int TG = G.nterms;   // planes
    for (int comp = 0; comp < nc; ++comp) {
      KX_TRY(bal(&G.last[comp], (size_t)TG * n1 * n1));
      if (d >= 2) KX_TRY(bal(&G.first[comp], (size_t)TG * nd * nd));
      for (int mu = 2; mu < d; ++mu) KX_TRY(bal(&G.mid[comp][mu - 1], (size_t)TG * c->n[mu - 1] * c->n[mu - 1]));
      for (int t = 0; t < TG / pl; ++t) {
        for (int part = 0; part < pl; ++part) {
          const int plane = t * pl + part;
          long long ld;
          const double* src = plane_src(refs[gi][comp][t][0], part, n1, &ld);
          KX_CUDA(c, cudaMemcpy2DAsync(G.last[comp] + plane * n1 * n1, n1 * 8, src, ld * 8, n1 * 8, n1,
                                       cudaMemcpyDeviceToDevice, c->cur));
          if (d >= 2) {
            src = plane_src(refs[gi][comp][t][d - 1], part, nd, &ld);
            KX_CUDA(c, cudaMemcpy2DAsync(G.first[comp] + plane * nd, (size_t)TG * nd * 8, src, ld * 8,
                                         nd * 8, nd, cudaMemcpyDeviceToDevice, c->cur));
          }
          for (int mu = 2; mu < d; ++mu) {
            const long long nm = c->n[mu - 1];
            src = plane_src(refs[gi][comp][t][mu - 1], part, nm, &ld);
            KX_CUDA(c, cudaMemcpy2DAsync(G.mid[comp][mu - 1] + plane * nm * nm, nm * 8, src, ld * 8,
                                         nm * 8, nm, cudaMemcpyDeviceToDevice, c->cur));
          }
        }
      }
    }
  }
  // Last-mode blocks: the real part of kappa * eta_t * (W_t x_1 P_t{1}) for a complex term is
  //   W_re x_1 Re(kappa eta P) + W_im x_1 (-Im(kappa eta P)),
  // so a term contributes the blocks [Re(kappa eta P); -Im(kappa eta P)] over its two slots.
  auto put_blocks = [&](double* dst, int gi, int comp, int t, double kre, double kim) -> kx_status {
    const long long m2 = n1 * n1;
    const Group& G = groups[gi];
    if (!cplx) {
      const double* src = G.last[comp] + t * m2;
      return run_other(c, [&] { return kx::launch_scale(dst, src, kre, m2, c->cur); });
    }
    const double* Pre = G.last[comp] + (2 * t) * m2;
    const double* Pim = G.last[comp] + (2 * t + 1) * m2;
    KX_TRY(run_other(c, [&] { return kx::launch_axpby(dst, kre, Pre, -kim, Pim, m2, c->cur); }));
    return run_other(c, [&] { return kx::launch_axpby(dst + m2, -kre, Pim, -kim, Pre, m2, c->cur); });
  };
  // phi stacks for kx_phi_apply: (Re part of) sum_t eta_t T(X, P_t)
  auto make_stack = [&](PhiStack& ps, int gi, int t0, int ell) -> kx_status {
    ps.group = gi;
    ps.t0 = t0 * pl;
    ps.nterms = T * pl;
    for (int comp = 0; comp < nc; ++comp) {
      KX_TRY(bal(&ps.B[comp], (size_t)T * pl * n1 * n1));
      for (int t = 0; t < T; ++t)
        KX_TRY(put_blocks(ps.B[comp] + (size_t)t * pl * n1 * n1, gi, comp, t0 + t, eta[ell - 1][t],
                          eta_im[ell - 1][t]));
    }
    return KX_OK;
  };
  if (etd3) {
    for (int st = 0; st < 3; ++st) KX_TRY(make_stack(c->phi[{1, st}], 0, st * T, 1));
    KX_TRY(make_stack(c->phi[{2, 1}], 1, 0, 2));
    KX_TRY(make_stack(c->phi[{2, 2}], 2, 0, 2));
  } else {
    KX_TRY(make_stack(c->phi[{1, 2}], 0, 0, 1));
    KX_TRY(make_stack(c->phi[{2, 2}], 1, 0, 2));
  }
  // stage stacks (eq:exprk3 P:586-594 scalars folded in): (group, term, slot of plane 0, kappa*eta)
  struct Seg { int gi, t, slot; double kre, kim; };
  auto make_stage = [&](Stage& S, const std::vector<Seg>& segs) -> kx_status {
    S.nseg = (int)segs.size() * pl;
    for (size_t k = 0; k < segs.size(); ++k)
      for (int part = 0; part < pl; ++part) S.slot[k * pl + part] = segs[k].slot + part;
    for (int comp = 0; comp < nc; ++comp) {
      KX_TRY(bal(&S.B[comp], (size_t)S.nseg * n1 * n1));
      for (size_t k = 0; k < segs.size(); ++k)
        KX_TRY(put_blocks(S.B[comp] + k * pl * n1 * n1, segs[k].gi, comp, segs[k].t, segs[k].kre, segs[k].kim));
    }
    return KX_OK;
  };
  if (etd3) {
    std::vector<Seg> s0, s1, s2;
    const double k0 = tau / 3.0, k1 = 2.0 * tau / 3.0, k1d = 4.0 * tau / 3.0, k2 = tau, k2d = 1.5 * tau;
    for (int i = 0; i < T; ++i) s0.push_back({0, i, i * pl, k0 * eta[0][i], k0 * eta_im[0][i]});
    for (int i = 0; i < T; ++i) s1.push_back({0, T + i, (T + i) * pl, k1 * eta[0][i], k1 * eta_im[0][i]});
    for (int i = 0; i < T; ++i) s1.push_back({1, i, (3 * T + i) * pl, k1d * eta[1][i], k1d * eta_im[1][i]});
    for (int i = 0; i < T; ++i) s2.push_back({0, 2 * T + i, (2 * T + i) * pl, k2 * eta[0][i], k2 * eta_im[0][i]});
    for (int i = 0; i < T; ++i) s2.push_back({2, i, (3 * T + i) * pl, k2d * eta[1][i], k2d * eta_im[1][i]});
    KX_TRY(make_stage(c->stages[0], s0));
    KX_TRY(make_stage(c->stages[1], s1));
    KX_TRY(make_stage(c->stages[2], s2));
    c->nstages = 3;
  } else {
    KX_TRY(make_stage(c->stages[0], {{0, 0, 0, tau * eta[0][0], 0.0}}));
    KX_TRY(make_stage(c->stages[1], {{1, 0, 1, tau * eta[1][0], 0.0}}));
    c->nstages = 2;
  }
  c->groups = groups;
  // workspaces
  const size_t N = (size_t)c->tN;
  auto wal = [&](double** p, size_t cnt) { return dalloc(c, p, cnt, c->ws_allocs); };
  for (int comp = 0; comp < nc; ++comp) {
    KX_TRY(wal(&c->G[comp], N));
    KX_TRY(wal(&c->F[comp], N));
    KX_TRY(wal(&c->D[comp], N));
    KX_TRY(wal(&c->Us[comp], N));
    if (d >= 2) KX_TRY(wal(&c->W1[comp], (size_t)c->nslots * N));
    if (d >= 3) KX_TRY(wal(&c->W2[comp], (size_t)c->nslots * N));
    if (c->dist) {
      KX_TRY(wal(&c->RA[comp], (size_t)c->nslots * N));
      KX_TRY(wal(&c->T1G_pack[comp], N));
      KX_TRY(wal(&c->U_pack[comp], N));
      KX_TRY(wal(&c->T1G_B[comp], N));
      KX_TRY(wal(&c->U_B[comp], N));
      KX_TRY(wal(&c->F_B[comp], N));
      KX_TRY(wal(&c->D_pack[comp], N));
      KX_TRY(wal(&c->D_B[comp], N));
    }
  }
  KX_CUDA(c, cudaStreamSynchronize(c->cur));
  c->bank_ready = true;
  c->bank_version += 1;
  return KX_OK;
}

kx_status collect_profile(kx_ctx* c) {
  if (c->recs.empty()) return KX_OK;
  KX_CUDA(c, cudaStreamSynchronize(c->stream));
  for (const auto& r : c->recs) {
    float ms = 0;
    KX_CUDA(c, cudaEventElapsedTime(&ms, c->ev_pool[r.e0], c->ev_pool[r.e1]));
    c->prof_ms[r.cls] += ms;
    c->prof_launches[r.cls] += 1;
    c->prof_flops += r.flops;
  }
  c->recs.clear();
  c->ev_used = c->gexec ? c->graph_ev_end : 0;
  return KX_OK;
}

kx_status check_ptr(kx_ctx* c, const void* p, const char* what) {
  if (!p) return fail(c, KX_ERR_INVALID, std::string(what) + " is NULL");
  if (reinterpret_cast<uintptr_t>(p) % 8 != 0)
    return fail(c, KX_ERR_INVALID, std::string(what) + " is not 8-byte aligned");
  return KX_OK;
}

kx_status step_impl(kx_ctx* c, double* const* U) {
  // The step is always replayed from a CUDA graph.  With profiling on, the graph also holds
  // an event-record node around every kernel; after each replay the stream is synchronised
  // and the per-kernel device times are accumulated (kx_get_profile).
  bool same = c->gexec && c->graph_version == c->bank_version && c->graph_prof == c->profiling;
  for (int s = 0; s < c->ncomp && same; ++s) same = c->graph_U[s] == U[s];
  if (!same) {
    drop_graph(c);
    KX_TRY(collect_profile(c));
    const kx_counters before = c->cnt;
    c->cur = c->cap;
    c->ev_used = 0;
    c->recs.clear();
    KX_CUDA(c, cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
    kx_status s = enqueue_step(c, U);
    cudaGraph_t gr = nullptr;
    cudaError_t e = cudaStreamEndCapture(c->cap, &gr);
    c->cur = c->stream;
    c->graph_recs = c->recs;
    c->graph_ev_end = c->ev_used;
    c->recs.clear();
    if (s != KX_OK) {
      if (gr) cudaGraphDestroy(gr);
      return s;
    }
    KX_CUDA(c, e);
    c->graph = gr;
    KX_CUDA(c, cudaGraphInstantiate(&c->gexec, c->graph, 0));
    c->graph_version = c->bank_version;
    c->graph_prof = c->profiling;
    for (int k = 0; k < c->ncomp; ++k) c->graph_U[k] = U[k];
    // capture counted one step's launches; remember the per-step deltas and undo
    kx_counters dl = c->cnt;
    dl.steps = 0;
    dl.tucker_ops -= before.tucker_ops;
    dl.mode_products -= before.mode_products;
    dl.kronsum_actions -= before.kronsum_actions;
    dl.phi_builds = 0;
    dl.gemm_launches -= before.gemm_launches;
    dl.other_launches -= before.other_launches;
    dl.mode_product_flops -= before.mode_product_flops;
    c->step_delta = dl;
    c->cnt = before;
  }
  KX_CUDA(c, cudaGraphLaunch(c->gexec, c->stream));
  c->cnt.steps += 1;
  c->cnt.tucker_ops += c->step_delta.tucker_ops;
  c->cnt.mode_products += c->step_delta.mode_products;
  c->cnt.kronsum_actions += c->step_delta.kronsum_actions;
  c->cnt.gemm_launches += c->step_delta.gemm_launches;
  c->cnt.other_launches += c->step_delta.other_launches;
  c->cnt.mode_product_flops += c->step_delta.mode_product_flops;
  if (c->graph_prof) {
    KX_CUDA(c, cudaStreamSynchronize(c->stream));
    for (const auto& r : c->graph_recs) {
      float ms = 0;
      KX_CUDA(c, cudaEventElapsedTime(&ms, c->ev_pool[r.e0], c->ev_pool[r.e1]));
      c->prof_ms[r.cls] += ms;
      c->prof_launches[r.cls] += 1;
      c->prof_flops += r.flops;
    }
  }
  return KX_OK;
}

}  // namespace


// ============================================================ distributed step ==========
// Slab decomposition along i_d over P ranks.  Layout A (i_d sharded) is the
// user layout; layout B (i_1 sharded) holds full i_d fibres.  Per exprk3ds step and component:
//   [A] G = g(U); (U x_1 A_1 + G) and U peer-packed          -> all-to-all -> layout B
//   [B] F_B = (U x_1 A_1 + G)_B + sum_{mu=d..2} U_B x_mu A_mu; first (mu = d) and middle modes
//       of the 3T F-terms                                    -> all-to-all of 3T slots -> A
//   [A] U2 = U + concat-K over (stage term, source rank) segments — the peer-major receive
//       layout is absorbed by the K segmentation, no unpack; D = g(U2) - G peer-packed
//   [B] D2 terms ... [A] U3 ... [B] D3 terms ... [A] U+
// 4 + 5T all-to-alls per component per step; every mode product runs on full fibres on one
// rank, so results match one GPU up to the summation order of F (rounding level).
namespace {

struct NcclApi {
  bool ok = false;
#ifdef KX_HAVE_NCCL
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
#endif
  std::string why;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
#ifdef KX_HAVE_NCCL
  const char* env = getenv("KX_NCCL_LIB");
  void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    api.why = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
    return api;
  }
  auto sym = [&](const char* n) { return dlsym(h, n); };
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
  api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
  api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
  api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
  api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
  api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv &&
           api.GroupStart && api.GroupEnd && api.GetErrorString;
  if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
#else
  api.why = "built without nccl.h";
#endif
  return api;
}

// Buffers one rank exchanges after a phase: for k < nbuf, chunk q (count doubles) of send[k]
// goes to rank q, which stores it at chunk `rank` of its recv[k].
struct Exchange {
  int nbuf = 0;
  size_t count = 0;
  const double* send[64];
  double* recv[64];
  void add(const double* sb, double* rb) {
    send[nbuf] = sb;
    recv[nbuf] = rb;
    ++nbuf;
  }
};

void set_layout(kx_ctx* c, bool B) {
  for (int mu = 0; mu < KX_MAXD; ++mu) c->tn[mu] = B ? c->nB[mu] : c->nA[mu];
  c->tN = c->Nloc;
}

// [A] G = g(U); T1G_pack = (U x_1 A_1 + G) peer-packed; U_pack = U peer-packed
kx_status dist_f_source(kx_ctx* c, double* const* U, Exchange& x) {
  set_layout(c, false);
  const int ns = c->ncomp, P = c->nranks;
  KX_TRY(nonlin(c, 0, U, c->G));
  const long long n1 = c->n[0], n1l = n1 / P, M = c->Nloc / n1, chunk = c->Nloc / P;
  GemmArgs g;
  g.arow = true;
  g.M = (int)M;
  g.N = (int)n1l;
  g.kseg = (int)n1;
  g.lda = n1;
  g.ldb = n1;
  g.ldc = n1l;
  g.ldd = n1;
  g.ns = ns;
  g.nt = P;                 // one batch per destination rank: columns [q n1l, (q+1) n1l)
  g.sB_t = n1l;
  g.sC_t = chunk;
  g.sD_t = n1l;
  g.beta = 1.0;
  for (int s = 0; s < ns; ++s) {
    g.A[s] = U[s];
    g.B[s] = c->A_dev[s][0];
    g.C[s] = c->T1G_pack[s];
    g.D[s] = c->G[s];
  }
  KX_TRY(run_gemm(c, g));
  c->cnt.mode_products += ns;
  for (int s = 0; s < ns; ++s)
    for (int q = 0; q < P; ++q)
      KX_CUDA(c, cudaMemcpy2DAsync(c->U_pack[s] + q * chunk, n1l * 8, U[s] + q * n1l, n1 * 8,
                                   n1l * 8, M, cudaMemcpyDeviceToDevice, c->cur));
  x.count = (size_t)chunk;
  for (int s = 0; s < ns; ++s) {
    x.add(c->T1G_pack[s], c->T1G_B[s]);
    x.add(c->U_pack[s], c->U_B[s]);
  }
  return KX_OK;
}

// [B] F_B = T1G_B + sum_{mu = d..2} U_B x_mu A_mu
kx_status dist_f_build(kx_ctx* c) {
  set_layout(c, true);
  const int ns = c->ncomp;
  const double* L[MAXS];
  const double* Ub[MAXS];
  double* Fb[MAXS];
  const double* Db[MAXS];
  for (int mu = c->d; mu >= 2; --mu) {
    for (int s = 0; s < ns; ++s) {
      L[s] = c->A_dev[s][mu - 1];
      Ub[s] = c->U_B[s];
      Fb[s] = c->F_B[s];
      Db[s] = mu == c->d ? c->T1G_B[s] : c->F_B[s];
    }
    KX_TRY(mode_product_multi(c, ns, Ub, Fb, mu, L, 1.0, 1.0, Db));
  }
  c->cnt.kronsum_actions += ns;
  return KX_OK;
}

// [B] first + middle modes of group gi on X_B; the term slots go back to layout A
kx_status nccl_exchange(kx_ctx* c, const Exchange& x, cudaStream_t st);

kx_status dist_group(kx_ctx* c, int gi, double* const* Xb, Exchange& x) {
  set_layout(c, true);
  const Group& G = c->groups[gi];
  double* const* ws = nullptr;
  if (c->dist == 1 && c->overlap && c->comm) {
    // f2: modes d..2 term by term; each term's slots go to the peers on the comm stream while
    // the next term's mode products run; the compute stream joins before the stage GEMM
    const int pl = c->cplx ? 2 : 1;
    const int nterm = G.nterms / pl;
    if (nterm > 64) return fail(c, KX_ERR_UNSUPPORTED, "too many terms");
    for (int t = 0; t < nterm; ++t) {
      KX_TRY(group_modes(c, G, t * pl, pl, Xb, G.slot0 + t * pl, &ws));
      KX_CUDA(c, cudaEventRecord(c->ev_term[t], c->cur));
      KX_CUDA(c, cudaStreamWaitEvent(c->comm, c->ev_term[t], 0));
      Exchange xt;
      xt.count = (size_t)(c->Nloc / c->nranks);
      for (int k = 0; k < pl; ++k)
        for (int s = 0; s < c->ncomp; ++s) {
          const long long slot = G.slot0 + t * pl + k;
          xt.add(ws[s] + slot * c->Nloc, c->RA[s] + slot * c->Nloc);
        }
      KX_TRY(nccl_exchange(c, xt, c->comm));
    }
    KX_CUDA(c, cudaEventRecord(c->ev_join, c->comm));
    KX_CUDA(c, cudaStreamWaitEvent(c->cur, c->ev_join, 0));
    x = Exchange{};
    return KX_OK;
  }
  KX_TRY(group_modes(c, G, 0, G.nterms, Xb, G.slot0, &ws));
  x.count = (size_t)(c->Nloc / c->nranks);
  for (int t = 0; t < G.nterms; ++t)
    for (int s = 0; s < c->ncomp; ++s)
      x.add(ws[s] + (long long)(G.slot0 + t) * c->Nloc, c->RA[s] + (long long)(G.slot0 + t) * c->Nloc);
  return KX_OK;
}

// [A] out = addend + sum over stage terms and source ranks of RA segments x_1 stacked B
kx_status dist_stage(kx_ctx* c, const Stage& S, double* const* out, const double* const* addend) {
  set_layout(c, false);
  const int P = c->nranks;
  const long long n1 = c->n[0], n1l = n1 / P;
  if (S.nseg * P > MAXSEG) return fail(c, KX_ERR_UNSUPPORTED, "too many K segments for this rank count");
  GemmArgs g;
  g.arow = true;
  g.M = (int)(c->Nloc / n1);
  g.N = (int)n1;
  g.kseg = (int)n1l;
  g.nseg = S.nseg * P;
  g.lda = n1l;
  g.ldb = n1;
  g.ldc = n1;
  g.ldd = n1;
  g.ns = c->ncomp;
  g.beta = 1.0;
  for (int k = 0; k < S.nseg; ++k)
    for (int q = 0; q < P; ++q)
      g.seg_off[k * P + q] = (long long)S.slot[k] * c->Nloc + (long long)q * (c->Nloc / P);
  for (int s = 0; s < c->ncomp; ++s) {
    g.A[s] = c->RA[s];
    g.B[s] = S.B[s];
    g.C[s] = out[s];
    g.D[s] = addend[s];
  }
  KX_TRY(run_gemm(c, g));
  c->cnt.mode_products += (long long)c->ncomp * S.nseg;
  return KX_OK;
}

// [A] D_pack = g(Us) - G, peer-packed
kx_status dist_d_source(kx_ctx* c, Exchange& x) {
  set_layout(c, false);
  kx::PointwiseArgs a;
  a.model = c->model;
  a.ncomp = c->ncomp;
  a.N = c->Nloc;
  a.pack_n1 = c->n[0];
  a.pack_n1l = c->n[0] / c->nranks;
  for (int s = 0; s < c->ncomp; ++s) {
    a.u[s] = c->Us[s];
    a.out[s] = c->D_pack[s];
    a.G[s] = c->G[s];
  }
  for (int i = 0; i < 8; ++i) a.p[i] = c->params[i];
  KX_TRY(run_other(c, [&] { return kx::launch_nonlinearity(a, 1, c->cur); }));
  x.count = (size_t)(c->Nloc / c->nranks);
  for (int s = 0; s < c->ncomp; ++s) x.add(c->D_pack[s], c->D_B[s]);
  return KX_OK;
}

int dist_phases(const kx_ctx* c) { return c->scheme == KX_ETD2RKDS ? 5 : 7; }

kx_status dist_phase(kx_ctx* c, double* const* U, int ph, Exchange& x) {
  x = Exchange{};
  const bool e3 = c->scheme != KX_ETD2RKDS;
  const double* Uc[MAXS];
  const double* Usc[MAXS];
  for (int s = 0; s < c->ncomp; ++s) {
    Uc[s] = U[s];
    Usc[s] = c->Us[s];
  }
  switch (ph) {
    case 0: return dist_f_source(c, U, x);
    case 1:
      KX_TRY(dist_f_build(c));
      return dist_group(c, 0, c->F_B, x);
    case 2:
      KX_TRY(dist_stage(c, c->stages[0], c->Us, Uc));
      return dist_d_source(c, x);
    case 3: return dist_group(c, 1, c->D_B, x);
    case 4:
      if (!e3) {
        KX_TRY(dist_stage(c, c->stages[1], U, Usc));
        c->cnt.tucker_ops += (long long)c->ncomp * 2;
        return KX_OK;
      }
      KX_TRY(dist_stage(c, c->stages[1], c->Us, Uc));
      return dist_d_source(c, x);
    case 5: return dist_group(c, 2, c->D_B, x);
    case 6:
      KX_TRY(dist_stage(c, c->stages[2], U, Uc));
      c->cnt.tucker_ops += (long long)c->ncomp * 5 * c->T;
      return KX_OK;
  }
  return fail(c, KX_ERR_INVALID, "bad phase");
}

kx_status nccl_exchange(kx_ctx* c, const Exchange& x, cudaStream_t st) {
#ifdef KX_HAVE_NCCL
  NcclApi& api = nccl();
  ncclComm_t comm = static_cast<ncclComm_t>(c->nccl_comm);
  auto chk = [&](ncclResult_t r) -> kx_status {
    if (r != ncclSuccess) return fail(c, KX_ERR_NCCL, std::string("NCCL: ") + api.GetErrorString(r));
    return KX_OK;
  };
  KX_TRY(chk(api.GroupStart()));
  for (int k = 0; k < x.nbuf; ++k)
    for (int q = 0; q < c->nranks; ++q) {
      KX_TRY(chk(api.Send(x.send[k] + q * x.count, x.count, ncclFloat64, q, comm, st)));
      KX_TRY(chk(api.Recv(x.recv[k] + q * x.count, x.count, ncclFloat64, q, comm, st)));
    }
  KX_TRY(chk(api.GroupEnd()));
  return KX_OK;
#else
  (void)x;
  return fail(c, KX_ERR_UNSUPPORTED, "built without NCCL");
#endif
}

kx_status dist_step_nccl(kx_ctx* c, double* const* U) {
  c->cur = c->stream;
  Exchange x;
  for (int ph = 0; ph < dist_phases(c); ++ph) {
    KX_TRY(dist_phase(c, U, ph, x));
    if (x.nbuf) KX_TRY(nccl_exchange(c, x, c->cur));
  }
  c->cnt.steps += 1;
  return KX_OK;
}

}  // namespace

namespace kx {
void gemm_prepare_all();
}

// ============================================================================ C ABI ======
extern "C" {

const char* kx_version(void) { return "kx 0.1 (sm_100a, fp64 DMMA mode products)"; }

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
  e = cudaSetDevice(device);
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
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  drop_bank(c);
  for (auto& v : c->A_dev)
    for (double* p : v) cudaFree(p);
  for (auto& v : c->A_tri)
    for (double* p : v) cudaFree(p);
  if (c->tmp1) cudaFree(c->tmp1);
  if (c->tmp2) cudaFree(c->tmp2);
  for (int s = 0; s < MAXS; ++s)
    if (c->hostU[s]) cudaFree(c->hostU[s]);
  if (c->flag) cudaFree(c->flag);
#ifdef KX_HAVE_NCCL
  if (c->nccl_comm && nccl().ok) nccl().CommDestroy(static_cast<ncclComm_t>(c->nccl_comm));
#endif
  if (c->comm) cudaStreamDestroy(c->comm);
  for (auto e : c->ev_term)
    if (e) cudaEventDestroy(e);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->sk_ws) cudaFree(c->sk_ws);
  if (c->sk_flags) cudaFree(c->sk_flags);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->cap) cudaStreamDestroy(c->cap);
  delete c;
}

const char* kx_last_error(const kx_ctx* c) { return c ? c->err.c_str() : "null context"; }

kx_status kx_set_grid(kx_ctx* c, int d, const long long* n, int ncomp) {
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
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  drop_bank(c);
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
  KX_TRY(need_grid(c));
  if (comp < 0 || comp >= c->ncomp) return fail(c, KX_ERR_INVALID, "comp out of range");
  if (mu < 1 || mu > c->d) return fail(c, KX_ERR_INVALID, "mu out of range 1..d");
  if (!A_host) return fail(c, KX_ERR_INVALID, "A_host is NULL");
  const long long n = c->n[mu - 1];
  for (long long i = 0; i < n * n; ++i)
    if (!std::isfinite(A_host[i])) return fail(c, KX_ERR_INVALID, "A has non-finite entries");
  cudaSetDevice(c->device);
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
  cudaSetDevice(c->device);
  KX_CUDA(c, cudaStreamSynchronize(c->stream));
  c->cur = c->stream;
  kx_status s = set_tau_impl(c, tau, scheme);
  if (s != KX_OK) drop_bank(c);
  return s;
}

kx_status kx_mode_product(kx_ctx* c, const double* X, double* Y, int mu, const double* L,
                          double alpha, double beta) {
  KX_TRY(need_grid(c));
  if (c->dist) return fail(c, KX_ERR_UNSUPPORTED, "single-GPU operator on a distributed context");
  if (mu < 1 || mu > c->d)
    return fail(c, KX_ERR_INVALID, "mode " + std::to_string(mu) + " outside 1.." + std::to_string(c->d));
  KX_TRY(check_ptr(c, X, "X"));
  KX_TRY(check_ptr(c, Y, "Y"));
  KX_TRY(check_ptr(c, L, "L"));
  if (X == Y) return fail(c, KX_ERR_INVALID, "X and Y must be distinct");
  c->cur = c->stream;
  const double* Xs[1] = {X};
  double* Ys[1] = {Y};
  const double* Ls[1] = {L};
  const double* Ds[1] = {Y};
  return mode_product_multi(c, 1, Xs, Ys, mu, Ls, alpha, beta, Ds);
}

kx_status kx_tucker(kx_ctx* c, const double* X, double* Y, const double* const* L, double alpha,
                    double beta) {
  KX_TRY(need_grid(c));
  if (c->dist) return fail(c, KX_ERR_UNSUPPORTED, "single-GPU operator on a distributed context");
  KX_TRY(check_ptr(c, X, "X"));
  KX_TRY(check_ptr(c, Y, "Y"));
  if (!L) return fail(c, KX_ERR_INVALID, "L is NULL");
  for (int mu = 0; mu < c->d; ++mu) KX_TRY(check_ptr(c, L[mu], "L[mu]"));
  if (X == Y) return fail(c, KX_ERR_INVALID, "X and Y must be distinct");
  c->cur = c->stream;
  const int d = c->d;
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

kx_status kx_kronsum(kx_ctx* c, int comp, const double* X, double* Y, double beta) {
  KX_TRY(need_grid(c));
  if (c->dist) return fail(c, KX_ERR_UNSUPPORTED, "single-GPU operator on a distributed context");
  if (comp < 0 || comp >= c->ncomp) return fail(c, KX_ERR_INVALID, "comp out of range");
  for (int mu = 1; mu <= c->d; ++mu)
    if (!c->A_dev[comp][mu - 1])
      return fail(c, KX_ERR_INVALID, "direction matrix mu=" + std::to_string(mu) + " not set");
  KX_TRY(check_ptr(c, X, "X"));
  KX_TRY(check_ptr(c, Y, "Y"));
  if (X == Y) return fail(c, KX_ERR_INVALID, "X and Y must be distinct");
  c->cur = c->stream;
  const double* Xs[1] = {X};
  double* Ys[1] = {Y};
  const double* Ds[1] = {Y};
  return kronsum_multi(c, comp, 1, Xs, Ys, beta, Ds);
}

kx_status kx_set_dist_overlap(kx_ctx* c, int on) {
  if (!c) return KX_ERR_INVALID;
  c->overlap = on != 0;
  return KX_OK;
}

kx_status kx_set_kronsum_mode(kx_ctx* c, int mode) {
  if (!c) return KX_ERR_INVALID;
  if (mode != 0 && mode != 1) return fail(c, KX_ERR_INVALID, "kronsum mode must be 0 or 1");
  if (c->kronsum_mode != mode) drop_graph(c);
  c->kronsum_mode = mode;
  return KX_OK;
}

kx_status kx_phi_apply(kx_ctx* c, int comp, int ell, int stage, const double* X, double* Y,
                       double alpha, double beta) {
  KX_TRY(need_grid(c));
  if (c->dist) return fail(c, KX_ERR_UNSUPPORTED, "single-GPU operator on a distributed context");
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

kx_status kx_integrate_host(kx_ctx* c, double t0, int nsteps, double* const* U_host) {
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
  double t = t0;
  for (int k = 0; k < nsteps; ++k) {
    KX_TRY(step_impl(c, c->hostU));
    t += c->tau;
  }
  for (int s = 0; s < c->ncomp; ++s)
    KX_CUDA(c, cudaMemcpyAsync(U_host[s], c->hostU[s], bytes, cudaMemcpyDeviceToHost, c->stream));
  KX_CUDA(c, cudaStreamSynchronize(c->stream));
  return KX_OK;
}

kx_status kx_get_counters(const kx_ctx* c, kx_counters* out) {
  if (!c || !out) return KX_ERR_INVALID;
  *out = c->cnt;
  return KX_OK;
}

kx_status kx_reset_counters(kx_ctx* c) {
  if (!c) return KX_ERR_INVALID;
  c->cnt = kx_counters{};
  return KX_OK;
}

kx_status kx_sync(kx_ctx* c) {
  if (!c) return KX_ERR_INVALID;
  KX_CUDA(c, cudaStreamSynchronize(c->stream));
  KX_CUDA(c, cudaGetLastError());
  return KX_OK;
}

kx_status kx_check_finite(kx_ctx* c, const double* X) {
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
  if (!c) return KX_ERR_INVALID;
  KX_TRY(collect_profile(c));
  c->profiling = on != 0;
  c->prof_ms[0] = c->prof_ms[1] = 0;
  c->prof_launches[0] = c->prof_launches[1] = 0;
  c->prof_flops = 0;
  return KX_OK;
}

kx_status kx_get_profile(kx_ctx* c, double* gemm_ms, double* other_ms, long long* gemm_launches,
                         long long* other_launches, double* gemm_flops) {
  if (!c) return KX_ERR_INVALID;
  KX_TRY(collect_profile(c));
  if (gemm_ms) *gemm_ms = c->prof_ms[0];
  if (other_ms) *other_ms = c->prof_ms[1];
  if (gemm_launches) *gemm_launches = c->prof_launches[0];
  if (other_launches) *other_launches = c->prof_launches[1];
  if (gemm_flops) *gemm_flops = c->prof_flops;
  return KX_OK;
}

kx_status kx_get_phi_matrix(kx_ctx* c, int comp, int ell, int stage, int term, int mu,
                            double* out_host) {
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
  std::vector<Exchange> xs(nranks);
  for (int ph = 0; ph < dist_phases(ctxs[0]); ++ph) {
    for (int r = 0; r < nranks; ++r) KX_TRY(dist_phase(ctxs[r], U + (size_t)r * nc, ph, xs[r]));
    // loopback all-to-all: device copies on the shared stream, after every rank's phase
    for (int r = 0; r < nranks; ++r) {
      const Exchange& xr = xs[r];
      for (int k = 0; k < xr.nbuf; ++k)
        for (int q = 0; q < nranks; ++q)
          KX_CUDA(ctxs[r], cudaMemcpyAsync(xs[q].recv[k] + (size_t)r * xr.count, xr.send[k] + (size_t)q * xr.count,
                                           xr.count * 8, cudaMemcpyDeviceToDevice, ctxs[r]->stream));
    }
  }
  for (int r = 0; r < nranks; ++r) ctxs[r]->cnt.steps += 1;
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
