// Internal definitions shared by the library's host translation units (not part of the ABI):
// the context, the phi-bank layout, and the helpers of kx_core.cpp (launch wrappers, mode
// products, Kronecker sums, split application), kx_bank.cpp (phi-bank formation), kx_step.cpp
// (one-GPU step schedules and graph capture) and kx_dist.cpp (slab-sharded steps).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "kx.h"
#include "kx_internal.h"
#ifdef KX_HAVE_NCCL
#include <nccl.h>
#endif

namespace kx::detail {

using kx::GemmArgs;
using kx::MAXS;
using kx::MAXSEG;

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
  int nterms = 0;                       // real planes (= terms; 2 per term for the complex split)
  int slot0 = 0;                        // first workspace slot of its intermediates
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

struct BlockRecipe {         // one scaled last-mode block: dst = kappa*eta * P_t{1} (Re/Im pair)
  int gi = 0, t = 0, comp = 0;
  double kre = 0.0, kim = 0.0;
  double* dst = nullptr;
};

struct F32State;             // fp32 variant's bank planes, workspaces and graph (kx_f32.cpp)

struct Chain {               // one phi-matrix family phi_{0,1,2}(sigma * A^c_mu)
  int c = 0, mu = 0;
  double sigma = 0.0;          // real part of the scale
  double sigma_im = 0.0;       // imaginary part (complex schemes: built on the real 2n x 2n
  int q = 0;                   //  embedding [[Re, -Im], [Im, Re]] of sigma A)
};

}  // namespace kx::detail

using kx::detail::BlockRecipe;
using kx::detail::Chain;
using kx::detail::Group;
using kx::detail::KX_MAXD;
using kx::detail::PhiStack;
using kx::detail::Stage;
using kx::MAXS;
using kx::MAXSEG;

constexpr int kTailMaxChunks = 8;

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
  int fused_small = 1;    // 1: small 2-D grids step in one cluster kernel (K*5, fused2d.cu)

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
  std::vector<BlockRecipe> recipes;   // how every stacked last-mode block was formed
  std::vector<double*> bank_allocs;
  int nslots = 0;

  // workspaces
  double* tmp1 = nullptr;
  double* tmp2 = nullptr;
  double* btmp[2] = {};          // kx_tucker_batched intermediates (grown on demand)
  size_t btmp_cap = 0;           // doubles per btmp buffer
  double* G[MAXS] = {};
  double* F[MAXS] = {};
  double* D[MAXS] = {};
  double* Us[MAXS] = {};
  double* W1[MAXS] = {};
  double* W2[MAXS] = {};
  std::vector<double*> ws_allocs;
  double* hostU[MAXS] = {};
  // kx_integrate_host: the last step's final stage GEMM runs in row chunks and each chunk's
  // rows are copied to the host on `copy` while the next chunk computes (one graph, cached per
  // host buffers and bank version)
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_tail[kTailMaxChunks + 1] = {};   // chunk k done; [kTailMaxChunks]: copies joined
  int tail_chunks = 4;
  bool tail_armed = false, tail_done = false;
  double* tail_host[MAXS] = {};
  cudaGraph_t tail_graph = nullptr;
  cudaGraphExec_t tail_gexec = nullptr;
  double* tail_key[MAXS] = {};   // host buffers the tail graph copies to
  double* tail_U[MAXS] = {};     // device state it steps
  long long tail_version = -1;
  kx_counters tail_delta{};
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
  double* halo_lo[MAXS] = {};   // tridiagonal K on a slab: the neighbours' boundary planes of U
  double* halo_hi[MAXS] = {};
  double* F_pack[MAXS] = {};
  // direct peer stores instead of exchanges (kx_group_set_p2p / kx_dist_ipc_import): every
  // rank's receive buffers, [rank][component]; valid until the workspaces are reallocated
  int p2p = 0;
  double* peerRA[kx::kMaxPeers][MAXS] = {};
  double* peerFB[kx::kMaxPeers][MAXS] = {};
  double* peerDB[kx::kMaxPeers][MAXS] = {};
  double* peerHlo[kx::kMaxPeers][MAXS] = {};
  double* peerHhi[kx::kMaxPeers][MAXS] = {};
  std::vector<void*> ipc_open;   // CUDA IPC mappings of the peers' buffers
  double* bar_buf = nullptr;     // scratch of the NCCL barrier
  // distributed operators (kx_tucker / kx_mode_product / kx_phi_apply on a sharded context):
  // pack, layout-B input, two layout-B intermediates, received chunks — Nloc doubles each
  double* dop[5] = {};
  std::vector<double*> dop_allocs;

  kx::detail::F32State* f32 = nullptr;   // fp32 variant (kx_*_f32), created on first use

  int nan_check = 0;             // per-step NaN/Inf watchdog inside the step graph
  int* watch = nullptr;          // device {steps completed, first bad step or -1}

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
  double prof_bytes = 0;        // algorithmic HBM bytes of the non-GEMM kernels
};

namespace kx::detail {

inline kx_status fail(kx_ctx* c, kx_status s, const std::string& m) {
  if (c) c->err = m;
  return s;
}

// Every ABI entry point runs on its context's device and leaves the caller's current device as
// it found it (distinct contexts on distinct devices in one process stay independent).
struct DevGuard {
  int prev = -1;
  explicit DevGuard(const kx_ctx* c) {
    int cur = -1;
    if (c && cudaGetDevice(&cur) == cudaSuccess && cur != c->device && cudaSetDevice(c->device) == cudaSuccess)
      prev = cur;
  }
  explicit DevGuard(int device) {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != device && cudaSetDevice(device) == cudaSuccess) prev = cur;
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DevGuard(const DevGuard&) = delete;
  DevGuard& operator=(const DevGuard&) = delete;
};

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

// ---- kx_core.cpp: launch wrappers, workspaces, tensor operations
cudaError_t record(kx_ctx* c, cudaEvent_t e);
cudaEvent_t pool_event(kx_ctx* c, int idx);
kx_status collect_profile(kx_ctx* c);
kx_status run_gemm(kx_ctx* c, const GemmArgs& g_in);
kx_status dalloc(kx_ctx* c, double** p, size_t count, std::vector<double*>& owner);
void free_list(std::vector<double*>& v);
void drop_graph(kx_ctx* c);
void drop_bank(kx_ctx* c);
long long prod_range(const kx_ctx* c, int lo, int hi);   // prod_{lo <= mu <= hi} tn_mu (1-based)
kx_status need_grid(kx_ctx* c);
kx_status mode_product_multi(kx_ctx* c, int ns, const double* const* X, double* const* Y,
                             int mu, const double* const* L, double alpha, double beta,
                             const double* const* Dd);
bool all_tridiag(const kx_ctx* c, int comp0, int ns);
kx_status kronsum_multi(kx_ctx* c, int comp0, int ns, const double* const* X, double* const* Y,
                        double beta, const double* const* Dd);
kx_status group_modes(kx_ctx* c, const Group& G, int t0, int nt, const double* const* X,
                      int slot, double* const** out_ws, const kx::PeerMap* peer = nullptr);
kx_status last_mode_concat(kx_ctx* c, double* const* ws, const double* const* src, int nseg,
                           const int* slots, double* const* B, double* const* Y, double alpha,
                           double beta, const double* const* Dd);
// the step's final stage GEMM: last_mode_concat, or (c->tail_armed) in row chunks, each copied
// to c->tail_host on c->copy as soon as it is written
kx_status final_concat(kx_ctx* c, double* const* ws, const double* const* src, int nseg,
                       const int* slots, double* const* B, double* const* Y, double alpha,
                       double beta, const double* const* Dd);
kx_status nonlin(kx_ctx* c, int mode, const double* const* u, double* const* out);
kx_status check_ptr(kx_ctx* c, const void* p, const char* what);
template <class F>
kx_status run_other(kx_ctx* c, F&& launch, double bytes = 0.0) {
  int e0 = -1;
  if (c->profiling) {
    e0 = c->ev_used;
    c->ev_used += 2;
    KX_CUDA(c, record(c, pool_event(c, e0)));
  }
  KX_CUDA(c, launch());
  if (c->profiling) {
    KX_CUDA(c, record(c, pool_event(c, e0 + 1)));
    c->recs.push_back({1, e0, e0 + 1, bytes});
  }
  c->cnt.other_launches += 1;
  return KX_OK;
}

// ---- kx_step.cpp: one-GPU schedules and graph capture
kx_status enqueue_step_etd3(kx_ctx* c, double* const* U);
kx_status enqueue_step_etd2(kx_ctx* c, double* const* U);
kx_status enqueue_step(kx_ctx* c, double* const* U);
kx_status enqueue_watch(kx_ctx* c, double* const* U);
bool fused_eligible(const kx_ctx* c);
kx_status enqueue_fused(kx_ctx* c, double* const* U, int nsteps);
kx_status step_impl(kx_ctx* c, double* const* U);
kx_status tail_step_impl(kx_ctx* c, double* const* U, double* const* U_host);
void drop_tail_graph(kx_ctx* c);
// ---- kx_bank.cpp: phi-bank formation
kx_status set_tau_impl(kx_ctx* c, double tau, kx_scheme scheme);
kx_status form_block(kx_ctx* c, const std::vector<Group>& groups, const BlockRecipe& r);
// ---- kx_f32.cpp: fp32 variant
void f32_drop_graph(kx_ctx* c);   // the captured fp32 step (model / settings changed)
void f32_drop(kx_ctx* c);         // + its bank planes and workspaces (bank changed)
void f32_free(kx_ctx* c);         // everything (context destroyed)
// ---- kx_dist.cpp: slab-sharded steps
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
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
#endif
  std::string why;
};
NcclApi& nccl();   // dlopen'ed once (the NCCL torch already loaded)
// Buffers one rank exchanges after a phase: for k < nbuf, chunk q (count doubles) of send[k]
// goes to rank q, which stores it at chunk `rank` of its recv[k].
// kind 0: all-to-all (above).  kind 1: halo — for each component s, send[2s] (this rank's
// first plane) goes to rank-1 and lands in its recv[2s+1]; send[2s+1] (last plane) goes to
// rank+1 and lands in its recv[2s]; the global end ranks skip the missing side.
struct Exchange {
  int kind = 0;   // 0 all-to-all, 1 halo, 2 none (direct peer stores: only a barrier)
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
void set_layout(kx_ctx* c, bool B);
bool p2p_on(const kx_ctx* c);
void p2p_close(kx_ctx* c);
kx_status dist_f_source(kx_ctx* c, double* const* U, Exchange& x);
kx_status dist_f_build(kx_ctx* c);
bool dist_banded(const kx_ctx* c);
kx_status dist_group(kx_ctx* c, int gi, double* const* Xb, Exchange& x);
kx_status dist_stage(kx_ctx* c, const Stage& S, double* const* out, const double* const* addend);
kx_status dist_d_source(kx_ctx* c, Exchange& x);
int dist_phases(const kx_ctx* c);
kx_status dist_phase(kx_ctx* c, double* const* U, int ph, Exchange& x);
kx_status nccl_exchange(kx_ctx* c, const Exchange& x, cudaStream_t st);
kx_status dist_step_nccl(kx_ctx* c, double* const* U);
// ---- kx_dist_ops.cpp: distributed operators (Tucker, mode product, split phi-action)
struct DistOp {
  int kind = 0;                      // 0 Tucker, 1 split phi-action, 2 mode product along mu = d,
                                     // 3 Kronecker-sum action (dense A_mu of component comp)
  const double* X = nullptr;         // layout-A slab (Nloc doubles)
  double* Y = nullptr;
  const double* L[KX_MAXD] = {};     // Tucker matrices / the mode-d matrix in L[d-1]
  double alpha = 1.0, beta = 0.0;
  int comp = 0;
  const PhiStack* ps = nullptr;
};
constexpr int kDistOpPhases = 3;
kx_status dist_op_phase(kx_ctx* c, const DistOp& op, int ph, Exchange& x);
kx_status dist_op_nccl(kx_ctx* c, const DistOp& op);
kx_status loopback_exchange(kx_ctx* const* ctxs, int nranks, const std::vector<Exchange>& xs);
void dop_free(kx_ctx* c);

}  // namespace kx::detail
