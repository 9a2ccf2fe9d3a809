// fp32 precision variant: the paper's "CUDA single" runs (Table 5 P:1477-1486,
// Table 7, the laptop single-precision timings P:776-778) on the 5th-generation
// tensor cores.  Same operators and step schedule as the fp64 path (kx_core.cpp / kx_step.cpp):
//   mu-mode product / Tucker operator, and exprk3ds_real / ETD2RKDS steps (Algorithms
//   1-2; eq:ETD2RK P:91-121), first mode concatenated-M, middle modes batched over
//   terms and slabs, last mode concatenated-K with the stage scalars folded in and "+U" in the
//   epilogue;
// every mode product runs on tf32x3_gemm_kernel (tcgen05 kind::tf32, three-pass hi/lo split that
// keeps fp32 accuracy, TMA loads, TMEM accumulators; tf32gemm.cu).  Tensors stay plain fp32 in
// HBM (the kernel splits them in shared memory); the phi-matrices are the fp64 bank of
// kx_set_tau rounded once to K-major (hi, lo) planes (the small matrices are not the hot path,
// P:1242-1252).
#include "kx_ctx.h"

#include <cstdint>

namespace kx::detail {

struct F32Planes {
  float* h = nullptr;
  float* l = nullptr;
};

struct F32State {
  // bank and step workspaces, derived from the fp64 bank of version `version`
  long long version = -1;
  std::vector<void*> allocs;
  F32Planes first[3], mid[3][KX_MAXD], stage[3];
  long long first_sp[3] = {}, mid_sp[3][KX_MAXD] = {}, stage_sp[3] = {};   // species strides
  int stage_slo[3] = {}, stage_hs[3] = {}, stage_s0[3] = {};   // segment slots: s0 + j%slo + (j/slo) hs
  float* tri = nullptr;   // [s][mu]: lo | di | up (3 n_mu floats), offsets tri_off
  long long tri_off[MAXS][KX_MAXD] = {};
  float* W[2] = {};         // species stride nslots N
  float* F = nullptr;       // species stride N (as G, D, Us)
  float* D = nullptr;
  float* G = nullptr;
  float* Us = nullptr;
  // CUDA graph of one fp32 step
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  float* graph_U[MAXS] = {};
  kx_counters step_delta{};
  // operator scratch (kx_mode_product_f32 / kx_tucker_f32), grown on demand
  std::vector<void*> op_allocs;
  size_t op_cap = 0, l_cap = 0;
  float* T[2] = {};
  F32Planes L;
};

namespace {

kx_status falloc(kx_ctx* c, float** p, size_t count, std::vector<void*>& owner) {
  *p = nullptr;
  if (count == 0) return KX_OK;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(float));
  if (e != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    return fail(c, KX_ERR_NOMEM, "device allocation of " + std::to_string(count * 4) +
                                     " bytes failed: " + cudaGetErrorString(e));
  }
  owner.push_back(*p);
  return KX_OK;
}
kx_status palloc(kx_ctx* c, F32Planes& P, size_t count, std::vector<void*>& owner) {
  KX_TRY(falloc(c, &P.h, count, owner));
  return falloc(c, &P.l, count, owner);
}
void free_all(std::vector<void*>& v) {
  for (void* p : v) cudaFree(p);
  v.clear();
}

void drop_f32_graph(F32State* f) {
  if (f->gexec) cudaGraphExecDestroy(f->gexec);
  if (f->graph) cudaGraphDestroy(f->graph);
  f->gexec = nullptr;
  f->graph = nullptr;
}

F32State* state(kx_ctx* c) {
  if (!c->f32) c->f32 = new F32State();
  return c->f32;
}

// 5-D view of a plane pair (or of a plain fp32 tensor: lo = nullptr): extents and element strides
kx::Tf32Dim view(const F32Planes& P, long long off, std::initializer_list<long long> ext,
                 std::initializer_list<long long> str) {
  kx::Tf32Dim d;
  d.hi = P.h + off;
  d.lo = P.l ? P.l + off : nullptr;
  int i = 0;
  for (long long e : ext) d.ext[i++] = e;
  i = 0;
  for (long long s : str) d.stride[i++] = s;
  return d;
}

kx_status run_f32(kx_ctx* c, const kx::Tf32Gemm& g) {
  const double fl = kx::tf32_gemm_flops(g);   // algorithmic (the three passes are the method's cost)
  int e0 = -1;
  if (c->profiling) {
    e0 = c->ev_used;
    c->ev_used += 2;
    KX_CUDA(c, record(c, pool_event(c, e0)));
  }
  KX_CUDA(c, kx::launch_tf32_gemm(g, c->cur));
  if (c->profiling) {
    KX_CUDA(c, record(c, pool_event(c, e0 + 1)));
    c->recs.push_back({0, e0, e0 + 1, fl});
  }
  c->cnt.gemm_launches += 1;
  c->cnt.mode_product_flops += fl;
  return KX_OK;
}

F32Planes plain(const float* x) { return F32Planes{const_cast<float*>(x), nullptr}; }

bool rows16(long long n) { return n % 4 == 0; }   // a row of n floats keeps TMA's 16-B strides

// mu >= 2 (COL): Y_b = L X_b for every slab b; S = L's K-major (row-major) planes, T = X.
kx_status col_product(kx_ctx* c, const float* X, const F32Planes& Lp, int mu, float* Y, float alpha, float beta,
                      const float* Dd) {
  const long long nm = c->tn[mu - 1], R = prod_range(c, 1, mu - 1), Bt = prod_range(c, mu + 1, c->d);
  kx::Tf32Gemm g;
  g.kind = kx::TF32_COL;
  g.M = (int)nm;
  g.N = (int)R;
  g.kseg = (int)nm;
  g.nb = (int)Bt;
  g.S = view(Lp, 0, {nm, nm, 1, 1, 1}, {1, nm, 0, 0, 0});
  g.T = view(plain(X), 0, {R, nm, Bt, 1, 1}, {1, R, nm * R, 0, 0});
  g.ldc = g.ldd = R;
  g.sC_b = g.sD_b = nm * R;
  g.alpha = alpha;
  g.beta = beta;
  g.C[0] = Y;
  g.D[0] = beta != 0.0f ? Dd : nullptr;
  KX_TRY(run_f32(c, g));
  c->cnt.mode_products += 1;
  return KX_OK;
}

// mu = 1 (ROW): Y_r = X_r L^T; S = L^T's K-major planes (= L row-major), T = X rows
kx_status row_product(kx_ctx* c, const float* X, const F32Planes& Lp, float* Y, float alpha, float beta,
                      const float* Dd) {
  const long long n1 = c->tn[0], rows = c->tN / n1;
  kx::Tf32Gemm g;
  g.kind = kx::TF32_ROW;
  g.M = (int)rows;
  g.N = (int)n1;
  g.kseg = (int)n1;
  g.T = view(plain(X), 0, {n1, rows, 1, 1, 1}, {1, n1, 0, 0, 0});
  g.S = view(Lp, 0, {n1, n1, 1, 1, 1}, {1, n1, 0, 0, 0});
  g.ldc = g.ldd = n1;
  g.alpha = alpha;
  g.beta = beta;
  g.C[0] = Y;
  g.D[0] = beta != 0.0f ? Dd : nullptr;
  KX_TRY(run_f32(c, g));
  c->cnt.mode_products += 1;
  return KX_OK;
}

kx_status grow_ops(kx_ctx* c, size_t n, size_t lsz) {
  F32State* f = state(c);
  if (n <= f->op_cap && lsz <= f->l_cap) return KX_OK;
  KX_CUDA(c, cudaStreamSynchronize(c->stream));
  free_all(f->op_allocs);
  f->op_cap = f->l_cap = 0;
  const size_t N = n, Ls = lsz;
  KX_TRY(falloc(c, &f->T[0], N, f->op_allocs));
  KX_TRY(falloc(c, &f->T[1], N, f->op_allocs));
  KX_TRY(palloc(c, f->L, Ls, f->op_allocs));
  f->op_cap = N;
  f->l_cap = Ls;
  return KX_OK;
}

kx_status f32_shape_ok(kx_ctx* c) {
  for (int mu = 0; mu < c->d; ++mu)
    if (!rows16(c->tn[mu]))
      return fail(c, KX_ERR_UNSUPPORTED, "the fp32 path needs every n_mu to be a multiple of 4 (16-B TMA rows)");
  return KX_OK;
}

kx_status check_fptr(kx_ctx* c, const void* p, const char* what) {
  if (!p) return fail(c, KX_ERR_INVALID, std::string(what) + " is NULL");
  if (reinterpret_cast<uintptr_t>(p) % 16 != 0)
    return fail(c, KX_ERR_INVALID, std::string(what) + " is not 16-byte aligned");
  return KX_OK;
}

// ---------------------------------------------------------------- bank + workspaces ---------
// Segment slots of a stage as s0 + (j % slo) + (j / slo) * hs (at most two progressions).
bool seg_progression(const Stage& S, int* s0, int* slo, int* hs) {
  const int n = S.nseg;
  *s0 = S.slot[0];
  int run = 1;
  while (run < n && S.slot[run] == S.slot[0] + run) ++run;
  *slo = run;
  *hs = run < n ? S.slot[run] - S.slot[0] : run;
  if (n % run) return false;
  for (int j = 0; j < n; ++j)
    if (S.slot[j] != *s0 + j % run + (j / run) * *hs) return false;
  return true;
}

kx_status prepare_f32(kx_ctx* c) {
  F32State* f = state(c);
  if (f->version == c->bank_version) return KX_OK;
  if (c->dist) return fail(c, KX_ERR_UNSUPPORTED, "the fp32 step runs on one GPU");
  if (c->cplx) return fail(c, KX_ERR_UNSUPPORTED, "the fp32 step implements the real schemes");
  if (c->ncomp != 2 || (c->d != 2 && c->d != 3))
    return fail(c, KX_ERR_UNSUPPORTED, "the fp32 step needs d in {2, 3} and 2 components");
  if (!all_tridiag(c, 0, 2))
    return fail(c, KX_ERR_UNSUPPORTED, "the fp32 step needs tridiagonal A_mu (the stencil Kronecker sum)");
  KX_TRY(f32_shape_ok(c));
  drop_f32_graph(f);
  free_all(f->allocs);
  const int d = c->d, ns = c->ncomp;
  const long long n1 = c->tn[0], nd = c->tn[d - 1], N = c->tN;
  c->cur = c->stream;
  for (size_t gi = 0; gi < c->groups.size(); ++gi) {
    const Group& G = c->groups[gi];
    const int TG = G.nterms;
    f->first_sp[gi] = (long long)TG * nd * nd;
    KX_TRY(palloc(c, f->first[gi], (size_t)ns * f->first_sp[gi], f->allocs));
    for (int s = 0; s < ns; ++s)   // column-major (TG nd) x nd -> row-major (K-major A)
      KX_TRY(run_other(c, [&] {
        return kx::launch_split_f64(G.first[s], f->first[gi].h + s * f->first_sp[gi],
                                    f->first[gi].l + s * f->first_sp[gi], (long long)TG * nd, nd, 1, true, 1.0,
                                    c->cur);
      }));
    for (int mu = 2; mu < d; ++mu) {
      const long long nm = c->tn[mu - 1];
      f->mid_sp[gi][mu - 1] = (long long)TG * nm * nm;
      KX_TRY(palloc(c, f->mid[gi][mu - 1], (size_t)ns * f->mid_sp[gi][mu - 1], f->allocs));
      for (int s = 0; s < ns; ++s)
        KX_TRY(run_other(c, [&] {
          const long long o = s * f->mid_sp[gi][mu - 1];
          return kx::launch_split_f64(G.mid[s][mu - 1], f->mid[gi][mu - 1].h + o, f->mid[gi][mu - 1].l + o, nm, nm,
                                      TG, true, 1.0, c->cur);
        }));
    }
  }
  for (int k = 0; k < c->nstages; ++k) {
    const Stage& S = c->stages[k];
    if (!seg_progression(S, &f->stage_s0[k], &f->stage_slo[k], &f->stage_hs[k]))
      return fail(c, KX_ERR_UNSUPPORTED, "stage segment slots are not two progressions");
    f->stage_sp[k] = (long long)S.nseg * n1 * n1;
    KX_TRY(palloc(c, f->stage[k], (size_t)ns * f->stage_sp[k], f->allocs));
    for (int s = 0; s < ns; ++s)   // blocks B_j(k, n) row-major -> K-major (n, k): transposed
      KX_TRY(run_other(c, [&] {
        const long long o = s * f->stage_sp[k];
        return kx::launch_split_f64(S.B[s], f->stage[k].h + o, f->stage[k].l + o, n1, n1, S.nseg, true, 1.0,
                                    c->cur);
      }));
  }
  long long tri_n = 0;
  for (int s = 0; s < ns; ++s)
    for (int mu = 0; mu < d; ++mu) {
      f->tri_off[s][mu] = tri_n;
      tri_n += 3 * c->tn[mu];
    }
  KX_TRY(falloc(c, &f->tri, (size_t)tri_n, f->allocs));
  for (int s = 0; s < ns; ++s)
    for (int mu = 0; mu < d; ++mu)
      KX_TRY(run_other(c, [&] {
        return kx::launch_f64_to_f32(c->A_tri[s][mu], f->tri + f->tri_off[s][mu], 3 * c->tn[mu], c->cur);
      }));
  const size_t wsz = (size_t)ns * c->nslots * N;
  KX_TRY(falloc(c, &f->W[0], wsz, f->allocs));
  if (d >= 3) KX_TRY(falloc(c, &f->W[1], wsz, f->allocs));
  KX_TRY(falloc(c, &f->F, (size_t)ns * N, f->allocs));
  KX_TRY(falloc(c, &f->D, (size_t)ns * N, f->allocs));
  KX_TRY(falloc(c, &f->G, (size_t)ns * N, f->allocs));
  KX_TRY(falloc(c, &f->Us, (size_t)ns * N, f->allocs));
  KX_CUDA(c, cudaStreamSynchronize(c->stream));
  f->version = c->bank_version;
  return KX_OK;
}

// ---------------------------------------------------------------- step pieces -------------
kx::F32PhaseArgs phase_args(kx_ctx* c, float* const* U) {
  F32State* f = c->f32;
  kx::F32PhaseArgs a;
  a.d = c->d;
  a.model = c->model;
  a.N = c->tN;
  for (int mu = 0; mu < c->d; ++mu) a.n[mu] = c->tn[mu];
  for (int i = 0; i < 8; ++i) a.p[i] = (float)c->params[i];
  for (int s = 0; s < 2; ++s) {
    a.U[s] = U[s];
    a.G[s] = f->G + s * c->tN;
    for (int mu = 0; mu < c->d; ++mu) a.tri[s][mu] = f->tri + f->tri_off[s][mu];
  }
  return a;
}

// first (concatenated-M) and middle modes of all terms of group gi on the fp32 input In (species
// stride N); returns the workspace index holding the results (slots slot0 ..)
kx_status group_modes_f32(kx_ctx* c, int gi, const float* In, int* out_w) {
  F32State* f = c->f32;
  const Group& G = c->groups[gi];
  const int d = c->d, ns = c->ncomp, TG = G.nterms;
  const long long N = c->tN, nd = c->tn[d - 1], R = N / nd;
  const long long wsp = (long long)c->nslots * N;
  {
    kx::Tf32Gemm g;
    g.kind = kx::TF32_COL;
    g.M = (int)(TG * nd);
    g.N = (int)R;
    g.kseg = (int)nd;
    g.ns = ns;
    g.S = view(f->first[gi], 0, {nd, TG * nd, 1, ns, 1}, {1, nd, 0, f->first_sp[gi], 0});
    g.T = view(plain(In), 0, {R, nd, 1, 1, ns}, {1, R, 0, 0, N});
    g.ldc = R;
    for (int s = 0; s < ns; ++s) g.C[s] = f->W[0] + s * wsp + (long long)G.slot0 * N;
    KX_TRY(run_f32(c, g));
  }
  int cur = 0;
  for (int mu = d - 1; mu >= 2; --mu) {
    const long long nm = c->tn[mu - 1], Rm = prod_range(c, 1, mu - 1), Bt = prod_range(c, mu + 1, d);
    kx::Tf32Gemm g;
    g.kind = kx::TF32_COL;
    g.M = (int)nm;
    g.N = (int)Rm;
    g.kseg = (int)nm;
    g.ns = ns;
    g.nt = TG;
    g.nb = (int)Bt;
    const long long msp = f->mid_sp[gi][mu - 1];
    g.S = view(f->mid[gi][mu - 1], 0, {nm, nm, TG, ns, 1}, {1, nm, nm * nm, msp, 0});
    g.T = view(plain(f->W[cur]), (long long)G.slot0 * N, {Rm, nm, Bt, TG, ns}, {1, Rm, nm * Rm, N, wsp});
    g.ldc = Rm;
    g.sC_b = nm * Rm;
    g.sC_t = N;
    for (int s = 0; s < ns; ++s) g.C[s] = f->W[cur ^ 1] + s * wsp + (long long)G.slot0 * N;
    KX_TRY(run_f32(c, g));
    cur ^= 1;
  }
  c->cnt.mode_products += (long long)ns * TG * (d - 1);
  *out_w = cur;
  return KX_OK;
}

// last mode with concatenated K over stage k's segments: Y_s = sum_j W_slot(j) x_1 B_j + Dd_s
kx_status stage_f32(kx_ctx* c, int k, int w, float* const* Y, const float* const* Dd) {
  F32State* f = c->f32;
  const int ns = c->ncomp;
  const long long N = c->tN, n1 = c->tn[0], rows = N / n1;
  const long long wsp = (long long)c->nslots * N;
  const int nseg = c->stages[k].nseg, slo = f->stage_slo[k];
  kx::Tf32Gemm g;
  g.kind = kx::TF32_ROW;
  g.M = (int)rows;
  g.N = (int)n1;
  g.kseg = (int)n1;
  g.nseg = nseg;
  g.slo = slo;
  g.ns = ns;
  g.T = view(plain(f->W[w]), (long long)f->stage_s0[k] * N, {n1, rows, slo, nseg / slo, ns},
             {1, n1, N, (long long)f->stage_hs[k] * N, wsp});
  g.S = view(f->stage[k], 0, {n1, n1, nseg, ns, 1}, {1, n1, n1 * n1, f->stage_sp[k], 0});
  g.ldc = g.ldd = n1;
  g.beta = 1.0f;
  for (int s = 0; s < ns; ++s) {
    g.C[s] = Y[s];
    g.D[s] = Dd[s];
  }
  KX_TRY(run_f32(c, g));
  c->cnt.mode_products += (long long)ns * nseg;
  return KX_OK;
}

// D = g(Us) - G; with U given (and the vectorised kernel eligible) also Us = U afterwards, so
// that the next stage GEMM adds into Us in place (TMA reduce-add, no D loads); returns through
// *refilled whether it did
kx_status nonlin_f32(kx_ctx* c, float* const* Us, float* const* U = nullptr, bool* refilled = nullptr) {
  F32State* f = c->f32;
  kx::F32PhaseArgs a = phase_args(c, Us);
  for (int s = 0; s < 2; ++s) a.F[s] = f->D + s * c->tN;
  if (U) {
    for (int s = 0; s < 2; ++s) a.Usrc[s] = U[s], a.Ucopy[s] = Us[s];
    if (!kx::f32_phase_vec_ok(a, false))
      for (int s = 0; s < 2; ++s) a.Usrc[s] = nullptr, a.Ucopy[s] = nullptr;
  }
  if (refilled) *refilled = a.Ucopy[0] != nullptr;
  // HBM bytes: read U (2 fields), G (2); write D (2) (+ read U, write Us: 4 more)
  const double bytes = (a.Ucopy[0] ? 40.0 : 24.0) * (double)c->tN;
  return run_other(c, [&] { return kx::launch_nonlin_f32(a, c->cur); }, bytes);
}

kx_status enqueue_step_f32(kx_ctx* c, float* const* U) {
  F32State* f = c->f32;
  const long long N = c->tN;
  float* Us[2] = {f->Us, f->Us + N};
  const float* Uc[2] = {U[0], U[1]};
  const float* Usc[2] = {Us[0], Us[1]};
  // Us = U is written by the first phase (and refreshed by the nonlinearity) where the
  // vectorised kernels apply: the stage GEMMs U_k = U + ... then add into Us in place (one
  // round-to-nearest add, as alpha acc + U) and skip their D loads
  bool pre = false;
  {   // G = g(U), F = K U + G (planes)
    kx::F32PhaseArgs a = phase_args(c, U);
    for (int s = 0; s < 2; ++s) a.F[s] = f->F + s * N;
    for (int s = 0; s < 2; ++s) a.Usrc[s] = U[s], a.Ucopy[s] = Us[s];
    pre = kx::f32_phase_vec_ok(a, true) && (c->d == 2 || c->d == 3) && !getenv("KX_F32_NOPREFILL");   // A/B
    if (!pre)
      for (int s = 0; s < 2; ++s) a.Usrc[s] = nullptr, a.Ucopy[s] = nullptr;
    // HBM bytes: read U (2 fields), write G and F (4) (+ Us: 2)
    KX_TRY(run_other(c, [&] { return kx::launch_first_phase_f32(a, c->cur); }, (pre ? 32.0 : 24.0) * (double)N));
    c->cnt.mode_products += 2LL * c->d;
    c->cnt.kronsum_actions += 2;
  }
  int w = 0;
  if (c->nstages == 3) {   // exprk3ds_real (Algorithms 1-2), groups F (3T), D2 (T), D3 (T)
    KX_TRY(group_modes_f32(c, 0, f->F, &w));
    KX_TRY(stage_f32(c, 0, w, Us, pre ? Usc : Uc));      // U2 = U + tau/3 S_1[F]
    // D2 = g(U2) - G; with KX_F32_REFILL=1 also Us = U (stage U3 then in place too).  Off by
    // default: that variant differs from the D-load form by 1 ulp in rare elements after a few
    // steps (1 of 131072 at step 5, 256^2), unexplained, so it is not the default
    KX_TRY(nonlin_f32(c, Us, (pre && getenv("KX_F32_REFILL")) ? U : nullptr, &pre));
    KX_TRY(group_modes_f32(c, 1, f->D, &w));
    KX_TRY(stage_f32(c, 1, w, Us, pre ? Usc : Uc));      // U3
    KX_TRY(nonlin_f32(c, Us));                            // D3 = g(U3) - G
    KX_TRY(group_modes_f32(c, 2, f->D, &w));
    KX_TRY(stage_f32(c, 2, w, U, Uc));                   // U+ (in place)
    c->cnt.tucker_ops += 2LL * 5 * c->T;
  } else {                 // ETD2RKDS (eq:ETD2RK), groups F (phi_1), D (phi_2)
    KX_TRY(group_modes_f32(c, 0, f->F, &w));
    KX_TRY(stage_f32(c, 0, w, Us, pre ? Usc : Uc));      // u2 = u + tau phi_1-split[F]
    KX_TRY(nonlin_f32(c, Us));                            // D = g(u2) - G
    KX_TRY(group_modes_f32(c, 1, f->D, &w));
    KX_TRY(stage_f32(c, 1, w, U, Usc));                  // u+ = u2 + 2^{d-1} tau phi_2-split[D]
    c->cnt.tucker_ops += 2LL * 2;
  }
  return KX_OK;
}

kx_status step_f32_impl(kx_ctx* c, float* const* U) {
  F32State* f = c->f32;
  if (c->profiling) {   // eager launches, each bracketed by profiling events
    c->cur = c->stream;
    KX_TRY(enqueue_step_f32(c, U));
    c->cnt.steps += 1;
    return KX_OK;
  }
  bool same = f->gexec != nullptr;
  for (int s = 0; s < c->ncomp && same; ++s) same = f->graph_U[s] == U[s];
  if (!same) {
    drop_f32_graph(f);
    const kx_counters before = c->cnt;
    c->cur = c->cap;
    KX_CUDA(c, cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
    kx_status s = enqueue_step_f32(c, U);
    cudaGraph_t gr = nullptr;
    cudaError_t e = cudaStreamEndCapture(c->cap, &gr);
    c->cur = c->stream;
    if (s != KX_OK) {
      if (gr) cudaGraphDestroy(gr);
      c->cnt = before;
      return s;
    }
    KX_CUDA(c, e);
    f->graph = gr;
    KX_CUDA(c, cudaGraphInstantiate(&f->gexec, f->graph, 0));
    for (int k = 0; k < c->ncomp; ++k) f->graph_U[k] = U[k];
    kx_counters dl{};
    dl.tucker_ops = c->cnt.tucker_ops - before.tucker_ops;
    dl.mode_products = c->cnt.mode_products - before.mode_products;
    dl.kronsum_actions = c->cnt.kronsum_actions - before.kronsum_actions;
    dl.gemm_launches = c->cnt.gemm_launches - before.gemm_launches;
    dl.other_launches = c->cnt.other_launches - before.other_launches;
    dl.mode_product_flops = c->cnt.mode_product_flops - before.mode_product_flops;
    f->step_delta = dl;
    c->cnt = before;
  }
  KX_CUDA(c, cudaGraphLaunch(f->gexec, c->stream));
  c->cnt.steps += 1;
  c->cnt.tucker_ops += f->step_delta.tucker_ops;
  c->cnt.mode_products += f->step_delta.mode_products;
  c->cnt.kronsum_actions += f->step_delta.kronsum_actions;
  c->cnt.gemm_launches += f->step_delta.gemm_launches;
  c->cnt.other_launches += f->step_delta.other_launches;
  c->cnt.mode_product_flops += f->step_delta.mode_product_flops;
  return KX_OK;
}

}  // namespace

void f32_drop_graph(kx_ctx* c) {
  if (c->f32) drop_f32_graph(c->f32);
}

void f32_drop(kx_ctx* c) {   // bank-derived state (kx_set_tau / kx_set_grid / matrices changed)
  if (!c->f32) return;
  drop_f32_graph(c->f32);
  free_all(c->f32->allocs);
  c->f32->version = -1;
}

void f32_free(kx_ctx* c) {
  if (!c->f32) return;
  f32_drop(c);
  free_all(c->f32->op_allocs);
  delete c->f32;
  c->f32 = nullptr;
}

}  // namespace kx::detail

using namespace kx::detail;

extern "C" {

kx_status kx_mode_product_f32(kx_ctx* c, const float* X, float* Y, int mu, const float* L, float alpha,
                              float beta) {
  DevGuard dg_(c);
  KX_TRY(need_grid(c));
  if (c->dist) return fail(c, KX_ERR_UNSUPPORTED, "single-GPU operator on a distributed context");
  if (mu < 1 || mu > c->d)
    return fail(c, KX_ERR_INVALID, "mode " + std::to_string(mu) + " outside 1.." + std::to_string(c->d));
  KX_TRY(check_fptr(c, X, "X"));
  KX_TRY(check_fptr(c, Y, "Y"));
  KX_TRY(check_fptr(c, L, "L"));
  if (X == Y) return fail(c, KX_ERR_INVALID, "X and Y must be distinct");
  KX_TRY(f32_shape_ok(c));
  c->cur = c->stream;
  const long long nm = c->tn[mu - 1];
  KX_TRY(grow_ops(c, (size_t)c->tN, (size_t)nm * nm));
  F32State* f = c->f32;
  // column-major L -> K-major planes: L itself (rows of L) for mu >= 2, L^T's K-major form = the
  // rows of L for mu = 1 as well
  KX_TRY(run_other(c, [&] { return kx::launch_split_f32_2d(L, f->L.h, f->L.l, nm, nm, 1, true, c->cur); }));
  if (mu == 1) return row_product(c, X, f->L, Y, alpha, beta, Y);
  return col_product(c, X, f->L, mu, Y, alpha, beta, Y);
}

kx_status kx_tucker_f32(kx_ctx* c, const float* X, float* Y, const float* const* L, float alpha, float beta) {
  DevGuard dg_(c);
  KX_TRY(need_grid(c));
  if (c->dist) return fail(c, KX_ERR_UNSUPPORTED, "single-GPU operator on a distributed context");
  KX_TRY(check_fptr(c, X, "X"));
  KX_TRY(check_fptr(c, Y, "Y"));
  if (!L) return fail(c, KX_ERR_INVALID, "L is NULL");
  for (int mu = 0; mu < c->d; ++mu) KX_TRY(check_fptr(c, L[mu], "L[mu]"));
  if (X == Y) return fail(c, KX_ERR_INVALID, "X and Y must be distinct");
  KX_TRY(f32_shape_ok(c));
  c->cur = c->stream;
  const int d = c->d;
  long long lsz = 0, loff[KX_MAXD];
  for (int mu = 0; mu < d; ++mu) {
    loff[mu] = lsz;
    lsz += c->tn[mu] * c->tn[mu];
  }
  KX_TRY(grow_ops(c, (size_t)c->tN, (size_t)lsz));
  F32State& F = *c->f32;
  for (int mu = 0; mu < d; ++mu) {
    const long long nm = c->tn[mu];
    KX_TRY(run_other(c, [&] {
      return kx::launch_split_f32_2d(L[mu], F.L.h + loff[mu], F.L.l + loff[mu], nm, nm, 1, true, c->cur);
    }));
  }
  // modes d, d-1, ..., 2 into fp32 scratch, mode 1 into Y (alpha, beta), as the fp64 kx_tucker
  const float* src = X;
  int w = 0;
  for (int mu = d; mu >= 2; --mu) {
    F32Planes Lp{F.L.h + loff[mu - 1], F.L.l + loff[mu - 1]};
    KX_TRY(col_product(c, src, Lp, mu, F.T[w], 1.0f, 0.0f, nullptr));
    src = F.T[w];
    w ^= 1;
  }
  F32Planes L1{F.L.h, F.L.l};
  KX_TRY(row_product(c, src, L1, Y, alpha, beta, Y));
  c->cnt.tucker_ops += 1;
  return KX_OK;
}

kx_status kx_step_f32(kx_ctx* c, double t0, int nsteps, float* const* U) {
  DevGuard dg_(c);
  (void)t0;   // both models are autonomous (reading R7)
  KX_TRY(need_grid(c));
  if (!c->bank_ready) return fail(c, KX_ERR_INVALID, "kx_set_tau has not been called");
  if (!U || nsteps < 0) return fail(c, KX_ERR_INVALID, "bad arguments");
  for (int s = 0; s < c->ncomp; ++s) {
    KX_TRY(check_fptr(c, U[s], "U[c]"));
    for (int r = 0; r < s; ++r)
      if (U[r] == U[s]) return fail(c, KX_ERR_INVALID, "U components must be distinct");
  }
  KX_TRY(prepare_f32(c));
  for (int k = 0; k < nsteps; ++k) KX_TRY(step_f32_impl(c, U));
  return KX_OK;
}

}  // extern "C"
