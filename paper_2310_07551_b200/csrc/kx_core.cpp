// Launch wrappers (profiling events), workspace helpers, and the tensor operations of the
// path as sequences of GEMM / pointwise launches: mu-mode products, Kronecker sums, the first
// and middle modes of a group of split terms, the concatenated-K last mode, g.
#include "kx_ctx.h"

namespace kx::detail {

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
  f32_drop_graph(c);
  drop_tail_graph(c);
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
  f32_drop(c);
  p2p_close(c);   // the peers' mappings point at buffers about to be reallocated
  free_list(c->bank_allocs);
  free_list(c->ws_allocs);
  c->groups.clear();
  c->phi.clear();
  c->recipes.clear();
  for (auto& s : c->stages) s = Stage{};
  c->nstages = 0;
  c->bank_ready = false;
  for (int s = 0; s < MAXS; ++s) {
    c->G[s] = c->F[s] = c->D[s] = c->Us[s] = c->W1[s] = c->W2[s] = nullptr;
    c->RA[s] = c->T1G_pack[s] = c->U_pack[s] = c->T1G_B[s] = c->U_B[s] = c->F_B[s] = nullptr;
    c->D_pack[s] = c->D_B[s] = nullptr;
    c->halo_lo[s] = c->halo_hi[s] = c->F_pack[s] = nullptr;
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
    const double bytes = 8.0 * (double)c->tN * ns * ((Dd && beta != 0.0) ? 3 : 2);
    KX_TRY(run_other(c, [&] { return kx::launch_kronsum_tridiag(a, c->cur); }, bytes));
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
                      int slot, double* const** out_ws, const kx::PeerMap* peer) {
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
    if (peer && d == 2) {   // the final product of the group: store straight into the peers
      g.peer = *peer;
      for (int s = 0; s < ns; ++s) g.peer.local_base[s] = c->W1[s];
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
    if (peer && mu == 2) {   // the final product of the group: store straight into the peers
      g.peer = *peer;
      for (int s = 0; s < ns; ++s) g.peer.local_base[s] = nxt[s];
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
namespace {
// rows [r0, r1) of the concatenated-K last-mode GEMM (row = one i_1 line of the output)
kx_status concat_rows(kx_ctx* c, double* const* ws, const double* const* src, int nseg,
                      const int* slots, double* const* B, double* const* Y, double alpha,
                      double beta, const double* const* Dd, long long r0, long long r1) {
  const long long n1 = c->tn[0];
  GemmArgs g;
  g.arow = true;
  g.M = (int)(r1 - r0);
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
  const long long off = r0 * n1;
  for (int s = 0; s < c->ncomp; ++s) {
    g.A[s] = (ws ? ws[s] : src[s]) + off;
    g.B[s] = B[s];
    g.C[s] = Y[s] + off;
    g.D[s] = (Dd && beta != 0.0) ? Dd[s] + off : nullptr;
  }
  return run_gemm(c, g);
}
}  // namespace

kx_status last_mode_concat(kx_ctx* c, double* const* ws, const double* const* src, int nseg,
                           const int* slots, double* const* B, double* const* Y, double alpha,
                           double beta, const double* const* Dd) {
  KX_TRY(concat_rows(c, ws, src, nseg, slots, B, Y, alpha, beta, Dd, 0, c->tN / c->tn[0]));
  c->cnt.mode_products += (long long)c->ncomp * nseg;
  return KX_OK;
}

kx_status final_concat(kx_ctx* c, double* const* ws, const double* const* src, int nseg,
                       const int* slots, double* const* B, double* const* Y, double alpha,
                       double beta, const double* const* Dd) {
  if (!c->tail_armed) return last_mode_concat(c, ws, src, nseg, slots, B, Y, alpha, beta, Dd);
  const long long n1 = c->tn[0], M = c->tN / n1;
  const int P = (int)std::max<long long>(1, std::min<long long>(std::min(c->tail_chunks, kTailMaxChunks), M));
  // shrinking chunks (weights P, P-1, ..., 1): each chunk's copy hides under the next chunk's
  // GEMM and the last, unhidden copy is the smallest.  Whole 128-row tile rows per chunk
  // (largest-remainder rounding); grids with fewer tile rows than chunks take one chunk.
  // Copy-bound tails (the copy of a chunk outlasts the next chunk's GEMM: C3) keep equal chunks.
  const double copy_us = 8.0 * c->ncomp * (double)c->tN / 50e3;   // ~50 GB/s D2H
  const double gemm_us = 2.0 * c->ncomp * (double)c->tN * n1 * nseg / 30e6;   // ~30 TF/s
  const bool shrink = copy_us < gemm_us;
  const long long TR = (M + 127) / 128, W = shrink ? (long long)P * (P + 1) / 2 : P;
  long long rows_of[kTailMaxChunks] = {}, used = 0;
  double rem[kTailMaxChunks];
  for (int k = 0; k < P; ++k) {
    const double want = (double)TR * (shrink ? P - k : 1) / (double)W;
    rows_of[k] = (long long)want;
    rem[k] = want - (double)rows_of[k];
    used += rows_of[k];
  }
  for (; used < TR; ++used) {
    int best = 0;
    for (int k = 1; k < P; ++k)
      if (rem[k] > rem[best]) best = k;
    rows_of[best] += 1;
    rem[best] = -1.0;
  }
  long long bound[kTailMaxChunks + 1];
  bound[0] = 0;
  for (int k = 0; k < P; ++k) bound[k + 1] = std::min(M, bound[k] + 128 * (TR < P ? (k == 0 ? TR : 0) : rows_of[k]));
  bound[P] = M;
  for (int k = 0; k < P; ++k) {
    const long long r0 = bound[k], r1 = bound[k + 1];
    if (r1 <= r0) continue;
    KX_TRY(concat_rows(c, ws, src, nseg, slots, B, Y, alpha, beta, Dd, r0, r1));
    KX_CUDA(c, cudaEventRecord(c->ev_tail[k], c->cur));
    KX_CUDA(c, cudaStreamWaitEvent(c->copy, c->ev_tail[k], 0));
    for (int s = 0; s < c->ncomp; ++s)
      KX_CUDA(c, cudaMemcpyAsync(c->tail_host[s] + r0 * n1, Y[s] + r0 * n1, (size_t)((r1 - r0) * n1) * 8,
                                 cudaMemcpyDeviceToHost, c->copy));
  }
  c->cnt.mode_products += (long long)c->ncomp * nseg;
  c->tail_done = true;
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
  // HBM bytes: read the ncomp fields (+ G for mode 1), write ncomp fields
  const double bytes = 8.0 * (double)c->tN * c->ncomp * (mode == 1 ? 3 : 2);
  return run_other(c, [&] { return kx::launch_nonlinearity(a, mode, c->cur); }, bytes);
}

kx_status collect_profile(kx_ctx* c) {
  if (c->recs.empty()) return KX_OK;
  KX_CUDA(c, cudaStreamSynchronize(c->stream));
  for (const auto& r : c->recs) {
    float ms = 0;
    KX_CUDA(c, cudaEventElapsedTime(&ms, c->ev_pool[r.e0], c->ev_pool[r.e1]));
    c->prof_ms[r.cls] += ms;
    c->prof_launches[r.cls] += 1;
    (r.cls == 0 ? c->prof_flops : c->prof_bytes) += r.flops;
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

}  // namespace kx::detail
