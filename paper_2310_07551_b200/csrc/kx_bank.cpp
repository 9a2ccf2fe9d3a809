// phi-bank formation on the device (kx_set_tau) and its layout.
#include "kx_ctx.h"

namespace kx::detail {

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

// Last-mode blocks: the real part of kappa * eta_t * (W_t x_1 P_t{1}) for a complex term is
//   W_re x_1 Re(kappa eta P) + W_im x_1 (-Im(kappa eta P)),
// so a term contributes the blocks [Re(kappa eta P); -Im(kappa eta P)] over its two slots.
kx_status form_block(kx_ctx* c, const std::vector<Group>& groups, const BlockRecipe& r) {
  const long long n1 = c->n[0];
  const long long m2 = n1 * n1;
  const Group& G = groups[r.gi];
  double* dst = r.dst;
  if (!c->cplx) {
    const double* src = G.last[r.comp] + r.t * m2;
    const double k = r.kre;
    return run_other(c, [&] { return kx::launch_scale(dst, src, k, m2, c->cur); });
  }
  const double* Pre = G.last[r.comp] + (2 * r.t) * m2;
  const double* Pim = G.last[r.comp] + (2 * r.t + 1) * m2;
  const double kre = r.kre, kim = r.kim;
  KX_TRY(run_other(c, [&] { return kx::launch_axpby(dst, kre, Pre, -kim, Pim, m2, c->cur); }));
  return run_other(c, [&] { return kx::launch_axpby(dst + m2, -kre, Pim, -kim, Pre, m2, c->cur); });
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
  // every scaled last-mode block is recorded (kx_set_phi_matrix re-forms it from the bank)
  c->recipes.clear();
  auto put_blocks = [&](double* dst, int gi, int comp, int t, double kre, double kim) -> kx_status {
    BlockRecipe r;
    r.gi = gi;
    r.t = t;
    r.comp = comp;
    r.kre = kre;
    r.kim = kim;
    r.dst = dst;
    c->recipes.push_back(r);
    return form_block(c, groups, r);
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
      KX_TRY(wal(&c->F_pack[comp], N));
      const size_t plane = N / (size_t)c->nA[d - 1];
      KX_TRY(wal(&c->halo_lo[comp], plane));
      KX_TRY(wal(&c->halo_hi[comp], plane));
    }
  }
  KX_CUDA(c, cudaStreamSynchronize(c->cur));
  c->bank_ready = true;
  c->bank_version += 1;
  return KX_OK;
}

}  // namespace kx::detail
