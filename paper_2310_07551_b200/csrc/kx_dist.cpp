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
#include <dlfcn.h>

#include "kx_ctx.h"

namespace kx::detail {

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
  api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv &&
           api.GroupStart && api.GroupEnd && api.GetErrorString && api.AllReduce;
  if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
#else
  api.why = "built without nccl.h";
#endif
  return api;
}


// ---- direct peer stores (P2P mode) ------------------------------------------------------
// The producing kernel of every exchange stores block q of its peer-packed output straight
// into rank q's receive buffer (kx::PeerMap); an exchange then reduces to a barrier between
// the producing and the consuming phase (stream order in an in-process group, a one-double
// NCCL all-reduce across processes).  Real schemes with the tridiagonal (halo) schedule.
bool dist_banded(const kx_ctx* c);
bool p2p_on(const kx_ctx* c) {
  // peer_redirect works in 32-bit offsets: every redirected buffer (nslots x Nloc) must fit
  return c->p2p && !c->cplx && dist_banded(c) && (long long)c->nslots * c->Nloc < (1LL << 31);
}

void p2p_close(kx_ctx* c) {
  for (void* p : c->ipc_open) cudaIpcCloseMemHandle(p);
  c->ipc_open.clear();
  c->p2p = 0;
  for (int q = 0; q < kx::kMaxPeers; ++q)
    for (int s = 0; s < MAXS; ++s)
      c->peerRA[q][s] = c->peerFB[q][s] = c->peerDB[q][s] = c->peerHlo[q][s] = c->peerHhi[q][s] = nullptr;
}

kx::PeerMap peer_map(const kx_ctx* c, double* const (*peers)[MAXS], double* const* local) {
  kx::PeerMap pm;
  pm.P = c->nranks;
  pm.rank = c->rank;
  pm.chunk = c->Nloc / c->nranks;
  pm.span = c->Nloc;
  for (int s = 0; s < c->ncomp; ++s) {
    pm.local_base[s] = local ? local[s] : nullptr;
    for (int q = 0; q < c->nranks; ++q) pm.peer_base[s][q] = peers[q][s];
  }
  return pm;
}

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
  if (p2p_on(c)) {   // the final mode product stores every term slot straight into the peers
    const kx::PeerMap pm = peer_map(c, c->peerRA, nullptr);
    KX_TRY(group_modes(c, G, 0, G.nterms, Xb, G.slot0, &ws, &pm));
    x.kind = 2;
    return KX_OK;
  }
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
  if (p2p_on(c)) a.peer = peer_map(c, c->peerDB, c->D_pack);
  KX_TRY(run_other(c, [&] { return kx::launch_nonlinearity(a, 1, c->cur); }));
  if (p2p_on(c)) {
    x.kind = 2;
    return KX_OK;
  }
  x.count = (size_t)(c->Nloc / c->nranks);
  for (int s = 0; s < c->ncomp; ++s) x.add(c->D_pack[s], c->D_B[s]);
  return KX_OK;
}

// Tridiagonal A_mu (the FD Laplacians of Sec. 3): the Kronecker sum is a stencil; on a slab
// only the two boundary planes of U cross ranks (a halo exchange with the neighbours), and F is
// formed locally in layout A and written peer-packed — one all-to-all instead of two, and no
// dense Kronecker-sum mode products.
bool dist_banded(const kx_ctx* c) { return all_tridiag(c, 0, c->ncomp); }

// [A] G = g(U); the boundary planes of U go to the neighbouring ranks
kx_status dist_f_halo(kx_ctx* c, double* const* U, Exchange& x) {
  set_layout(c, false);
  KX_TRY(nonlin(c, 0, U, c->G));
  const long long ndl = c->nA[c->d - 1];
  const long long plane = c->Nloc / ndl;
  if (p2p_on(c)) {   // boundary planes straight into the neighbours' halo buffers (copy engine)
    for (int s = 0; s < c->ncomp; ++s) {
      if (c->rank > 0)
        KX_CUDA(c, cudaMemcpyAsync(c->peerHhi[c->rank - 1][s], U[s], plane * 8, cudaMemcpyDeviceToDevice, c->cur));
      if (c->rank + 1 < c->nranks)
        KX_CUDA(c, cudaMemcpyAsync(c->peerHlo[c->rank + 1][s], U[s] + (ndl - 1) * plane, plane * 8,
                                   cudaMemcpyDeviceToDevice, c->cur));
    }
    x.kind = 2;
    return KX_OK;
  }
  x.kind = 1;
  x.count = (size_t)plane;
  for (int s = 0; s < c->ncomp; ++s) {
    x.add(U[s], c->halo_lo[s]);
    x.add(U[s] + (ndl - 1) * plane, c->halo_hi[s]);
  }
  return KX_OK;
}

// [A] F = G + sum_mu U x_mu A_mu (stencil, halos for the sharded direction), peer-packed
kx_status dist_f_stencil(kx_ctx* c, double* const* U, Exchange& x) {
  set_layout(c, false);
  kx::StencilArgs a;
  a.d = c->d;
  a.ns = c->ncomp;
  a.N = c->Nloc;
  a.beta = 1.0;
  for (int mu = 0; mu < c->d; ++mu) a.n[mu] = c->nA[mu];
  a.d_off = (long long)c->rank * c->nA[c->d - 1];
  a.n_glob_d = c->n[c->d - 1];
  a.pack_n1 = c->n[0];
  a.pack_n1l = c->n[0] / c->nranks;
  for (int s = 0; s < c->ncomp; ++s) {
    a.X[s] = U[s];
    a.Y[s] = c->F_pack[s];
    a.Dd[s] = c->G[s];
    a.halo_lo[s] = c->halo_lo[s];
    a.halo_hi[s] = c->halo_hi[s];
    for (int mu = 0; mu < c->d; ++mu) {
      const double* t = c->A_tri[s][mu];
      const long long n = c->n[mu];
      a.lo[s][mu] = t;
      a.di[s][mu] = t + n;
      a.up[s][mu] = t + 2 * n;
    }
  }
  if (p2p_on(c)) a.peer = peer_map(c, c->peerFB, c->F_pack);
  KX_TRY(run_other(c, [&] { return kx::launch_kronsum_tridiag(a, c->cur); }));
  c->cnt.mode_products += (long long)c->ncomp * c->d;
  c->cnt.kronsum_actions += c->ncomp;
  if (p2p_on(c)) {
    x.kind = 2;
    return KX_OK;
  }
  x.count = (size_t)(c->Nloc / c->nranks);
  for (int s = 0; s < c->ncomp; ++s) x.add(c->F_pack[s], c->F_B[s]);
  return KX_OK;
}

int dist_phases(const kx_ctx* c) {
  return (c->scheme == KX_ETD2RKDS ? 5 : 7) + (dist_banded(c) ? 1 : 0);
}

kx_status dist_phase(kx_ctx* c, double* const* U, int ph, Exchange& x) {
  x = Exchange{};
  const bool e3 = c->scheme != KX_ETD2RKDS;
  const double* Uc[MAXS];
  const double* Usc[MAXS];
  for (int s = 0; s < c->ncomp; ++s) {
    Uc[s] = U[s];
    Usc[s] = c->Us[s];
  }
  if (dist_banded(c)) {
    if (ph == 0) return dist_f_halo(c, U, x);
    if (ph == 1) return dist_f_stencil(c, U, x);
    if (ph == 2) return dist_group(c, 0, c->F_B, x);
    ph -= 1;   // the remaining phases are those of the dense schedule
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
  if (x.kind == 2) {   // direct peer stores: every rank's producers are done before anyone reads
    if (c->nranks == 1) return KX_OK;
    if (!c->bar_buf) {
      std::vector<double*> keep;
      KX_TRY(dalloc(c, &c->bar_buf, 1, keep));
      KX_CUDA(c, cudaMemsetAsync(c->bar_buf, 0, 8, st));
    }
    return chk(api.AllReduce(c->bar_buf, c->bar_buf, 1, ncclFloat64, ncclSum, comm, st));
  }
  KX_TRY(chk(api.GroupStart()));
  if (x.kind == 1) {
    for (int k = 0; k + 1 < x.nbuf; k += 2) {
      if (c->rank > 0) {
        KX_TRY(chk(api.Send(x.send[k], x.count, ncclFloat64, c->rank - 1, comm, st)));
        KX_TRY(chk(api.Recv(x.recv[k], x.count, ncclFloat64, c->rank - 1, comm, st)));
      }
      if (c->rank + 1 < c->nranks) {
        KX_TRY(chk(api.Send(x.send[k + 1], x.count, ncclFloat64, c->rank + 1, comm, st)));
        KX_TRY(chk(api.Recv(x.recv[k + 1], x.count, ncclFloat64, c->rank + 1, comm, st)));
      }
    }
    KX_TRY(chk(api.GroupEnd()));
    return KX_OK;
  }
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
    if (x.nbuf || x.kind == 2) KX_TRY(nccl_exchange(c, x, c->cur));
  }
  KX_TRY(enqueue_watch(c, U));
  c->cnt.steps += 1;
  return KX_OK;
}

}  // namespace kx::detail
