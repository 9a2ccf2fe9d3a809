// Distributed operators: the Tucker operator, the mu-mode product, the
// split phi-action (eq:split2d / eq:splitnd3 via eq:krontomu) and the
// Kronecker-sum action (eq:kronsumv: the mode-d term through the exchange, the other
// terms local, summed into Y by the unpack) on a slab-sharded context (BASELINE.json configs[4], the Tucker sweep at 2-8 GPUs).
//
// The user's tensors are layout-A slabs (i_d sharded, n_d / P planes per rank).  Modes 1..d-1
// are local in layout A; mode d needs whole i_d fibres, which layout B (i_1 sharded) holds.  An
// operator that contracts along mode d therefore runs in three phases with two all-to-alls:
//   [A] pack X by destination i_1 block (one strided copy)            -> all-to-all -> layout B
//   [B] modes d, d-1, ..., 2 on full fibres (for the split action: the first mode of every term
//       as one concatenated-M GEMM, then the batched middle modes)    -> all-to-all -> peer-major A
//   [A] mode 1 as ONE concatenated-K GEMM over (term, source rank) segments, which absorbs the
//       peer-major receive layout (no unpack), with alpha / beta in its epilogue; a lone mode-d
//       product unpacks instead (Y = alpha R + beta Y, strided copy).
// Modes are applied in descending mu as on one GPU (reading R2), and every product runs on full
// fibres on one rank, so the result equals the single-GPU one up to the split of the mode-1
// K-sum into P segments (rounding level).
#include "kx_ctx.h"

namespace kx::detail {

namespace {

kx_status dop_buffers(kx_ctx* c) {
  if (c->dop[0]) return KX_OK;
  for (double*& p : c->dop) KX_TRY(dalloc(c, &p, (size_t)c->Nloc, c->dop_allocs));
  return KX_OK;
}

// View a multi-component context as one component (comp) for the group / stage helpers.
struct CompView {
  kx_ctx* c;
  int nc;
  double* W1[MAXS];
  double* W2[MAXS];
  double* RA[MAXS];
  CompView(kx_ctx* ctx, int comp) : c(ctx), nc(ctx->ncomp) {
    for (int s = 0; s < MAXS; ++s) {
      W1[s] = c->W1[s];
      W2[s] = c->W2[s];
      RA[s] = c->RA[s];
    }
    c->ncomp = 1;
    c->W1[0] = W1[comp];
    c->W2[0] = W2[comp];
    c->RA[0] = RA[comp];
  }
  ~CompView() {
    c->ncomp = nc;
    for (int s = 0; s < MAXS; ++s) {
      c->W1[s] = W1[s];
      c->W2[s] = W2[s];
      c->RA[s] = RA[s];
    }
  }
};

}  // namespace

void dop_free(kx_ctx* c) {
  free_list(c->dop_allocs);
  for (double*& p : c->dop) p = nullptr;
}

kx_status dist_op_phase(kx_ctx* c, const DistOp& op, int ph, Exchange& x) {
  x = Exchange{};
  KX_TRY(dop_buffers(c));
  const int P = c->nranks, d = c->d;
  const long long n1 = c->n[0], n1l = n1 / P, rows = c->Nloc / n1, chunk = c->Nloc / P;
  x.count = (size_t)chunk;
  if (ph == 0) {   // [A] pack: chunk q = columns [q n1l, (q+1) n1l) of every row of the slab
    set_layout(c, false);
    KX_TRY(run_other(c, [&] {
      return kx::launch_copy2d_axpby(c->dop[0], n1l, chunk, op.X, n1, n1l, rows, n1l, P, 1.0, 0.0, c->cur);
    }, 16.0 * (double)c->Nloc));
    x.add(c->dop[0], c->dop[1]);
    return KX_OK;
  }
  if (ph == 1) {   // [B] modes d..2 on full fibres
    set_layout(c, true);
    if (op.kind == 1) {
      const PhiStack& ps = *op.ps;
      CompView v(c, op.comp);
      const Group& G = c->groups[ps.group];
      Group Gc;
      Gc.nterms = G.nterms;
      Gc.first[0] = G.first[op.comp];
      for (int mu = 0; mu < KX_MAXD; ++mu) Gc.mid[0][mu] = G.mid[op.comp][mu];
      const double* Xs[1] = {c->dop[1]};
      double* const* ws = nullptr;
      KX_TRY(group_modes(c, Gc, ps.t0, ps.nterms, Xs, 0, &ws));
      for (int t = 0; t < ps.nterms; ++t) x.add(ws[0] + (long long)t * c->Nloc, c->RA[0] + (long long)t * c->Nloc);
      return KX_OK;
    }
    if (op.kind == 3) {   // the mode-d term of the Kronecker sum
      const double* Xs[1] = {c->dop[1]};
      double* Ys[1] = {c->dop[2]};
      const double* Ls[1] = {c->A_dev[op.comp][d - 1]};
      KX_TRY(mode_product_multi(c, 1, Xs, Ys, d, Ls, 1.0, 0.0, nullptr));
      x.add(c->dop[2], c->dop[4]);
      return KX_OK;
    }
    const double* src = c->dop[1];
    double* bufs[2] = {c->dop[2], c->dop[3]};
    int w = 0;
    const int last = op.kind == 2 ? d : 2;
    for (int mu = d; mu >= last; --mu) {
      const double* Xs[1] = {src};
      double* Ys[1] = {bufs[w]};
      const double* Ls[1] = {op.L[mu - 1]};
      // a lone mode-d product carries alpha here; its beta is applied by the unpack
      KX_TRY(mode_product_multi(c, 1, Xs, Ys, mu, Ls, op.kind == 2 ? op.alpha : 1.0, 0.0, nullptr));
      src = bufs[w];
      w ^= 1;
    }
    x.add(src, c->dop[4]);
    return KX_OK;
  }
  // [A] ph == 2
  set_layout(c, false);
  if (op.kind == 3) {   // Y = beta Y + sum_{mu < d} X x_mu A_mu (local), then + the mode-d term
    double beta = op.beta;
    for (int mu = 1; mu < d; ++mu) {
      const double* Xs[1] = {op.X};
      double* Ys[1] = {op.Y};
      const double* Ls[1] = {c->A_dev[op.comp][mu - 1]};
      const double* Ds[1] = {op.Y};
      KX_TRY(mode_product_multi(c, 1, Xs, Ys, mu, Ls, 1.0, beta, Ds));
      beta = 1.0;
    }
    KX_TRY(run_other(c, [&] {
      return kx::launch_copy2d_axpby(op.Y, n1, n1l, c->dop[4], n1l, chunk, rows, n1l, P, 1.0, beta, c->cur);
    }, 24.0 * (double)c->Nloc));
    c->cnt.kronsum_actions += 1;
    return KX_OK;
  }
  if (op.kind == 2) {   // unpack: Y[row, q n1l + j] = R_q[row, j] + beta Y
    KX_TRY(run_other(c, [&] {
      return kx::launch_copy2d_axpby(op.Y, n1, n1l, c->dop[4], n1l, chunk, rows, n1l, P, 1.0, op.beta, c->cur);
    }, (op.beta != 0.0 ? 24.0 : 16.0) * (double)c->Nloc));
    return KX_OK;
  }
  const int nterm = op.kind == 1 ? op.ps->nterms : 1;
  if (nterm * P > MAXSEG) return fail(c, KX_ERR_UNSUPPORTED, "too many K segments for this rank count");
  GemmArgs g;
  g.arow = true;
  g.M = (int)rows;
  g.N = (int)n1;
  g.kseg = (int)n1l;
  g.nseg = nterm * P;
  g.lda = n1l;
  g.ldb = n1;
  g.ldc = n1;
  g.ldd = n1;
  g.ns = 1;
  g.alpha = op.alpha;
  g.beta = op.beta;
  for (int t = 0; t < nterm; ++t)
    for (int q = 0; q < P; ++q) g.seg_off[t * P + q] = (long long)t * c->Nloc + (long long)q * chunk;
  g.A[0] = op.kind == 1 ? c->RA[op.comp] : c->dop[4];
  g.B[0] = op.kind == 1 ? op.ps->B[op.comp] : op.L[0];   // stacked eta_t P_t{1} / L (= L^T row-major)
  g.C[0] = op.Y;
  g.D[0] = op.beta != 0.0 ? op.Y : nullptr;
  KX_TRY(run_gemm(c, g));
  c->cnt.mode_products += nterm;
  return KX_OK;
}

kx_status dist_op_nccl(kx_ctx* c, const DistOp& op) {
  c->cur = c->stream;
  Exchange x;
  for (int ph = 0; ph < kDistOpPhases; ++ph) {
    KX_TRY(dist_op_phase(c, op, ph, x));
    if (x.nbuf) KX_TRY(nccl_exchange(c, x, c->cur));
  }
  return KX_OK;
}

// Loopback group (one device, shared stream): the exchanges of one phase as device copies
// issued after every rank's phase (no kernel ever waits on another rank).
kx_status loopback_exchange(kx_ctx* const* ctxs, int nranks, const std::vector<Exchange>& xs) {
  for (int r = 0; r < nranks; ++r) {
    const Exchange& xr = xs[r];
    if (xr.kind == 2) continue;   // the producers stored straight into the peers
    if (xr.kind == 1) {   // halo: first plane -> rank-1's upper halo, last plane -> rank+1's lower
      for (int k = 0; k + 1 < xr.nbuf; k += 2) {
        if (r > 0)
          KX_CUDA(ctxs[r], cudaMemcpyAsync(xs[r - 1].recv[k + 1], xr.send[k], xr.count * 8,
                                           cudaMemcpyDeviceToDevice, ctxs[r]->stream));
        if (r + 1 < nranks)
          KX_CUDA(ctxs[r], cudaMemcpyAsync(xs[r + 1].recv[k], xr.send[k + 1], xr.count * 8,
                                           cudaMemcpyDeviceToDevice, ctxs[r]->stream));
      }
      continue;
    }
    for (int k = 0; k < xr.nbuf; ++k)
      for (int q = 0; q < nranks; ++q)
        KX_CUDA(ctxs[r], cudaMemcpyAsync(xs[q].recv[k] + (size_t)r * xr.count, xr.send[k] + (size_t)q * xr.count,
                                         xr.count * 8, cudaMemcpyDeviceToDevice, ctxs[r]->stream));
  }
  return KX_OK;
}

}  // namespace kx::detail
