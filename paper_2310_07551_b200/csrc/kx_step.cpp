// One-GPU step schedules (ETD2RKDS, exprk3ds) and their CUDA-graph capture / replay.
#include "kx_ctx.h"

#include <cstdint>
#include <cstdio>
#include <cstdlib>

namespace kx::detail {

// ---------------------------------------------------------------- time steps --------------
// G = g(U); F = K(U, A) + G.  One fused pass (launch_g_kronsum) when both species have
// tridiagonal A_mu on a 2-D / 3-D grid with even n_1; else the nonlinearity kernel and the
// Kronecker-sum action (stencil or dense mode products).
kx_status first_phase(kx_ctx* c, double* const* U) {
  const int ns = c->ncomp;
  bool fuse = ns == 2 && (c->d == 2 || c->d == 3) && c->tn[0] % 2 == 0 && c->tN < (1LL << 30) &&
              all_tridiag(c, 0, ns);
  for (int s = 0; s < ns && fuse; ++s)
    fuse = ((reinterpret_cast<uintptr_t>(U[s]) | reinterpret_cast<uintptr_t>(c->G[s]) |
             reinterpret_cast<uintptr_t>(c->F[s])) & 15) == 0;
  if (!fuse) {
    KX_TRY(nonlin(c, 0, U, c->G));
    return kronsum_multi(c, 0, ns, U, c->F, 1.0, c->G);
  }
  kx::GKronArgs a;
  a.d = c->d;
  a.model = c->model;
  a.N = (int)c->tN;
  for (int mu = 0; mu < c->d; ++mu) a.n[mu] = (int)c->tn[mu];
  for (int i = 0; i < 8; ++i) a.p[i] = c->params[i];
  for (int s = 0; s < 2; ++s) {
    a.U[s] = U[s];
    a.G[s] = c->G[s];
    a.F[s] = c->F[s];
    for (int mu = 0; mu < c->d; ++mu) a.tri[s][mu] = c->A_tri[s][mu];
  }
  // HBM bytes: read U (2 fields), write G and F (4 fields)
  KX_TRY(run_other(c, [&] { return kx::launch_g_kronsum(a, c->cur); }, 48.0 * (double)c->tN));
  c->cnt.mode_products += (long long)ns * c->d;
  c->cnt.kronsum_actions += ns;
  return KX_OK;
}

// exprk3ds_real, Algorithm 1 (d = 2) / Algorithm 2 (d > 2), P:2229-2264 / P:2302-2342,
// fused schedule of SURVEY.md §3 CS2.  Groups: 0 = F (3T terms), 1 = D2 (T), 2 = D3 (T).
kx_status enqueue_step_etd3(kx_ctx* c, double* const* U) {
  const int ns = c->ncomp;
  // G = g(t, U); F = K(U, A) + G
  KX_TRY(first_phase(c, U));
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
  KX_TRY(final_concat(c, ws, nullptr, c->stages[2].nseg, c->stages[2].slot, c->stages[2].B,
                      U, 1.0, 1.0, U));
  c->cnt.tucker_ops += (long long)ns * 5 * c->T;   // 3T on F, T on D2, T on D3
  return KX_OK;
}

// ETD2RKDS (eq:ETD2RK with eq:phisplit).  Groups: 0 = F (phi_1), 1 = D (phi_2).
kx_status enqueue_step_etd2(kx_ctx* c, double* const* U) {
  const int ns = c->ncomp;
  KX_TRY(first_phase(c, U));
  double* const* ws = nullptr;
  KX_TRY(group_modes(c, c->groups[0], 0, 1, c->F, c->groups[0].slot0, &ws));
  KX_TRY(last_mode_concat(c, ws, c->F, 1, c->stages[0].slot, c->stages[0].B, c->Us, 1.0, 1.0, U));
  KX_TRY(nonlin(c, 1, c->Us, c->D));
  KX_TRY(group_modes(c, c->groups[1], 0, 1, c->D, c->groups[1].slot0, &ws));
  KX_TRY(final_concat(c, ws, c->D, 1, c->stages[1].slot, c->stages[1].B, U, 1.0, 1.0, c->Us));
  c->cnt.tucker_ops += (long long)ns * 2;
  return KX_OK;
}

kx_status enqueue_watch(kx_ctx* c, double* const* U) {
  if (!c->nan_check) return KX_OK;
  for (int s = 0; s < c->ncomp; ++s)
    KX_TRY(run_other(c, [&] { return kx::launch_watch_finite(U[s], c->tN, c->watch, c->cur); },
                     8.0 * (double)c->tN));
  return run_other(c, [&] { return kx::launch_watch_tick(c->watch, c->cur); });
}

// ---------------------------------------------------------------- small 2-D grids (K*5) ---
// Eligible: one GPU, d = 2, real scheme, <= 2 species, 8 <= n_2 <= 64, n_1 <= 64, every A_mu
// tridiagonal (the stencil form of the Kronecker sum).
bool fused_eligible(const kx_ctx* c) {
  if (!c->fused_small || c->dist || c->cplx || c->d != 2 || c->ncomp < 1 || c->ncomp > 2) return false;
  if (c->scheme != KX_ETD2RKDS && c->scheme != KX_ETD3RKDS_REAL) return false;
  const long long n1 = c->tn[0], n2 = c->tn[1];
  if (n1 < 1 || n1 > kx::kFusedNMax || n2 < kx::kFusedCluster || n2 > kx::kFusedNMax) return false;
  if (!all_tridiag(c, 0, c->ncomp)) return false;
  for (int k = 0; k < c->nstages; ++k)
    if (c->stages[k].nseg > kx::kFusedMaxSeg) return false;
  return c->nstages == 2 || c->nstages == 3;
}

// nsteps steps of the current scheme in one cluster launch.  The stage banks are the ones the
// general path uses: stage k's segment sg reads group gi's term t (first-mode matrix
// group.first + t n_2, leading dimension nterms n_2) and the scaled mode-1 block
// stage.B + sg n_1^2.
kx_status enqueue_fused(kx_ctx* c, double* const* U, int nsteps) {
  kx::Fused2dArgs a;
  const long long n1 = c->tn[0], n2 = c->tn[1];
  const bool etd3 = c->nstages == 3;
  a.n1 = (int)n1;
  a.n2 = (int)n2;
  a.ncomp = c->ncomp;
  a.model = c->model;
  a.nsteps = nsteps;
  a.nstages = c->nstages;
  for (int i = 0; i < 8; ++i) a.p[i] = c->params[i];
  for (int s = 0; s < c->ncomp; ++s) {
    a.U[s] = U[s];
    for (int mu = 0; mu < 2; ++mu) a.tri[s][mu] = c->A_tri[s][mu];
  }
  const Group& F = c->groups[0];
  for (int k = 0; k < c->nstages; ++k) {
    const Stage& st = c->stages[k];
    a.nseg[k] = st.nseg;
    a.base[k] = (!etd3 && k == 1) ? 1 : 0;
    for (int sg = 0; sg < st.nseg; ++sg) {
      const int slot = st.slot[sg];
      const bool from_f = slot < F.slot0 + F.nterms;
      const Group& G = from_f ? F : c->groups[etd3 ? k : 1];
      const int t = slot - G.slot0;
      a.seg_in[k][sg] = from_f ? 0 : 1;
      a.ld2[k][sg] = (long long)G.nterms * n2;
      for (int s = 0; s < c->ncomp; ++s) {
        a.P2[k][sg][s] = G.first[s] + t * n2;
        a.B[k][sg][s] = st.B[s] + (long long)sg * n1 * n1;
      }
    }
  }
  // algorithmic work of the steps, counted as on the general path
  const long long tuckers = (long long)c->ncomp * (etd3 ? 5 * c->T : 2) * nsteps;
  const double fl = 2.0 * (double)c->tN * (double)(n1 + n2) * (double)tuckers;
  int e0 = -1;
  if (c->profiling) {
    e0 = c->ev_used;
    c->ev_used += 2;
    KX_CUDA(c, record(c, pool_event(c, e0)));
  }
  // diagnostics only: KX_FUSED_PROF=1 prints phase clocks of eager (not captured) launches
  static long long* prof_buf = nullptr;
  long long* prof = nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(c->cur, &cap);
  if (getenv("KX_FUSED_PROF") && cap == cudaStreamCaptureStatusNone) {
    if (!prof_buf && cudaMallocManaged(&prof_buf, 64 * sizeof(long long)) != cudaSuccess) prof_buf = nullptr;
    prof = prof_buf;
  }
  a.prof = prof;
  KX_CUDA(c, kx::launch_fused2d(a, c->cur));
  if (prof) {
    KX_CUDA(c, cudaStreamSynchronize(c->cur));
    fprintf(stderr, "kx-fused phases (cycles):");
    for (int i = 1; i < 64 && prof[i] > prof[i - 1]; ++i) fprintf(stderr, " %lld", prof[i] - prof[i - 1]);
    fprintf(stderr, "\n");
  }
  if (c->profiling) {
    KX_CUDA(c, record(c, pool_event(c, e0 + 1)));
    c->recs.push_back({0, e0, e0 + 1, fl});
  }
  c->cnt.gemm_launches += 1;
  c->cnt.tucker_ops += tuckers;
  c->cnt.mode_products += 2 * tuckers + (long long)c->ncomp * 2 * nsteps;
  c->cnt.kronsum_actions += (long long)c->ncomp * nsteps;
  c->cnt.mode_product_flops += fl;
  return KX_OK;
}

kx_status enqueue_step(kx_ctx* c, double* const* U) {
  if (fused_eligible(c)) KX_TRY(enqueue_fused(c, U, 1));
  else if (c->scheme == KX_ETD3RKDS_REAL || c->scheme == KX_ETD3RKDS_CPLX) KX_TRY(enqueue_step_etd3(c, U));
  else KX_TRY(enqueue_step_etd2(c, U));
  return enqueue_watch(c, U);
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
      (r.cls == 0 ? c->prof_flops : c->prof_bytes) += r.flops;
    }
  }
  return KX_OK;
}

// ---------------------------------------------------------------- host-buffer tail -------
void drop_tail_graph(kx_ctx* c) {
  if (c->tail_gexec) cudaGraphExecDestroy(c->tail_gexec);
  if (c->tail_graph) cudaGraphDestroy(c->tail_graph);
  c->tail_gexec = nullptr;
  c->tail_graph = nullptr;
  c->tail_version = -1;
}

// The last step of kx_integrate_host with the device -> host copy of U overlapped with its
// final stage GEMM (final_concat in row chunks); a plain copy after the step when the step has
// no such GEMM (the one-kernel small-grid path).  Captured once per (U, U_host, bank) and
// replayed; the counters advance by one step per replay as in step_impl.
kx_status tail_step_impl(kx_ctx* c, double* const* U, double* const* U_host) {
  bool same = c->tail_gexec && c->tail_version == c->bank_version;
  for (int s = 0; s < c->ncomp && same; ++s) same = c->tail_key[s] == U_host[s] && c->tail_U[s] == U[s];
  if (!same) {
    drop_tail_graph(c);
    if (!c->copy) KX_CUDA(c, cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    for (cudaEvent_t& e : c->ev_tail)
      if (!e) KX_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const kx_counters before = c->cnt;
    c->cur = c->cap;
    for (int s = 0; s < c->ncomp; ++s) c->tail_host[s] = U_host[s];
    c->tail_armed = true;
    c->tail_done = false;
    KX_CUDA(c, cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
    kx_status st = enqueue_step(c, U);
    c->tail_armed = false;
    const size_t bytes = (size_t)c->tN * 8;
    if (st == KX_OK && c->tail_done) {   // join the copy stream back into the capture
      if (cudaEventRecord(c->ev_tail[kTailMaxChunks], c->copy) != cudaSuccess ||
          cudaStreamWaitEvent(c->cap, c->ev_tail[kTailMaxChunks], 0) != cudaSuccess)
        st = fail(c, KX_ERR_CUDA, "tail join");
    } else if (st == KX_OK) {
      for (int s = 0; s < c->ncomp && st == KX_OK; ++s)
        if (cudaMemcpyAsync(U_host[s], U[s], bytes, cudaMemcpyDeviceToHost, c->cap) != cudaSuccess)
          st = fail(c, KX_ERR_CUDA, "tail copy");
    }
    cudaGraph_t gr = nullptr;
    const cudaError_t e = cudaStreamEndCapture(c->cap, &gr);
    c->cur = c->stream;
    c->recs.clear();
    if (st != KX_OK) {
      if (gr) cudaGraphDestroy(gr);
      c->cnt = before;
      return st;
    }
    KX_CUDA(c, e);
    c->tail_graph = gr;
    KX_CUDA(c, cudaGraphInstantiate(&c->tail_gexec, c->tail_graph, 0));
    c->tail_version = c->bank_version;
    for (int s = 0; s < c->ncomp; ++s) c->tail_key[s] = U_host[s], c->tail_U[s] = U[s];
    kx_counters dl = c->cnt;
    dl.steps = 0;
    dl.tucker_ops -= before.tucker_ops;
    dl.mode_products -= before.mode_products;
    dl.kronsum_actions -= before.kronsum_actions;
    dl.phi_builds = 0;
    dl.gemm_launches -= before.gemm_launches;
    dl.other_launches -= before.other_launches;
    dl.mode_product_flops -= before.mode_product_flops;
    c->tail_delta = dl;
    c->cnt = before;
  }
  KX_CUDA(c, cudaGraphLaunch(c->tail_gexec, c->stream));
  c->cnt.steps += 1;
  c->cnt.tucker_ops += c->tail_delta.tucker_ops;
  c->cnt.mode_products += c->tail_delta.mode_products;
  c->cnt.kronsum_actions += c->tail_delta.kronsum_actions;
  c->cnt.gemm_launches += c->tail_delta.gemm_launches;
  c->cnt.other_launches += c->tail_delta.other_launches;
  c->cnt.mode_product_flops += c->tail_delta.mode_product_flops;
  return KX_OK;
}

}  // namespace kx::detail
