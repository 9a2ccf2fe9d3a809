// One-GPU step schedules (ETD2RKDS, exprk3ds) and their CUDA-graph capture / replay.
#include "kx_ctx.h"

namespace kx::detail {

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

kx_status enqueue_watch(kx_ctx* c, double* const* U) {
  if (!c->nan_check) return KX_OK;
  for (int s = 0; s < c->ncomp; ++s)
    KX_TRY(run_other(c, [&] { return kx::launch_watch_finite(U[s], c->tN, c->watch, c->cur); }));
  return run_other(c, [&] { return kx::launch_watch_tick(c->watch, c->cur); });
}

kx_status enqueue_step(kx_ctx* c, double* const* U) {
  if (c->scheme == KX_ETD3RKDS_REAL || c->scheme == KX_ETD3RKDS_CPLX) KX_TRY(enqueue_step_etd3(c, U));
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
      c->prof_flops += r.flops;
    }
  }
  return KX_OK;
}

}  // namespace kx::detail
