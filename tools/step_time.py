"""ms per step of a config (CUDA events, L2 flushed between steps, graph replay) — for A/B runs
of GEMM schedule settings (KX_GEMM_* environment variables).  Diagnostics, not the bench."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import inputs  # noqa: E402
from paper_2310_07551_b200 import kx  # noqa: E402

for cfg_name in sys.argv[1:] or ["C2", "C3"]:
    k = inputs.CONFIGS[cfg_name]
    prob = inputs.make_problem(k["model"], k["d"], k["n"], seed=0)
    ctx = kx.Context(0)
    ctx.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(prob.d):
            ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    ctx.set_model(prob.model, prob.params)
    ctx.set_tau(k["T"] / k["m"], k["scheme"])
    U = [torch.from_numpy(u.copy()).cuda() for u in prob.U0]
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
    for _ in range(3):
        ctx.step(U)
    torch.cuda.synchronize()
    ms = []
    for rep in range(3):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
        for i in range(20):
            flush.fill_(float(i))
            ev[i][0].record()
            ctx.step(U)
            ev[i][1].record()
        torch.cuda.synchronize()
        ms.append(sum(a.elapsed_time(b) for a, b in ev) / 20)
    print(f"{cfg_name} {os.environ.get('KX_TAG', '')} ms/step best {min(ms):.4f} all {[round(m, 4) for m in ms]}", flush=True)
    ctx.close()
