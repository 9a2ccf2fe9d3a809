"""End-to-end ms per step through kx_integrate_host with page-locked host buffers (the bench's
e2e protocol: L2 flushed, one step per call), for A/B runs of KX_TAIL_CHUNKS.  Diagnostics."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import inputs  # noqa: E402
from paper_2310_07551_b200 import kx  # noqa: E402

for cfg_name in sys.argv[1:] or ["C2"]:
    k = inputs.CONFIGS[cfg_name]
    prob = inputs.make_problem(k["model"], k["d"], k["n"], seed=0)
    ctx = kx.Context(0)
    ctx.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(prob.d):
            ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    ctx.set_model(prob.model, prob.params)
    ctx.set_tau(k["T"] / k["m"], k["scheme"])
    Uh = [torch.from_numpy(u.copy()).pin_memory() for u in prob.U0]
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
    ms = []
    for rep in range(23):
        flush.fill_(float(rep))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.integrate_host([u.numpy() for u in Uh], 1)
        if rep >= 3:
            ms.append((time.perf_counter() - t0) * 1e3)
    ctx.close()
    ms.sort()
    print(f"{cfg_name} chunks={os.environ.get('KX_TAIL_CHUNKS', '4')} e2e ms/step median {ms[len(ms) // 2]:.4f} "
          f"min {ms[0]:.4f} -> {1e3 / ms[len(ms) // 2]:.1f} steps/s", flush=True)
