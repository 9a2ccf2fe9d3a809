"""Small 2-D grids: microseconds per step of the fused one-cluster kernel (K*5) against the
general multi-launch path, per-step launches (graph replays) and kx_step_n (all steps in one
launch).  No L2 flush (the state is kilobytes).

    python tools/fused_bench.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_2310_07551_b200 import kx  # noqa: E402


def run(n, scheme, fused, multi, steps=400):
    prob = inputs.make_problem("schnakenberg", 2, n, seed=0)
    stream = torch.cuda.Stream()
    c = kx.Context(0, stream)
    c.set_grid(prob.n, 2)
    for k in range(2):
        for mu in range(2):
            c.set_direction_matrix(k, mu + 1, prob.A[k][mu])
    c.set_model(prob.model, prob.params)
    c.set_tau(1e-4, scheme)
    c.set_fused_small(fused)
    U = [torch.from_numpy(u.copy()).cuda() for u in prob.U0]
    for _ in range(3):
        c.step(U)
    c.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(3):
        with torch.cuda.stream(stream):
            e0.record()
            if multi:
                c.step_n(U, steps)
            else:
                for _ in range(steps):
                    c.step(U)
            e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / steps)
    c.close()
    return round(best, 2)


out = {}
for n in (32, 64):
    for scheme in ("etd2rkds", "etd3rkds"):
        out[f"{scheme}_{n}"] = {"general_us": run(n, scheme, False, False),
                                "fused_step_us": run(n, scheme, True, False),
                                "fused_step_n_us": run(n, scheme, True, True)}
print(json.dumps(out, indent=1))
