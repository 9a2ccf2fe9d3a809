"""Profiling driver (run under ncu on one GPU): set up a config and run a few steps, or a
Tucker operator.  Not a benchmark (numbers printed under ncu are never bench values).

    python tools/prof_step.py --config C2 --steps 2
    python tools/prof_step.py --tucker 3 512
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_2310_07551_b200 import kx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--eager", action="store_true")
ap.add_argument("--tucker", nargs=2, type=int, default=None)
ap.add_argument("--n", type=int, default=None, help="override the config's grid extent")
ap.add_argument("--scheme", default=None)
a = ap.parse_args()

ctx = kx.Context(0)
if a.tucker:
    d, n = a.tucker
    ctx.set_grid([n] * d, 1)
    X = torch.rand(n ** d, dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    L = torch.rand(n * n, dtype=torch.float64, device="cuda") / n
    ctx.tucker(X, Y, [L] * d)
    ctx.sync()
    torch.cuda.profiler.start()
    for _ in range(a.steps):
        ctx.tucker(X, Y, [L] * d)
    ctx.sync()
    torch.cuda.profiler.stop()
else:
    cfg = dict(inputs.CONFIGS[a.config])
    if a.n:
        cfg["n"] = a.n
    if a.scheme:
        cfg["scheme"] = a.scheme
    prob = inputs.make_problem(cfg["model"], cfg["d"], cfg["n"])
    ctx.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(prob.d):
            ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    ctx.set_model(prob.model, prob.params)
    ctx.set_tau(cfg["T"] / cfg["m"], cfg["scheme"])
    U = [torch.from_numpy(u.copy()).cuda() for u in prob.U0]
    if a.eager:
        ctx.set_profiling(True)
    ctx.step(U)                      # capture the graph outside the profiled range
    ctx.sync()
    torch.cuda.profiler.start()      # ncu --profile-from-start off
    for k in range(a.steps):
        ctx.step(U)
    ctx.sync()
    torch.cuda.profiler.stop()
ctx.sync()
print("done")
