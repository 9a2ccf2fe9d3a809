"""fp32-variant throughput: C2 / C3 steps/s (kx_step_f32) and Tucker TF/s (kx_tucker_f32), with
the per-kernel profile.  Diagnostics; bench.py reports the same numbers in its JSON line."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import inputs  # noqa: E402
from paper_2310_07551_b200 import kx  # noqa: E402


def timed(fn, reps):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def steps(cfg, nsteps=20):
    k = inputs.CONFIGS[cfg]
    prob = inputs.make_problem(k["model"], k["d"], k["n"], seed=0)
    ctx = kx.Context(0)
    ctx.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(prob.d):
            ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    ctx.set_model(prob.model, prob.params)
    ctx.set_tau(k["T"] / k["m"], k["scheme"])
    U = [torch.from_numpy(u.astype(np.float32)).cuda() for u in prob.U0]
    ctx.step_f32(U, 3)
    ms = timed(lambda: ctx.step_f32(U, 1), nsteps)
    ctx.set_profiling(True)
    ctx.step_f32(U, 5)
    ctx.sync()
    pr = ctx.profile()
    ctx.close()
    fl = pr["gemm_flops"] / 5
    return dict(cfg=cfg, ms_per_step=ms, steps_per_s=1e3 / ms, gemm_ms=pr["gemm_ms"] / 5, other_ms=pr["other_ms"] / 5,
                gemm_tflops_alg=fl / (pr["gemm_ms"] / 5) / 1e9, gemm_tflops_tc=3 * fl / (pr["gemm_ms"] / 5) / 1e9)


def tucker(n, reps=20):
    N = int(np.prod(n))
    ctx = kx.Context(0)
    ctx.set_grid(n, 1)
    X = torch.randn(N, device="cuda")
    Y = torch.zeros(N, device="cuda")
    Ls = [torch.randn(m, m, device="cuda") for m in n]
    ctx.tucker_f32(X, Y, Ls)
    ms = timed(lambda: ctx.tucker_f32(X, Y, Ls), reps)
    ctx.set_profiling(True)
    ctx.tucker_f32(X, Y, Ls)
    ctx.sync()
    pr = ctx.profile()
    ctx.close()
    fl = 2.0 * N * sum(n)
    return dict(n=n, ms=ms, tflops_alg=fl / ms / 1e9, gemm_ms=pr["gemm_ms"], gemm_tflops_alg=fl / pr["gemm_ms"] / 1e9)


if __name__ == "__main__":
    rows = []
    for cfg in ("C2", "C3"):
        rows.append(steps(cfg))
        print(rows[-1], flush=True)
    for n in ([1024, 1024], [2048, 2048], [4096, 4096], [256, 256, 256], [512, 512, 512]):
        rows.append(tucker(n))
        print(rows[-1], flush=True)
    if len(sys.argv) > 1:
        json.dump(rows, open(sys.argv[1], "w"), indent=1)
