"""Steps/s of the GPU integrators at the paper's own grid sizes (plain step graph, CUDA events,
L2 flushed between steps): 2D Schnakenberg n = 150/300/450/600 (Tables 4-5), 3D FHN
n = 64/100/150/200 (Tables 6-7)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_2310_07551_b200 import kx  # noqa: E402

cases = [("schnakenberg", 2, n, 2.0 / 6000) for n in (150, 300, 450, 600)] + \
        [("fhn", 3, n, 0.015) for n in (64, 100, 150, 200)]
s = torch.cuda.Stream()
flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
for scheme in sys.argv[1:] or ["etd3rkds"]:
    for model, d, n, tau in cases:
        prob = inputs.make_problem(model, d, n)
        ctx = kx.Context(0, s)
        ctx.set_grid(prob.n, 2)
        for c in range(2):
            for mu in range(d):
                ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
        ctx.set_model(model, prob.params)
        ctx.set_tau(tau, scheme)
        U = [torch.from_numpy(u.copy()).cuda() for u in prob.U0]
        for _ in range(3):
            ctx.step(U)
        ctx.sync()
        ctx.reset_counters()
        ts = []
        for k in range(20):
            with torch.cuda.stream(s):
                flush.fill_(1.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ctx.step(U)
                e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.mean(ts))
        cnt = ctx.counters()
        fl = cnt["mode_product_flops"] / max(1, cnt["steps"])
        print(f"{scheme:14s} {model:13s} n={n:4d}  {1e3 / ms:9.1f} steps/s  {ms * 1e3:9.1f} us/step  "
              f"{fl / ms / 1e9:6.2f} TF/s (GEMM flops / step time)", flush=True)
        ctx.close()
        del U
