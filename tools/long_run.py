"""The headline workload integrated to the paper's final time on one B200: C2 (2-D Schnakenberg
1024^2, exprk3ds_real, T = 2) with m = 6000 steps (the bench's step size) and with m = 12000 and
24000 (self-convergence: the differences shrink ~8x per halving for a third-order method), plus
the pattern that forms (dominant cosine mode of u).  Prints one JSON object.

    python tools/long_run.py > profiles/long_run_c2_r01.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_2310_07551_b200 import kx  # noqa: E402


def run(prob, T, m):
    ctx = kx.Context(0)
    ctx.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(prob.d):
            ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    ctx.set_model(prob.model, prob.params)
    ctx.set_tau(T / m, "etd3rkds")
    U = [torch.from_numpy(u.copy()).cuda() for u in prob.U0]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.step_n(U, m)
    ctx.sync()
    el = time.perf_counter() - t0
    out = [u.cpu().numpy() for u in U]
    ctx.close()
    return out, el


def main():
    cfg = inputs.CONFIGS["C2"]
    prob = inputs.make_problem(cfg["model"], cfg["d"], cfg["n"], seed=0)
    T = cfg["T"]
    res = {"workload": "C2 " + cfg["desc"], "runs": {}}
    sols = {}
    for m in (6000, 12000, 24000):
        u, el = run(prob, T, m)
        sols[m] = u
        res["runs"][m] = {"seconds": round(el, 2), "steps_per_s": round(m / el, 1),
                          "finite": bool(all(np.isfinite(x).all() for x in u)),
                          "u_min": float(u[0].min()), "u_max": float(u[0].max())}
        print(json.dumps({m: res["runs"][m]}), file=sys.stderr, flush=True)
    ref = sols[24000]
    scale = max(np.abs(ref[c]).max() for c in range(2))
    d1 = max(np.abs(sols[6000][c] - ref[c]).max() for c in range(2)) / scale
    d2 = max(np.abs(sols[12000][c] - ref[c]).max() for c in range(2)) / scale
    res["self_convergence"] = {"rel_diff_6000_vs_24000": d1, "rel_diff_12000_vs_24000": d2,
                               "ratio": d1 / d2 if d2 > 0 else None}
    # the pattern: dominant 2-D cosine mode of u - mean(u)
    n = prob.n
    u = sols[24000][0].reshape(n[1], n[0])
    h = u - u.mean()
    best, kbest = 0.0, None
    for k2 in range(0, 16):
        c2 = np.cos(k2 * np.pi * np.arange(n[1]) / (n[1] - 1))
        for k1 in range(0, 16):
            if k1 == 0 and k2 == 0:
                continue
            c1 = np.cos(k1 * np.pi * np.arange(n[0]) / (n[0] - 1))
            a = abs(float(c2 @ h @ c1)) / (np.linalg.norm(c2) * np.linalg.norm(c1))
            if a > best:
                best, kbest = a, (k1, k2)
    res["pattern_dominant_mode"] = kbest
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
