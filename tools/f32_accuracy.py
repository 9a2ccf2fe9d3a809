"""Accuracy of the fp32 variant against the fp64 oracle, next to the error of the oracle's own
algorithm run in fp32 arithmetic (numpy sgemm, RN accumulation) on the same fp32 data.
Writes a JSON table (profiles/f32_accuracy_r02.json by default).  Diagnostics, not a test."""
import dataclasses
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import inputs  # noqa: E402
from oracle.etd import integrate  # noqa: E402  (oracle: test infrastructure)
from oracle.tensor import tucker, unvec, vec  # noqa: E402
from paper_2310_07551_b200 import kx  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_f32 import _cast_bank, relerr  # noqa: E402


def dev32(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def tucker_row(n):
    N = int(np.prod(n))
    x = inputs.uniform_sym(31, 0, N).astype(np.float32)
    Ls = [(inputs.uniform_sym(32, mu, m * m).reshape(m, m) / np.sqrt(m)).astype(np.float32) for mu, m in enumerate(n)]
    ref = vec(tucker(unvec(x.astype(np.float64), n), [L.astype(np.float64) for L in Ls]))
    r32 = vec(tucker(unvec(x, n), Ls))
    ctx = kx.Context(0)
    ctx.set_grid(n, 1)
    Y = torch.zeros(N, dtype=torch.float32, device="cuda")
    ctx.tucker_f32(dev32(x), Y, [dev32(L.T.copy()) for L in Ls])
    e = relerr(Y.cpu().numpy(), ref)
    ctx.close()
    return dict(n=n, gpu=e, np_f32=relerr(r32, ref), ratio=e / max(relerr(r32, ref), 1e-30))


def step_row(model, d, n, scheme, tau, steps=20):
    prob = inputs.make_problem(model, d, n, seed=3)
    prob = dataclasses.replace(prob, U0=[u.astype(np.float32).astype(np.float64) for u in prob.U0])
    ref, bank = integrate(prob, scheme, T=tau * steps, m=steps, steps=steps)
    p32 = dataclasses.replace(prob, A=[[A.astype(np.float32) for A in Ac] for Ac in prob.A],
                              U0=[u.astype(np.float32) for u in prob.U0])
    r32, _ = integrate(p32, scheme, T=tau * steps, m=steps, steps=steps, bank=_cast_bank(bank))
    ctx = kx.Context(0)
    ctx.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(d):
            ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    ctx.set_model(prob.model, prob.params)
    ctx.set_tau(tau, scheme)
    U = [dev32(u) for u in prob.U0]
    ctx.step_f32(U, steps)
    ctx.sync()
    e = max(relerr(U[c].cpu().numpy(), ref[c]) for c in range(2))
    e32 = max(relerr(r32[c], ref[c]) for c in range(2))
    ctx.close()
    return dict(model=model, n=n, scheme=scheme, tau=tau, steps=steps, gpu=e, np_f32=e32, ratio=e / e32)


if __name__ == "__main__":
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "f32_accuracy_r02.json")
    t0 = time.time()
    rows = {"tucker": [], "steps": []}
    for n in ([64, 64], [256, 256], [1024, 1024], [32, 32, 32], [128, 128, 128]):
        rows["tucker"].append(tucker_row(n))
        print(rows["tucker"][-1], flush=True)
    for case in [("schnakenberg", 2, 64, "etd3rkds", 2.0 / 6000), ("schnakenberg", 2, 64, "etd2rkds", 0.25 / 3000),
                 ("fhn", 3, 32, "etd3rkds", 0.015), ("fhn", 3, 32, "etd2rkds", 0.015),
                 ("fhn", 3, 64, "etd3rkds", 0.015), ("schnakenberg", 2, 256, "etd3rkds", 2.0 / 6000)]:
        rows["steps"].append(step_row(*case))
        print(rows["steps"][-1], flush=True)
    rows["wall_s"] = time.time() - t0
    with open(out, "w") as f:
        json.dump(rows, f, indent=1, default=float)
