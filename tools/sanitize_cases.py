"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck): every GEMM layout,
the stream-K schedule, the stencil, the nonlinearity, phi-bank formation, both steps, the
loopback sharded step.  Exits non-zero on a parity failure."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_2310_07551_b200 import kx  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


ctx = kx.Context(0)
for n in ([33, 17, 9], [64, 48], [300, 280]):      # ragged, vector path, stream-K tail
    ctx.set_grid(n, 1)
    X = dev(inputs.uniform_sym(1, 0, int(np.prod(n))))
    Y = torch.zeros_like(X)
    Ls = [dev(inputs.uniform_sym(2, mu, m * m)) for mu, m in enumerate(n)]
    ctx.tucker(X, Y, Ls)
    for mu in range(1, len(n) + 1):
        ctx.mode_product(X, Y, mu, Ls[mu - 1], 1.0, 0.5)
ctx.sync()
for model, d, n, scheme, tau in [("schnakenberg", 2, 24, "etd3rkds", 1e-4), ("fhn", 3, 10, "etd3rkds", 0.015),
                                 ("schnakenberg", 2, 20, "etd2rkds", 1e-4)]:
    prob = inputs.make_problem(model, d, n)
    ctx.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(d):
            ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    ctx.set_model(model, prob.params)
    ctx.set_tau(tau, scheme)
    U = [dev(u) for u in prob.U0]
    for _ in range(2):
        ctx.step(U)
    ctx.set_kronsum_mode(True)
    ctx.step(U)
    ctx.set_kronsum_mode(False)
    ctx.sync()
grp = kx.Group(2)
prob = inputs.make_problem("fhn", 3, [8, 6, 4])
for c_ in grp.ctx:
    c_.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(3):
            c_.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    c_.set_model("fhn", prob.params)
    c_.set_tau(0.015, "etd3rkds")
Ug = [[dev(u.reshape(4, 6, 8)[2 * r:2 * r + 2].ravel()) for u in prob.U0] for r in range(2)]
grp.step(Ug)
grp.ctx[0].sync()
print("sanitize cases done")
