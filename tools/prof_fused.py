"""Profiling driver for the fused small-grid kernel (run under ncu): kx_step_n of N steps."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_2310_07551_b200 import kx  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
scheme = sys.argv[2] if len(sys.argv) > 2 else "etd3rkds"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
prob = inputs.make_problem("schnakenberg", 2, n, seed=0)
c = kx.Context(0)
c.set_grid(prob.n, 2)
for k in range(2):
    for mu in range(2):
        c.set_direction_matrix(k, mu + 1, prob.A[k][mu])
c.set_model(prob.model, prob.params)
c.set_tau(1e-4, scheme)
U = [torch.from_numpy(u.copy()).cuda() for u in prob.U0]
c.step(U)
c.sync()
torch.cuda.profiler.start()
c.step_n(U, steps)
c.sync()
torch.cuda.profiler.stop()
print("done")
