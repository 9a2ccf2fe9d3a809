import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, inputs
from paper_2310_07551_b200 import kx
k = inputs.CONFIGS[sys.argv[1]]
prob = inputs.make_problem(k["model"], k["d"], k["n"], seed=0)
ctx = kx.Context(0); ctx.set_grid(prob.n, 2)
for c in range(2):
    for mu in range(prob.d): ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
ctx.set_model(prob.model, prob.params); ctx.set_tau(k["T"] / k["m"], k["scheme"])
U = [torch.from_numpy(u.astype(np.float32)).cuda() for u in prob.U0]
ctx.step_f32(U, 2); ctx.sync()
torch.cuda.profiler.start(); ctx.step_f32(U, 1); ctx.sync(); torch.cuda.profiler.stop()
print("done")
