import os, sys, time
sys.path.insert(0, "/root/repo")
import torch, numpy as np, inputs
from paper_2310_07551_b200 import kx
cfg = inputs.CONFIGS[sys.argv[1]]
prob = inputs.make_problem(cfg["model"], cfg["d"], cfg["n"])
s = torch.cuda.Stream()
ctx = kx.Context(0, s)
ctx.set_grid(prob.n, 2)
for c in range(2):
    for mu in range(prob.d): ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
ctx.set_model(prob.model, prob.params); ctx.set_tau(cfg["T"] / cfg["m"], cfg["scheme"])
U = [torch.from_numpy(u.copy()).cuda() for u in prob.U0]
flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
for prof in (False, True, False, True):
    ctx.set_profiling(prof)
    for _ in range(3): ctx.step(U)
    ctx.sync()
    ts = []
    for k in range(20):
        with torch.cuda.stream(s):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); ctx.step(U); e1.record()
        e1.synchronize(); ts.append(e0.elapsed_time(e1))
    print(sys.argv[1], "profiling" if prof else "plain    ", f"{np.mean(ts)*1e3:8.1f} us", flush=True)
