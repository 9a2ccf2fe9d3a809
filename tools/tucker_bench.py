"""Tucker-operator throughput (dense flops / CUDA-event time) for a list of shapes."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2310_07551_b200 import kx  # noqa: E402

shapes = [[int(x) for x in a.split("x")] for a in (sys.argv[1:] or ["1024x1024", "4096x4096", "256x256x256", "512x512x512", "128x128x128"])]
ctx = kx.Context(0)
for n in shapes:
    N = 1
    for m in n:
        N *= m
    ctx.set_grid(n, 1)
    X = torch.rand(N, dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    Ls = [torch.rand(m * m, dtype=torch.float64, device="cuda") / m for m in n]
    for _ in range(2):
        ctx.tucker(X, Y, Ls)
    fl = 2.0 * N * sum(n)
    reps = max(2, min(20, int(2e12 / fl)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ctx.tucker(X, Y, Ls)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{'x'.join(map(str, n)):>14s}  {ms:9.3f} ms  {fl / ms / 1e9:6.2f} TF/s", flush=True)
