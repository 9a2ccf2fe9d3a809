"""Tucker-operator throughput (dense flops / CUDA-event time) for a list of shapes; R Tuckers
captured in a CUDA graph and replayed between events (no host launch overhead).

    python tools/tucker_bench.py 512x512 256x256x256 ...      (KX_GEMM_CFG=0|1|2 forces a tile)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2310_07551_b200 import kx  # noqa: E402

shapes = [[int(x) for x in a.split("x")] for a in (sys.argv[1:] or ["1024x1024", "4096x4096", "256x256x256", "512x512x512", "128x128x128"])]
stream = torch.cuda.Stream()
out = {}
for n in shapes:
    N = 1
    for m in n:
        N *= m
    ctx = kx.Context(0, stream)
    ctx.set_grid(n, 1)
    X = torch.rand(N, dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    Ls = [torch.rand(m * m, dtype=torch.float64, device="cuda") / m for m in n]
    for _ in range(2):
        ctx.tucker(X, Y, Ls)
    ctx.sync()
    fl = 2.0 * N * sum(n)
    reps = int(min(200, max(3, 2e10 / fl)))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream, capture_error_mode="relaxed"):
        for _ in range(reps):
            ctx.tucker(X, Y, Ls)
    g.replay()
    stream.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(3):
        with torch.cuda.stream(stream):
            e0.record()
            g.replay()
            e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    key = "x".join(map(str, n))
    out[key] = {"us": round(best * 1e3, 2), "tflops": round(fl / best / 1e9, 2)}
    del g
    ctx.close()
print(json.dumps({"cfg": os.environ.get("KX_GEMM_CFG", "auto"), **out}))
