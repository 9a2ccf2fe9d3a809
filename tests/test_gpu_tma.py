"""The TMA-fed variant of the fp64 GEMM (csrc/gemm.cu, VEC = 3: fragment-ordered boxes, the
last warp out of a stage issues its refill) forced on every eligible launch (KX_GEMM_TMA=1, read
once per process, hence a subprocess) against the oracle: mode products of both layouts, Tucker
operators with ragged M / N tiles, the concatenated-K split action over several segments, and
steps; and bitwise agreement with the cp.async pipeline (KX_GEMM_TMA=0) — the same DMMA order."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import inputs
from paper_2310_07551_b200 import kx
from oracle.tensor import mode_product, tucker, unvec, vec
out = {}
def dev(a): return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()
def rel(x, r): return float(np.max(np.abs(x - r)) / np.max(np.abs(r)))
ctx = kx.Context(0)
for n in ([1000, 264], [264, 1024], [512, 40, 520]):
    N = int(np.prod(n)); ctx.set_grid(n, 1)
    x = inputs.uniform_sym(1, 0, N); Ls = [inputs.uniform_sym(2, m, k * k).reshape(k, k) for m, k in enumerate(n)]
    Y = dev(np.zeros(N)); ctx.tucker(dev(x), Y, [dev(L.T.copy()) for L in Ls]); ctx.sync()
    y = Y.cpu().numpy(); out["tucker_%s" % n] = [rel(y, vec(tucker(unvec(x, n), Ls))), y[:64].tolist()]
    for mu in range(1, len(n) + 1):
        Y = dev(np.zeros(N)); ctx.mode_product(dev(x), Y, mu, dev(Ls[mu - 1].T.copy()), 1.0, 0.0); ctx.sync()
        out["mp_%s_%d" % (n, mu)] = [rel(Y.cpu().numpy(), vec(mode_product(unvec(x, n), Ls[mu - 1], mu))), 0]
prob = inputs.make_problem("schnakenberg", 2, [1024, 256], seed=2)
ctx.set_grid(prob.n, 2)
for c in range(2):
    for mu in range(2): ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
ctx.set_model(prob.model, prob.params); ctx.set_tau(1e-4, "etd3rkds")
U = [dev(u) for u in prob.U0]
for k in range(3): ctx.step(U)
ctx.sync()
out["step"] = [0.0, U[0].cpu().numpy()[:4096:7].tolist() + U[1].cpu().numpy()[:4096:7].tolist()]
print(json.dumps(out))
"""


@pytest.fixture(scope="module")
def runs():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2310_07551_b200 import build
    build.build()
    res = {}
    for mode in ("1", "0"):
        env = dict(os.environ, KX_GEMM_TMA=mode)
        r = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[mode] = json.loads(r.stdout.strip().splitlines()[-1])
    return res


def test_tma_forced_matches_oracle(runs):
    for key, (err, _) in runs["1"].items():
        if key != "step":
            assert err <= 1e-12, (key, err)


def test_tma_bitwise_equals_cp_async(runs):
    """Same operand values reach the same DMMA sequence, so results are bit-identical."""
    for key in runs["1"]:
        assert runs["1"][key][1] == runs["0"][key][1], key
