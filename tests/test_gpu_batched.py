"""GPU parity of the batched Tucker operator (kx_tucker_batched): nbatch independent Tucker
operators T(X_b, {L_mu}) sharing the matrices, one GEMM launch per mode, against the
oracle's Tucker of every batch element (1e-12 relative inf-norm, north_star)."""
import math

import numpy as np
import pytest

import inputs
from oracle.tensor import tucker, unvec, vec

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def kx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2310_07551_b200 import build
    build.build()
    from paper_2310_07551_b200 import kx as mod
    return mod


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def relerr(x, ref):
    return np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300)


@pytest.mark.parametrize("n,nb", [([7], 3), ([256, 256], 4), ([100, 150], 3), ([65, 33], 5),
                                  ([1, 9], 2), ([16, 24, 32], 3), ([33, 17, 65], 2),
                                  ([3, 4, 5, 6], 4), ([512, 512], 2), ([64, 64, 64], 1)])
def test_tucker_batched_parity(kx, n, nb):
    ctx = kx.Context(0)
    try:
        ctx.set_grid(n, 1)
        N = int(np.prod(n))
        x = inputs.uniform_sym(31, 0, nb * N)
        y0 = inputs.uniform_sym(32, 0, nb * N)
        Ls = [inputs.uniform_sym(40 + mu, 0, m * m).reshape(m, m) / math.sqrt(m)
              for mu, m in enumerate(n)]
        Y = dev(y0)
        ctx.tucker_batched(dev(x), Y, [dev(L.T.copy()) for L in Ls], nb, alpha=0.5, beta=-1.25)
        out = Y.cpu().numpy()
        for b in range(nb):
            ref = 0.5 * vec(tucker(unvec(x[b * N:(b + 1) * N], n), Ls)) - 1.25 * y0[b * N:(b + 1) * N]
            assert relerr(out[b * N:(b + 1) * N], ref) <= 1e-12, b
        cnt = ctx.counters()
        assert cnt["tucker_ops"] == nb and cnt["gemm_launches"] == len(n)
    finally:
        ctx.close()


def test_tucker_batched_matches_single(kx):
    """The batched launch and nbatch single kx_tucker calls agree to rounding."""
    n, nb = [256, 256], 6
    ctx = kx.Context(0)
    try:
        ctx.set_grid(n, 1)
        N = n[0] * n[1]
        X = dev(inputs.uniform_sym(5, 0, nb * N))
        Ls = [dev(inputs.uniform_sym(6 + mu, 0, 256 * 256) / 16.0) for mu in range(2)]
        Yb = torch.zeros_like(X)
        ctx.tucker_batched(X, Yb, Ls, nb)
        Ys = torch.zeros_like(X)
        for b in range(nb):
            ctx.tucker(X[b * N:(b + 1) * N], Ys[b * N:(b + 1) * N], Ls)
        ctx.sync()
        assert relerr(Yb.cpu().numpy(), Ys.cpu().numpy()) <= 1e-14
    finally:
        ctx.close()


def test_tucker_batched_rejects_bad_args(kx):
    ctx = kx.Context(0)
    try:
        ctx.set_grid([8, 8], 1)
        X = dev(np.zeros(64 * 2))
        L = dev(np.eye(8))
        with pytest.raises(ValueError):
            ctx.tucker_batched(X, torch.zeros_like(X), [L, L], 3)   # too small for 3 tensors
        with pytest.raises(kx.KxError):
            ctx.tucker_batched(X, X, [L, L], 2)                     # aliasing
    finally:
        ctx.close()
