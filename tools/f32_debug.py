"""Diagnostics for the fp32 tcgen05 mode-product GEMM: per-mode errors with identity / random /
structured matrices, and where the wrong entries sit (rows, columns, k-ranges).  Not a test."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_07551_b200 import kx  # noqa: E402


def col32(M):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(M, np.float32).T)).cuda()


def mp_ref(x, L, mu, n):
    T = x.astype(np.float64).reshape(n[::-1])           # C-order (n_d, ..., n_1)
    ax = len(n) - mu
    return np.moveaxis(np.tensordot(L.astype(np.float64), T, axes=([1], [ax])), 0, ax).reshape(-1)


def run(n, mu, kind):
    N = int(np.prod(n))
    m = n[mu - 1]
    rng = np.random.default_rng(0)
    x = rng.standard_normal(N).astype(np.float32)
    if kind == "eye":
        L = np.eye(m, dtype=np.float32)
    elif kind == "shift":
        L = np.roll(np.eye(m, dtype=np.float32), 1, axis=1)
    elif kind == "ones":
        L = np.ones((m, m), np.float32)
    else:
        L = rng.standard_normal((m, m)).astype(np.float32)
    ctx = kx.Context(0)
    ctx.set_grid(n, 1)
    X = torch.from_numpy(x).cuda()
    Y = torch.zeros(N, dtype=torch.float32, device="cuda")
    ctx.mode_product_f32(X, Y, mu, col32(L), 1.0, 0.0)
    y = Y.cpu().numpy().astype(np.float64)
    ref = mp_ref(x, L, mu, n)
    err = np.abs(y - ref)
    rel = err.max() / max(np.abs(ref).max(), 1e-30)
    out = f"n={n} mu={mu} {kind:5s} rel={rel:.3e}"
    if rel > 1e-5:
        E = err.reshape(n[::-1]) > 1e-4 * np.abs(ref).max()
        # fraction wrong along each axis (C-order axes: n_d ... n_1)
        for ax in range(len(n)):
            other = tuple(a for a in range(len(n)) if a != ax)
            frac = E.mean(axis=other)
            bad = np.nonzero(frac > 0)[0]
            out += f"\n   axis i_{len(n) - ax}: wrong at {len(bad)}/{E.shape[ax]} idx, first {bad[:12].tolist()}"
        if kind in ("eye", "shift"):
            yy = y.reshape(n[::-1])
            rr = ref.reshape(n[::-1])
            idx = np.argwhere(E)[:4]
            for ii in idx:
                out += f"\n   at {tuple(ii)} got {yy[tuple(ii)]:.4f} want {rr[tuple(ii)]:.4f}"
    print(out, flush=True)
    ctx.close()


if __name__ == "__main__":
    for n in ([128, 128], [64, 64], [256, 128], [128, 256]):
        for mu in (1, 2):
            for kind in ("eye", "shift", "ones", "rand"):
                run(n, mu, kind)
