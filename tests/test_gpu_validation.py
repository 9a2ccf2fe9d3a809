"""Paper-protocol validation of the GPU integrators, all through the C ABI:
self-convergence orders (the slope-2 / slope-3 lines of Figs. 1-8) and the Turing patterns of
Fig. 3 (Schnakenberg modes (3,5)/(5,3), colour bar 0.6-1.8) and Fig. 7 (FHN mode
(2,2,2) with u within about +-0.107)."""
import itertools
import math

import numpy as np
import pytest

import inputs
from oracle.tensor import unvec

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


def integrate_gpu(kx, prob, scheme, T, m):
    ctx = kx.Context(0)
    ctx.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(prob.d):
            ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    ctx.set_model(prob.model, prob.params)
    ctx.set_tau(T / m, scheme)
    U = [torch.from_numpy(u.copy()).cuda() for u in prob.U0]
    for k in range(m):
        ctx.step(U, k * T / m)
    ctx.sync()
    out = [u.cpu().numpy() for u in U]
    ctx.close()
    return out


@pytest.mark.parametrize("scheme,lo,hi,ladder", [("etd2rkds", 1.75, 2.25, [200, 400, 800]),
                                                 ("etd3rkds", 2.75, 3.25, [200, 400, 800]),
                                                 # the complex split is pre-asymptotic at 200 steps
                                                 # (the oracle gives the same ratios 6.1, 6.9, 7.5)
                                                 ("exprk3ds_cplx", 2.75, 3.25, [400, 800, 1600])])
def test_self_convergence_order(kx, scheme, lo, hi, ladder):
    prob = inputs.make_problem("schnakenberg", 2, 64, seed=1)
    T = 0.1
    ref = integrate_gpu(kx, prob, scheme, T, 8 * ladder[-1])
    errs = []
    for m in ladder:
        out = integrate_gpu(kx, prob, scheme, T, m)
        errs.append(max(np.max(np.abs(out[c] - ref[c])) for c in range(2)))
    slope = -np.polyfit(np.log(ladder), np.log(errs), 1)[0]
    assert lo <= slope <= hi, (slope, errs)


def modes(U, kmax):
    n, d = U.shape, U.ndim
    W = U - U.mean()
    out = []
    for k in itertools.product(range(kmax + 1), repeat=d):
        if sum(k) == 0:
            continue
        b = unvec(inputs.kron_vec([inputs.cosine_mode(n[mu], k[mu]) for mu in range(d)]), list(n))
        out.append((abs(np.sum(W * b)) / np.sum(b * b), k))
    return sorted(out, reverse=True)


def test_schnakenberg_turing_pattern(kx):
    prob = inputs.make_problem("schnakenberg", 2, 64, seed=2)
    out = integrate_gpu(kx, prob, "etd3rkds", 2.0, 2000)
    u = unvec(out[0], [64, 64])
    top = modes(u, 8)
    assert top[0][1] in ((3, 5), (5, 3)), top[:3]
    assert 0.55 < u.min() and u.max() < 1.85


def test_fhn_turing_pattern(kx):
    prob = inputs.make_problem("fhn", 3, 32, seed=2)
    out = integrate_gpu(kx, prob, "etd3rkds", 150.0, 10000)
    u = unvec(out[0], [32, 32, 32])
    top = modes(u, 4)
    assert top[0][1] == (2, 2, 2), top[:3]
    assert 0.09 < np.max(np.abs(u)) < 0.12


@pytest.mark.parametrize("case", [("schnakenberg", 2, 128, "etd3rkds", 2.0, 6000),
                                  ("fhn", 3, 32, "etd3rkds", 150.0, 10000)])
def test_full_integration_parity(kx, case):
    """north_star: GPU vs oracle within 1e-10 after a FULL integration to the paper's final
    times (T = 2; T = 150) at reduced n, where the dynamics do not
    amplify rounding (1-ulp floor <= 1e-14)."""
    from oracle.etd import integrate
    model, d, n, scheme, T, m = case
    prob = inputs.make_problem(model, d, n, seed=0)
    out = integrate_gpu(kx, prob, scheme, T, m)
    ref, _ = integrate(prob, scheme, T=T, m=m)
    err = max(np.max(np.abs(out[c] - ref[c])) / np.max(np.abs(ref[c])) for c in range(2))
    assert err <= 1e-10, err


@pytest.mark.parametrize("case", [("C2", 2), ("C3", 3)])
def test_full_size_config_steps(kx, case):
    """BASELINE.json configs[1] (1024^2 Schnakenberg) and configs[2] (128^3 FHN) at their full
    size, in the launch configuration bench.py times (graph replay), vs the oracle — whose
    phi-bank at n = 1024 alone is ~5 TFLOP on the host (~30 s)."""
    from oracle.etd import integrate
    name, steps = case
    cfg = inputs.CONFIGS[name]
    prob = inputs.make_problem(cfg["model"], cfg["d"], cfg["n"], seed=0)
    out = integrate_gpu(kx, prob, cfg["scheme"], cfg["T"] * steps / cfg["m"], steps)
    ref, _ = integrate(prob, cfg["scheme"], T=cfg["T"], m=cfg["m"], steps=steps)
    err = max(np.max(np.abs(out[c] - ref[c])) / np.max(np.abs(ref[c])) for c in range(2))
    assert err <= 1e-10, err


@pytest.mark.parametrize("scheme", ["etd3rkds", "exprk3ds_cplx"])
def test_c4_size_linear_closed_form(kx, scheme):
    """configs[3] size (512^3 FHN delta_v, tau = 0.015), g = 0, cosine-mode data: one step is
    the scalar recurrence of SURVEY §8(c) (no oracle run needed at this size)."""
    from oracle import coeffs
    n, delta, tau = 512, 42.1887, 0.015
    A = inputs.laplacian_neumann(n, math.pi, delta)
    ks = (2, 37, 130)
    x = inputs.kron_vec([inputs.cosine_mode(n, k) for k in ks])
    lams = [inputs.cosine_eigenvalue(n, math.pi, delta, k) for k in ks]
    ctx = kx.Context(0)
    ctx.set_grid([n, n, n], 2)
    for c in range(2):
        for mu in (1, 2, 3):
            ctx.set_direction_matrix(c, mu, A)
    ctx.set_model("none")
    ctx.set_tau(tau, scheme)
    U = [torch.from_numpy(x).cuda(), torch.from_numpy(x).cuda()]
    ctx.step(U)
    ctx.sync()
    s = coeffs.table3(1, 3) if scheme == "etd3rkds" else coeffs.table2(1, 3)

    def phis(ell, z):
        import cmath
        e = cmath.exp(z)
        return [e, (e - 1) / z, (e - 1 - z) / (z * z)][ell]

    split = sum(eta * np.prod([phis(li, tau * al[m] * lams[m]) for m in range(3)])
                for eta, li, al in zip(s.etas, s.inner, s.alphas))
    expect = np.real(1.0 + tau * sum(lams) * split) * x
    got = U[0].cpu().numpy()
    assert np.max(np.abs(got - expect)) / np.max(np.abs(expect)) <= 1e-11
    ctx.close()


def test_c_client_example(kx):
    """examples/schnakenberg_2d.c drives the library through the C ABI alone (no Python in the
    loop) and reaches the Turing pattern's range at T = 2 (colour bar 0.6-1.8)."""
    import os
    import re
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build", "schnakenberg_2d")
    assert os.path.exists(exe)
    r = subprocess.run([exe, "64", "2000", "2"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lo, hi = map(float, re.findall(r"u in \[([0-9.]+), ([0-9.]+)\]", r.stdout)[-1])
    assert 0.55 < lo < 0.8 and 1.5 < hi < 1.85, r.stdout
    assert "40000 Tucker operators" in r.stdout    # 2000 steps x 2 species x 10
