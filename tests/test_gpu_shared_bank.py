"""GPU parity with a SHARED phi-bank (SURVEY §8(c) ledger row 8, run (i)): the oracle's own
phi-matrices are uploaded into the library's bank with kx_set_phi_matrix, so the hot path —
the term-fused split actions (concat-M first mode, batched middle modes, concat-K last mode with
the eta and stage scalars folded into the blocks, the "+U" epilogues) and whole steps — is
compared with the oracle independently of the two phi algorithms (reading R8).  The bar is
north_star's 1e-12 relative inf-norm per split application (a sum of Tucker operators), and
1e-11 after 20 full-size steps.  The independent-bank tests (test_gpu_parity.py) stay.

Bank correspondence (Algorithms 1-2, "Needed phi-functions", P:2212-2228 / P:2285-2301):
kx (ell, stage) = (1, 0) <-> P_{i,2}^{(1)} (c = 1/3); (1, 1) <-> P_{i,3}^{(1)}; (1, 2) <-> P_{i,f}^{(1)};
(2, 1) <-> P_{i,3}^{(2)} (c = 2/3); (2, 2) <-> P_{i,f}^{(2)} (c = 1).  Complex terms (Table 2) are
two real planes: term 2i = Re, 2i+1 = Im."""
import numpy as np
import pytest

import inputs
from oracle.etd import (etd2rkds_precompute, exprk3ds_precompute, integrate, split_apply)
from oracle.tensor import unvec, vec

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

KEYS = {(1, 0): ("2", 1), (1, 1): ("3", 1), (1, 2): ("f", 1), (2, 1): ("3", 2), (2, 2): ("f", 2)}


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
    x, ref = np.asarray(x), np.asarray(ref)
    return np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300)


def oracle_bank(prob, scheme, tau):
    if scheme == "etd2rkds":
        return etd2rkds_precompute(prob.A, tau)
    return exprk3ds_precompute(prob.A, tau, "cplx" if scheme == "exprk3ds_cplx" else "real")


def bank_terms(bank, scheme, c, ell, stage):
    """(etas, P[i][mu-1]) of the oracle bank for the library's (ell, stage)."""
    if scheme == "etd2rkds":
        return ([bank.eta1], bank.P1[c]) if ell == 1 else ([bank.eta2], bank.P2[c])
    etas = bank.s1.etas if ell == 1 else bank.s2.etas
    return etas, bank.P[c][KEYS[(ell, stage)]]


def pairs(scheme):
    return [(1, 2), (2, 2)] if scheme == "etd2rkds" else list(KEYS)


def upload(ctx, bank, scheme, d):
    cplx = scheme == "exprk3ds_cplx"
    for c in range(2):
        for ell, stage in pairs(scheme):
            _, P = bank_terms(bank, scheme, c, ell, stage)
            for i, Pi in enumerate(P):
                for mu in range(1, d + 1):
                    M = Pi[mu - 1]
                    if cplx:
                        ctx.set_phi_matrix(c, ell, stage, 2 * i, mu, np.real(M))
                        ctx.set_phi_matrix(c, ell, stage, 2 * i + 1, mu, np.imag(M))
                    else:
                        ctx.set_phi_matrix(c, ell, stage, i, mu, M)


def make_ctx(kx, prob, scheme, tau, bank):
    ctx = kx.Context(0)
    ctx.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(prob.d):
            ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    ctx.set_model(prob.model, prob.params)
    ctx.set_tau(tau, scheme)
    upload(ctx, bank, scheme, prob.d)
    return ctx


def check_phi_apply(ctx, prob, scheme, bank, seed=8):
    x = inputs.uniform_sym(seed, 0, prob.N)
    y0 = inputs.uniform_sym(seed, 1, prob.N)
    X = dev(x)
    worst = 0.0
    for c in range(2):
        for ell, stage in pairs(scheme):
            etas, P = bank_terms(bank, scheme, c, ell, stage)
            ref = vec(split_apply(etas, P, unvec(x, prob.n)))
            if scheme == "exprk3ds_cplx":
                ref = np.real(ref)
            Y = dev(y0)
            ctx.phi_apply(c, ell, stage, X, Y, alpha=0.5, beta=1.0)
            worst = max(worst, relerr(Y.cpu().numpy(), 0.5 * ref + y0))
            # the round trip of the upload is exact
            P0 = ctx.phi_matrix(c, ell, stage, 0, 1)
            assert np.array_equal(P0, np.real(P[0][0]))
    return worst


@pytest.mark.parametrize("case", [("schnakenberg", 2, 64, "etd3rkds", 1.0 / 3000),
                                  ("schnakenberg", 2, 100, "etd3rkds", 1e-3),          # ragged n
                                  ("schnakenberg", 2, [48, 80], "exprk3ds_cplx", 1e-3),
                                  ("schnakenberg", 2, 64, "etd2rkds", 0.25 / 3000),
                                  ("fhn", 3, 32, "etd3rkds", 0.015),
                                  ("fhn", 3, [24, 20, 28], "exprk3ds_cplx", 0.015),
                                  ("fhn", 3, 33, "etd3rkds", 0.015)])                  # ragged n
def test_phi_apply_shared_bank(kx, case):
    """kx_phi_apply with the oracle's phi-matrices vs the oracle's split_apply: 1e-12."""
    model, d, n, scheme, tau = case
    prob = inputs.make_problem(model, d, n, seed=0)
    bank = oracle_bank(prob, scheme, tau)
    ctx = make_ctx(kx, prob, scheme, tau, bank)
    try:
        assert check_phi_apply(ctx, prob, scheme, bank) <= 1e-12
    finally:
        ctx.close()


@pytest.mark.parametrize("case", [("schnakenberg", 2, 64, "etd3rkds", 2.0, 6000, 20),
                                  ("schnakenberg", 2, 64, "etd2rkds", 0.25, 3000, 20),
                                  ("schnakenberg", 2, 100, "exprk3ds_cplx", 0.25, 1000, 10),
                                  ("fhn", 3, 32, "etd3rkds", 150.0, 10000, 20),
                                  ("fhn", 3, 24, "exprk3ds_cplx", 150.0, 10000, 10)])
@pytest.mark.parametrize("fused_small", [True, False])
def test_steps_shared_bank(kx, case, fused_small):
    """Whole steps on the shared bank: the stage GEMMs (concat-K over 2T / 3T segments with the
    folded c*eta scalars) and the nonlinearity against Algorithms 1-2 step by step."""
    model, d, n, scheme, T, m, steps = case
    prob = inputs.make_problem(model, d, n, seed=0)
    tau = T / m
    bank = oracle_bank(prob, scheme, tau)
    ctx = make_ctx(kx, prob, scheme, tau, bank)
    try:
        ctx.set_fused_small(fused_small)
        U = [dev(u) for u in prob.U0]
        ctx.step(U)
        ctx.sync()
        ref1, _ = integrate(prob, scheme, T=T, m=m, steps=1, bank=bank)
        assert max(relerr(U[c].cpu().numpy(), ref1[c]) for c in range(2)) <= 1e-12
        for k in range(1, steps):
            ctx.step(U, k * tau)
        ctx.sync()
        ref, _ = integrate(prob, scheme, T=T, m=m, steps=steps, bank=bank)
        assert max(relerr(U[c].cpu().numpy(), ref[c]) for c in range(2)) <= 1e-11
    finally:
        ctx.close()


@pytest.fixture(scope="module", params=["C2", "C3"])
def full_size(request, kx):
    """BASELINE.json configs[1] / configs[2] at their full size with the oracle's bank (the
    oracle's phi-bank at n = 1024 is ~6 TFLOP of host BLAS)."""
    cfg = inputs.CONFIGS[request.param]
    prob = inputs.make_problem(cfg["model"], cfg["d"], cfg["n"], seed=0)
    tau = cfg["T"] / cfg["m"]
    bank = oracle_bank(prob, cfg["scheme"], tau)
    return request.param, cfg, prob, tau, bank


def test_phi_apply_shared_bank_full_size(kx, full_size):
    name, cfg, prob, tau, bank = full_size
    ctx = make_ctx(kx, prob, cfg["scheme"], tau, bank)
    try:
        assert check_phi_apply(ctx, prob, cfg["scheme"], bank) <= 1e-12, name
    finally:
        ctx.close()


def test_steps_shared_bank_full_size(kx, full_size):
    """20 steps of C2 / C3 in the launch configuration bench.py times (graph replay) vs the
    oracle on the same bank: 1e-11."""
    name, cfg, prob, tau, bank = full_size
    ctx = make_ctx(kx, prob, cfg["scheme"], tau, bank)
    try:
        U = [dev(u) for u in prob.U0]
        for k in range(20):
            ctx.step(U, k * tau)
        ctx.sync()
        ref, _ = integrate(prob, cfg["scheme"], T=cfg["T"], m=cfg["m"], steps=20, bank=bank)
        err = max(relerr(U[c].cpu().numpy(), ref[c]) for c in range(2))
        assert err <= 1e-11, (name, err)
    finally:
        ctx.close()
