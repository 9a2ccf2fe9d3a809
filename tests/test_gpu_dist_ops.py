"""The distributed operators (kx_tucker / kx_mode_product / kx_phi_apply on slab-sharded
contexts; csrc/kx_dist_ops.cpp) on in-process loopback groups of P = 2, 4 ranks and on a
one-rank NCCL context: the assembled slabs equal the oracle at north_star's 1e-12 relative
inf-norm per operator and the single-GPU operator to rounding (BASELINE.json configs[4]: the
Tucker sweep at 2-8 GPUs)."""
import numpy as np
import pytest

import inputs
from oracle.etd import split_apply
from oracle.tensor import mode_product, tucker, unvec, vec

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


def dmat(A):
    return dev(np.asarray(A, dtype=np.float64).T.copy())


def relerr(x, ref):
    return np.max(np.abs(np.asarray(x) - ref)) / max(np.max(np.abs(ref)), 1e-300)


def slab(u, n, r, P):
    T = unvec(u, n)
    nd = n[-1] // P
    return vec(T[..., r * nd:(r + 1) * nd])


def assemble(parts, n, P):
    return vec(np.concatenate([unvec(p.cpu().numpy(), n[:-1] + [n[-1] // P]) for p in parts], axis=-1))


def make_group(kx, n, P, ncomp=1):
    g = kx.Group(P)
    for c in g.ctx:
        c.set_grid(n, ncomp)
    return g


@pytest.mark.parametrize("case", [([64, 48], 2), ([128, 96], 4), ([24, 20, 32], 2), ([16, 12, 16], 4),
                                  ([36, 20, 28], 2), ([8, 6, 5, 4], 2), ([64, 24, 32], 8), ([128, 64], 8)])
def test_tucker_group(kx, case):
    n, P = case
    N = int(np.prod(n))
    x = inputs.uniform_sym(21, 0, N)
    y0 = inputs.uniform_sym(22, 0, N)
    Ls = [inputs.uniform_sym(23, mu, m * m).reshape(m, m) for mu, m in enumerate(n)]
    g = make_group(kx, n, P)
    Xs = [dev(slab(x, n, r, P)) for r in range(P)]
    Ys = [dev(slab(y0, n, r, P)) for r in range(P)]
    g.tucker(Xs, Ys, [dmat(L) for L in Ls], alpha=0.5, beta=-1.5)
    g.ctx[0].sync()
    ref = 0.5 * vec(tucker(unvec(x, n), Ls)) - 1.5 * y0
    out = assemble(Ys, n, P)
    assert relerr(out, ref) <= 1e-12
    # and the single-GPU operator to rounding
    one = kx.Context(0)
    one.set_grid(n, 1)
    Y1 = dev(y0)
    one.tucker(dev(x), Y1, [dmat(L) for L in Ls], alpha=0.5, beta=-1.5)
    assert relerr(out, Y1.cpu().numpy()) <= 1e-13
    assert all(c.counters()["tucker_ops"] == 1 for c in g.ctx)
    one.close()
    g.close()


@pytest.mark.parametrize("case", [([64, 48], 2), ([24, 20, 32], 4)])
def test_mode_product_group(kx, case):
    n, P = case
    N = int(np.prod(n))
    x = inputs.uniform_sym(31, 0, N)
    y0 = inputs.uniform_sym(32, 0, N)
    g = make_group(kx, n, P)
    for mu in range(1, len(n) + 1):
        m = n[mu - 1]
        L = inputs.uniform_sym(33, mu, m * m).reshape(m, m)
        Xs = [dev(slab(x, n, r, P)) for r in range(P)]
        Ys = [dev(slab(y0, n, r, P)) for r in range(P)]
        g.mode_product(Xs, Ys, mu, dmat(L), alpha=2.0, beta=0.25)
        g.ctx[0].sync()
        ref = 2.0 * vec(mode_product(unvec(x, n), L, mu)) + 0.25 * y0
        assert relerr(assemble(Ys, n, P), ref) <= 1e-12, mu
    g.close()


@pytest.mark.parametrize("case", [("schnakenberg", 2, [64, 48], "etd3rkds", 1e-3, 2),
                                  ("schnakenberg", 2, [48, 40], "exprk3ds_cplx", 1e-3, 4),
                                  ("fhn", 3, [24, 20, 32], "etd3rkds", 0.015, 2),
                                  ("fhn", 3, [16, 12, 16], "exprk3ds_cplx", 0.015, 4),
                                  ("fhn", 3, [16, 12, 8], "etd2rkds", 0.01, 2)])
def test_phi_apply_group_shared_bank(kx, case):
    """Split phi-action on the sharded context with the oracle's phi-matrices uploaded (shared
    bank, as tests/test_gpu_shared_bank.py) — the term-fused first/middle modes on layout B and
    the concatenated-K last mode over (term, source rank) segments, at 1e-12."""
    from test_gpu_shared_bank import bank_terms, oracle_bank, pairs, upload
    model, d, n, scheme, tau, P = case
    prob = inputs.make_problem(model, d, n, seed=9)
    bank = oracle_bank(prob, scheme, tau)
    g = kx.Group(P)
    for c in g.ctx:
        c.set_grid(prob.n, 2)
        for s in range(2):
            for mu in range(d):
                c.set_direction_matrix(s, mu + 1, prob.A[s][mu])
        c.set_model(prob.model, prob.params)
        c.set_tau(tau, scheme)
        upload(c, bank, scheme, d)
    x = inputs.uniform_sym(41, 0, prob.N)
    y0 = inputs.uniform_sym(42, 0, prob.N)
    worst = 0.0
    for comp in range(2):
        for ell, stage in pairs(scheme):
            etas, Pm = bank_terms(bank, scheme, comp, ell, stage)
            ref = vec(split_apply(etas, Pm, unvec(x, prob.n)))
            if scheme == "exprk3ds_cplx":
                ref = np.real(ref)
            Xs = [dev(slab(x, prob.n, r, P)) for r in range(P)]
            Ys = [dev(slab(y0, prob.n, r, P)) for r in range(P)]
            g.phi_apply(comp, ell, stage, Xs, Ys, alpha=0.5, beta=1.0)
            g.ctx[0].sync()
            worst = max(worst, relerr(assemble(Ys, prob.n, P), 0.5 * ref + y0))
    assert worst <= 1e-12, worst
    g.close()


def test_nccl_one_rank_operators(kx):
    """The NCCL path of the distributed operators (kx_create_dist, one rank: self-exchange
    through NCCL) equals the single-GPU operators to rounding."""
    n = [24, 20, 16]
    N = int(np.prod(n))
    x = inputs.uniform_sym(51, 0, N)
    Ls = [inputs.uniform_sym(52, mu, m * m).reshape(m, m) for mu, m in enumerate(n)]
    d = kx.Context(0, dist=(kx.nccl_unique_id(), 0, 1))
    d.set_grid(n, 1)
    one = kx.Context(0)
    one.set_grid(n, 1)
    Yd, Y1 = dev(np.zeros(N)), dev(np.zeros(N))
    d.tucker(dev(x), Yd, [dmat(L) for L in Ls])
    one.tucker(dev(x), Y1, [dmat(L) for L in Ls])
    d.sync()
    one.sync()
    assert relerr(Yd.cpu().numpy(), Y1.cpu().numpy()) <= 1e-13
    assert relerr(Yd.cpu().numpy(), vec(tucker(unvec(x, n), Ls))) <= 1e-12
    for mu in (1, 3):
        d.mode_product(dev(x), Yd, mu, dmat(Ls[mu - 1]), 1.0, 0.0)
        d.sync()
        assert relerr(Yd.cpu().numpy(), vec(mode_product(unvec(x, n), Ls[mu - 1], mu))) <= 1e-12
    d.close()
    one.close()


def test_group_ops_no_out_of_bounds_writes(kx):
    """Guard bands around every rank's output slab: the distributed operators' pack, exchange
    copies, concat-K GEMM over source-rank segments and unpack stay inside the slabs."""
    n, P, G = [36, 20, 16], 2, 512
    N = int(np.prod(n))
    Nl = N // P
    g = make_group(kx, n, P)
    x = inputs.uniform_sym(71, 0, N)
    Ls = [dmat(inputs.uniform_sym(72, mu, m * m).reshape(m, m)) for mu, m in enumerate(n)]
    bigs = [torch.full((Nl + 2 * G,), 4321.0, dtype=torch.float64, device="cuda") for _ in range(P)]
    Ys = [b[G:G + Nl] for b in bigs]
    Xs = [dev(slab(x, n, r, P)) for r in range(P)]
    g.tucker(Xs, Ys, Ls, 1.0, 0.5)
    for mu in range(1, len(n) + 1):
        g.mode_product(Xs, Ys, mu, Ls[mu - 1], 1.0, 1.0)
    g.ctx[0].sync()
    for b in bigs:
        v = b[:G].cpu().numpy().tolist() + b[G + Nl:].cpu().numpy().tolist()
        assert len(set(v)) == 1, "guard band overwritten"
    g.close()


@pytest.mark.parametrize("case", [([64, 48], 2), ([24, 20, 32], 4), ([8, 6, 5, 4], 2)])
def test_kronsum_group(kx, case):
    """Kronecker-sum action on slabs (eq:kronsumv): modes 1..d-1 local, the mode-d
    term through the two exchanges; dense random A_mu (no stencil shortcut)."""
    from oracle.tensor import kronsum_apply
    n, P = case
    N = int(np.prod(n))
    x = inputs.uniform_sym(81, 0, N)
    y0 = inputs.uniform_sym(82, 0, N)
    As = [inputs.uniform_sym(83, mu, m * m).reshape(m, m) for mu, m in enumerate(n)]
    g = kx.Group(P)
    for c in g.ctx:
        c.set_grid(n, 1)
        for mu in range(len(n)):
            c.set_direction_matrix(0, mu + 1, As[mu])
    Xs = [dev(slab(x, n, r, P)) for r in range(P)]
    Ys = [dev(slab(y0, n, r, P)) for r in range(P)]
    g.kronsum(0, Xs, Ys, beta=0.5)
    g.ctx[0].sync()
    ref = vec(kronsum_apply(unvec(x, n), As)) + 0.5 * y0
    assert relerr(assemble(Ys, n, P), ref) <= 1e-12
    g.close()


@pytest.mark.parametrize("scheme", ["etd3rkds", "exprk3ds_cplx"])
def test_nccl_one_rank_phi_apply_and_kronsum(kx, scheme):
    """kx_phi_apply and kx_kronsum through the NCCL path of a one-rank distributed context equal
    the single-GPU calls to rounding (every (ell, stage) of the bank, both components)."""
    prob = inputs.make_problem("fhn", 3, [24, 20, 16], seed=4)
    tau = 0.015
    uid = kx.nccl_unique_id()
    ctxs = [kx.Context(0, dist=(uid, 0, 1)), kx.Context(0)]
    for c in ctxs:
        c.set_grid(prob.n, 2)
        for s in range(2):
            for mu in range(3):
                c.set_direction_matrix(s, mu + 1, prob.A[s][mu])
        c.set_model(prob.model, prob.params)
        c.set_tau(tau, scheme)
    x = dev(inputs.uniform_sym(91, 0, prob.N))
    y0 = inputs.uniform_sym(92, 0, prob.N)
    for comp in range(2):
        for ell, stage in [(1, 0), (1, 1), (1, 2), (2, 1), (2, 2)]:
            Ys = [dev(y0), dev(y0)]
            for c, Y in zip(ctxs, Ys):
                c.phi_apply(comp, ell, stage, x, Y, 0.5, 1.0)
                c.sync()
            assert relerr(Ys[0].cpu().numpy(), Ys[1].cpu().numpy()) <= 1e-13, (comp, ell, stage)
        Ys = [dev(y0), dev(y0)]
        for c, Y in zip(ctxs, Ys):
            c.set_kronsum_mode(True)     # dense A_mu on both (the sharded kronsum is dense)
            c.kronsum(comp, x, Y, 0.25)
            c.sync()
        assert relerr(Ys[0].cpu().numpy(), Ys[1].cpu().numpy()) <= 1e-13
    for c in ctxs:
        c.close()
