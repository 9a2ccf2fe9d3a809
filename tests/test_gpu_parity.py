"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs.  Tolerances (BASELINE.json north_star): 1e-12 relative inf-norm per Tucker
application / mode product / Kronecker-sum action; phi-bank and split actions with two
INDEPENDENT phi algorithms (library: Taylor theta=1 + doubling on the GPU; oracle: Taylor
theta=2 + doubling on the CPU) agree to the phi-bank limit of DESIGN.md (1e-11 at stiff
settings); integrations to 1e-10 relative."""
import math

import numpy as np
import pytest

import inputs
from oracle import coeffs
from oracle.etd import exprk3ds_precompute, integrate, split_apply, split_phi_matrices
from oracle.phi import phi_matrices
from oracle.tensor import kronsum_apply, mode_product, tucker, unvec, vec

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


@pytest.fixture
def ctx(kx):
    c = kx.Context(0)
    yield c
    c.close()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def dmat(A):
    """Device column-major copy of a dense matrix."""
    return dev(np.asarray(A).T.copy())


def relerr(x, ref):
    x, ref = np.asarray(x), np.asarray(ref)
    return np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300)


def tensor(n, seed, stream=0):
    return inputs.uniform_sym(seed, stream, int(np.prod(n)))


SHAPES = [[1], [7], [64], [3, 5], [65, 33], [100, 150], [128, 128], [1, 9], [9, 1],
          [5, 6, 7], [16, 24, 32], [33, 17, 65], [64, 64, 64], [3, 4, 5, 6], [2, 3, 2, 3, 2]]


@pytest.mark.parametrize("n", SHAPES, ids=lambda n: "x".join(map(str, n)))
def test_mode_product_parity(ctx, n):
    ctx.set_grid(n, 1)
    x = tensor(n, 1)
    X = dev(x)
    Xo = unvec(x, n)
    for mu in range(1, len(n) + 1):
        L = inputs.uniform_sym(10 + mu, 0, n[mu - 1] ** 2).reshape(n[mu - 1], n[mu - 1])
        y0 = tensor(n, 2)
        Y = dev(y0)
        ctx.mode_product(X, Y, mu, dmat(L), alpha=0.75, beta=-0.5)
        ref = 0.75 * vec(mode_product(Xo, L, mu)) - 0.5 * y0
        assert relerr(Y.cpu().numpy(), ref) <= 1e-13, mu


@pytest.mark.parametrize("n", SHAPES, ids=lambda n: "x".join(map(str, n)))
def test_tucker_parity(ctx, n):
    ctx.set_grid(n, 1)
    x = tensor(n, 3)
    Ls = [inputs.uniform_sym(20 + mu, 0, m * m).reshape(m, m) / math.sqrt(m)
          for mu, m in enumerate(n)]
    Y = dev(np.zeros(int(np.prod(n))))
    ctx.tucker(dev(x), Y, [dmat(L) for L in Ls])
    ref = vec(tucker(unvec(x, n), Ls))
    assert relerr(Y.cpu().numpy(), ref) <= 1e-12


@pytest.mark.parametrize("n", [[6], [64, 64], [100, 150], [33, 17, 65], [32, 32, 32], [4, 5, 3, 6]],
                         ids=lambda n: "x".join(map(str, n)))
def test_kronsum_parity(ctx, n):
    ctx.set_grid(n, 2)
    As = [[inputs.laplacian_neumann(m, 1.0, 1.0 + 9.0 * c) + 0.1 * inputs.uniform_sym(5, mu, m * m).reshape(m, m)
           for mu, m in enumerate(n)] for c in range(2)]
    for c in range(2):
        for mu in range(len(n)):
            ctx.set_direction_matrix(c, mu + 1, As[c][mu])
    x = tensor(n, 4)
    for c in range(2):
        y0 = tensor(n, 6 + c)
        Y = dev(y0)
        ctx.kronsum(c, dev(x), Y, beta=2.0)
        ref = vec(kronsum_apply(unvec(x, n), As[c])) + 2.0 * y0
        assert relerr(Y.cpu().numpy(), ref) <= 1e-12


@pytest.mark.parametrize("n", [[7], [64, 64], [100, 150], [33, 17, 65], [32, 32, 32], [4, 5, 3, 6]],
                         ids=lambda n: "x".join(map(str, n)))
@pytest.mark.parametrize("dense", [False, True])
def test_kronsum_tridiagonal_parity(ctx, n, dense):
    """FD Neumann Laplacians (tridiagonal): the stencil path and the dense-GEMM path."""
    ctx.set_grid(n, 2)
    ctx.set_kronsum_mode(dense)
    As = [[inputs.laplacian_neumann(m, 1.0, 1.0 + 9.0 * c + mu) for mu, m in enumerate(n)]
          for c in range(2)]
    for c in range(2):
        for mu in range(len(n)):
            ctx.set_direction_matrix(c, mu + 1, As[c][mu])
    x = tensor(n, 14)
    for c in range(2):
        for beta in (0.0, -1.5):
            y0 = tensor(n, 15 + c)
            Y = dev(y0)
            ctx.kronsum(c, dev(x), Y, beta=beta)
            ref = vec(kronsum_apply(unvec(x, n), As[c])) + beta * y0
            assert relerr(Y.cpu().numpy(), ref) <= 1e-12


def setup_problem(ctx, prob, scheme, tau):
    ctx.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(prob.d):
            ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    ctx.set_model(prob.model, prob.params)
    ctx.set_tau(tau, scheme)


@pytest.mark.parametrize("case", [("schnakenberg", 2, 64, 1.0 / 3000), ("schnakenberg", 2, 150, 0.25 / 1000),
                                  ("fhn", 3, 32, 0.015), ("fhn", 3, 65, 0.015)])
def test_phi_bank_vs_oracle(ctx, case):
    """Every phi-matrix of the ETD3RKDS bank against the oracle's independent phi."""
    model, d, n, tau = case
    prob = inputs.make_problem(model, d, n)
    setup_problem(ctx, prob, "etd3rkds", tau)
    s = {1: coeffs.etd3_scheme(1, d), 2: coeffs.etd3_scheme(2, d)}
    cs = {0: 1 / 3, 1: 2 / 3, 2: 1.0}
    worst = 0.0
    for c in range(2):
        for (ell, stage) in [(1, 0), (1, 1), (1, 2), (2, 1), (2, 2)]:
            for i in range(s[ell].nterms):
                for mu in range(1, d + 1):
                    P = ctx.phi_matrix(c, ell, stage, i, mu)
                    X = cs[stage] * tau * s[ell].alphas[i][mu - 1] * prob.A[c][mu - 1]
                    ref = phi_matrices(X, 2)[s[ell].inner[i]]
                    worst = max(worst, relerr(P, ref))
                    rs = P.sum(axis=1) * math.factorial(s[ell].inner[i])   # row sums = 1/l!
                    assert np.max(np.abs(rs - 1.0)) <= 1e-11
    assert worst <= 1e-11, worst


def _phi_pade(X, ell):
    """phi_ell(X) by the block (Van Loan) exponential, computed with scipy's Pade-13 scaling and
    squaring: expm([[X, I, 0], [0, 0, I], [0, 0, 0]]) holds phi_1(X) / phi_2(X) in its first block
    row (P:619-625 defines the phi-functions; a different algorithm family from both the
    library's and the oracle's Taylor + doubling)."""
    from scipy.linalg import expm
    n = X.shape[0]
    if ell == 0:
        return expm(X)
    W = np.zeros(((ell + 1) * n, (ell + 1) * n))
    W[:n, :n] = X
    for k in range(ell):
        W[k * n:(k + 1) * n, (k + 1) * n:(k + 2) * n] = np.eye(n)
    return expm(W)[:n, ell * n:(ell + 1) * n]


@pytest.mark.parametrize("case", [("schnakenberg", 2, 64, 1.0 / 3000), ("fhn", 3, 65, 0.015),
                                  ("schnakenberg", 2, 1024, 2.0 / 6000)],
                         ids=["schnakenberg64", "fhn65", "C2_1024"])
def test_phi_bank_vs_pade(ctx, case):
    """The GPU phi-bank against a Pade-based phi (not Taylor): every matrix at the small sizes,
    one phi_1 and one phi_2 matrix of each species at the full C2 size."""
    model, d, n, tau = case
    prob = inputs.make_problem(model, d, n)
    setup_problem(ctx, prob, "etd3rkds", tau)
    s = {1: coeffs.etd3_scheme(1, d), 2: coeffs.etd3_scheme(2, d)}
    cs = {0: 1 / 3, 1: 2 / 3, 2: 1.0}
    entries = [(c, ell, stage, i, mu) for c in range(2) for (ell, stage) in [(1, 0), (1, 1), (1, 2), (2, 1), (2, 2)]
               for i in range(s[ell].nterms) for mu in range(1, d + 1)]
    if n > 200:   # full size: the first term of each scheme part at the full step, both species
        entries = [(c, ell, 2, 0, 1) for c in range(2) for ell in (1, 2)]
    worst = 0.0
    for (c, ell, stage, i, mu) in entries:
        P = ctx.phi_matrix(c, ell, stage, i, mu)
        X = cs[stage] * tau * s[ell].alphas[i][mu - 1] * prob.A[c][mu - 1]
        worst = max(worst, relerr(P, _phi_pade(X, s[ell].inner[i])))
    assert worst <= 1e-11, worst


@pytest.mark.parametrize("case", [("schnakenberg", 2, 64, 1.0 / 3000), ("fhn", 3, 24, 0.015),
                                  ("schnakenberg", 2, 100, 1e-3)])
def test_phi_apply_parity(ctx, case):
    model, d, n, tau = case
    prob = inputs.make_problem(model, d, n)
    setup_problem(ctx, prob, "etd3rkds", tau)
    x = tensor(prob.n, 8)
    cs = {0: 1 / 3, 1: 2 / 3, 2: 1.0}
    for c in range(2):
        for (ell, stage) in [(1, 0), (1, 1), (1, 2), (2, 1), (2, 2)]:
            s = coeffs.etd3_scheme(ell, d)
            P = split_phi_matrices(s, cs[stage] * tau, prob.A[c])
            ref = vec(split_apply(s.etas, P, unvec(x, prob.n)))
            y0 = tensor(prob.n, 9)
            Y = dev(y0)
            ctx.phi_apply(c, ell, stage, dev(x), Y, alpha=0.5, beta=1.0)
            assert relerr(Y.cpu().numpy(), 0.5 * ref + y0) <= 1e-11


def run_gpu(ctx, prob, scheme, tau, steps):
    U = [dev(u) for u in prob.U0]
    for k in range(steps):
        ctx.step(U, k * tau)
    ctx.sync()
    return [u.cpu().numpy() for u in U]


@pytest.mark.parametrize("case", [
    ("schnakenberg", 2, 64, "etd2rkds", 0.25, 3000, 20),      # C1
    ("schnakenberg", 2, 64, "etd3rkds", 2.0, 6000, 20),
    ("schnakenberg", 2, 100, "etd3rkds", 0.25, 1000, 10),     # ragged n
    ("fhn", 3, 32, "etd3rkds", 150.0, 10000, 20),
    ("fhn", 3, 24, "etd2rkds", 5.0, 60000, 20),
    ("fhn", 3, 33, "etd3rkds", 150.0, 10000, 5),              # ragged n
])
def test_step_parity(ctx, case):
    model, d, n, scheme, T, m, steps = case
    prob = inputs.make_problem(model, d, n, seed=0)
    tau = T / m
    setup_problem(ctx, prob, scheme, tau)
    out = run_gpu(ctx, prob, scheme, tau, steps)
    ref, _ = integrate(prob, scheme, T=T, m=m, steps=steps)
    err = max(relerr(out[c], ref[c]) for c in range(2))
    assert err <= 1e-10, err
    cnt = ctx.counters()
    per = 2 if scheme == "etd2rkds" else (10 if d == 2 else 15)
    assert cnt["steps"] == steps
    assert cnt["tucker_ops"] == steps * 2 * per
    assert cnt["kronsum_actions"] == steps * 2


def test_linear_cosine_closed_form_full_size(ctx):
    """C2 size (1024^2), g = 0, cosine-mode initial data: one ETD3RKDS step is the scalar
    recurrence of SURVEY §8(c) — a full-size check that needs no oracle run."""
    n, delta, tau = 1024, 10.0, 1.0 / 3000
    A = inputs.laplacian_neumann(n, 1.0, delta)
    ks = (3, 200)
    x = inputs.kron_vec([inputs.cosine_mode(n, k) for k in ks])
    lams = [inputs.cosine_eigenvalue(n, 1.0, delta, k) for k in ks]
    ctx.set_grid([n, n], 2)
    for c in range(2):
        for mu in (1, 2):
            ctx.set_direction_matrix(c, mu, A)
    ctx.set_model("none")
    ctx.set_tau(tau, "etd3rkds")
    U = [dev(x), dev(x)]
    ctx.step(U)
    ctx.sync()
    s = coeffs.table1(1)

    def phis(ell, z):
        return [math.exp(z), math.expm1(z) / z, (math.expm1(z) - z) / (z * z)][ell]

    split = sum(eta * phis(li, tau * al[0] * lams[0]) * phis(li, tau * al[1] * lams[1])
                for eta, li, al in zip(s.etas, s.inner, s.alphas))
    expect = (1.0 + tau * sum(lams) * split) * x
    assert relerr(U[0].cpu().numpy(), expect) <= 1e-11


def test_full_size_tucker_sampled(ctx):
    """C2 size Tucker (1024^2) and C3-size (128^3): sampled outputs computed one by one."""
    for n in ([1024, 1024], [128, 128, 128]):
        ctx.set_grid(n, 1)
        x = tensor(n, 11)
        Ls = [inputs.uniform_sym(30 + mu, 0, m * m).reshape(m, m) / math.sqrt(m) for mu, m in enumerate(n)]
        Y = dev(np.zeros(x.size))
        ctx.tucker(dev(x), Y, [dmat(L) for L in Ls])
        y = unvec(Y.cpu().numpy(), n)
        X = unvec(x, n)
        rs = np.random.default_rng(0)
        for _ in range(64):
            idx = [int(rs.integers(0, m)) for m in n]
            # s_{i} = sum_j t_j prod_mu l^mu_{i_mu j_mu}
            val = X
            for mu in range(len(n) - 1, -1, -1):
                val = np.tensordot(val, Ls[mu][idx[mu]], axes=([mu], [0]))
            assert abs(y[tuple(idx)] - val) <= 1e-12 * np.max(np.abs(y))


def test_graph_replay_matches_eager(ctx):
    prob = inputs.make_problem("fhn", 3, 20, seed=2)
    setup_problem(ctx, prob, "etd3rkds", 0.015)
    Ug = [dev(u) for u in prob.U0]
    Ue = [dev(u) for u in prob.U0]
    for _ in range(3):
        ctx.step(Ug)
    ctx.set_profiling(True)
    for _ in range(3):
        ctx.step(Ue)
    prof = ctx.profile()
    ctx.set_profiling(False)
    ctx.sync()
    for c in range(2):
        assert torch.equal(Ug[c], Ue[c])
    assert prof["gemm_launches"] > 0 and prof["gemm_ms"] > 0


def test_integrate_host_matches_device(ctx):
    prob = inputs.make_problem("schnakenberg", 2, 48, seed=3)
    setup_problem(ctx, prob, "etd3rkds", 1e-4)
    Ud = [dev(u) for u in prob.U0]
    for _ in range(4):
        ctx.step(Ud)
    Uh = [u.copy() for u in prob.U0]
    ctx.integrate_host(Uh, 4)
    for c in range(2):
        assert np.array_equal(Uh[c], Ud[c].cpu().numpy())


@pytest.mark.parametrize("case", [("schnakenberg", 2, [160, 96], "etd3rkds"), ("fhn", 3, [24, 20, 16], "etd2rkds"),
                                  ("schnakenberg", 2, [1024, 1024], "etd3rkds"), ("schnakenberg", 2, [48, 40], "etd3rkds"),
                                  ("fhn", 3, [32, 32, 32], "exprk3ds_cplx")],
                         ids=["160x96_etd3", "24x20x16_etd2", "C2_1024", "48x40_one_kernel", "32cube_cplx"])
def test_integrate_host_pinned_tail(ctx, case):
    """kx_integrate_host with page-locked host buffers: the last step's final stage GEMM runs in
    row chunks whose rows are copied back while the next chunk computes.  Equal to the device
    path up to the rounding of that GEMM's k-split (<= 1e-14 relative); counters advance by the
    steps taken; a second call replays the cached graph with the same result."""
    model, d, n, scheme = case
    prob = inputs.make_problem(model, d, n, seed=3)
    tau = 1e-4 if model == "schnakenberg" else 0.01
    setup_problem(ctx, prob, scheme, tau)
    Ud = [dev(u) for u in prob.U0]
    for _ in range(3):
        ctx.step(Ud)
    ref = [u.cpu().numpy() for u in Ud]
    pinned = [torch.from_numpy(u.copy()).pin_memory() for u in prob.U0]
    for rep in range(2):
        for c in range(2):
            pinned[c].copy_(torch.from_numpy(prob.U0[c]))
        ctx.reset_counters()
        ctx.integrate_host([p.numpy() for p in pinned], 3)
        assert ctx.counters()["steps"] == 3
        for c in range(2):
            assert relerr(pinned[c].numpy(), ref[c]) <= 1e-14, (rep, c)


def test_equilibrium_and_finite(ctx):
    prob = inputs.make_problem("fhn", 3, 16, amplitude=0.0)
    setup_problem(ctx, prob, "etd3rkds", 0.015)
    U = [dev(u) for u in prob.U0]
    for _ in range(5):
        ctx.step(U)
    ctx.sync()
    assert float(U[0].abs().max()) == 0.0 and float(U[1].abs().max()) == 0.0
    assert ctx.check_finite(U[0])
    bad = dev(np.array([0.0] * 16 ** 3))
    bad[5] = float("nan")
    assert not ctx.check_finite(bad)


def test_invalid_arguments(ctx, kx):
    ctx.set_grid([4, 5], 1)
    X = dev(np.zeros(20))
    with pytest.raises(kx.KxError, match="mode 3"):
        ctx.mode_product(X, dev(np.zeros(20)), 3, dmat(np.eye(4)))
    with pytest.raises(kx.KxError, match="distinct"):
        ctx.mode_product(X, X, 1, dmat(np.eye(4)))
    with pytest.raises(kx.KxError, match="set_tau"):
        ctx.step([X])
    with pytest.raises(kx.KxError):
        ctx.set_tau(-1.0, "etd3rkds")


@pytest.mark.parametrize("n", [[1000, 1000], [700, 1500], [1024, 1024], [256, 200, 300], [520, 96, 40],
                               [256, 256], [512, 512], [384, 320], [640, 384], [300, 260], [128, 1000]],
                         ids=lambda n: "x".join(map(str, n)))
def test_streamk_shapes_parity_and_determinism(ctx, n):
    """Shapes whose tile count is not a multiple of the SM count take the hybrid
    data-parallel + stream-K schedule (partials reduced in fixed k order): parity with the
    oracle and bitwise run-to-run determinism."""
    ctx.set_grid(n, 1)
    x = tensor(n, 12)
    X = dev(x)
    Xo = unvec(x, n)
    for mu in range(1, len(n) + 1):
        L = inputs.uniform_sym(40 + mu, 0, n[mu - 1] ** 2).reshape(n[mu - 1], n[mu - 1])
        Ld = dmat(L)
        Y1 = dev(np.zeros(x.size))
        ctx.mode_product(X, Y1, mu, Ld)
        ref = vec(mode_product(Xo, L, mu))
        assert relerr(Y1.cpu().numpy(), ref) <= 1e-13, mu
        # few-tile launches are split over many CTAs whose partials several reducers sum in
        # contributor order: repeated launches must agree bitwise
        for _ in range(4):
            Y2 = dev(np.zeros(x.size))
            ctx.mode_product(X, Y2, mu, Ld)
            assert torch.equal(Y1, Y2)


def slab(u, n, r, P):
    """Rank r's slab (i_d in its block) of a vec-order global tensor, as vec-order flat."""
    T = unvec(u, n)
    nd = n[-1] // P
    return vec(T[..., r * nd:(r + 1) * nd])


@pytest.mark.parametrize("case", [("schnakenberg", 2, [64, 64], "etd3rkds", 2.0 / 6000, 2),
                                  ("schnakenberg", 2, [48, 40], "etd3rkds", 1e-4, 4),
                                  ("fhn", 3, [24, 20, 32], "etd3rkds", 0.015, 2),
                                  ("fhn", 3, [16, 16, 16], "etd3rkds", 0.015, 4),
                                  ("schnakenberg", 2, [64, 64], "etd2rkds", 0.25 / 3000, 4),
                                  ("fhn", 3, [16, 12, 8], "etd2rkds", 0.01, 2)])
@pytest.mark.parametrize("dense_kronsum", [False, True], ids=["halo-stencil", "dense-kronsum"])
@pytest.mark.parametrize("p2p", [False, True], ids=["exchange-copies", "direct-peer-stores"])
def test_sharded_step_loopback(kx, case, dense_kronsum, p2p):
    """The slab-sharded schedule (layouts A/B, peer-packed all-to-alls, concat-K over
    (term, source rank) segments; the Kronecker sum either as a stencil with a halo exchange
    of the boundary planes or as dense mode products across layouts) on an in-process loopback
    group: equals the single-GPU step to rounding and the oracle to 1e-10."""
    model, d, n, scheme, tau, P = case
    prob = inputs.make_problem(model, d, n, seed=5)
    one = kx.Context(0)
    setup_problem(one, prob, scheme, tau)
    U1 = [dev(u) for u in prob.U0]
    grp = kx.Group(P)
    for c in grp.ctx:
        setup_problem(c, prob, scheme, tau)
        c.set_kronsum_mode(dense_kronsum)
    if p2p:   # the producers store straight into the other ranks' receive buffers
        grp.set_p2p(True)
    Ug = [[dev(slab(prob.U0[s], n, r, P)) for s in range(2)] for r in range(P)]
    steps = 3
    for k in range(steps):
        one.step(U1)
        grp.step(Ug)
    one.sync()
    grp.ctx[0].sync()
    ref, _ = integrate(prob, scheme, T=tau * 100, m=100, steps=steps)
    for s in range(2):
        u1 = U1[s].cpu().numpy()
        # assemble the global tensor from the slabs
        parts = [unvec(Ug[r][s].cpu().numpy(), n[:-1] + [n[-1] // P]) for r in range(P)]
        ug = vec(np.concatenate(parts, axis=-1))
        assert relerr(ug, u1) <= 1e-13
        assert relerr(ug, ref[s]) <= 1e-10
    cnt = grp.ctx[1].counters()
    per = 2 if scheme == "etd2rkds" else (10 if d == 2 else 15)
    assert cnt["tucker_ops"] == steps * 2 * per and cnt["steps"] == steps
    grp.close()
    one.close()


@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("scheme", ["etd3rkds", "exprk3ds_cplx"])
def test_nccl_single_rank_dist_context(kx, overlap, scheme):
    """kx_create_dist with one rank (NCCL self-exchange): the distributed code path end to
    end through NCCL on one GPU, with and without the term-by-term overlapped exchange (f2),
    equal to the single-GPU step to rounding."""
    prob = inputs.make_problem("fhn", 3, [16, 12, 8], seed=7)
    tau = 0.015
    uid = kx.nccl_unique_id()
    dctx = kx.Context(0, dist=(uid, 0, 1))
    dctx.set_dist_overlap(overlap)
    setup_problem(dctx, prob, scheme, tau)
    one = kx.Context(0)
    setup_problem(one, prob, scheme, tau)
    Ud = [dev(u) for u in prob.U0]
    U1 = [dev(u) for u in prob.U0]
    for _ in range(3):
        dctx.step(Ud)
        one.step(U1)
    dctx.sync()
    one.sync()
    for s in range(2):
        assert relerr(Ud[s].cpu().numpy(), U1[s].cpu().numpy()) <= 1e-13
    with pytest.raises(kx.KxError, match="distributed"):   # still one-GPU only
        dctx.tucker_batched(Ud[0], U1[0], [dmat(np.eye(m)) for m in prob.n], 1)
    dctx.close()
    one.close()


@pytest.mark.parametrize("G", [4096, 4097], ids=["aligned", "offset8B"])
@pytest.mark.parametrize("n", [[33, 17, 9], [65, 33], [300, 280], [7], [128, 96, 24]],
                         ids=lambda n: "x".join(map(str, n)))
def test_no_out_of_bounds_writes(ctx, n, G):
    """compute-sanitizer is unavailable on this pool: outputs live inside a larger buffer whose
    guard bands hold a sentinel; every operator must leave the guards bit-identical."""
    N = int(np.prod(n))
    ctx.set_grid(n, 2)
    As = [[inputs.laplacian_neumann(m, 1.0, 1.0 + c) for m in n] for c in range(2)]
    for c in range(2):
        for mu in range(len(n)):
            ctx.set_direction_matrix(c, mu + 1, As[c][mu])
    ctx.set_tau(1e-4, "etd3rkds" if len(n) >= 2 else "etd2rkds")
    X = dev(tensor(n, 21))
    big = torch.full((N + 2 * G,), 12345.678, dtype=torch.float64, device="cuda")
    Y = big[G:G + N]
    Ls = [dmat(inputs.uniform_sym(22, mu, m * m).reshape(m, m)) for mu, m in enumerate(n)]
    ctx.tucker(X, Y, Ls)
    for mu in range(1, len(n) + 1):
        ctx.mode_product(X, Y, mu, Ls[mu - 1], 1.0, 1.0)
    ctx.kronsum(0, X, Y, 1.0)
    ctx.set_kronsum_mode(True)
    ctx.kronsum(1, X, Y, 1.0)
    ctx.set_kronsum_mode(False)
    ctx.phi_apply(0, 1, 2, X, Y, 1.0, 1.0)
    bigU = [torch.full((N + 2 * G,), -777.0, dtype=torch.float64, device="cuda") for _ in range(2)]
    U = [b[G:G + N] for b in bigU]
    for c in range(2):
        U[c].copy_(X)
    ctx.step(U)
    ctx.sync()
    for b in [big] + bigU:
        v = b[:G].cpu().numpy().tolist() + b[G + N:].cpu().numpy().tolist()
        assert len(set(v)) == 1, "guard band overwritten"


@pytest.mark.parametrize("case", [("schnakenberg", 2, 48, 1e-4), ("fhn", 3, 20, 0.015), ("fhn", 3, 17, 0.01)])
def test_complex_bank_and_phi_apply(ctx, case):
    """exprk3ds_cplx (Table 2): complex phi-matrices via the real 2n x 2n embedding on the GPU
    against the oracle's complex Taylor/doubling phi, and the real part of the split action."""
    model, d, n, tau = case
    prob = inputs.make_problem(model, d, n)
    setup_problem(ctx, prob, "exprk3ds_cplx", tau)
    s = {1: coeffs.table2(1, d), 2: coeffs.table2(2, d)}
    cs = {0: 1 / 3, 1: 2 / 3, 2: 1.0}
    x = tensor(prob.n, 31)
    for c in range(2):
        for (ell, stage) in [(1, 0), (1, 1), (1, 2), (2, 1), (2, 2)]:
            for i in range(2):
                for mu in range(1, d + 1):
                    X = cs[stage] * tau * s[ell].alphas[i][mu - 1] * prob.A[c][mu - 1]
                    ref = phi_matrices(X, 2)[s[ell].inner[i]]
                    re = ctx.phi_matrix(c, ell, stage, 2 * i, mu)
                    im = ctx.phi_matrix(c, ell, stage, 2 * i + 1, mu)
                    assert relerr(re + 1j * im, ref) <= 1e-11
            P = split_phi_matrices(s[ell], cs[stage] * tau, prob.A[c])
            ref = np.real(vec(split_apply(s[ell].etas, P, unvec(x, prob.n))))
            Y = dev(np.zeros(x.size))
            ctx.phi_apply(c, ell, stage, dev(x), Y)
            assert relerr(Y.cpu().numpy(), ref) <= 1e-11


@pytest.mark.parametrize("case", [("schnakenberg", 2, 64, 2.0, 6000, 10), ("fhn", 3, 24, 150.0, 10000, 10),
                                  ("schnakenberg", 2, 50, 0.25, 1000, 5)])
def test_complex_step_parity(ctx, case):
    model, d, n, T, m, steps = case
    prob = inputs.make_problem(model, d, n, seed=4)
    tau = T / m
    setup_problem(ctx, prob, "exprk3ds_cplx", tau)
    out = run_gpu(ctx, prob, "exprk3ds_cplx", tau, steps)
    ref, _ = integrate(prob, "exprk3ds_cplx", T=T, m=m, steps=steps)
    err = max(relerr(out[c], ref[c]) for c in range(2))
    assert err <= 1e-10, err
    cnt = ctx.counters()
    assert cnt["tucker_ops"] == steps * 2 * 10 and cnt["kronsum_actions"] == steps * 2


def test_complex_sharded_loopback(kx):
    prob = inputs.make_problem("fhn", 3, [16, 12, 16], seed=6)
    tau, P = 0.015, 2
    one = kx.Context(0)
    setup_problem(one, prob, "exprk3ds_cplx", tau)
    grp = kx.Group(P)
    for c in grp.ctx:
        setup_problem(c, prob, "exprk3ds_cplx", tau)
    U1 = [dev(u) for u in prob.U0]
    Ug = [[dev(slab(prob.U0[s], prob.n, r, P)) for s in range(2)] for r in range(P)]
    for _ in range(2):
        one.step(U1)
        grp.step(Ug)
    one.sync()
    grp.ctx[0].sync()
    for s in range(2):
        parts = [unvec(Ug[r][s].cpu().numpy(), prob.n[:-1] + [prob.n[-1] // P]) for r in range(P)]
        assert relerr(vec(np.concatenate(parts, axis=-1)), U1[s].cpu().numpy()) <= 1e-13
    grp.close()
    one.close()


@pytest.mark.parametrize("case", [("fhn", [6, 5, 4, 7], "etd3rkds", 0.015, 4),
                                  ("fhn", [4, 3, 5, 2, 3], "etd3rkds", 0.01, 3),
                                  ("schnakenberg", [5, 6, 4, 3], "etd2rkds", 1e-4, 4),
                                  ("fhn", [8, 6, 4, 4], "exprk3ds_cplx", 0.01, 2),
                                  ("schnakenberg", [40], "etd2rkds", 1e-4, 5)])
def test_step_parity_other_dimensions(ctx, case):
    """d = 1, 4, 5 (Table 3 carries 2^{d-3}; Table 2 2^{d-2}; middle modes mu = d-1..2)."""
    model, n, scheme, tau, steps = case
    prob = inputs.make_problem(model, len(n), n, seed=9)
    setup_problem(ctx, prob, scheme, tau)
    out = run_gpu(ctx, prob, scheme, tau, steps)
    ref, _ = integrate(prob, scheme, T=tau * 10, m=10, steps=steps)
    err = max(relerr(out[c], ref[c]) for c in range(2))
    assert err <= 1e-10, err


def test_out_of_memory_is_reported(ctx, kx):
    """A grid whose exprk3ds workspaces exceed HBM (1024^3: ~0.4 TB) fails with KX_ERR_NOMEM at
    kx_set_tau, frees what it allocated, and the context stays usable."""
    n = [1024, 1024, 1024]
    ctx.set_grid(n, 2)
    A = inputs.laplacian_neumann(1024, math.pi, 1.0)
    for c in range(2):
        for mu in (1, 2, 3):
            ctx.set_direction_matrix(c, mu, A)
    with pytest.raises(kx.KxError) as ei:
        ctx.set_tau(0.015, "etd3rkds")
    assert ei.value.status == kx.KX_ERR_NOMEM
    ctx.set_grid([16, 16], 1)
    X = dev(tensor([16, 16], 1))
    Y = dev(np.zeros(256))
    ctx.tucker(X, Y, [dmat(np.eye(16)), dmat(np.eye(16))])
    ctx.sync()
    assert torch.equal(X, Y)


def test_degenerate_and_invalid_grids(ctx, kx):
    """Empty / oversized / unsupported grids are rejected synchronously; K = 0 (A_mu = 0) turns
    exprk3ds into a pointwise ODE solver (phi_l(0) = I/l! exactly), matching the oracle; a tiny
    tau gives phi-matrices equal to I/l! to rounding."""
    for bad in ([0, 4], [4, 0, 3], [1 << 16, 1 << 16]):
        with pytest.raises(kx.KxError):
            ctx.set_grid(bad, 2)
    with pytest.raises(kx.KxError):
        ctx.set_grid([2] * 7, 2)
    # K = 0
    n = [12, 10]
    prob = inputs.make_problem("fhn", 2, n, seed=4, amplitude=0.5)
    prob.A = [[np.zeros((m, m)) for m in n] for _ in range(2)]
    setup_problem(ctx, prob, "etd3rkds", 0.01)
    out = run_gpu(ctx, prob, "etd3rkds", 0.01, 5)
    ref, _ = integrate(prob, "etd3rkds", T=0.1, m=10, steps=5)
    assert max(relerr(out[c], ref[c]) for c in range(2)) <= 1e-13
    # tiny tau
    prob = inputs.make_problem("schnakenberg", 2, 16)
    setup_problem(ctx, prob, "etd3rkds", 1e-14)
    P = ctx.phi_matrix(0, 2, 2, 1, 1)        # phi_2-term (l_2 = 2) at c = 1
    assert np.max(np.abs(P - np.eye(16) / 2)) <= 1e-9


def test_nan_watchdog(ctx, kx):
    """kx_set_nan_check: a blow-up (tau far beyond the stable range of an explicit-like
    reaction, rho = 1e8) is reported by kx_sync as KX_ERR_NUMERIC with the step index."""
    prob = inputs.make_problem("fhn", 2, [16, 16], seed=1, amplitude=1.0)
    prob.params = dict(prob.params, rho=1e8)
    setup_problem(ctx, prob, "etd3rkds", 0.5)
    ctx.set_nan_check(True)
    U = [dev(u) for u in prob.U0]
    with pytest.raises(kx.KxError) as ei:
        for _ in range(20):
            ctx.step(U)
        ctx.sync()
    assert ei.value.status == kx.KX_ERR_NUMERIC and "step" in str(ei.value)
    # a healthy run stays silent
    prob = inputs.make_problem("fhn", 2, [16, 16], seed=1)
    setup_problem(ctx, prob, "etd3rkds", 0.01)
    ctx.set_nan_check(True)
    U = [dev(u) for u in prob.U0]
    for _ in range(5):
        ctx.step(U)
    ctx.sync()


# ---------------------------------------------------------------- K*5: fused small 2-D grids
@pytest.mark.parametrize("case", [("schnakenberg", [64, 64], "etd2rkds", 1.0 / 3000, 1.0),
                                  ("schnakenberg", [64, 64], "etd3rkds", 1.0 / 3000, 1.0),
                                  ("fhn", [48, 40], "etd3rkds", 0.01, 1.0),
                                  ("fhn", [33, 20], "etd2rkds", 0.01, 1.0),
                                  ("schnakenberg", [7, 8], "etd3rkds", 1e-5, 1.0),
                                  ("schnakenberg", [64, 9], "etd2rkds", 1e-5, 1.0)])
def test_fused_small_vs_general_and_oracle(kx, case):
    """The one-cluster step kernel (kx_set_fused_small, default on) against the general
    multi-launch path and against the oracle: 3 steps, element by element."""
    from oracle import etd
    model, n, scheme, tau, amp = case
    prob = inputs.make_problem(model, 2, n, seed=11, amplitude=amp)
    out = {}
    for fused in (True, False):
        c = kx.Context(0)
        setup_problem(c, prob, scheme, tau)
        c.set_fused_small(fused)
        U = [dev(u) for u in prob.U0]
        c.reset_counters()
        for _ in range(3):
            c.step(U)
        c.sync()
        out[fused] = [u.cpu().numpy() for u in U]
        cnt = c.counters()
        per = 10 if scheme == "etd3rkds" else 2
        assert cnt["tucker_ops"] == 3 * 2 * per and cnt["kronsum_actions"] == 3 * 2
        if fused:
            assert cnt["gemm_launches"] == 3 and cnt["other_launches"] == 0
        c.close()
    ref, _ = etd.integrate(prob, scheme, 3 * tau, 3, steps=3)
    for k in range(2):
        assert relerr(out[True][k], out[False][k]) < 1e-13
        assert relerr(out[True][k], ref[k]) < 1e-12


def test_fused_small_step_n(kx):
    """kx_step_n runs all steps in one launch on the fused path: equal to repeated kx_step."""
    prob = inputs.make_problem("schnakenberg", 2, 64, seed=5)
    res = []
    for multi in (True, False):
        c = kx.Context(0)
        setup_problem(c, prob, "etd2rkds", 1.0 / 3000)
        U = [dev(u) for u in prob.U0]
        c.reset_counters()
        if multi:
            c.step_n(U, 20)
        else:
            for _ in range(20):
                c.step(U)
        c.sync()
        cnt = c.counters()
        assert cnt["steps"] == 20 and cnt["tucker_ops"] == 20 * 2 * 2
        if multi:
            assert cnt["gemm_launches"] == 1
        res.append([u.cpu().numpy() for u in U])
        c.close()
    for k in range(2):
        assert np.array_equal(res[0][k], res[1][k])


def test_fused_small_not_eligible_falls_back(kx):
    """Grids outside the fused kernel's range (n_2 < 8, n > 64, dense A) take the general path."""
    for n, dense in (([16, 7], False), ([65, 16], False), ([32, 32], True)):
        prob = inputs.make_problem("schnakenberg", 2, n, seed=2)
        c = kx.Context(0)
        setup_problem(c, prob, "etd3rkds", 1e-3)
        if dense:
            c.set_kronsum_mode(True)
        U = [dev(u) for u in prob.U0]
        c.reset_counters()
        c.step(U)
        c.sync()
        assert c.counters()["gemm_launches"] > 1
        c.close()


def test_p2p_requires_every_member(kx):
    """kx_set_tau disables direct peer stores on that member: the group refuses to step until
    kx_group_set_p2p is called again (no stale peer pointers)."""
    prob = inputs.make_problem("fhn", 3, [16, 12, 8], seed=7)
    grp = kx.Group(2)
    for c in grp.ctx:
        setup_problem(c, prob, "etd3rkds", 0.015)
    grp.set_p2p(True)
    Ug = [[dev(slab(prob.U0[s], prob.n, r, 2)) for s in range(2)] for r in range(2)]
    grp.step(Ug)
    grp.ctx[1].set_tau(0.01, "etd3rkds")
    with pytest.raises(kx.KxError, match="kx_group_set_p2p"):
        grp.step(Ug)
    grp.set_p2p(True)
    grp.step(Ug)
    grp.ctx[0].sync()
    grp.close()


def test_nccl_single_rank_ipc_p2p(kx):
    """NCCL rank with direct peer stores (IPC export/import round trip on one rank; the
    exchanges become barriers): equal to the single-GPU step to rounding."""
    prob = inputs.make_problem("fhn", 3, [16, 12, 8], seed=7)
    tau = 0.015
    dctx = kx.Context(0, dist=(kx.nccl_unique_id(), 0, 1))
    setup_problem(dctx, prob, "etd3rkds", tau)
    blob = dctx.ipc_export()
    assert len(blob) == 5 * 2 * 64
    dctx.ipc_import([blob])
    one = kx.Context(0)
    setup_problem(one, prob, "etd3rkds", tau)
    Ud = [dev(u) for u in prob.U0]
    U1 = [dev(u) for u in prob.U0]
    for _ in range(3):
        dctx.step(Ud)
        one.step(U1)
    dctx.sync()
    one.sync()
    for s in range(2):
        assert relerr(Ud[s].cpu().numpy(), U1[s].cpu().numpy()) <= 1e-13
    dctx.close()
    one.close()


@pytest.mark.parametrize("n", [[64, 64], [128, 128], [1, 7], [7, 1], [33, 100], [128, 9], [5, 128]],
                         ids=lambda n: "x".join(map(str, n)))
def test_tucker2d_small_one_launch(kx, n):
    """d = 2, n <= 128: the Tucker operator as one launch (intermediate in shared memory),
    with alpha/beta, against the oracle and against the general two-launch path."""
    x = tensor(n, 31)
    Ls = [inputs.uniform_sym(40 + mu, 0, m * m).reshape(m, m) / math.sqrt(m) for mu, m in enumerate(n)]
    y0 = tensor(n, 32)
    out = {}
    for fused in (True, False):
        c = kx.Context(0)
        c.set_grid(n, 1)
        c.set_fused_small(fused)
        Y = dev(y0)
        c.reset_counters()
        c.tucker(dev(x), Y, [dmat(L) for L in Ls], alpha=0.5, beta=-2.0)
        c.sync()
        assert c.counters()["gemm_launches"] == (1 if fused else 2)
        out[fused] = Y.cpu().numpy()
        c.close()
    ref = 0.5 * vec(tucker(unvec(x, n), Ls)) - 2.0 * y0
    assert relerr(out[True], ref) <= 1e-12
    assert relerr(out[True], out[False]) <= 1e-13


@pytest.mark.parametrize("scheme", ["etd2rkds", "etd3rkds"])
def test_fused_small_single_component_linear(kx, scheme):
    """One component, no reaction (u' = K u, K = A_2 (+) A_1 Neumann Laplacians): the fused
    small-grid kernel with a single species equals the general path (1e-13) and tracks the
    exact exp(t K) u0 (scipy expm of the assembled K) to the splitting error."""
    import scipy.linalg
    from oracle.tensor import kronsum_assemble
    n = [24, 16]
    A = [inputs.laplacian_neumann(m, 1.0, 0.5) for m in n]
    u0 = inputs.kron_vec([inputs.cosine_mode(n[0], 2), inputs.cosine_mode(n[1], 1)]) + 0.3
    tau, steps = 1e-3, 10
    out = {}
    for fused in (True, False):
        c = kx.Context(0)
        c.set_grid(n, 1)
        for mu in range(2):
            c.set_direction_matrix(0, mu + 1, A[mu])
        c.set_model("none")
        c.set_tau(tau, scheme)
        c.set_fused_small(fused)
        U = [dev(u0)]
        c.reset_counters()
        for _ in range(steps):
            c.step(U)
        c.sync()
        if fused:
            assert c.counters()["gemm_launches"] == steps
        out[fused] = U[0].cpu().numpy()
        c.close()
    assert relerr(out[True], out[False]) <= 1e-13
    K = kronsum_assemble(A)
    exact = scipy.linalg.expm(steps * tau * K) @ u0
    assert relerr(out[True], exact) <= (1e-5 if scheme == "etd2rkds" else 1e-6)


def test_new_entry_points_reject_bad_use(kx):
    """Error paths of kx_step_n, kx_set_fused_small, kx_group_set_p2p and the IPC calls."""
    prob = inputs.make_problem("schnakenberg", 2, [16, 16], seed=1)
    c = kx.Context(0)
    U = [dev(u) for u in prob.U0]
    with pytest.raises(kx.KxError):          # no grid / no bank yet
        c.step_n(U, 3)
    setup_problem(c, prob, "etd3rkds", 1e-4)
    with pytest.raises(kx.KxError):          # negative step count
        c.step_n(U, -1)
    with pytest.raises(kx.KxError):          # aliased components
        c.step_n([U[0], U[0]], 1)
    c.step_n(U, 0)                           # zero steps: a no-op
    with pytest.raises(kx.KxError, match="NCCL"):   # IPC export needs an NCCL rank
        c.ipc_export()
    c.close()
    grp = kx.Group(2)
    with pytest.raises(kx.KxError):          # p2p before set_tau
        grp.set_p2p(True)
    grp.close()


def test_fused_small_integrate_host_watchdog_profile(kx):
    """The small-grid kernel through the other entry points: kx_integrate_host (all steps in
    one launch) equals kx_step on the device; with the NaN watchdog on, kx_step_n falls back
    to per-step launches and stays silent on a healthy run; profiling records the fused kernel
    as a mode-product launch."""
    prob = inputs.make_problem("fhn", 2, [40, 32], seed=4)
    tau, steps = 0.01, 7
    c = kx.Context(0)
    setup_problem(c, prob, "etd3rkds", tau)
    Uh = [np.ascontiguousarray(u.copy()) for u in prob.U0]
    c.integrate_host(Uh, steps)
    U = [dev(u) for u in prob.U0]
    for _ in range(steps):
        c.step(U)
    c.sync()
    for k in range(2):
        assert np.array_equal(Uh[k], U[k].cpu().numpy())
    c.set_nan_check(True)
    c.reset_counters()
    c.step_n(U, 3)
    c.sync()
    assert c.counters()["gemm_launches"] == 3     # one fused launch per step
    c.set_nan_check(False)
    c.set_profiling(True)
    c.step(U)
    c.sync()
    prof = c.profile()
    c.set_profiling(False)
    assert prof["gemm_launches"] >= 1 and prof["gemm_flops"] > 0
    c.close()


def test_integrate_host_tail_graph_follows_bank_and_buffers(ctx):
    """The cached host-copy tail graph is rebuilt when the phi bank changes (kx_set_tau) and
    when other host buffers are passed: results equal the device path at the new tau, and the
    first host buffers are not written by the second call."""
    prob = inputs.make_problem("schnakenberg", 2, [160, 96], seed=8)
    setup_problem(ctx, prob, "etd3rkds", 1e-4)
    a = [torch.from_numpy(u.copy()).pin_memory() for u in prob.U0]
    ctx.integrate_host([p.numpy() for p in a], 2)
    ctx.set_tau(3e-4, "etd3rkds")
    Ud = [dev(u) for u in prob.U0]
    for _ in range(2):
        ctx.step(Ud)
    b = [torch.from_numpy(u.copy()).pin_memory() for u in prob.U0]
    snap = [p.clone() for p in a]
    ctx.integrate_host([p.numpy() for p in b], 2)
    for c in range(2):
        assert relerr(b[c].numpy(), Ud[c].cpu().numpy()) <= 1e-14
        assert torch.equal(a[c], snap[c])
