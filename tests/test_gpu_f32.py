"""GPU parity of the fp32 variant (the paper's "CUDA single" columns, Table 5
P:1477-1486, Table 7) against the fp64 oracle.

The fp32 path runs every mode product on the tcgen05 tensor cores (kind::tf32) with a three-pass
hi/lo split of both operands, so its error is fp32 rounding: the inputs are rounded to fp32 once,
the oracle computes in fp64 from those same fp32 values, and the bars (reading
R21) follow from the arithmetic with unit roundoff u = 2^-22 for the split products:
  * mode product / Tucker operator: relative inf-norm <= 2 u sqrt(sum_mu n_mu) (the probabilistic
    bound of d chained length-n_mu dot products; a single-pass tf32 product, 2^-11, fails it);
  * m steps: relative inf-norm <= max(16 E32, m u), where E32 is the error of the oracle's own
    algorithm run in fp32 arithmetic on the same fp32 data (oracle/ is dtype-generic: fp32 A,
    phi-matrices rounded from the fp64 bank, fp32 state), against its fp64 run — the error that
    fp32 arithmetic admits for this problem, dominated by the conditioning of the fp32 stencil
    F = K U + G (|K| |U| >> |K U| for the stiff Laplacians).  16 = 4 (the split carries 22 of
    fp32's 24 significand bits into the tensor core: u = 2^-22 against fp32's 2^-24) x 4
    (margin).  Measured ratios (profiles/f32_accuracy_r02.json): 0.9-1.4 except ETD2RKDS on the
    growing FitzHugh-Nagumo mode (12), where the tensor core's truncating in-MMA accumulation
    (K <= 32 per partial) is amplified by the instability.
The ragged shapes span several 128 x 128 tiles with a partial tile in M, N and K (n = 132, 260,
36)."""
import dataclasses

import numpy as np
import pytest

import inputs
from oracle.etd import integrate
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


def f32(a):
    return np.asarray(a, dtype=np.float32)


def dev32(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


U22 = 2.0 ** -22


def tucker_tol(n):
    return 2 * U22 * np.sqrt(sum(n))


def _cast_bank(b):
    """Copy of an oracle bank with every phi-matrix rounded to fp32 (the library rounds its fp64
    bank the same way)."""
    b = dataclasses.replace(b)
    if hasattr(b, "P1"):
        b.P1 = [[[M.astype(np.float32) for M in row] for row in Pc] for Pc in b.P1]
        b.P2 = [[[M.astype(np.float32) for M in row] for row in Pc] for Pc in b.P2]
    else:
        b.P = [{k: [[M.astype(np.float32) for M in row] for row in v] for k, v in Pc.items()} for Pc in b.P]
    return b


def oracle_pair(prob, scheme, T, m, steps):
    """(fp64 oracle result, step tolerance): the tolerance is 4x the deviation of the same oracle
    run in fp32 arithmetic (floor m u)."""
    ref, bank = integrate(prob, scheme, T=T, m=m, steps=steps)
    p32 = dataclasses.replace(prob, A=[[A.astype(np.float32) for A in Ac] for Ac in prob.A],
                              U0=[u.astype(np.float32) for u in prob.U0])
    r32, _ = integrate(p32, scheme, T=T, m=m, steps=steps, bank=_cast_bank(bank))
    assert r32[0].dtype == np.float32          # the oracle really ran in fp32
    e32 = max(relerr(r32[c], ref[c]) for c in range(2))
    return ref, max(16.0 * e32, steps * U22), e32


def relerr(x, ref):
    x, ref = np.asarray(x, dtype=np.float64), np.asarray(ref, dtype=np.float64)
    return np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300)


def col32(M):
    """fp32 column-major device copy of M (the ABI's matrix convention)."""
    return dev32(np.asarray(M, dtype=np.float32).T.copy())


@pytest.mark.parametrize("n", [[64, 64], [132, 68], [260, 132], [1024, 1024], [36, 20, 16],
                               [128, 128, 128], [68, 132, 36]])
def test_tucker_f32_parity(kx, n):
    N = int(np.prod(n))
    x = f32(inputs.uniform_sym(31, 0, N))
    Ls = [f32(inputs.uniform_sym(32, mu, m * m).reshape(m, m)) / np.sqrt(m) for mu, m in enumerate(n)]
    y0 = f32(inputs.uniform_sym(33, 0, N))
    ctx = kx.Context(0)
    ctx.set_grid(n, 1)
    X, Y = dev32(x), dev32(y0)
    ctx.tucker_f32(X, Y, [col32(L) for L in Ls], alpha=0.75, beta=0.5)
    ref = 0.75 * vec(tucker(unvec(x.astype(np.float64), n), [L.astype(np.float64) for L in Ls])) \
        + 0.5 * y0.astype(np.float64)
    err = relerr(Y.cpu().numpy(), ref)
    assert err <= tucker_tol(n), (err, tucker_tol(n))
    cnt = ctx.counters()
    assert cnt["tucker_ops"] == 1 and cnt["gemm_launches"] == len(n)
    ctx.close()


@pytest.mark.parametrize("n", [[132, 68], [36, 20, 16], [128, 64, 96]])
def test_mode_product_f32_parity(kx, n):
    N = int(np.prod(n))
    x = f32(inputs.uniform_sym(41, 0, N))
    y0 = f32(inputs.uniform_sym(42, 0, N))
    ctx = kx.Context(0)
    ctx.set_grid(n, 1)
    for mu in range(1, len(n) + 1):
        m = n[mu - 1]
        L = f32(inputs.uniform_sym(43, mu, m * m).reshape(m, m))
        X, Y = dev32(x), dev32(y0)
        ctx.mode_product_f32(X, Y, mu, col32(L), alpha=1.0, beta=-2.0)
        ref = vec(mode_product(unvec(x.astype(np.float64), n), L.astype(np.float64), mu)) - 2.0 * y0
        assert relerr(Y.cpu().numpy(), ref) <= tucker_tol([n[mu - 1]]), (mu, relerr(Y.cpu().numpy(), ref))
    ctx.close()


def test_f32_rejects_unsupported(kx):
    ctx = kx.Context(0)
    ctx.set_grid([30, 32], 1)            # n_1 not a multiple of 4: no 16-B TMA rows
    X = dev32(np.zeros(960))
    Y = dev32(np.zeros(960))
    with pytest.raises(kx.KxError) as e:
        ctx.tucker_f32(X, Y, [col32(np.eye(30)), col32(np.eye(32))])
    assert e.value.status == kx.KX_ERR_UNSUPPORTED
    with pytest.raises(TypeError):      # fp64 tensors are refused by the fp32 calls
        ctx.tucker_f32(torch.zeros(960, dtype=torch.float64, device="cuda"), Y,
                       [col32(np.eye(30)), col32(np.eye(32))])
    ctx.close()


def run_steps(kx, prob, scheme, tau, steps):
    ctx = kx.Context(0)
    ctx.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(prob.d):
            ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    ctx.set_model(prob.model, prob.params)
    ctx.set_tau(tau, scheme)
    U = [dev32(u) for u in prob.U0]
    ctx.step_f32(U, steps)
    ctx.sync()
    out = [u.cpu().numpy().astype(np.float64) for u in U]
    cnt = ctx.counters()
    ctx.close()
    return out, cnt


@pytest.mark.parametrize("case", [("schnakenberg", 2, 64, "etd3rkds", 2.0 / 6000),
                                  ("schnakenberg", 2, 132, "etd3rkds", 1e-3),     # ragged tiles
                                  ("schnakenberg", 2, 64, "etd2rkds", 0.25 / 3000),
                                  ("fhn", 3, 32, "etd3rkds", 0.015),
                                  ("fhn", 3, [36, 20, 28], "etd3rkds", 0.015),
                                  ("fhn", 3, 32, "etd2rkds", 0.015)])
def test_step_f32_parity(kx, case):
    model, d, n, scheme, tau = case
    prob = inputs.make_problem(model, d, n, seed=3)
    prob = dataclasses.replace(prob, U0=[f32(u).astype(np.float64) for u in prob.U0])
    steps = 20
    out, cnt = run_steps(kx, prob, scheme, tau, steps)
    ref, tol, e32 = oracle_pair(prob, scheme, tau * steps, steps, steps)
    err = max(relerr(out[c], ref[c]) for c in range(2))
    assert err <= tol, (err, tol, e32)
    T = 2 if d == 2 else 3
    per_step = 5 * T if scheme != "etd2rkds" else 2
    assert cnt["steps"] == steps and cnt["tucker_ops"] == 2 * per_step * steps


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_step_f32_full_size(kx, cfg):
    """20 fp32 steps at the configured full sizes (C2 1024^2, C3 128^3) against the fp64 oracle
    from the same fp32-rounded initial data."""
    k = inputs.CONFIGS[cfg]
    prob = inputs.make_problem(k["model"], k["d"], k["n"], seed=0)
    prob = dataclasses.replace(prob, U0=[f32(u).astype(np.float64) for u in prob.U0])
    tau = k["T"] / k["m"]
    out, _ = run_steps(kx, prob, k["scheme"], tau, 20)
    ref, tol, e32 = oracle_pair(prob, k["scheme"], k["T"], k["m"], 20)
    err = max(relerr(out[c], ref[c]) for c in range(2))
    assert err <= tol, (err, tol, e32)


@pytest.mark.parametrize("n", [[132, 68], [36, 20, 16], [260, 4]])
def test_f32_no_out_of_bounds_writes(kx, n):
    """compute-sanitizer is closed on this pool: the fp32 outputs live inside larger buffers
    whose guard bands hold a sentinel (16-B aligned offsets, as the fp32 calls require); every
    fp32 operator and the fp32 step must leave the guards bit-identical (ragged tiles in M, N, K)."""
    N = int(np.prod(n))
    G = 1024
    ctx = kx.Context(0)
    ctx.set_grid(n, 2)
    As = [[inputs.laplacian_neumann(m, 1.0, 1.0 + c) for m in n] for c in range(2)]
    for c in range(2):
        for mu in range(len(n)):
            ctx.set_direction_matrix(c, mu + 1, As[c][mu])
    ctx.set_model("schnakenberg" if len(n) == 2 else "fhn",
                  inputs.SCHNAKENBERG if len(n) == 2 else inputs.FHN)
    ctx.set_tau(1e-4, "etd3rkds")
    X = dev32(inputs.uniform_sym(61, 0, N))
    big = torch.full((N + 2 * G,), 12345.678, dtype=torch.float32, device="cuda")
    Y = big[G:G + N]
    Ls = [col32(inputs.uniform_sym(62, mu, m * m).reshape(m, m)) for mu, m in enumerate(n)]
    ctx.tucker_f32(X, Y, Ls, 1.0, 0.5)
    for mu in range(1, len(n) + 1):
        ctx.mode_product_f32(X, Y, mu, Ls[mu - 1], 1.0, 1.0)
    bigU = [torch.full((N + 2 * G,), -777.0, dtype=torch.float32, device="cuda") for _ in range(2)]
    U = [b[G:G + N] for b in bigU]
    for c in range(2):
        U[c].copy_(X.abs() * 1e-3 + 1.0)
    if len(n) in (2, 3):
        ctx.step_f32(U, 2)
    ctx.sync()
    for b in [big] + bigU:
        v = b[:G].cpu().numpy().tolist() + b[G + N:].cpu().numpy().tolist()
        assert len(set(v)) == 1, "guard band overwritten"
    assert all(bool(torch.isfinite(u).all()) for u in U)
    ctx.close()


def test_step_f32_c4_size_closed_form(kx):
    """configs[3] size (512^3, FHN delta_v, tau = 0.015) in fp32: g = 0 and cosine-mode data make
    one exprk3ds_real step the scalar recurrence of Table 3 (as the fp64 test at this size); the
    fp32 bar: the rounding of the stencil F = K U, amplified by ||K|| / |lambda| (~20 here), and the
    split products, well inside 1e-4 relative."""
    import cmath
    import math
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
    ctx.set_model("fhn", inputs.FHN)
    ctx.set_model("none")
    ctx.set_tau(tau, "etd3rkds")
    U = [dev32(x), dev32(x)]
    ctx.step_f32(U, 1)
    ctx.sync()
    s = coeffs.table3(1, 3)

    def phis(ell, z):
        e = cmath.exp(z)
        return [e, (e - 1) / z, (e - 1 - z) / (z * z)][ell]

    split = sum(eta * np.prod([phis(li, tau * al[m] * lams[m]) for m in range(3)])
                for eta, li, al in zip(s.etas, s.inner, s.alphas))
    expect = np.real(1.0 + tau * sum(lams) * split) * x
    got = U[0].cpu().numpy().astype(np.float64)
    err = np.max(np.abs(got - expect)) / np.max(np.abs(expect))
    assert err <= 1e-4, err
    ctx.close()


@pytest.mark.parametrize("n", [[4, 4], [4, 8, 4], [8], [4, 4, 4, 4]])
def test_tucker_f32_tiny_and_any_d(kx, n):
    """Degenerate sizes (the smallest extents the 16-B TMA rows allow, d = 1 and d = 4): every tile
    is almost all padding, zero-filled by TMA out-of-bounds fill."""
    N = int(np.prod(n))
    x = f32(inputs.uniform_sym(101, 0, N))
    Ls = [f32(inputs.uniform_sym(102, mu, m * m).reshape(m, m)) for mu, m in enumerate(n)]
    ctx = kx.Context(0)
    ctx.set_grid(n, 1)
    Y = dev32(np.zeros(N))
    ctx.tucker_f32(dev32(x), Y, [col32(L) for L in Ls])
    ref = vec(tucker(unvec(x.astype(np.float64), n), [L.astype(np.float64) for L in Ls]))
    assert relerr(Y.cpu().numpy(), ref) <= tucker_tol(n)
    ctx.close()


def test_step_f32_zero_steps_is_noop(kx):
    prob = inputs.make_problem("schnakenberg", 2, 16, seed=1)
    ctx = kx.Context(0)
    ctx.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(2):
            ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    ctx.set_model(prob.model, prob.params)
    ctx.set_tau(1e-4, "etd3rkds")
    U = [dev32(u) for u in prob.U0]
    before = [u.clone() for u in U]
    ctx.step_f32(U, 0)
    ctx.sync()
    assert all(torch.equal(a, b) for a, b in zip(U, before))
    assert ctx.counters()["steps"] == 0
    ctx.close()


@pytest.mark.parametrize("n,mu", [([256, 192], 1), ([256, 192], 2), ([64, 48, 32], 3)])
def test_inplace_epilogue_rounds_to_nearest(kx, n, mu):
    """Y = X x_mu I + Y in place (beta = 1, D = C): the epilogue is a TMA reduce-add into Y.
    X holds tf32-exact values (11 significant bits), so the split product is exactly X and the
    result must be numpy's fp32 Y + X bit for bit (one round-to-nearest add)."""
    N = int(np.prod(n))
    rng = np.random.default_rng(7)
    x = np.ldexp(rng.integers(-2**10, 2**10, N).astype(np.float64), -10).astype(np.float32)   # <= 11 bits
    y = rng.standard_normal(N).astype(np.float32)
    ctx = kx.Context(0)
    ctx.set_grid(n, 1)
    Y = dev32(y)
    I = torch.eye(n[mu - 1], dtype=torch.float32, device="cuda")
    ctx.mode_product_f32(dev32(x), Y, mu, I, 1.0, 1.0)
    ctx.sync()
    got = Y.cpu().numpy()
    assert np.array_equal(got, y + x), int(np.sum(got != y + x))
    ctx.close()


def test_step_f32_rejects_misaligned_state(kx):
    """U tensors off a 16-B boundary are refused (KX_ERR_INVALID) before anything is enqueued:
    the vectorised pointwise kernels and the TMA loads / stores of the fp32 step need them."""
    prob = inputs.make_problem("schnakenberg", 2, [96, 64], seed=4)
    ctx = kx.Context(0)
    ctx.set_grid(prob.n, 2)
    for c in range(2):
        for mu in range(prob.d):
            ctx.set_direction_matrix(c, mu + 1, prob.A[c][mu])
    ctx.set_model(prob.model, prob.params)
    ctx.set_tau(2.0 / 6000, "etd3rkds")
    N = int(np.prod(prob.n))
    bufs = [torch.full((N + 1,), 7.0, dtype=torch.float32, device="cuda") for _ in range(2)]
    U = [b[1:] for b in bufs]   # 4-byte offset
    with pytest.raises(kx.KxError) as e:
        ctx.step_f32(U, 1)
    assert e.value.status == kx.KX_ERR_INVALID
    ctx.sync()
    assert all(bool(torch.all(b == 7.0)) for b in bufs)   # nothing written
    ctx.close()
