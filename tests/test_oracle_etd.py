"""Pins for oracle/etd.py (split phi-actions, ETD2RKDS, Algorithms 1-2).

* observed splitting order vs the exact dense phi_l(tau K) v (scipy expm on the Van Loan
  block of the assembled K): error ratio ~8 per tau-halving for Tables 1-3 (third order,
  eq:split2d/eq:splitnd/eq:splitnd3), ~4 for eq:secondord;
* tau = 0 / scalar-case closed forms; cosine-mode closed forms at realistic sizes;
* per-step cost accounting; equilibria;
* linear-problem local order and nonlinear self-convergence slopes (Figs. 1-8 slope lines);
* Turing patterns."""
import math

import numpy as np
import pytest
import scipy.linalg

import inputs
from oracle import coeffs
from oracle.etd import (Counters, exprk3ds_precompute, exprk3ds_step, integrate,
                        split_apply, split_phi_matrices, etd2rkds_precompute)
from oracle.models import g_fhn, g_schnakenberg
from oracle.tensor import kronsum_assemble, unvec, vec


def dense_phi_action(ell, K, v):
    N = K.shape[0]
    B = np.zeros((3 * N, 3 * N), dtype=complex if np.iscomplexobj(K) else float)
    B[:N, :N] = K
    B[:N, N:2 * N] = np.eye(N)
    B[N:2 * N, 2 * N:] = np.eye(N)
    E = scipy.linalg.expm(B)
    return E[:N, ell * N:(ell + 1) * N] @ v


def split_error(scheme, As, V, tau):
    P = split_phi_matrices(scheme, tau, As)
    S = vec(split_apply(scheme.etas, P, V))
    ref = dense_phi_action(scheme.ell, tau * kronsum_assemble(As), vec(V))
    return np.max(np.abs(S - ref))


SCHEMES = [("t1", 1, 2), ("t1", 2, 2), ("t2", 1, 2), ("t2", 2, 3), ("t3", 1, 3), ("t3", 2, 3),
           ("t3", 1, 2), ("so", 1, 2), ("so", 2, 3)]


@pytest.mark.parametrize("name,ell,d", SCHEMES)
def test_split_order(name, ell, d):
    s = {"t1": lambda: coeffs.table1(ell), "t2": lambda: coeffs.table2(ell, d),
         "t3": lambda: coeffs.table3(ell, d), "so": lambda: coeffs.second_order(ell, d)}[name]()
    rs = np.random.default_rng(ell * 10 + d)
    As = [rs.uniform(-1, 1, (4, 4)) for _ in range(d)]
    V = rs.uniform(-1, 1, [4] * d)
    errs = [split_error(s, As, V, tau) for tau in (0.1, 0.05, 0.025)]
    ratios = [errs[i] / errs[i + 1] for i in range(2)]
    lo, hi = (3.4, 4.6) if name == "so" else (6.5, 9.5)
    assert all(lo <= r <= hi for r in ratios), (errs, ratios)


def test_split_at_tau_zero_is_identity_over_lfact():
    for s in (coeffs.table1(1), coeffs.table1(2), coeffs.table3(1, 3), coeffs.table3(2, 3)):
        As = [inputs.laplacian_neumann(5, 1.0, 1.0)] * s.d
        V = unvec(inputs.uniform_sym(1, 1, 5 ** s.d), [5] * s.d)
        out = split_apply(s.etas, split_phi_matrices(s, 0.0, As), V)
        assert np.max(np.abs(out - V / math.factorial(s.ell))) <= 1e-13


def phi_cf(ell, z):
    """Closed-form scalar phi written here independently of oracle.phi."""
    if z == 0.0:
        return 1.0 / math.factorial(ell)
    if ell == 0:
        return math.exp(z)
    if ell == 1:
        return math.expm1(z) / z
    if abs(z) < 1e-4:
        return 0.5 + z / 6 + z * z / 24 + z ** 3 / 120
    return (math.expm1(z) - z) / (z * z)


def scalar_split(s, ctau, lams):
    return sum(eta * np.prod([phi_cf(li, ctau * al[mu] * lams[mu]) for mu in range(s.d)])
               for eta, li, al in zip(s.etas, s.inner, s.alphas))


@pytest.mark.parametrize("case", [("t1", 1, 2, 256, 1.0), ("t1", 2, 2, 128, 10.0),
                                  ("t3", 1, 3, 48, 42.1887), ("t3", 2, 3, 40, 1.0)])
def test_cosine_mode_closed_form(case):
    """FD Neumann A has exact eigenvectors cos(k pi i/(n-1)); the split action
    on a tensor of modes is a scalar multiple given by the closed form."""
    name, ell, d, n, delta = case
    s = coeffs.table1(ell) if name == "t1" else coeffs.table3(ell, d)
    L = math.pi
    A = inputs.laplacian_neumann(n, L, delta)
    ks = [3, n // 4, 7][:d]
    X = unvec(inputs.kron_vec([inputs.cosine_mode(n, k) for k in ks]), [n] * d)
    lams = [inputs.cosine_eigenvalue(n, L, delta, k) for k in ks]
    tau = 0.015 if d == 3 else 1.0 / 3000
    for c in (1 / 3, 2 / 3, 1.0):
        out = split_apply(s.etas, split_phi_matrices(s, c * tau, [A] * d), X)
        expect = scalar_split(s, c * tau, lams) * X
        assert np.max(np.abs(out - expect)) <= 1e-11 * np.max(np.abs(expect))


def test_scalar_case_not_exact_but_third_order():
    """Reading R11: with n_mu = 1 the third-order split is NOT exact; it deviates from
    phi_l(tau sum a_mu) at O(tau^3) (ratio ~8 per halving)."""
    a = [-1.3, -0.4, -2.0]
    for s in (coeffs.table3(1, 3), coeffs.table3(2, 3)):
        errs = []
        for tau in (0.2, 0.1, 0.05):
            As = [np.array([[x]]) for x in a]
            out = split_apply(s.etas, split_phi_matrices(s, tau, As), np.ones((1, 1, 1)))[0, 0, 0]
            errs.append(abs(out - phi_cf(s.ell, tau * sum(a))))
        assert errs[0] > 1e-6
        assert 6.0 < errs[0] / errs[1] < 9.5 and 6.0 < errs[1] / errs[2] < 9.5


def zero_g(t, u, v, p):
    return np.zeros_like(u), np.zeros_like(v)


@pytest.mark.parametrize("d", [2, 3])
def test_step_counts(d):
    prob = inputs.make_problem("fhn", d, 6)
    c = Counters()
    integrate(prob, "etd3rkds", T=0.1, m=10, steps=3, counters=c)
    per = 10 if d == 2 else 15
    assert c.steps == 3 and c.tucker_ops == 3 * 2 * per and c.kronsum_actions == 3 * 2
    c2 = Counters()
    integrate(prob, "etd2rkds", T=0.1, m=10, steps=4, counters=c2)
    assert c2.tucker_ops == 4 * 2 * 2 and c2.kronsum_actions == 4 * 2


@pytest.mark.parametrize("model,d", [("schnakenberg", 2), ("fhn", 3)])
@pytest.mark.parametrize("scheme", ["etd2rkds", "etd3rkds"])
def test_equilibrium_is_stationary(model, d, scheme):
    # short horizon: the Schnakenberg equilibrium is Turing-unstable, so rounding-level
    # residuals of K u_e (~1e-14) grow like e^{lambda t}
    prob = inputs.make_problem(model, d, 8, amplitude=0.0)
    out, _ = integrate(prob, scheme, T=0.005, m=50, steps=5)
    for c in range(2):
        assert np.max(np.abs(out[c] - prob.U0[c])) <= 1e-12


@pytest.mark.parametrize("d", [2, 3])
def test_linear_local_order(d):
    """g = 0: one exprk3ds step is U + tau S_1^tau[K U] = exp(tau K) U + O(tau^4)."""
    rs = np.random.default_rng(5 + d)
    n = 4
    A1 = [rs.uniform(-1, 1, (n, n)) for _ in range(d)]
    A = [A1, A1]
    U0 = [rs.uniform(-1, 1, [n] * d) for _ in range(2)]
    errs = []
    for tau in (0.1, 0.05, 0.025):
        bank = exprk3ds_precompute(A, tau)
        U1 = exprk3ds_step(U0, 0.0, bank, A, zero_g, {})
        ref = scipy.linalg.expm(tau * kronsum_assemble(A1)) @ vec(U0[0])
        errs.append(np.max(np.abs(vec(U1[0]) - ref)))
    r = [errs[0] / errs[1], errs[1] / errs[2]]
    assert all(12.0 < x < 20.0 for x in r), (errs, r)


def test_linear_step_cosine_closed_form():
    """g = 0, U = cosine-mode tensor: the whole step is a scalar recurrence."""
    n, delta, tau = 96, 10.0, 1.0 / 3000
    A1 = inputs.laplacian_neumann(n, 1.0, delta)
    ks = (5, 17)
    X = unvec(inputs.kron_vec([inputs.cosine_mode(n, k) for k in ks]), [n, n])
    lams = [inputs.cosine_eigenvalue(n, 1.0, delta, k) for k in ks]
    lam = sum(lams)
    bank = exprk3ds_precompute([[A1, A1], [A1, A1]], tau)
    U1 = exprk3ds_step([X, X], 0.0, bank, [[A1, A1], [A1, A1]], zero_g, {})
    s1 = coeffs.table1(1)
    expect = (1.0 + tau * lam * scalar_split(s1, tau, lams)) * X
    assert np.max(np.abs(U1[0] - expect)) <= 1e-12 * np.max(np.abs(X))
    # ETD2RKDS: u2 = u + tau phi1-split(K u); D = 0
    b2 = etd2rkds_precompute([[A1, A1], [A1, A1]], tau)
    from oracle.etd import etd2rkds_step
    U1 = etd2rkds_step([X, X], 0.0, b2, [[A1, A1], [A1, A1]], zero_g, {})
    expect = (1.0 + tau * lam * phi_cf(1, tau * lams[0]) * phi_cf(1, tau * lams[1])) * X
    assert np.max(np.abs(U1[0] - expect)) <= 1e-12 * np.max(np.abs(X))


def self_convergence_slope(scheme, steps_list, model="schnakenberg", d=2, n=32, T=0.1):
    prob = inputs.make_problem(model, d, n, seed=1)
    ref, _ = integrate(prob, scheme, T=T, m=8 * steps_list[-1])
    errs = []
    for m in steps_list:
        out, _ = integrate(prob, scheme, T=T, m=m)
        errs.append(max(np.max(np.abs(out[c] - ref[c])) for c in range(2)))
    x = np.log(np.array(steps_list, dtype=float))
    y = np.log(np.array(errs))
    return -np.polyfit(x, y, 1)[0], errs


def test_self_convergence_etd3():
    slope, errs = self_convergence_slope("etd3rkds", [200, 400, 800])
    assert 2.75 <= slope <= 3.25, (slope, errs)


def test_self_convergence_etd2():
    slope, errs = self_convergence_slope("etd2rkds", [200, 400, 800])
    assert 1.75 <= slope <= 2.25, (slope, errs)


def test_self_convergence_cplx():
    """Algorithm 1 with the complex Table 2, real part kept after each
    stage combination (reading R19): the scheme must still be third order (Fig. 1's slope-3
    line for exprk3ds_cplx).  A dropped term, a wrong eta/alpha branch or a truncation in the
    wrong place breaks the order.  The ladder starts at 400 steps: at 200 the complex split is
    pre-asymptotic (ratios 6.1, 6.9, 7.5 per halving)."""
    slope, errs = self_convergence_slope("exprk3ds_cplx", [400, 800, 1600])
    assert 2.75 <= slope <= 3.25, (slope, errs)


def phi_cf_c(ell, z):
    """Closed-form complex scalar phi_ell, written here independently of oracle.phi."""
    import cmath
    if z == 0:
        return 1.0 / math.factorial(ell)
    e = cmath.exp(z)
    return [e, (e - 1) / z, (e - 1 - z) / (z * z)][ell]


def scalar_split_c(s, ctau, lams):
    return sum(eta * np.prod([phi_cf_c(li, ctau * al[mu] * lams[mu]) for mu in range(s.d)])
               for eta, li, al in zip(s.etas, s.inner, s.alphas))


@pytest.mark.parametrize("d,n,delta,tau,ks", [(2, 64, 10.0, 1.0 / 3000, (5, 17)),
                                              (3, 20, 42.1887, 0.015, (2, 3, 7))])
def test_linear_step_cosine_closed_form_cplx(d, n, delta, tau, ks):
    """g = 0, cosine-mode data: one exprk3ds_cplx step of the oracle is the scalar
    Re(1 + tau lam S_1^tau) with S_1^tau = sum_i eta_i prod_mu phi_{l_i}(tau alpha_{i,mu} lam_mu)
    from the complex Table 2 — eq:exprk3's last line with D3 = 0,
    Re taken after the stage combination (R19)."""
    L = 1.0 if d == 2 else math.pi
    A1 = inputs.laplacian_neumann(n, L, delta)
    X = unvec(inputs.kron_vec([inputs.cosine_mode(n, k) for k in ks]), [n] * d)
    lams = [inputs.cosine_eigenvalue(n, L, delta, k) for k in ks]
    A = [[A1] * d, [A1] * d]
    bank = exprk3ds_precompute(A, tau, "cplx")
    U1 = exprk3ds_step([X, X], 0.0, bank, A, zero_g, {})
    s1 = coeffs.table2(1, d)
    expect = np.real(1.0 + tau * sum(lams) * scalar_split_c(s1, tau, lams)) * X
    assert not np.iscomplexobj(U1[0])
    assert np.max(np.abs(U1[0] - expect)) <= 1e-12 * np.max(np.abs(X))


def test_linear_reaction_cosine_recurrence_cplx():
    """Linear reaction g(u) = sigma u on cosine-mode data: every stage of Algorithm 1 (complex
    Table 2) acts on the single mode, so the step is a scalar recurrence in
    (lam, sigma) built from closed-form complex phi values — it checks that the imaginary part
    is dropped after EACH stage combination (reading R19), which g = 0 cannot see."""
    n, delta, tau, sigma, ks = 48, 10.0, 1.0 / 200, -3.0, (3, 11)
    A1 = inputs.laplacian_neumann(n, 1.0, delta)
    X = unvec(inputs.kron_vec([inputs.cosine_mode(n, k) for k in ks]), [n, n])
    lams = [inputs.cosine_eigenvalue(n, 1.0, delta, k) for k in ks]
    lam = sum(lams)
    A = [[A1, A1], [A1, A1]]

    def g_lin(t, u, v, p):
        return sigma * u, sigma * v

    bank = exprk3ds_precompute(A, tau, "cplx")
    U1 = exprk3ds_step([X, X], 0.0, bank, A, g_lin, {})
    S = {(ell, c): scalar_split_c(coeffs.table2(ell, 2), c * tau, lams)
         for ell in (1, 2) for c in (1 / 3, 2 / 3, 1.0)}
    u0, f = 1.0, (lam + sigma)
    u2 = np.real(u0 + tau / 3 * S[(1, 1 / 3)] * f)
    u3 = np.real(u0 + 2 * tau / 3 * S[(1, 2 / 3)] * f + 4 * tau / 3 * S[(2, 2 / 3)] * sigma * (u2 - u0))
    u1 = np.real(u0 + tau * S[(1, 1.0)] * f + 1.5 * tau * S[(2, 1.0)] * sigma * (u3 - u0))
    # negative control: keeping the imaginary parts of U2, U3 changes u1 by ~1.5e-6 relative
    v2 = u0 + tau / 3 * S[(1, 1 / 3)] * f
    v3 = u0 + 2 * tau / 3 * S[(1, 2 / 3)] * f + 4 * tau / 3 * S[(2, 2 / 3)] * sigma * (v2 - u0)
    v1 = np.real(u0 + tau * S[(1, 1.0)] * f + 1.5 * tau * S[(2, 1.0)] * sigma * (v3 - u0))
    assert abs(v1 - u1) > 1e-7 * abs(u1)
    assert np.max(np.abs(U1[0] - u1 * X)) <= 1e-12 * np.max(np.abs(X))


def dominant_modes(U, L, kmax=8):
    """Project U - mean onto cos(k pi x / L) products, k_mu <= kmax (SPEC dominant_modes)."""
    n = U.shape
    d = U.ndim
    W = U - U.mean()
    out = []
    import itertools
    for k in itertools.product(range(kmax + 1), repeat=d):
        if sum(k) == 0:
            continue
        basis = inputs.kron_vec([inputs.cosine_mode(n[mu], k[mu]) for mu in range(d)])
        basis = unvec(basis, list(n))
        out.append((abs(np.sum(W * basis)) / np.sum(basis * basis), k))
    out.sort(reverse=True)
    return out


def test_schnakenberg_pattern():
    """Fig. 3 / P:1163-1164: Turing pattern with modes (3,5),(5,3) at T = 2 (n reduced)."""
    prob = inputs.make_problem("schnakenberg", 2, 48, seed=1)
    out, _ = integrate(prob, "etd3rkds", T=2.0, m=2000)
    u = unvec(out[0], [48, 48])
    top = dominant_modes(u, 1.0)
    assert top[0][1] in ((3, 5), (5, 3)), top[:3]
    assert 0.55 < u.min() and u.max() < 1.85      # colour bar 0.6-1.8


def test_fhn_pattern():
    """Fig. 7 / P:1823-1824: FHN mode (2,2,2), u within about +-0.107 at T = 150."""
    prob = inputs.make_problem("fhn", 3, 24, seed=1)
    out, _ = integrate(prob, "etd3rkds", T=150.0, m=10000)
    u = unvec(out[0], [24, 24, 24])
    top = dominant_modes(u, math.pi, kmax=4)
    assert top[0][1] == (2, 2, 2), top[:3]
    assert 0.09 < np.max(np.abs(u)) < 0.12
