"""Pins for oracle/coeffs.py against what the paper fixes independently of the tables:
the order-condition systems eq:phi1phi22d, eq:phi1phi2nd,
eq:phi1phi2nd3t + eq:addcond, and the Groebner bases of the proof of
Theorem 3.  The moment form used here is the Taylor matching the paper states:
the coefficient of prod_mu (tau A_mu)^{k_mu} in sum_i eta_i (x)_mu phi_{l_i}(alpha_{i,mu} tau A_mu)
is sum_i eta_i prod_mu alpha_{i,mu}^{k_mu}/(k_mu+l_i)!, and in phi_l(tau K) it is
multinomial(|k|; k)/(|k|+l)!  (the A_mu commute).  E.g. k=(1,1) gives eq:deg2ab exactly."""
import itertools
from decimal import Decimal
from math import factorial

import pytest

from oracle import coeffs

D = Decimal


class C:
    """Minimal complex Decimal."""

    def __init__(self, re, im=D(0)):
        self.re, self.im = D(re), D(im)

    def __add__(self, o):
        o = o if isinstance(o, C) else C(o)
        return C(self.re + o.re, self.im + o.im)

    __radd__ = __add__

    def __sub__(self, o):
        o = o if isinstance(o, C) else C(o)
        return C(self.re - o.re, self.im - o.im)

    def __mul__(self, o):
        o = o if isinstance(o, C) else C(o)
        return C(self.re * o.re - self.im * o.im, self.re * o.im + self.im * o.re)

    __rmul__ = __mul__

    def __truediv__(self, o):
        return C(self.re / D(o), self.im / D(o))

    def __abs__(self):
        return (self.re * self.re + self.im * self.im).sqrt()


def as_c(x):
    if isinstance(x, tuple):
        return C(x[0], x[1])
    if isinstance(x, complex):
        return C(D(x.real), D(x.imag))
    return C(D(x))


def moment_residual(s: coeffs.Scheme, k):
    split = C(0)
    for eta, li, al in zip(s.etas, s.inner, s.alphas):
        t = as_c(eta)
        for mu, km in enumerate(k):
            a = as_c(al[mu])
            for _ in range(km):
                t = t * a
            t = t / factorial(km + li)
        split = split + t
    K = sum(k)
    multi = factorial(K)
    for km in k:
        multi //= factorial(km)
    exact = C(D(multi) / D(factorial(K + s.ell)))
    return abs(split - exact)


def conditions(d, third_order_extra):
    """Multi-indices of the order systems: all |k| <= 2; plus eq:addcond when asked."""
    ks = [k for k in itertools.product(range(3), repeat=d) if sum(k) <= 2]
    if third_order_extra:
        for mu in range(d):
            k = [0] * d
            k[mu] = 3
            ks.append(tuple(k))
        for c in itertools.combinations(range(d), 3):
            k = [0] * d
            for m in c:
                k[m] = 1
            ks.append(tuple(k))
    return ks


def max_residual(s, third=False):
    return max(moment_residual(s, k) for k in conditions(s.d, third))


@pytest.mark.parametrize("ell", [1, 2])
@pytest.mark.parametrize("branch", [1, -1])
def test_table1_solves_system(ell, branch):
    assert max_residual(coeffs.table1(ell, branch, exact=True)) < D("1e-45")
    assert max_residual(coeffs.table1(ell, branch)) < D("1e-14")


@pytest.mark.parametrize("ell", [1, 2])
@pytest.mark.parametrize("branch", [1, -1])
@pytest.mark.parametrize("d", [2, 3, 4, 5])
def test_table2_solves_system(ell, branch, d):
    assert max_residual(coeffs.table2(ell, d, branch, exact=True)) < D("1e-45")
    assert max_residual(coeffs.table2(ell, d, branch)) < D("1e-13")


@pytest.mark.parametrize("ell", [1, 2])
@pytest.mark.parametrize("branch", [1, -1])
@pytest.mark.parametrize("d", [2, 3, 4, 5])
def test_table3_solves_system_with_cubic_conditions(ell, branch, d):
    assert max_residual(coeffs.table3(ell, d, branch, exact=True), third=True) < D("1e-44")
    assert max_residual(coeffs.table3(ell, d, branch), third=True) < D("2e-13")


def test_mixed_sign_pairing_fails():
    """Negative control (reading R4): pairing the upper sign of alpha_{1,1} with the upper sign
    of the -+ entry alpha_{1,2} (i.e. alpha_{1,1} = alpha_{1,2}) leaves residual O(1)."""
    s = coeffs.table1(1, exact=True)
    s.alphas[0][1] = s.alphas[0][0]
    assert max_residual(s) > D("0.01")


def test_second_order_scheme_is_only_second_order():
    for d in (2, 3):
        for ell in (1, 2):
            s = coeffs.second_order(ell, d)
            assert all(moment_residual(s, k) < D("1e-15")
                       for k in itertools.product(range(2), repeat=d) if sum(k) <= 1)
            assert max_residual(s) > D("1e-3")


def test_groebner_basis_vanishes_table3():
    """Proof of Theorem 3, d = 3, both branches."""
    for branch in (1, -1):
        s = coeffs.table3(1, 3, branch, exact=True)
        e1, e2, e3 = s.etas
        a1, a2, a3 = (s.alphas[i][0] for i in range(3))
        polys = [D(570887639987) - D(724578693084) * e3 + D(218051991900) * e3 * e3,
                 12544 + 675 * e2, -2243 + 675 * e1 + 675 * e3, -45 + 28 * a2,
                 D(6486012633) + D(13981255498) * a3 - D(12113999550) * e3,
                 D(-33768359205) + D(13981255498) * a1 + D(12113999550) * e3]
        assert max(abs(p) for p in polys) < D("1e-35")
        s = coeffs.table3(2, 3, branch, exact=True)
        e1, e2, e3 = s.etas
        a1, a2, a3 = (s.alphas[i][0] for i in range(3))
        polys = [840350 - 2453166 * e3 + 1743039 * e3 * e3, 196 + 27 * e2,
                 -38 + 27 * e1 + 27 * e3, 81474 + 73990 * a3 - 193671 * e3,
                 -9 + 7 * a2, -191100 + 73990 * a1 + 193671 * e3]
        assert max(abs(p) for p in polys) < D("1e-38")


def test_printed_values():
    """SPEC examples / Table entries that are rational."""
    t1 = coeffs.table1(1)
    assert t1.etas == [-1.25, 9.0]
    assert t1.inner == [1, 2]
    t3 = coeffs.table3(1, 3)
    assert t3.alphas[1][0] == 45 / 28 and t3.etas[1] == -12544 / 675
    assert coeffs.table3(2, 4).etas[1] == -196 / 27 * 2
    t2 = coeffs.table2(2, 3)
    # '+' in alpha_{1,mu}: alpha_1 = 3/4 + sqrt3/4 i
    assert t2.alphas[0][0].imag > 0 and t2.etas[1] == 2 * complex(-2 / 3, 8 * 3 ** 0.5 / 3)
    # Table 2 at d = 2 equals Table 1's complex column -- checked via residual above;
    # eta_2 scaling 2^{d-2}:
    assert coeffs.table2(1, 4).etas[1] == 4 * coeffs.table2(1, 2).etas[1]


def test_correctly_rounded():
    """Float coefficients are the correctly rounded doubles of the 50-digit values (R18)."""
    for s_exact, s in [(coeffs.table1(1, exact=True), coeffs.table1(1)),
                       (coeffs.table1(2, exact=True), coeffs.table1(2)),
                       (coeffs.table3(1, 3, exact=True), coeffs.table3(1, 3)),
                       (coeffs.table3(2, 3, exact=True), coeffs.table3(2, 3))]:
        for a, b in zip(s_exact.etas + sum(s_exact.alphas, []), s.etas + sum(s.alphas, [])):
            assert b == float(a)
