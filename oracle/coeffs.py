"""Directional-splitting coefficients (oracle; test infrastructure only).

A split scheme approximates phi_ell(tau K) by
    sum_i eta_i  phi_{l_i}(alpha_{i,d} tau A_d) (x) ... (x) phi_{l_i}(alpha_{i,1} tau A_1)
(eq:split2d P:302-312, eq:splitnd P:383-392, eq:splitnd3 P:460-472).

Values are evaluated from the radical forms printed in Tables 1-3 with 50-digit decimal
arithmetic and rounded once to fp64 (reading R18).  Branch: the paper always uses "the
choice of the symbol + in alpha_{1,1} or alpha_{1,mu}".  For Tables 1 and 3
that is the upper sign of every +-/-+ pair (pairing upper-with-upper, reading R4); for the
complex Table 2 the "+" in alpha_{1,mu} = 12/11 -+ 4 sqrt2/11 i is the LOWER sign, and the
other entries take the lower sign with it (reading R3).
"""
from __future__ import annotations

from dataclasses import dataclass
from decimal import Decimal, getcontext
from math import factorial

getcontext().prec = 50


def _D(x) -> Decimal:
    return Decimal(x)


def _sqrt(x: int) -> Decimal:
    return Decimal(x).sqrt()


@dataclass
class Scheme:
    """One split rule: terms (eta_i, l_i, [alpha_{i,1}, ..., alpha_{i,d}])."""
    name: str
    ell: int                      # target phi_ell
    d: int
    etas: list                    # complex or float
    inner: list[int]              # l_i
    alphas: list[list]            # alphas[i][mu-1]

    @property
    def nterms(self) -> int:
        return len(self.etas)


def _f(x: Decimal) -> float:
    return float(x)


def second_order(ell: int, d: int) -> Scheme:
    """eq:secondord: phi_ell(tau K) ~ ell!^{d-1} (x)_mu phi_ell(tau A_mu)."""
    return Scheme("second_order", ell, d, [float(factorial(ell) ** (d - 1))], [ell],
                  [[1.0] * d])


def table1(ell: int, branch: int = +1, exact: bool = False) -> Scheme:
    """Table 1, real columns, d = 2, l_1 = 1, l_2 = 2.  branch=+1: upper signs."""
    s = _D(branch)
    if ell == 1:
        r = _sqrt(10)
        eta1, eta2 = _D(-5) / 4, _D(9)
        a11 = s * 4 * r / 15 + _D(4) / 3
        a12 = -s * 4 * r / 15 + _D(4) / 3
        a21 = s * 2 * r / 9 + _D(16) / 9
        a22 = -s * 2 * r / 9 + _D(16) / 9
    elif ell == 2:
        r = _sqrt(33)
        eta1, eta2 = _D(-4) / 3, _D(22) / 3
        a11 = s * r / 8 + _D(9) / 8
        a12 = -s * r / 8 + _D(9) / 8
        a21 = s * 3 * r / 22 + _D(3) / 2
        a22 = -s * 3 * r / 22 + _D(3) / 2
    else:
        raise ValueError(ell)
    cv = (lambda x: x) if exact else _f
    return Scheme("table1", ell, 2, [cv(eta1), cv(eta2)], [1, 2],
                  [[cv(a11), cv(a12)], [cv(a21), cv(a22)]])


def table2(ell: int, d: int, branch: int = -1, exact: bool = False) -> Scheme:
    """Table 2, complex, d >= 2, l_1 = 1, l_2 = 2, alpha independent of mu.
    branch=-1 (default) is the paper's '+ in alpha_{1,mu}' choice (lower sign of -+)."""
    s = _D(branch)          # +1 -> upper sign of +- (and upper of -+ i.e. minus)
    two = _D(2) ** (d - 2)
    if ell == 1:
        r = _sqrt(2)
        eta1 = (_D(7) / 4, s * 3 * r / 2)
        a1 = (_D(12) / 11, -s * 4 * r / 11)
        eta2 = (two * -3, two * (-s * 6 * r))
        a2 = (_D(4) / 3, -s * 2 * r / 3)
    elif ell == 2:
        r = _sqrt(3)
        eta1 = (_D(2) / 3, s * 2 * r / 3)
        a1 = (_D(3) / 4, -s * r / 4)
        eta2 = (two * (_D(-2) / 3), two * (-s * 8 * r / 3))
        a2 = (_D(6) / 7, -s * 3 * r / 7)
    else:
        raise ValueError(ell)
    if exact:
        cv = lambda p: p
    else:
        cv = lambda p: complex(float(p[0]), float(p[1]))
    return Scheme("table2", ell, d, [cv(eta1), cv(eta2)], [1, 2],
                  [[cv(a1)] * d, [cv(a2)] * d])


def table3(ell: int, d: int, branch: int = +1, exact: bool = False) -> Scheme:
    """Table 3, real, d >= 2 (used for d > 2, Algorithm 2), l = (1, 2, 1)."""
    s = _D(branch)
    two = _D(2) ** (d - 3) if d >= 3 else _D(1) / _D(2) ** (3 - d)
    if ell == 1:
        r = _sqrt(2991111)
        eta1 = _D(2243) / 1350 + s * _D(440521) / (675 * r)
        a1 = 3 * (5161 + s * r) / 15869
        eta2 = _D(-12544) / 675 * two
        a2 = _D(45) / 28
        eta3 = _D(2243) / 1350 - s * _D(440521) / (675 * r)
        a3 = 3 * (5161 - s * r) / 15869
    elif ell == 2:
        r = _sqrt(2391)
        eta1 = _D(19) / 27 + s * _D(151) / (27 * r)
        a1 = 3 * (121 + s * r) / 490
        eta2 = _D(-196) / 27 * two
        a2 = _D(9) / 7
        eta3 = _D(19) / 27 - s * _D(151) / (27 * r)
        a3 = 3 * (121 - s * r) / 490
    else:
        raise ValueError(ell)
    cv = (lambda x: x) if exact else _f
    return Scheme("table3", ell, d, [cv(eta1), cv(eta2), cv(eta3)], [1, 2, 1],
                  [[cv(a1)] * d, [cv(a2)] * d, [cv(a3)] * d])


def etd3_scheme(ell: int, d: int, variant: str = "real") -> Scheme:
    """Scheme used by exprk3ds: real -> Table 1 if d == 2 (Algorithm 1 caption, P:2192-2196,
    reading R10) else Table 3 (Algorithm 2); cplx -> Table 2."""
    if variant == "real":
        return table1(ell) if d == 2 else table3(ell, d)
    if variant == "cplx":
        return table2(ell, d)
    raise ValueError(variant)
