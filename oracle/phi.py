"""phi-functions of small dense matrices (oracle; test infrastructure only).

phi_l(X) = sum_{k>=0} X^k / (k+l)!.

The paper forms the small phi-matrices with "a rational Pade approach with modified scaling
and squaring [SW09]" and gives no further detail.  Reading R8: the
oracle uses the same *modified squaring* structure with a Taylor base approximant:

  1. s = max(0, ceil(log2(||X||_1 / theta))), theta = 2, Y = X / 2^s;
  2. phi_l(Y) for l = 0..lmax by the Taylor series itself, 40 terms (truncation
     2^40/40! ~ 1e-36, far below fp64 rounding);
  3. s times the doubling identities (SW09; derived from e^{2Y} = e^Y e^Y and
     z phi_1(z) = e^z - 1, z^2 phi_2(z) = e^z - 1 - z):
        phi_0(2Y) = phi_0(Y)^2
        phi_1(2Y) = 1/2 phi_1(Y) (phi_0(Y) + I)
        phi_2(2Y) = 1/4 (phi_1(Y)^2 + 2 phi_2(Y))
"""
from __future__ import annotations

import math

import numpy as np

THETA = 2.0
TAYLOR_TERMS = 40


def scaling_exponent(X: np.ndarray, theta: float = THETA) -> int:
    nrm = np.abs(X).sum(axis=0).max() if X.size else 0.0   # induced 1-norm
    if nrm <= theta:
        return 0
    return int(math.ceil(math.log2(nrm / theta)))


def phi_taylor_unscaled(X: np.ndarray, lmax: int, terms: int = TAYLOR_TERMS) -> list[np.ndarray]:
    """[phi_0(X), ..., phi_lmax(X)] straight from the series (use only for small ||X||)."""
    n = X.shape[0]
    Xk = np.eye(n, dtype=X.dtype)               # X^k
    out = [np.zeros_like(Xk) for _ in range(lmax + 1)]
    for k in range(terms):
        for ell in range(lmax + 1):
            out[ell] = out[ell] + Xk / math.factorial(k + ell)
        Xk = Xk @ X
    return out


def phi_matrices(X: np.ndarray, lmax: int = 2) -> list[np.ndarray]:
    """[phi_0(X), phi_1(X), ..., phi_lmax(X)], lmax <= 2, via Taylor + doubling (reading R8)."""
    if lmax > 2:
        raise ValueError("doubling identities implemented for l <= 2")
    X = np.asarray(X)
    s = scaling_exponent(X)
    phis = phi_taylor_unscaled(X / (2.0 ** s), 2)
    I = np.eye(X.shape[0], dtype=phis[0].dtype)
    for _ in range(s):
        p0, p1, p2 = phis
        phis = [p0 @ p0,
                0.5 * (p1 @ (p0 + I)),
                0.25 * (p1 @ p1 + 2.0 * p2)]
    return phis[: lmax + 1]


def phi(ell: int, X: np.ndarray) -> np.ndarray:
    """phi_ell(X) for ell in {0, 1, 2}."""
    return phi_matrices(X, ell)[ell]


def phi_scalar(ell: int, z: complex | float) -> complex | float:
    """Closed forms phi_0 = e^z, phi_1 = (e^z-1)/z, phi_2 = (e^z-1-z)/z^2, with the series
    near 0 (used only by tests as an independent pin and by closed-form expectations)."""
    if abs(z) < 1e-3:
        return sum(z ** k / math.factorial(k + ell) for k in range(12))
    if isinstance(z, complex) or np.iscomplexobj(z):
        e = np.exp(z)
        em1 = e - 1.0
    else:
        e = math.exp(z)
        em1 = math.expm1(z)
    if ell == 0:
        return e
    if ell == 1:
        return em1 / z
    if ell == 2:
        return (em1 - z) / (z * z)
    raise ValueError(ell)
