"""Pins for oracle/phi.py: scipy's expm on the Van Loan block (independent library routine),
closed-form scalar phi-functions, diagonal and nilpotent matrices, the recurrence
phi_l(X) X = phi_{l-1}(X) - I/(l-1)!, and the exact row sums for zero-row-sum generators."""
import math

import numpy as np
import pytest
import scipy.linalg

from inputs import laplacian_neumann, uniform_sym
from oracle.phi import phi, phi_matrices, phi_scalar


def vanloan_phis(X):
    """phi_1, phi_2 as the top-right blocks of expm([[X, I, 0], [0, 0, I], [0, 0, 0]])."""
    n = X.shape[0]
    B = np.zeros((3 * n, 3 * n), dtype=X.dtype)
    B[:n, :n] = X
    B[:n, n:2 * n] = np.eye(n)
    B[n:2 * n, 2 * n:] = np.eye(n)
    E = scipy.linalg.expm(B)
    return E[:n, :n], E[:n, n:2 * n], E[:n, 2 * n:]


@pytest.mark.parametrize("scale", [0.1, 1.0, 5.0, 20.0])
@pytest.mark.parametrize("seed", range(4))
def test_phi_vs_vanloan_random(scale, seed):
    X = scale * uniform_sym(seed, 11, 36).reshape(6, 6)
    ours = phi_matrices(X, 2)
    ref = vanloan_phis(X)
    for ell in range(3):
        rel = np.max(np.abs(ours[ell] - ref[ell])) / np.max(np.abs(ref[ell]))
        assert rel <= 1e-12, (ell, rel)


@pytest.mark.parametrize("n,delta,ctau", [(16, 1.0, 1e-3), (32, 10.0, 1e-3), (64, 42.1887, 0.02)])
def test_phi_vs_vanloan_stiff_laplacian(n, delta, ctau):
    X = ctau * laplacian_neumann(n, math.pi, delta)
    ours = phi_matrices(X, 2)
    ref = vanloan_phis(X)
    for ell in range(3):
        rel = np.max(np.abs(ours[ell] - ref[ell])) / np.max(np.abs(ref[ell]))
        assert rel <= 1e-11, (ell, rel)


@pytest.mark.parametrize("z", [-40.0, -3.0, -0.5, -1e-4, 0.0, 1e-6, 0.7, 2.5])
def test_scalar_closed_forms(z):
    ours = [phi(ell, np.array([[z]]))[0, 0] for ell in range(3)]
    e = math.exp(z)
    if z == 0.0:
        ref = [1.0, 1.0, 0.5]
    else:
        ref = [e, math.expm1(z) / z, (math.expm1(z) - z) / (z * z) if abs(z) > 1e-3
               else 0.5 + z / 6 + z * z / 24]
    for ell in range(3):
        assert abs(ours[ell] - ref[ell]) <= 1e-13 * abs(ref[ell]) + 1e-300


def test_zero_gives_inverse_factorials():
    for ell in range(3):
        assert np.array_equal(phi(ell, np.zeros((5, 5))), np.eye(5) / math.factorial(ell))


def test_diagonal_matrix():
    lam = np.array([-30.0, -2.0, 0.0, 0.3, 1.5])
    P = phi_matrices(np.diag(lam), 2)
    for ell in range(3):
        ref = [phi_scalar(ell, z) if z != 0 else 1.0 / math.factorial(ell) for z in lam]
        assert np.max(np.abs(np.diag(P[ell]) - ref)) <= 1e-13 * np.max(np.abs(ref))
        assert np.max(np.abs(P[ell] - np.diag(np.diag(P[ell])))) == 0.0


def test_nilpotent_series_terminates():
    A = np.array([[0.0, 1.0], [0.0, 0.0]])
    assert np.allclose(phi(1, A), np.eye(2) + A / 2, rtol=0, atol=1e-16)
    assert np.allclose(phi(2, A), np.eye(2) / 2 + A / 6, rtol=0, atol=1e-16)
    N3 = np.diag([3.0, -2.0], k=1)      # 3x3 strictly upper, N^3 = 0
    N2 = N3 @ N3
    assert np.allclose(phi(0, N3), np.eye(3) + N3 + N2 / 2, rtol=0, atol=1e-15)


@pytest.mark.parametrize("seed", range(5))
def test_recurrence(seed):
    X = 3.0 * uniform_sym(seed, 12, 25).reshape(5, 5)
    P = phi_matrices(X, 2)
    for ell in (1, 2):
        res = P[ell] @ X - P[ell - 1] + np.eye(5) / math.factorial(ell - 1)
        assert np.max(np.abs(res)) <= 1e-12 * max(1.0, np.max(np.abs(P[ell - 1])))


@pytest.mark.parametrize("n,delta,ctau", [(32, 1.0, 0.01), (100, 42.1887, 0.015), (128, 10.0, 1e-3)])
def test_row_sums_neumann(n, delta, ctau):
    """Zero-row-sum A: phi_l(c A) 1 = 1/l! exactly; entries >= 0 for c > 0 (Metzler A)."""
    X = ctau * laplacian_neumann(n, 1.0, delta)
    P = phi_matrices(X, 2)
    for ell in range(3):
        rs = P[ell].sum(axis=1)
        assert np.max(np.abs(rs - 1.0 / math.factorial(ell))) <= 1e-11
        assert np.min(P[ell]) >= -1e-15
