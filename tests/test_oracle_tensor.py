"""Pins for oracle/tensor.py: brute force, dense Kronecker algebra written independently
here from index formulas, the d=2 BLAS identities and the exact exp split
 with scipy's expm."""
import itertools

import numpy as np
import pytest
import scipy.linalg

from inputs import laplacian_neumann, uniform_sym
from oracle.tensor import (kron_assemble, kronsum_apply, kronsum_assemble, mode_product,
                           tucker, unvec, vec)


def rnd(seed, *shape):
    n = int(np.prod(shape))
    return uniform_sym(seed, 7, n).reshape(shape)


def lin(idx, n):
    """vec index of multi-index idx (first fastest)."""
    k, stride = 0, 1
    for i, m in zip(idx, n):
        k += i * stride
        stride *= m
    return k


def brute_kron(Ls):
    """K[(i),(j)] = prod_mu L_mu[i_mu, j_mu] with vec linear indices (eq:krontomu)."""
    n = [L.shape[0] for L in Ls]
    N = int(np.prod(n))
    K = np.zeros((N, N))
    for I in itertools.product(*[range(m) for m in n]):
        for J in itertools.product(*[range(m) for m in n]):
            K[lin(I, n), lin(J, n)] = np.prod([Ls[m][I[m], J[m]] for m in range(len(n))])
    return K


def test_mode_product_brute_force():
    T = rnd(1, 3, 4, 5)
    for mu in (1, 2, 3):
        L = rnd(10 + mu, T.shape[mu - 1], T.shape[mu - 1])
        S = mode_product(T, L, mu)
        E = np.zeros_like(T)
        for i1, i2, i3 in itertools.product(range(3), range(4), range(5)):
            idx = [i1, i2, i3]
            acc = 0.0
            for j in range(T.shape[mu - 1]):
                jdx = list(idx)
                jdx[mu - 1] = j
                acc += T[tuple(jdx)] * L[idx[mu - 1], j]
            E[i1, i2, i3] = acc
        assert np.max(np.abs(S - E)) <= 1e-14


def test_mode_product_d2_is_matrix_product():
    T = rnd(2, 5, 7)
    L1, L2 = rnd(3, 5, 5), rnd(4, 7, 7)
    assert np.allclose(mode_product(T, L1, 1), L1 @ T, rtol=0, atol=1e-14)
    assert np.allclose(mode_product(T, L2, 2), T @ L2.T, rtol=0, atol=1e-14)
    # eq:exp2d shape: T x_1 L1 x_2 L2 = L1 T L2^T
    assert np.allclose(tucker(T, [L1, L2]), L1 @ T @ L2.T, rtol=0, atol=1e-13)


def test_mode_product_shape_error_names_mu():
    with pytest.raises(ValueError, match="mode 2"):
        mode_product(rnd(5, 3, 4), np.eye(3), 2)


@pytest.mark.parametrize("seed", range(40))
def test_tucker_equals_dense_kronecker(seed):
    rs = np.random.default_rng(seed)
    d = int(rs.integers(1, 4))
    n = [int(rs.integers(1, 6)) for _ in range(d)]
    T = rnd(100 + seed, *n)
    Ls = [rnd(200 + seed * 7 + mu, m, m) for mu, m in enumerate(n)]
    K = brute_kron(Ls)
    assert np.allclose(kron_assemble(Ls), K, rtol=0, atol=1e-15)
    lhs = vec(tucker(T, Ls))
    rhs = K @ vec(T)
    assert np.max(np.abs(lhs - rhs)) <= 1e-13 * max(1.0, np.max(np.abs(rhs)))


@pytest.mark.parametrize("seed", range(40))
def test_kronsum_equals_dense(seed):
    rs = np.random.default_rng(1000 + seed)
    d = int(rs.integers(1, 4))
    n = [int(rs.integers(1, 6)) for _ in range(d)]
    T = rnd(300 + seed, *n)
    As = [rnd(400 + seed * 7 + mu, m, m) for mu, m in enumerate(n)]
    N = int(np.prod(n))
    K = np.zeros((N, N))      # sum_mu I(x)..(x)A_mu(x)..(x)I, by index formula
    for I in itertools.product(*[range(m) for m in n]):
        for J in itertools.product(*[range(m) for m in n]):
            for mu in range(d):
                if all(I[nu] == J[nu] for nu in range(d) if nu != mu):
                    K[lin(I, n), lin(J, n)] += As[mu][I[mu], J[mu]]
    assert np.allclose(kronsum_assemble(As), K, rtol=0, atol=1e-15)
    assert np.max(np.abs(vec(kronsum_apply(T, As)) - K @ vec(T))) <= 1e-13


def test_identity_and_zero_cases():
    T = rnd(9, 3, 4, 2)
    assert np.array_equal(tucker(T, [np.eye(3), np.eye(4), np.eye(2)]), T)
    assert np.array_equal(kronsum_apply(T, [np.zeros((3, 3)), np.zeros((4, 4)), np.zeros((2, 2))]),
                          np.zeros_like(T))


def test_neumann_kills_constants():
    As = [laplacian_neumann(m, 1.0, 3.0) for m in (5, 6, 7)]
    T = np.full((5, 6, 7), 2.5)
    assert np.max(np.abs(kronsum_apply(T, As))) <= 1e-9   # entries ~ 3*2*36*2.5; exact 0 up to rounding
    for A in As:
        assert np.all(A.sum(axis=1) == 0.0)


def test_mode_order_commutes():
    T = rnd(11, 4, 3, 5)
    Ls = [rnd(12, 4, 4), rnd(13, 3, 3), rnd(14, 5, 5)]
    ref = tucker(T, Ls)
    S = T
    for mu in (3, 1, 2):
        S = mode_product(S, Ls[mu - 1], mu)
    assert np.max(np.abs(S - ref)) <= 1e-14 * np.max(np.abs(ref)) * 10


def test_exp_split_is_exact():
    """eq:expTucker: exp(tau K) v = vec(V x_1 e^{tau A_1} ... x_d e^{tau A_d})."""
    n = [3, 4, 5]
    As = [rnd(20 + i, m, m) for i, m in enumerate(n)]
    V = rnd(30, *n)
    tau = 0.3
    lhs = vec(tucker(V, [scipy.linalg.expm(tau * A) for A in As]))
    rhs = scipy.linalg.expm(tau * kronsum_assemble(As)) @ vec(V)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(rhs))


def test_vec_roundtrip():
    v = uniform_sym(3, 3, 60)
    assert np.array_equal(vec(unvec(v, [3, 4, 5])), v)
    T = unvec(v, [3, 4, 5])
    assert T[1, 2, 3] == v[1 + 3 * (2 + 4 * 3)]
