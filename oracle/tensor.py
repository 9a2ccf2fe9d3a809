"""Tensor algebra of PAPER.md §2 (oracle; test infrastructure only).

Tensors are numpy arrays indexed T[i_1, ..., i_d] (0-based); ``vec`` stacks by columns,
i.e. first index fastest: vec(T) = T.reshape(-1, order="F").
"""
from __future__ import annotations

import numpy as np


def vec(T: np.ndarray) -> np.ndarray:
    """vec operator, "stacks by columns the input tensor"."""
    return T.reshape(-1, order="F")


def unvec(v: np.ndarray, n: list[int]) -> np.ndarray:
    return np.asarray(v).reshape(list(n), order="F")


def mode_product(T: np.ndarray, L: np.ndarray, mu: int) -> np.ndarray:
    """mu-mode product S = T x_mu L:

        s_{i_1..i_d} = sum_{j_mu} t_{i_1..i_{mu-1} j_mu i_{mu+1}..i_d} * l^mu_{i_mu j_mu}

    mu is 1-based.  Computed as one contraction over axis mu-1 ("a single GEMM").
    """
    d = T.ndim
    if not 1 <= mu <= d:
        raise ValueError(f"mu={mu} outside 1..{d}")
    if L.shape != (T.shape[mu - 1], T.shape[mu - 1]):
        raise ValueError(f"mode {mu}: matrix {L.shape} does not match extent {T.shape[mu - 1]}")
    S = np.tensordot(L, T, axes=([1], [mu - 1]))       # axis 0 of S is i_mu
    return np.moveaxis(S, 0, mu - 1)


def tucker(T: np.ndarray, Ls: list[np.ndarray]) -> np.ndarray:
    """Tucker operator T x_1 L_1 x_2 ... x_d L_d, modes in ascending order
    (reading R2: order is free in exact arithmetic since the mode products commute)."""
    if len(Ls) != T.ndim:
        raise ValueError("need one matrix per direction")
    S = T
    for mu, L in enumerate(Ls, start=1):
        S = mode_product(S, L, mu)
    return S


def kronsum_apply(T: np.ndarray, As: list[np.ndarray]) -> np.ndarray:
    """Kronecker-sum action in tensor form, eq:kronsumv:
        K t = vec( sum_mu T x_mu A_mu ),  K = A_d (+) ... (+) A_1."""
    out = np.zeros_like(T, dtype=np.result_type(T, *As))
    for mu, A in enumerate(As, start=1):
        out = out + mode_product(T, A, mu)
    return out


ORACLE_CAP = 4096


def kron_assemble(Ls: list[np.ndarray]) -> np.ndarray:
    """Dense L_d (x) ... (x) L_1, N <= ORACLE_CAP."""
    N = int(np.prod([L.shape[0] for L in Ls]))
    if N > ORACLE_CAP:
        raise ValueError(f"N={N} exceeds the dense oracle cap {ORACLE_CAP}")
    K = np.array([[1.0]])
    for L in Ls:               # L_1 innermost (rightmost factor)
        K = np.kron(L, K)
    return K


def kronsum_assemble(As: list[np.ndarray]) -> np.ndarray:
    """Dense K = A_d (+) ... (+) A_1 = sum_mu I_d (x) .. (x) A_mu (x) .. (x) I_1 (eq:kronsum,
    P:58-66), N <= ORACLE_CAP."""
    ns = [A.shape[0] for A in As]
    N = int(np.prod(ns))
    if N > ORACLE_CAP:
        raise ValueError(f"N={N} exceeds the dense oracle cap {ORACLE_CAP}")
    K = np.zeros((N, N), dtype=np.result_type(*As))
    for mu in range(len(As)):
        factors = [As[nu] if nu == mu else np.eye(ns[nu]) for nu in range(len(As))]
        K = K + kron_assemble(factors)
    return K
