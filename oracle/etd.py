"""Split phi-actions and the directionally split exponential integrators (oracle; test infra).

Written step by step in the paper's order and notation:
  * ETD2RKDS: eq:ETD2RK with the second-order split eq:phisplit / eq:secondord
    (P:114-121);
  * exprk3ds_real: scheme eq:exprk3 realised by Algorithm 1 (d = 2, Table 1;
    P:2191-2265) and Algorithm 2 (d > 2, Table 3);
  * exprk3ds_cplx (Algorithm 1 with Table 2) is included for completeness (reading R3/R19:
    imaginary parts are discarded after each full stage combination).

States are lists of per-component tensors T[i_1..i_d]; A[c][mu-1] are the direction matrices
of component c (block-diagonal K = diag(K_1, K_2), eq:twocompdisc P:700-724).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import coeffs
from .phi import phi
from .tensor import kronsum_apply, tucker, unvec, vec


@dataclass
class Counters:
    """Cost accounting of P:671-673 (one Kronecker-sum action + 10/15 Tuckers per step and
    component)."""
    steps: int = 0
    tucker_ops: int = 0
    kronsum_actions: int = 0
    phi_builds: int = 0


def split_phi_matrices(scheme: coeffs.Scheme, c_tau: float, A: list[np.ndarray],
                       counters: Counters | None = None) -> list[list[np.ndarray]]:
    """P_i{mu} = phi_{l_i}(c_tau * alpha_{i,mu} * A_mu) for every term i and direction mu."""
    out = []
    for i in range(scheme.nterms):
        row = []
        for mu in range(scheme.d):
            row.append(phi(scheme.inner[i], c_tau * scheme.alphas[i][mu] * A[mu]))
            if counters is not None:
                counters.phi_builds += 1
        out.append(row)
    return out


def split_apply(etas, P: list[list[np.ndarray]], X: np.ndarray,
                counters: Counters | None = None) -> np.ndarray:
    """sum_i eta_i T(X, P_i)  — the tensor form of eq:split2d / eq:splitnd / eq:splitnd3 via
    eq:krontomu."""
    out = None
    for eta, Pi in zip(etas, P):
        term = eta * tucker(X, Pi)
        if counters is not None:
            counters.tucker_ops += 1
        out = term if out is None else out + term
    return out


# ------------------------------------------------------------------------------------------
# ETD2RKDS
# ------------------------------------------------------------------------------------------
@dataclass
class Etd2Bank:
    tau: float
    P1: list          # P1[c] = [[phi_1(tau A_1), ..., phi_1(tau A_d)]]  (single term)
    P2: list          # P2[c] = [[phi_2(tau A_mu)]]
    eta1: float
    eta2: float


def etd2rkds_precompute(A: list[list[np.ndarray]], tau: float,
                        counters: Counters | None = None) -> Etd2Bank:
    d = len(A[0])
    s1, s2 = coeffs.second_order(1, d), coeffs.second_order(2, d)
    P1 = [split_phi_matrices(s1, tau, Ac, counters) for Ac in A]
    P2 = [split_phi_matrices(s2, tau, Ac, counters) for Ac in A]
    return Etd2Bank(tau, P1, P2, s1.etas[0], s2.etas[0])


def etd2rkds_step(U: list[np.ndarray], t: float, bank: Etd2Bank, A, g, params,
                  counters: Counters | None = None) -> list[np.ndarray]:
    """eq:ETD2RK with phi_1, phi_2 replaced by the second-order split:
        u_n2   = u_n + tau phi_1(tau K) f(t_n, u_n)
        u_n+1  = u_n2 + tau phi_2(tau K) (g(t_n+1, u_n2) - g(t_n, u_n))."""
    tau = bank.tau
    G = g(t, U[0], U[1], params)
    F = [kronsum_apply(U[c], A[c]) + G[c] for c in range(2)]
    if counters is not None:
        counters.kronsum_actions += 2
    U2 = [U[c] + tau * split_apply([bank.eta1], bank.P1[c], F[c], counters) for c in range(2)]
    G2 = g(t + tau, U2[0], U2[1], params)
    D = [G2[c] - G[c] for c in range(2)]
    Un = [U2[c] + tau * split_apply([bank.eta2], bank.P2[c], D[c], counters) for c in range(2)]
    if counters is not None:
        counters.steps += 1
    return Un


# ------------------------------------------------------------------------------------------
# exprk3ds (Algorithms 1 and 2)
# ------------------------------------------------------------------------------------------
@dataclass
class Exprk3Bank:
    tau: float
    s1: coeffs.Scheme           # scheme approximating phi_1
    s2: coeffs.Scheme           # scheme approximating phi_2
    # P[c][key] = list over terms i of [P_i{1}, ..., P_i{d}],
    # key in {("2",1), ("3",1), ("3",2), ("f",1), ("f",2)}   (P_{i,2}^{(1)}, P_{i,3}^{(l)}, P_{i,f}^{(l)})
    P: list = field(default_factory=list)


def exprk3ds_precompute(A: list[list[np.ndarray]], tau: float, variant: str = "real",
                        counters: Counters | None = None) -> Exprk3Bank:
    """"Needed phi-functions" loop of Algorithms 1-2."""
    d = len(A[0])
    s = {1: coeffs.etd3_scheme(1, d, variant), 2: coeffs.etd3_scheme(2, d, variant)}
    bank = Exprk3Bank(tau, s[1], s[2])
    for Ac in A:
        Pc = {}
        Pc[("2", 1)] = split_phi_matrices(s[1], tau / 3.0, Ac, counters)       # P_{i,2}^{(1)}
        for ell in (1, 2):
            Pc[("3", ell)] = split_phi_matrices(s[ell], 2.0 * tau / 3.0, Ac, counters)
            Pc[("f", ell)] = split_phi_matrices(s[ell], tau, Ac, counters)
        bank.P.append(Pc)
    return bank


def _re(x, real: bool):
    return np.real(x) if real else x


def exprk3ds_step(U: list[np.ndarray], t: float, bank: Exprk3Bank, A, g, params,
                  counters: Counters | None = None) -> list[np.ndarray]:
    """One pass of the time loop of Algorithm 1 / 2."""
    tau = bank.tau
    e1, e2 = bank.s1.etas, bank.s2.etas
    real = not np.iscomplexobj(U[0])
    G = g(t, U[0], U[1], params)
    F = [kronsum_apply(U[c], A[c]) + G[c] for c in range(2)]        # F = K(U, A) + G
    if counters is not None:
        counters.kronsum_actions += 2
    # Stage U_n2
    U2 = [_re(U[c] + tau / 3.0 * split_apply(e1, bank.P[c][("2", 1)], F[c], counters), real)
          for c in range(2)]
    # Stage U_n3
    G2 = g(t + tau / 3.0, U2[0], U2[1], params)
    D2 = [G2[c] - G[c] for c in range(2)]
    U3 = [_re(U[c]
              + 2.0 * tau / 3.0 * split_apply(e1, bank.P[c][("3", 1)], F[c], counters)
              + 4.0 * tau / 3.0 * split_apply(e2, bank.P[c][("3", 2)], D2[c], counters), real)
          for c in range(2)]
    # Final approximation U_n+1
    G3 = g(t + 2.0 * tau / 3.0, U3[0], U3[1], params)
    D3 = [G3[c] - G[c] for c in range(2)]
    Un = [_re(U[c]
              + tau * split_apply(e1, bank.P[c][("f", 1)], F[c], counters)
              + 1.5 * tau * split_apply(e2, bank.P[c][("f", 2)], D3[c], counters), real)
          for c in range(2)]
    if counters is not None:
        counters.steps += 1
    return Un


# ------------------------------------------------------------------------------------------
# Drivers
# ------------------------------------------------------------------------------------------
def integrate(problem, scheme: str, T: float, m: int, steps: int | None = None,
              U0=None, counters: Counters | None = None, bank=None):
    """Integrate ``problem`` (inputs.Problem) with tau = T/m for ``steps`` steps
    (default m).  Returns the final state as vec-order flat arrays, plus the bank."""
    from .models import g_of
    g = g_of(problem.model)
    tau = T / m
    A = problem.A
    U = [unvec(u, problem.n) for u in (U0 if U0 is not None else problem.U0)]
    if bank is None:
        if scheme == "etd2rkds":
            bank = etd2rkds_precompute(A, tau, counters)
        elif scheme in ("etd3rkds", "exprk3ds_real"):
            bank = exprk3ds_precompute(A, tau, "real", counters)
        elif scheme == "exprk3ds_cplx":
            bank = exprk3ds_precompute(A, tau, "cplx", counters)
        else:
            raise ValueError(scheme)
    stepf = etd2rkds_step if scheme == "etd2rkds" else exprk3ds_step
    t = 0.0
    for _ in range(m if steps is None else steps):
        U = stepf(U, t, bank, A, g, problem.params, counters)
        t = t + tau
    return [vec(u) for u in U], bank
