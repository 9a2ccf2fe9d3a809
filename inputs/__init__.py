"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the CPU oracle.

This module holds NONE of the method's arithmetic (no mode products, no phi-functions, no
splitting coefficients, no integrator stages).  It only builds the problem data the paper's
experiments feed to the method:

* a counter-based uniform generator (SplitMix64 -> 53-bit doubles), because the paper's
  initial data are draws from U(0,1) with no stated generator or seed (PAPER.md l.839-841,
  l.1516-1517; reading R6);
* the second-order centred finite-difference Laplacian with homogeneous Neumann boundary
  conditions built into the matrix (reading R5: nodes
  x_i = i*h, h = L/(n-1), ghost-point boundary rows (delta/h^2)[-2, 2]);
* the model parameters of Sec. 3 (Schnakenberg l.821-842, FitzHugh-Nagumo l.1497-1518)
  and their initial-data recipes;
* closed-form test vectors (discrete cosine modes) and the named configurations C1-C5
  of BASELINE.json / SURVEY.md §8(d).

Tensors are numpy arrays in *vec order*: a flat fp64 buffer whose first index is fastest
("stacks by columns").  ``flat.reshape(n, order="F")`` gives the
oracle's T[i_1, ..., i_d] view; the CUDA path sees the same bytes as a C-contiguous
array of shape (n_d, ..., n_1).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix64(z: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser (Steele, Lea, Flood 2014), elementwise on uint64 arrays."""
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform01(seed: int, stream: int, count: int) -> np.ndarray:
    """``count`` doubles in [0, 1) from SplitMix64, stream ``stream`` of ``seed``.

    value_i = (mix64(base + (i+1)*golden) >> 11) * 2^-53 with
    base = mix64(seed*golden + stream + 1).  Counter-based: any slice is reproducible
    independently (used to generate per-rank slabs without generating the whole field).
    """
    return uniform01_range(seed, stream, 0, count)


def uniform01_range(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        base = _mix64(np.array([np.uint64(seed) * _GOLDEN + np.uint64(stream + 1)],
                               dtype=np.uint64))[0]
        idx = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = _mix64(base + idx * _GOLDEN)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform_sym(seed: int, stream: int, count: int) -> np.ndarray:
    """U(-1, 1) doubles (used for Tucker sweep inputs)."""
    return 2.0 * uniform01(seed, stream, count) - 1.0


def laplacian_neumann(n: int, length: float, delta: float) -> np.ndarray:
    """delta * (1-D second-order FD Laplacian) with homogeneous Neumann BCs, n x n, dense.

    PAPER.md l.695-699 ("second order uniform centered finite differences ... homogeneous
    Neumann ... directly in the relevant matrices").  Reading R5: nodes x_i = i*h,
    h = length/(n-1); interior rows (delta/h^2)[1, -2, 1]; boundary rows from the ghost
    point u_{-1} = u_1: (delta/h^2)[-2, 2] and [2, -2].  Row sums are exactly zero.
    For n == 1 the matrix is [[0]] (a single node has no diffusion).
    """
    if n == 1:
        return np.zeros((1, 1))
    h = length / (n - 1)
    c = delta / (h * h)
    a = np.zeros((n, n))
    for i in range(n):
        if i == 0:
            a[0, 0], a[0, 1] = -2.0 * c, 2.0 * c
        elif i == n - 1:
            a[i, i - 1], a[i, i] = 2.0 * c, -2.0 * c
        else:
            a[i, i - 1], a[i, i], a[i, i + 1] = c, -2.0 * c, c
    return a


def cosine_mode(n: int, k: int) -> np.ndarray:
    """v_k[i] = cos(k*pi*i/(n-1)): an exact eigenvector of laplacian_neumann(n, L, delta)
    with eigenvalue -(4 delta/h^2) sin^2(k pi / (2(n-1)))  (SURVEY.md §8(c) cosine pin)."""
    i = np.arange(n, dtype=np.float64)
    return np.cos(k * math.pi * i / (n - 1))


def cosine_eigenvalue(n: int, length: float, delta: float, k: int) -> float:
    h = length / (n - 1)
    return -(4.0 * delta / (h * h)) * math.sin(k * math.pi / (2 * (n - 1))) ** 2


def kron_vec(vectors_first_fastest: list[np.ndarray]) -> np.ndarray:
    """vec(v_1 o v_2 o ... o v_d) with v_1 varying fastest (outer product in vec order)."""
    out = np.array([1.0])
    for v in vectors_first_fastest:
        out = np.kron(v, out)
    return out


# ----------------------------------------------------------------------------------------
# Models of Sec. 3 (parameters only; the reaction terms themselves are method inputs that
# each side implements on its own: oracle/models.py and the CUDA nonlinearity kernel).
# ----------------------------------------------------------------------------------------
SCHNAKENBERG = dict(du=1.0, dv=10.0, rho=1000.0, au=0.1, av=0.9)
FHN = dict(du=1.0, dv=42.1887, rho=24.649, a1=11.0, a2=0.1)


@dataclass
class Problem:
    """A two-component reaction-diffusion problem u' = K_c u + g(u, v) (eq:twocompdisc)."""
    model: str                      # "schnakenberg" | "fhn"
    d: int
    n: list[int]                    # n_1..n_d
    length: float
    params: dict
    A: list[list[np.ndarray]] = field(default_factory=list)   # A[c][mu-1], dense n_mu x n_mu
    U0: list[np.ndarray] = field(default_factory=list)        # vec-order fp64, per component

    @property
    def N(self) -> int:
        return int(np.prod(self.n))


def make_problem(model: str, d: int, n: int | list[int], seed: int = 0,
                 amplitude: float | None = None, slab: tuple[int, int] | None = None) -> Problem:
    """Build the Sec. 3 problem with the initial-data recipe of DESIGN.md (R6).

    Schnakenberg: Omega = (0,1)^d, u0 = u_e + 1e-5 U(0,1),
    v0 = v_e + 1e-5 U(0,1), (u_e, v_e) = (a^u + a^v, a^v/(a^u+a^v)^2).
    FitzHugh-Nagumo (l.1497-1518): Omega = (0,pi)^d, u0, v0 = 1e-3 U(0,1).
    Stream 0 -> u, stream 1 -> v.
    slab=(r, P): only rank r's i_d-slab of the initial data (a contiguous vec-order range,
    produced by the counter-based generator without generating the rest).
    """
    ns = [n] * d if isinstance(n, int) else list(n)
    assert len(ns) == d
    N = int(np.prod(ns))
    if model == "schnakenberg":
        p = dict(SCHNAKENBERG)
        length = 1.0
        ue = p["au"] + p["av"]
        ve = p["av"] / (p["au"] + p["av"]) ** 2
        amp = 1e-5 if amplitude is None else amplitude
        base = (ue, ve)
    elif model == "fhn":
        p = dict(FHN)
        length = math.pi
        amp = 1e-3 if amplitude is None else amplitude
        base = (0.0, 0.0)
    else:
        raise ValueError(model)
    deltas = (p["du"], p["dv"])
    A = [[laplacian_neumann(nm, length, deltas[c]) for nm in ns] for c in range(2)]
    if slab is None:
        U0 = [base[c] + amp * uniform01(seed, c, N) for c in range(2)]
    else:
        r, P = slab
        cnt = N // P
        U0 = [base[c] + amp * uniform01_range(seed, c, r * cnt, cnt) for c in range(2)]
    return Problem(model=model, d=d, n=ns, length=length, params=p, A=A, U0=U0)


# Named configurations (BASELINE.json "configs").
CONFIGS = {
    "C1": dict(model="schnakenberg", d=2, n=64, scheme="etd2rkds", T=0.25, m=3000, steps=20,
               desc="2D Schnakenberg 64^2, ETD2RKDS, tau = 0.25/3000, 20 steps"),
    "C2": dict(model="schnakenberg", d=2, n=1024, scheme="etd3rkds", T=2.0, m=6000, steps=20,
               desc="2D Schnakenberg 1024^2, ETD3RKDS real (Table 1), T=2, m=6000"),
    "C3": dict(model="fhn", d=3, n=128, scheme="etd3rkds", T=150.0, m=10000, steps=20,
               desc="3D FitzHugh-Nagumo 128^3, ETD3RKDS real (Table 3), T=150, m=10000"),
    "C4": dict(model="fhn", d=3, n=512, scheme="etd3rkds", T=150.0, m=10000, steps=20,
               desc="3D FitzHugh-Nagumo 512^3, ETD3RKDS real (Table 3), slab-sharded"),
}
