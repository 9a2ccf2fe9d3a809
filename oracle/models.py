"""Reaction terms g = (g^1, g^2) of the two models of PAPER.md §3 (oracle; test infra only).

Both are autonomous; t is accepted and ignored (reading R7).
"""
from __future__ import annotations

import numpy as np


def g_schnakenberg(t, u: np.ndarray, v: np.ndarray, p: dict):
    """eq:Schnakenberg_2d: g^1 = rho (a^u - u + u^2 v), g^2 = rho (a^v - u^2 v)."""
    u2v = u * u * v
    return p["rho"] * (p["au"] - u + u2v), p["rho"] * (p["av"] - u2v)


def g_fhn(t, u: np.ndarray, v: np.ndarray, p: dict):
    """FitzHugh-Nagumo: g^1 = rho (-u (u^2 - 1) - v),
    g^2 = rho a_1^v (u - a_2^v v)."""
    return p["rho"] * (-u * (u * u - 1.0) - v), p["rho"] * p["a1"] * (u - p["a2"] * v)


def g_of(model: str):
    return {"schnakenberg": g_schnakenberg, "fhn": g_fhn}[model]
