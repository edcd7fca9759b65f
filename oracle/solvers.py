"""Oracle: block-layer, full-QGT and NTK (MinSR) solves (stage 5 and comparison paths).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §2 "Block-layer QGT": "Each block S_l is inverted independently, using a
uniform diagonal shift lambda to stabilize the inversion, S~_l = S_l + lambda I_l,
and delta theta_l = -eta S~_l^{-1} F_l"; BASELINE.json north_star step (5):
"(S_b + lambda I) dtheta_b = -F_b" (eta = 1, reading R6).

Full QGT (§2, "S . delta theta = -F"): (S + lambda I) dtheta = -F.
NTK / MinSR (§1, "inverting the neural tangent kernel (NTK)-like matrix
whose size depends on the number of Monte Carlo samples"): with S = A^H A,
F = A^H e (estimators.scaled_centered),

    dtheta = -A^H (A A^H + lambda I)^{-1} e

which equals the full-QGT solution by the push-through identity.
The linear systems are solved with numpy's dense LU solver (a library step).
"""
from __future__ import annotations

import numpy as np


def shifted_solve(S, rhs, lam):
    return np.linalg.solve(S + lam * np.eye(S.shape[0]), rhs)


def block_solve(blocks, F, offsets, lam):
    out = np.empty_like(F)
    for l, S_l in enumerate(blocks):
        s = slice(offsets[l], offsets[l + 1])
        out[s] = -shifted_solve(S_l, F[s], lam)
    return out


def full_solve(S, F, lam):
    return -shifted_solve(S, F, lam)


def ntk_solve(A, e, lam):
    y = shifted_solve(A @ A.conj().T, e, lam)
    return -(A.conj().T @ y)
