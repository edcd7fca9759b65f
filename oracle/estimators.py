"""Oracle: centring, energy, force, block/full QGT and NTK (stages 3-4).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Sample weights w_k (sum 1): uniform 1/N_s for Monte-Carlo batches (BASELINE.json
north_star: "F = Obar^dagger (E_loc - <E_loc>)/N_s", "S_b = Obar_b^dagger Obar_b / N_s"),
Born weights |psi(x)|^2/Z when the whole sector is enumerated (§2:
expectations over p_theta(x) = |psi_theta(x)|^2).

    <O_i>      = sum_k w_k O_ki                     (Eq. 2, Delta O_i = O_i - <O_i>)
    Obar_ki    = O_ki - <O_i>
    E          = sum_k w_k E_loc(x_k)               (Eq. 1)
    F_i        = sum_k w_k conj(Obar_ki) (E_loc(x_k) - E)
    S_ij       = sum_k w_k conj(Obar_ki) Obar_kj     (Eq. 2)
    S_l        = S restricted to layer l's columns   (Eq. 3)
    T_kk'      = sqrt(w_k) (sum_i Obar_ki conj(Obar_k'i)) sqrt(w_k')   (NTK, §1)
"""
from __future__ import annotations

import numpy as np


def uniform_weights(n):
    return np.full(n, 1.0 / n)


def _w(O, w):
    return uniform_weights(O.shape[0]) if w is None else np.asarray(w, dtype=np.float64)


def mean_O(O, w=None):
    w = _w(O, w)
    return np.array([np.sum(w * O[:, i]) for i in range(O.shape[1])])


def center(O, w=None):
    return O - mean_O(O, w)[None, :]


def energy(e_loc, w=None):
    w = uniform_weights(len(e_loc)) if w is None else np.asarray(w)
    return np.sum(w * e_loc)


def force(O, e_loc, w=None):
    w = _w(O, w)
    ob = center(O, w)
    eps = e_loc - energy(e_loc, w)
    return np.array([np.sum(w * np.conj(ob[:, i]) * eps) for i in range(O.shape[1])])


def qgt_full(O, w=None):
    w = _w(O, w)
    ob = center(O, w)
    return ob.conj().T @ (w[:, None] * ob)


def qgt_blocks(O, offsets, w=None):
    """[S_l] computed from each layer's own columns (never forming the full S)."""
    w = _w(O, w)
    ob = center(O, w)
    out = []
    for l in range(len(offsets) - 1):
        a = ob[:, offsets[l]:offsets[l + 1]]
        out.append(a.conj().T @ (w[:, None] * a))
    return out


def ntk(O, w=None):
    w = _w(O, w)
    a = np.sqrt(w)[:, None] * center(O, w)
    return a @ a.conj().T


def scaled_centered(O, e_loc, w=None):
    """(A, e) with A_k = sqrt(w_k) Obar_k and e_k = sqrt(w_k)(E_loc,k - E), so that
    S = A^H A, F = A^H e and T = A A^H (the factorised form both solvers share)."""
    w = _w(O, w)
    sw = np.sqrt(w)
    return sw[:, None] * center(O, w), sw * (e_loc - energy(e_loc, w))
