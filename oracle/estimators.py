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

Centring precision (reading R7): <O_i> and E are accumulated in extended
precision (numpy longdouble) and O_ki - <O_i>, E_loc,k - E are rounded to complex128
once.  For sum-pooled lncosh networks at the BASELINE.json initialisation the last-layer
bias derivatives are nearly constant over samples (|<O_i>| / std(O_i) up to ~1e6), so a
double-rounded mean would cost ~6 of the 16 digits of Obar before any estimator is formed.
"""
from __future__ import annotations

import numpy as np


def uniform_weights(n):
    return np.full(n, 1.0 / n)


def _w(O, w):
    return uniform_weights(O.shape[0]) if w is None else np.asarray(w, dtype=np.float64)


_LD = np.clongdouble


def _mean_ld(x, w):
    """sum_k w_k x_k in extended precision (longdouble accumulation); w = None means the
    uniform mean (sum_k x_k) / N with the division also in extended precision."""
    xl = np.asarray(x).astype(_LD)
    if w is None:
        return np.sum(xl, axis=0) / np.longdouble(xl.shape[0])
    return np.sum(np.asarray(w, dtype=np.longdouble)[:, None] * xl, axis=0)


def mean_O(O, w=None):
    return _mean_ld(O, w).astype(np.complex128)


def center(O, w=None):
    """Obar = O - <O>, the difference taken in extended precision and rounded once."""
    return (np.asarray(O).astype(_LD) - _mean_ld(O, w)[None, :]).astype(np.complex128)


def _energy_ld(e_loc, w):
    return _mean_ld(np.asarray(e_loc)[:, None], w)[0]


def energy(e_loc, w=None):
    return complex(_energy_ld(e_loc, w))


def centered_energies(e_loc, w=None):
    """E_loc,k - E with E in extended precision, rounded once."""
    return (np.asarray(e_loc).astype(_LD) - _energy_ld(e_loc, w)).astype(np.complex128)


def force(O, e_loc, w=None):
    ob = center(O, w)
    eps = centered_energies(e_loc, w)
    w = _w(O, w)
    return np.array([np.sum(w * np.conj(ob[:, i]) * eps) for i in range(O.shape[1])])


def qgt_full(O, w=None):
    ob = center(O, w)
    w = _w(O, w)
    return ob.conj().T @ (w[:, None] * ob)


def qgt_blocks(O, offsets, w=None):
    """[S_l] computed from each layer's own columns (never forming the full S)."""
    ob = center(O, w)
    w = _w(O, w)
    out = []
    for l in range(len(offsets) - 1):
        a = ob[:, offsets[l]:offsets[l + 1]]
        out.append(a.conj().T @ (w[:, None] * a))
    return out


def ntk(O, w=None):
    a = np.sqrt(_w(O, w))[:, None] * center(O, w)
    return a @ a.conj().T


def scaled_centered(O, e_loc, w=None):
    """(A, e) with A_k = sqrt(w_k) Obar_k and e_k = sqrt(w_k)(E_loc,k - E), so that
    S = A^H A, F = A^H e and T = A A^H (the factorised form both solvers share)."""
    sw = np.sqrt(_w(O, w))
    return sw[:, None] * center(O, w), sw * centered_energies(e_loc, w)
