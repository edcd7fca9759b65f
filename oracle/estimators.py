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

Centring precision (readings R7, R11): the uniform mean <O_i> = (sum_k O_ki)/N
and E are carried as unevaluated double-double pairs (error-free TwoSum accumulation, the
quotient by N with its remainder), and O_ki - <O_i>, E_loc,k - E are rounded to complex128
once; weighted means use numpy longdouble.  For sum-pooled lncosh networks at the
BASELINE.json initialisation the deep-layer derivatives are nearly constant over samples
(|<O_i>| / std(O_i) up to ~1e6 at configs[2], ~1e9 at configs[3]), so a double-rounded
mean would cost up to 9 of the 16 digits of Obar before any estimator is formed, and a
64-bit long-double mean still several.
"""
from __future__ import annotations

import numpy as np


def uniform_weights(n):
    return np.full(n, 1.0 / n)


def _w(O, w):
    return uniform_weights(O.shape[0]) if w is None else np.asarray(w, dtype=np.float64)


_LD = np.clongdouble


def _two_sum(a, b):
    """s + e = a + b exactly (Knuth's TwoSum, elementwise on float64 arrays)."""
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def _dd_mean(x):
    """Uniform column mean of a real float64 array [N, m] as a double-double (hi, lo):
    the column sums are accumulated by TwoSum with the rounding errors summed separately
    (cascaded summation: accurate to ~N 2^-106 relative to sum |x|), renormalised, then
    divided by N as hi/N plus (the remainder hi - N q, exact by TwoSum of the product
    split) + lo, over N."""
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[0]
    hi = np.zeros(x.shape[1:])
    lo = np.zeros(x.shape[1:])
    for k in range(n):
        hi, e = _two_sum(hi, x[k])
        lo = lo + e
    hi, lo = _two_sum(hi, lo)
    q = hi / n
    # r = hi - n q exactly: n q = p + pe with p = n * q rounded and pe its error (Dekker's
    # product split; n is an integer below 2^26 so the split of n is exact)
    p = n * q
    c = 134217729.0 * q   # 2^27 + 1
    qh = c - (c - q)
    ql = q - qh
    pe = ((n * qh - p) + n * ql)
    r = (hi - p) - pe + lo
    return q, r / n


def _mean_ld(x, w):
    """sum_k w_k x_k in extended precision (longdouble accumulation) for weighted means."""
    xl = np.asarray(x).astype(_LD)
    return np.sum(np.asarray(w, dtype=np.longdouble)[:, None] * xl, axis=0)


def _center_cols(x, w):
    """x_k - <x> rounded once, for complex columns x [N, m]."""
    x = np.asarray(x)
    if w is None:
        out = np.empty(x.shape, dtype=np.complex128)
        for part, dst in ((x.real, "real"), (x.imag, "imag")):
            q, r = _dd_mean(part)
            d, de = _two_sum(part, -q)       # exact difference of x and the leading part
            setattr(out, dst, d + (de - r))
        return out
    return (x.astype(_LD) - _mean_ld(x, w)[None, :]).astype(np.complex128)


def mean_O(O, w=None):
    if w is None:
        O = np.asarray(O)
        qr, rr = _dd_mean(O.real)
        qi, ri = _dd_mean(O.imag)
        return (qr + rr) + 1j * (qi + ri)
    return _mean_ld(O, w).astype(np.complex128)


def center(O, w=None):
    """Obar = O - <O>, the mean beyond double precision, the difference rounded once."""
    return _center_cols(O, w)


def energy(e_loc, w=None):
    return complex(mean_O(np.asarray(e_loc)[:, None], w)[0])


def centered_energies(e_loc, w=None):
    """E_loc,k - E with E beyond double precision, rounded once."""
    return _center_cols(np.asarray(e_loc)[:, None], w)[:, 0]


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
