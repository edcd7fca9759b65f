"""Bond lists of the paper's two lattices (host-side problem set-up, no arithmetic of the step).

PAPER.md §3: periodic Heisenberg chain, H = sum_i S_i.S_{i+1}; periodic square lattice
J1-J2 model, H = J1 sum_<i,j> S_i.S_j + J2 sum_<<i,j>> S_i.S_j.  Site index x + Lx*y.
Couplings are returned in the Pauli convention of the C ABI (H = sum_b J_b sigma_i.sigma_j,
DESIGN.md reading R3); pass ``spin_units=True`` for S = sigma/2 units (J/4).
"""
from __future__ import annotations

import numpy as np


def _unique(pairs):
    seen, out = set(), []
    for i, j, J in pairs:
        key = (min(i, j), max(i, j))
        if i != j and key not in seen:
            seen.add(key)
            out.append((key[0], key[1], J))
    return out


def chain(L: int, J: float = 1.0):
    return _unique([(i, (i + 1) % L, J) for i in range(L)])


def square(Lx: int, Ly: int, J1: float = 1.0, J2: float = 0.0):
    idx = lambda x, y: (x % Lx) + Lx * (y % Ly)
    nn = [(idx(x, y), idx(x + 1, y), J1) for y in range(Ly) for x in range(Lx)]
    nn += [(idx(x, y), idx(x, y + 1), J1) for y in range(Ly) for x in range(Lx)]
    nnn = []
    if J2 != 0.0:
        nnn = [(idx(x, y), idx(x + 1, y + 1), J2) for y in range(Ly) for x in range(Lx)]
        nnn += [(idx(x, y), idx(x + 1, y - 1), J2) for y in range(Ly) for x in range(Lx)]
    return _unique(nn) + _unique(nnn)


def bond_arrays(bonds, spin_units: bool = False):
    """(int32 [n_bonds, 2], float64 [n_bonds]) in the C ABI layout."""
    ij = np.array([[i, j] for i, j, _ in bonds], dtype=np.int32).reshape(-1, 2)
    jj = np.array([J for *_, J in bonds], dtype=np.float64)
    return ij, (jj / 4.0 if spin_units else jj)


def for_workload(w, spin_units: bool = False):
    b = chain(w.extent[0], w.j1) if w.lattice == "chain" else square(w.extent[0], w.extent[1], w.j1, w.j2)
    return bond_arrays(b, spin_units)
