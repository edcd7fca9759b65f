"""Oracle: Heisenberg / J1-J2 Hamiltonians, local energies, dense H and ED (stage 2).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §3: "H = sum_i S_i . S_{i+1}" (chain, periodic) and
"H = J1 sum_<i,j> S_i.S_j + J2 sum_<<i,j>> S_i.S_j" (square lattice, periodic).
Units (reading R3): matrix elements are written in Pauli units,
sigma_i . sigma_j = 4 S_i . S_j, which is the convention PAPER.md Table 2's energy
(-28.5685(3) for the L=16 chain) is quoted in; pass J/4 for S = sigma/2 units.

Local energy (§2 Eq. 1: "E = E_{x~p}[<x|H|psi>/<x|psi>]"):

    E_loc(x) = sum_{x'} <x|H|x'> psi(x')/psi(x)
             = sum_{(i,j,J)} J [ s_i s_j + (1 - s_i s_j) psi(x^{ij})/psi(x) ]

since sigma_i.sigma_j = Z_i Z_j + 2 (S+_i S-_j + S-_i S+_j) flips an anti-aligned pair
with amplitude 2J and leaves an aligned pair alone; x^{ij} is x with s_i, s_j swapped.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import network


def _dedupe(bonds):
    seen, out = set(), []
    for i, j, J in bonds:
        key = (min(i, j), max(i, j))
        if i != j and key not in seen:
            seen.add(key)
            out.append((key[0], key[1], float(J)))
    return out


def chain_bonds(L, J=1.0):
    """Periodic chain: bonds (i, i+1 mod L)."""
    return _dedupe([(i, (i + 1) % L, J) for i in range(L)])


def square_bonds(Lx, Ly, J1=1.0, J2=0.0):
    """Periodic Lx x Ly square lattice, site = x + Lx*y.

    Nearest neighbours (x+1,y), (x,y+1) with J1; next-nearest (diagonal)
    neighbours (x+1,y+1), (x+1,y-1) with J2 (§3 <i,j> and <<i,j>>)."""
    site = lambda x, y: (x % Lx) + Lx * (y % Ly)
    nn, nnn = [], []
    for y in range(Ly):
        for x in range(Lx):
            nn.append((site(x, y), site(x + 1, y), J1))
            nn.append((site(x, y), site(x, y + 1), J1))
            if J2 != 0.0:
                nnn.append((site(x, y), site(x + 1, y + 1), J2))
                nnn.append((site(x, y), site(x + 1, y - 1), J2))
    return _dedupe(nn) + _dedupe(nnn)


def bonds_for(workload):
    if workload.lattice == "chain":
        return chain_bonds(workload.extent[0], workload.j1)
    return square_bonds(workload.extent[0], workload.extent[1], workload.j1, workload.j2)


def connected(x, bonds):
    """[(x', <x|H|x'>)]: the diagonal element first, then one entry per flipped bond."""
    x = np.asarray(x)
    diag = 0.0
    out = []
    for i, j, J in bonds:
        diag += J * x[i] * x[j]
        if x[i] != x[j]:
            xp = x.copy()
            xp[i], xp[j] = x[j], x[i]
            out.append((xp, 2.0 * J))
    return [(x.copy(), diag)] + out


def local_energy_fn(log_amp, x, bonds):
    """E_loc(x) for an arbitrary log-amplitude function log_amp(config)."""
    lp = log_amp(x)
    e = 0.0 + 0.0j
    for xp, amp in connected(x, bonds):
        e += amp * np.exp(log_amp(xp) - lp)
    return e


def local_energies(params, xs, bonds):
    """E_loc for every row of xs with the MLP wavefunction."""
    f = lambda c: network.forward(params, c)[0]
    return np.array([local_energy_fn(f, x, bonds) for x in np.asarray(xs)], dtype=np.complex128)


# ---------------------------------------------------------------------------
# Dense Hamiltonian from Pauli Kronecker products (independent of `connected`).
# Basis index: bit i set <=> s_i = +1; site 0 is the least-significant bit.
# ---------------------------------------------------------------------------
_SX = sp.csr_matrix(np.array([[0, 1], [1, 0]], dtype=np.complex128))
_SY = sp.csr_matrix(np.array([[0, 1j], [-1j, 0]], dtype=np.complex128))   # basis (down, up)
_SZ = sp.csr_matrix(np.array([[-1, 0], [0, 1]], dtype=np.complex128))
_ID = sp.identity(2, dtype=np.complex128, format="csr")


def _site_op(op, i, n):
    out = sp.identity(1, dtype=np.complex128, format="csr")
    for s in reversed(range(n)):              # kron(op_{n-1}, ..., op_0)
        out = sp.kron(out, op if s == i else _ID, format="csr")
    return out


def dense_hamiltonian(n, bonds):
    """Sparse 2^n x 2^n matrix sum_b J_b (X_i X_j + Y_i Y_j + Z_i Z_j)."""
    h = sp.csr_matrix((1 << n, 1 << n), dtype=np.complex128)
    for i, j, J in bonds:
        for op in (_SX, _SY, _SZ):
            h = h + J * (_site_op(op, i, n) @ _site_op(op, j, n))
    return h.tocsr()


def basis_index(x):
    return int(sum(1 << i for i, s in enumerate(np.asarray(x)) if s > 0))


def sector_indices(n, total=0):
    up = (n + total) // 2
    return np.array([k for k in range(1 << n) if bin(k).count("1") == up], dtype=np.int64)


def ground_state(n, bonds, total=0):
    """Lowest eigenpair of H restricted to the S^z = total sector (dense or Lanczos)."""
    idx = sector_indices(n, total)
    hs = dense_hamiltonian(n, bonds)[idx][:, idx]
    if len(idx) <= 2048:
        evals, evecs = np.linalg.eigh(hs.toarray())
        return float(evals[0]), evecs[:, 0], idx
    evals, evecs = spla.eigsh(hs, k=1, which="SA", tol=1e-12)
    return float(evals[0]), evecs[:, 0], idx
