"""Oracle: full-sector enumeration (exact energy, exact QGT by PAPER.md Eq. 2's first form).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

These are the independent routes used to pin the sample estimators:

* exact_energy: <psi|H|psi>/<psi|psi> with the dense Kronecker Hamiltonian
  (Eq. 1, left-hand form).
* exact_qgt_wavefunction: PAPER.md Eq. 2, first form,
      S_ij = <d_i psi|d_j psi>/<psi|psi> - <d_i psi|psi><psi|d_j psi>/<psi|psi>^2,
  with d_i psi obtained by central finite differences of the amplitude vector in
  theta_i (never through network.log_derivative_row).
"""
from __future__ import annotations

import numpy as np

from . import hamiltonian, network


def sector_configs(n, total=0):
    idx = hamiltonian.sector_indices(n, total)
    xs = np.array([[1 if (k >> i) & 1 else -1 for i in range(n)] for k in idx], dtype=np.int8)
    return idx, xs


def amplitudes(params, xs):
    return np.exp(network.log_psi(params, xs))


def born_weights(params, xs):
    lp = network.log_psi(params, xs)
    p = np.exp(2.0 * (lp.real - lp.real.max()))
    return p / p.sum()


def exact_energy(params, n, bonds, total=0):
    idx, xs = sector_configs(n, total)
    psi = amplitudes(params, xs)
    h = hamiltonian.dense_hamiltonian(n, bonds)[idx][:, idx]
    return np.vdot(psi, h @ psi) / np.vdot(psi, psi)


def exact_energy_theta(theta, like, n, bonds, total=0):
    return exact_energy(network.unflatten(theta, like), n, bonds, total)


def exact_qgt_wavefunction(params, n, total=0, h=1e-5):
    _, xs = sector_configs(n, total)
    theta = network.flatten(params)
    psi = amplitudes(params, xs)
    dpsi = np.empty((len(theta), len(xs)), dtype=np.complex128)
    for i in range(len(theta)):
        tp, tm = theta.copy(), theta.copy()
        tp[i] += h
        tm[i] -= h
        dpsi[i] = (amplitudes(network.unflatten(tp, params), xs)
                   - amplitudes(network.unflatten(tm, params), xs)) / (2 * h)
    nrm = np.vdot(psi, psi)
    overlap = dpsi.conj() @ psi                      # <d_i psi|psi>
    return (dpsi.conj() @ dpsi.T) / nrm - np.outer(overlap, overlap.conj()) / nrm ** 2
