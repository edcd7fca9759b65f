"""Pins for oracle/hamiltonian.py (stage 2: local energies, ED)."""
import os

import numpy as np
import pytest

import workloads
from oracle import hamiltonian, network

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    vals = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                k, v = line.split()
                vals[k] = float(v)
    return vals


def test_bond_counts():
    assert len(hamiltonian.chain_bonds(10)) == 10
    assert len(hamiltonian.chain_bonds(2)) == 1          # the two periodic bonds coincide
    b = hamiltonian.square_bonds(6, 6, 1.0, 0.5)
    assert sum(1 for *_, J in b if J == 1.0) == 72 and sum(1 for *_, J in b if J == 0.5) == 72
    assert len(hamiltonian.square_bonds(10, 10, 1.0, 0.5)) == 400
    for i, j, _ in b:
        assert i != j


def test_connected_neel_and_ferro():
    # Pauli units: Neel state on the L=4 ring, every bond anti-aligned:
    # diagonal = 4 * (-1), four flips of amplitude 2 (S-units: -1 and 1/2, SPEC example x4)
    bonds = hamiltonian.chain_bonds(4)
    c = hamiltonian.connected(np.array([1, -1, 1, -1]), bonds)
    assert c[0][1] == -4.0 and len(c) == 5 and all(a == 2.0 for _, a in c[1:])
    c = hamiltonian.connected(np.array([1, 1, 1, 1]), bonds)
    assert len(c) == 1 and c[0][1] == 4.0


def test_local_energy_constant_state_closed_form():
    # psi = const: every bond contributes s_i s_j + (1 - s_i s_j) = 1  =>  E_loc = #bonds
    bonds = hamiltonian.square_bonds(4, 4, 1.0, 0.5)
    for x in workloads.draw_spins(16, 5, seed=2):
        e = hamiltonian.local_energy_fn(lambda c: 0.0, x, bonds)
        np.testing.assert_allclose(e, sum(J for *_, J in bonds), rtol=1e-15)


@pytest.mark.parametrize("geom", [("chain", 8), ("square", (4, 2)), ("square", (4, 4))])
def test_local_energy_equals_dense_H_ratio(geom):
    # E_loc(x) = (H psi)(x) / psi(x) with H built from Pauli Kronecker products
    if geom[0] == "chain":
        n, bonds = geom[1], hamiltonian.chain_bonds(geom[1])
    else:
        (lx, ly) = geom[1]
        n, bonds = lx * ly, hamiltonian.square_bonds(lx, ly, 1.0, 0.5)
    rng = np.random.default_rng(11)
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    hpsi = hamiltonian.dense_hamiltonian(n, bonds) @ psi
    log_amp = lambda c: np.log(psi[hamiltonian.basis_index(c)])
    for x in workloads.draw_spins(n, 6, seed=4):
        k = hamiltonian.basis_index(x)
        e = hamiltonian.local_energy_fn(log_amp, x, bonds)
        np.testing.assert_allclose(e, hpsi[k] / psi[k], rtol=1e-12)


def test_mlp_local_energies_equal_dense_ratio():
    n = 10
    params = workloads.draw_params((10, 20, 20), seed=0, scale=1.0)
    bonds = hamiltonian.chain_bonds(n)
    allx = np.array([[1 if (k >> i) & 1 else -1 for i in range(n)] for k in range(1 << n)])
    psi = np.exp(network.log_psi(params, allx))
    hpsi = hamiltonian.dense_hamiltonian(n, bonds) @ psi
    xs = workloads.draw_spins(n, 8, seed=9)
    e = hamiltonian.local_energies(params, xs, bonds)
    ks = [hamiltonian.basis_index(x) for x in xs]
    np.testing.assert_allclose(e, hpsi[ks] / psi[ks], rtol=1e-12)


def test_ed_small_closed_forms():
    # singlet: sigma.sigma = -3 ; L=4 ring: 4 * (-2) = -8 (S-units E0 = -2J)
    assert abs(hamiltonian.ground_state(2, hamiltonian.chain_bonds(2))[0] + 3.0) < 1e-12
    assert abs(hamiltonian.ground_state(4, hamiltonian.chain_bonds(4))[0] + 8.0) < 1e-10


def test_zero_variance_at_ground_state():
    n = 8
    bonds = hamiltonian.square_bonds(4, 2, 1.0, 0.5)
    e0, vec, idx = hamiltonian.ground_state(n, bonds)
    table = {int(k): v for k, v in zip(idx, vec)}
    log_amp = lambda c: np.log(table[hamiltonian.basis_index(c)] + 0j)
    for x in workloads.draw_spins(n, 10, seed=1):
        if abs(table[hamiltonian.basis_index(x)]) < 1e-8:
            continue
        e = hamiltonian.local_energy_fn(log_amp, x, bonds)
        assert abs(e - e0) < 1e-9


def test_table2_heisenberg_L16_ground_state():
    g = _golden("table2_heisenberg_L16.txt")
    e0, _, _ = hamiltonian.ground_state(16, hamiltonian.chain_bonds(16))
    # variational bound: both Table 2 energies lie above E0 (within their error bars)
    assert e0 <= g["energy_block_layer"] + g["energy_block_layer_err"]
    assert e0 <= g["energy_full_qgt"] + g["energy_full_qgt_err"]
    # and only slightly above (infidelity 1.6e-5): relative gap below 1e-4
    assert (g["energy_block_layer"] - e0) / abs(e0) < 1e-4
