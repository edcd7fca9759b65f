"""Pins for oracle/estimators.py and oracle/exact.py (stages 3-4)."""
import numpy as np
import pytest

import workloads
from oracle import estimators, exact, hamiltonian, network

N = 10
SMALL = (10, 6, 4)        # small net so the finite-difference routes stay fast


@pytest.fixture(scope="module")
def sector_batch():
    params = workloads.draw_params(SMALL, seed=21, scale=2.0)
    _, xs = exact.sector_configs(N)
    O = network.jacobian(params, xs)
    w = exact.born_weights(params, xs)
    bonds = hamiltonian.chain_bonds(N)
    e_loc = hamiltonian.local_energies(params, xs, bonds)
    return params, xs, O, w, bonds, e_loc


def test_qgt_covariance_equals_wavefunction_form(sector_batch):
    # PAPER.md Eq. 2: the covariance estimator with exact Born weights over the whole
    # sector equals the <d psi|d psi> form computed from finite-difference amplitudes.
    params, xs, O, w, _, _ = sector_batch
    s_cov = estimators.qgt_full(O, w)
    s_wf = exact.exact_qgt_wavefunction(params, N)
    assert np.linalg.norm(s_cov - s_wf) / np.linalg.norm(s_wf) < 1e-7


def test_energy_equals_dense_expectation(sector_batch):
    params, xs, O, w, bonds, e_loc = sector_batch
    e = estimators.energy(e_loc, w)
    np.testing.assert_allclose(e, exact.exact_energy(params, N, bonds), rtol=1e-12)
    # variational principle against exact diagonalisation
    assert e.real >= hamiltonian.ground_state(N, bonds)[0] - 1e-10


def test_force_equals_energy_gradient(sector_batch):
    # F_i = dE/d conj(theta_i) = (dE/da + i dE/db)/2 for theta = a + i b (holomorphic psi)
    params, xs, O, w, bonds, e_loc = sector_batch
    F = estimators.force(O, e_loc, w)
    theta = network.flatten(params)
    h = 1e-6
    rng = np.random.default_rng(3)
    for i in rng.choice(len(theta), 12, replace=False):
        def e_at(d):
            t = theta.copy()
            t[i] += d
            return exact.exact_energy_theta(t, params, N, bonds).real
        dre = (e_at(h) - e_at(-h)) / (2 * h)
        dim = (e_at(1j * h) - e_at(-1j * h)) / (2 * h)
        g = 0.5 * (dre + 1j * dim)
        assert abs(F[i] - g) <= 1e-6 * max(abs(g), 1e-3)


def test_blocks_are_diagonal_subblocks_and_psd(sector_batch):
    params, xs, O, w, _, _ = sector_batch
    off = network.layer_offsets(params)
    full = estimators.qgt_full(O, w)
    blocks = estimators.qgt_blocks(O, off, w)
    for l, S in enumerate(blocks):
        sub = full[off[l]:off[l + 1], off[l]:off[l + 1]]
        assert np.max(np.abs(S - sub)) <= 1e-14 * np.max(np.abs(sub))
        assert np.max(np.abs(S - S.conj().T)) <= 1e-15 * np.max(np.abs(S))
        ev = np.linalg.eigvalsh(S)
        assert ev.min() >= -1e-12 * ev.max()


def test_centering_and_two_sample_closed_form():
    O = np.array([[1.0 + 2j, 3.0], [-1.0, 1j]])
    ob = estimators.center(O)
    np.testing.assert_allclose(ob.sum(axis=0), 0, atol=1e-15)
    S = estimators.qgt_full(O)
    # two uniform samples: Obar = +-(a - b)/2, so S = conj(d) d^T / 4 with d = O_0 - O_1
    d = O[0] - O[1]
    np.testing.assert_allclose(S, np.outer(d.conj(), d) / 4, rtol=1e-15)
    # a constant column has a zero row/column in S
    O2 = np.column_stack([O, np.full(2, 5 - 1j)])
    assert np.all(estimators.qgt_full(O2)[2] == 0)


def test_ntk_shares_nonzero_spectrum_with_qgt():
    rng = np.random.default_rng(5)
    O = rng.standard_normal((12, 30)) + 1j * rng.standard_normal((12, 30))
    s = np.sort(np.linalg.eigvalsh(estimators.qgt_full(O)))[::-1][:11]
    t = np.sort(np.linalg.eigvalsh(estimators.ntk(O)))[::-1][:11]
    np.testing.assert_allclose(s, t, rtol=1e-9)
    # Ns = 1: a single sample centres to zero
    assert np.all(estimators.ntk(O[:1]) == 0)


def test_scaled_centered_factorisation():
    rng = np.random.default_rng(6)
    O = rng.standard_normal((20, 7)) + 1j * rng.standard_normal((20, 7))
    e = rng.standard_normal(20) + 1j * rng.standard_normal(20)
    w = rng.random(20)
    w /= w.sum()
    A, ev = estimators.scaled_centered(O, e, w)
    np.testing.assert_allclose(A.conj().T @ A, estimators.qgt_full(O, w), rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(A.conj().T @ ev, estimators.force(O, e, w), rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(A @ A.conj().T, estimators.ntk(O, w), rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("scale,n", [(1e-7, 33), (1e-9, 4096), (1e-12, 500)])
def test_centering_is_exact_to_double_rounding_under_cancellation(scale, n):
    # columns nearly constant over samples (as the deep-layer derivatives are: |<O>|/std up
    # to ~1e9 at configs[3], ~1e12 here): the centred values must equal the exactly computed
    # (rational-arithmetic) ones up to one double rounding (R7, R11), where a
    # double-rounded mean would give errors of ~1e-4 relative and a 64-bit long-double
    # mean still ~1e-7
    from fractions import Fraction
    rng = np.random.default_rng(8)
    base = 0.731 - 0.25j
    O = base + scale * (rng.standard_normal((n, 2)) + 1j * rng.standard_normal((n, 2)))
    ob = estimators.center(O)
    for c in range(2):
        for part in ("real", "imag"):
            col = [Fraction(float(getattr(v, part))) for v in O[:, c]]
            mean = sum(col) / len(col)
            exact = np.array([float(v - mean) for v in col])
            got = getattr(ob[:, c], part)
            assert np.all(np.abs(got - exact) <= 2.0 ** -52 * np.abs(exact))
    # the mean itself, and the energy path, to double rounding as well
    m = estimators.mean_O(O)
    for c in range(2):
        exact = sum(Fraction(float(v.real)) for v in O[:, c]) / n
        assert abs(m[c].real - float(exact)) <= 2.0 ** -52 * abs(float(exact))
