"""Pins for oracle/solvers.py (stage 5 and the full-QGT / NTK comparison paths)."""
import numpy as np
import pytest

from oracle import estimators, solvers


def _rand(shape, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def test_two_by_two_hand_solution():
    # S = diag(2, 0), F = (2, 1), lambda = 0.1: dtheta = -(2/2.1, 1/0.1)
    S = np.diag([2.0, 0.0]).astype(complex)
    d = solvers.full_solve(S, np.array([2.0, 1.0 + 0j]), 0.1)
    np.testing.assert_allclose(d, [-2 / 2.1, -10.0], rtol=1e-15)
    # two 1x1 blocks of a 2x2 block-diagonal metric give the same answer
    d2 = solvers.block_solve([S[:1, :1], S[1:, 1:]], np.array([2.0, 1.0 + 0j]), [0, 1, 2], 0.1)
    np.testing.assert_allclose(d2, d, rtol=1e-15)


@pytest.mark.parametrize("ns,np_", [(40, 12), (12, 40)])
def test_push_through_identity(ns, np_):
    # (A^H A + lam)^{-1} A^H e = A^H (A A^H + lam)^{-1} e
    A = _rand((ns, np_), 1) / np.sqrt(ns)
    e = _rand(ns, 2) / np.sqrt(ns)
    for lam in (1e-3, 1e-1):
        full = solvers.full_solve(A.conj().T @ A, A.conj().T @ e, lam)
        ntk = solvers.ntk_solve(A, e, lam)
        assert np.linalg.norm(full - ntk) / np.linalg.norm(full) < 1e-10


def test_block_solve_equals_full_when_off_blocks_zero():
    O = _rand((64, 17), 3)
    e = _rand(64, 4)
    off = [0, 5, 12, 17]
    blocks = estimators.qgt_blocks(O, off)
    F = estimators.force(O, e)
    S = np.zeros((17, 17), complex)
    for l, B in enumerate(blocks):
        S[off[l]:off[l + 1], off[l]:off[l + 1]] = B
    a = solvers.block_solve(blocks, F, off, 1e-3)
    b = solvers.full_solve(S, F, 1e-3)
    assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-12
    # single-layer partition: block solve is the full solve
    c = solvers.block_solve([estimators.qgt_full(O)], F, [0, 17], 1e-3)
    d = solvers.full_solve(estimators.qgt_full(O), F, 1e-3)
    assert np.linalg.norm(c - d) / np.linalg.norm(d) < 1e-14


def test_residual_and_large_shift_limit():
    O = _rand((30, 20), 7)
    e = _rand(30, 8)
    S, F = estimators.qgt_full(O), estimators.force(O, e)
    d = solvers.full_solve(S, F, 1e-3)
    assert np.linalg.norm((S + 1e-3 * np.eye(20)) @ d + F) / np.linalg.norm(F) < 1e-11
    big = 1e9
    np.testing.assert_allclose(solvers.full_solve(S, F, big), -F / big, rtol=1e-6)
