"""Pins for oracle/network.py (stage 1: log psi and log-derivatives)."""
import numpy as np
import pytest

import workloads
from oracle import network


def test_lncosh_closed_forms():
    # cosh(0) = 1; cosh(i x) = cos x; cosh(x) real for real x
    assert network.lncosh(0.0 + 0.0j) == 0.0
    np.testing.assert_allclose(network.lncosh(1j * np.pi / 3), np.log(0.5), atol=1e-15)
    np.testing.assert_allclose(network.lncosh(0.7 + 0j), np.log((np.exp(0.7) + np.exp(-0.7)) / 2), rtol=1e-15)


def test_lncosh_small_argument_series_and_branch():
    # log cosh z = z^2/2 - z^4/12 + z^6/45 - ...: full relative accuracy for small z
    for z in (1e-8 + 3e-9j, 0.003 + 0.002j, -0.02 + 0.01j):
        series = z ** 2 / 2 - z ** 4 / 12 + z ** 6 / 45 - 17 * z ** 8 / 2520
        assert abs(network.lncosh(z) - series) <= 4e-16 * abs(series)
    # moderate z: agrees with the literal definition; principal branch (|Im| <= pi)
    rng = np.random.default_rng(1)
    z = rng.normal(0, 2, 50) + 1j * rng.normal(0, 2, 50)
    np.testing.assert_allclose(network.lncosh(z), np.log(np.cosh(z)), rtol=1e-12, atol=1e-14)
    assert np.all(np.abs(network.lncosh(z).imag) <= np.pi)
    # d lncosh / dz = tanh z (central difference), tanh accurate at small z
    h = 1e-6
    for z0 in (0.3 + 0.2j, -1.1 + 0.7j):
        fd = (network.lncosh(z0 + h) - network.lncosh(z0 - h)) / (2 * h)
        assert abs(fd - np.tanh(z0)) < 1e-9
    z = 0.003 + 0.002j
    assert abs(np.tanh(z) - (z - z ** 3 / 3 + 2 * z ** 5 / 15)) <= 4e-16 * abs(z)


def test_single_unit_closed_form():
    # ln psi = lncosh(w s + b): O_w = tanh(w s + b) s, O_b = tanh(w s + b)  (hand derivation)
    w, b = 0.3 + 0.1j, -0.2 + 0.05j
    params = [(np.array([[w]]), np.array([b]))]
    for s in (-1, 1):
        row = network.log_derivative_row(params, np.array([s]))
        t = np.tanh(w * s + b)
        np.testing.assert_allclose(row, [t * s, t], rtol=1e-15)
        lp = network.forward(params, np.array([s]))[0]
        np.testing.assert_allclose(lp, np.log(np.cosh(w * s + b)), rtol=1e-13)   # literal form: ~eps/|z|^2


@pytest.mark.parametrize("widths", [(10, 20, 20), (8, 6, 5, 4)])
def test_jacobian_matches_finite_differences(widths):
    params = workloads.draw_params(widths, seed=3, scale=1.0)   # larger weights: non-trivial curvature
    xs = workloads.draw_spins(widths[0], 4, seed=5)
    theta = network.flatten(params)
    h = 1e-6
    rng = np.random.default_rng(0)
    for x in xs:
        row = network.log_derivative_row(params, x)
        idx = rng.choice(len(theta), size=min(40, len(theta)), replace=False)
        for i in idx:
            tp, tm = theta.copy(), theta.copy()
            tp[i] += h
            tm[i] -= h
            fd = (network.forward(network.unflatten(tp, params), x)[0]
                  - network.forward(network.unflatten(tm, params), x)[0]) / (2 * h)
            assert abs(fd - row[i]) <= 1e-6 * (abs(row[i]) + 1e-12) + 1e-9
            # holomorphy: an imaginary step gives i * O_i (no conjugation anywhere)
            tp, tm = theta.copy(), theta.copy()
            tp[i] += 1j * h
            tm[i] -= 1j * h
            fdi = (network.forward(network.unflatten(tp, params), x)[0]
                   - network.forward(network.unflatten(tm, params), x)[0]) / (2 * h)
            assert abs(fdi - 1j * row[i]) <= 1e-6 * (abs(row[i]) + 1e-12) + 1e-9


def test_layer_blocks_partition_matches_baseline_counts():
    # BASELINE.json configs: n_p ~640, ~16k, ~67k, ~95k; blocks (W+b each)
    expected = [640, 16240, 67968, 95488, 196480]
    for w, n_p in zip(workloads.CONFIGS, expected):
        assert w.n_params == n_p
        assert len(w.layer_sizes) == w.n_layers
    params = workloads.draw_params((10, 20, 20), seed=0)
    off = network.layer_offsets(params)
    assert off == [0, 220, 640]
    row = network.log_derivative_row(params, workloads.draw_spins(10, 1, 0)[0])
    assert row.shape == (640,)
    # bias block of the last layer equals tanh(z_L) (sum pooling), by the chain rule
    _, hs, zs = network.forward(params, workloads.draw_spins(10, 1, 0)[0])
    np.testing.assert_allclose(row[620:640], np.tanh(zs[-1]), rtol=1e-14)
    # W block of layer l is the outer product of its bias block with h_{l-1}
    np.testing.assert_allclose(row[0:200].reshape(20, 10), np.outer(row[200:220], hs[0]), rtol=1e-14)


def test_flatten_roundtrip():
    params = workloads.draw_params((6, 4, 3), seed=1)
    back = network.unflatten(network.flatten(params), params)
    for (w, b), (w2, b2) in zip(params, back):
        assert np.array_equal(w, w2) and np.array_equal(b, b2)
