"""Oracle: complex lncosh MLP wavefunction and its log-derivatives (stage 1).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Network (BASELINE.json configs: "complex128 MLP N->h_1->...->h_L with lncosh
activations, sum-pooled to ln psi"; §2 "the neural network ... takes as
input a configuration x in {-1,+1}^N and outputs a complex amplitude psi_theta(x)"):

    h_0 = x,   z_l = W_l h_{l-1} + b_l,   h_l = lncosh(z_l)   (l = 1..L)
    ln psi(x) = sum_j h_L[j]

lncosh(z) = log(cosh z) on the principal branch of the complex logarithm
(reading R2), evaluated through the identity cosh z = 1 + 2 sinh^2(z/2) as
log1p(2 sinh^2(z/2)) so that small activations (h ~ z^2/2, the regime of the BASELINE.json
initialisation) keep full relative accuracy; log(cosh z) taken literally loses
~eps/|z|^2 of it (2e-12 relative at |z| = 0.004).

Log-derivatives (§2 Eq. 2: "O_i(x) = d_{theta_i} log psi_theta(x)").  The
network is holomorphic in its complex parameters, so O_i is the complex
derivative.  Layer blocks (§2 Eq. 3: "O_l is the Jacobian of the
log-wavefunction with respect to layer parameters theta_l"): block l holds
W_l (row-major, index j*fan_in + i) followed by b_l (index fan_out*fan_in + j);
blocks are concatenated in layer order.  Chain rule, written out:

    delta_L = tanh(z_L)                         (d ln psi / d z_L; d lncosh/dz = tanh)
    O[W_l][j, i] = delta_l[j] * h_{l-1}[i],     O[b_l][j] = delta_l[j]
    delta_{l-1} = tanh(z_{l-1}) * (W_l^T delta_l)
"""
from __future__ import annotations

import numpy as np


def log1p_complex(w):
    """Principal log(1 + w): log|1 + w| = log1p(2 Re w + |w|^2)/2, arg(1 + w) = atan2(Im w, 1 + Re w)."""
    w = np.asarray(w, dtype=np.complex128)
    return 0.5 * np.log1p(2.0 * w.real + np.abs(w) ** 2) + 1j * np.arctan2(w.imag, 1.0 + w.real)


def lncosh(z):
    """Principal-branch log(cosh z) = log(1 + 2 sinh^2(z/2))."""
    s = np.sinh(np.asarray(z, dtype=np.complex128) / 2.0)
    return log1p_complex(2.0 * s * s)


def forward(params, x):
    """Return (ln psi(x), [h_0..h_L], [z_1..z_L]) for one configuration x."""
    h = np.asarray(x, dtype=np.complex128)
    hs, zs = [h], []
    for w, b in params:
        z = w @ h + b
        h = lncosh(z)
        zs.append(z)
        hs.append(h)
    return h.sum(), hs, zs


def log_psi(params, xs):
    """ln psi for every row of xs (one forward pass per configuration)."""
    return np.array([forward(params, x)[0] for x in np.asarray(xs)], dtype=np.complex128)


def layer_sizes(params):
    return [w.shape[0] * (w.shape[1] + 1) for w, _ in params]


def layer_offsets(params):
    sizes = layer_sizes(params)
    return list(np.concatenate([[0], np.cumsum(sizes)]).astype(int))


def log_derivative_row(params, x):
    """O(x): complex row of length n_p, blocks in layer order (W_l then b_l)."""
    _, hs, zs = forward(params, x)
    n_layers = len(params)
    blocks = [None] * n_layers
    g = np.ones_like(zs[-1])                      # d ln psi / d h_L (sum pooling)
    for l in reversed(range(n_layers)):
        delta = g * np.tanh(zs[l])                # d ln psi / d z_l
        blocks[l] = np.concatenate([np.outer(delta, hs[l]).ravel(), delta])
        g = params[l][0].T @ delta                # d ln psi / d h_{l-1} (no conjugation)
    return np.concatenate(blocks)


def jacobian(params, xs):
    """O matrix [N_s, n_p]: row k is O(x_k)."""
    return np.stack([log_derivative_row(params, x) for x in np.asarray(xs)])


def flatten(params):
    """theta as one complex vector in the O column order."""
    return np.concatenate([np.concatenate([w.ravel(), b]) for w, b in params])


def unflatten(theta, like):
    """Inverse of flatten, shapes taken from ``like``."""
    out, pos = [], 0
    for w, b in like:
        nw = w.size
        out.append((theta[pos:pos + nw].reshape(w.shape).copy(),
                    theta[pos + nw:pos + nw + b.size].copy()))
        pos += nw + b.size
    return out
