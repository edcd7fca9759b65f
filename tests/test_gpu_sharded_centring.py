"""Sample-sharded stage (3) through the real kernels (sr_column_moments + sr_center_force_global
with n_parts > 1) on one GPU, against the oracle and the unsharded sr_center_force.

This is what parallel.ShardedStep runs on every rank (Eq. 2 centring over ALL
samples, north_star "samples shard naturally"): each shard writes its double-double moment
row, the rows of all shards are stacked (the all-gather), and each shard centres its own
rows against the summed moments and forms its partial force; the partial forces sum to F.
No collective is needed to check this: the shards are slices of one matrix on one GPU.

Tolerances as tests/test_gpu_parity.py: A and e_tilde 1e-11 (relative L2), F 1e-9, E 1e-13.
The ill-conditioned column (|<O>|/std ~ 1e9, readings R7/R11) checks that the
cross-shard sum keeps the low parts of the double-double moments: a mean rounded to double
would move that column of A by ~1e-7 relative.
"""
import numpy as np
import pytest
import torch

import workloads
from oracle import estimators, hamiltonian, network

pytestmark = pytest.mark.gpu

C128 = torch.complex128


@pytest.fixture(scope="module")
def sr():
    import paper_2510_08430_b200 as pkg
    pkg.load()
    return pkg


def dev():
    return torch.device("cuda:0")


def T(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev())


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _bounds(n, parts):
    from paper_2510_08430_b200.parallel import shard_range
    return [shard_range(n, r, parts) for r in range(parts)]


def sharded_center_force(sr, O, e, parts, weights=None):
    """Run the sharded stage (3) over `parts` row shards of O (in place) and return
    (energy, e_tilde, F) with F the sum of the partial forces."""
    ns, n_p = O.shape
    rows = torch.empty(parts, 2 * n_p + 2, dtype=C128, device=dev())
    bounds = _bounds(ns, parts)
    for r, (lo, hi) in enumerate(bounds):
        sr.sr_column_moments(O[lo:hi], e[lo:hi], ns, rows[r],
                             weights=None if weights is None else weights[lo:hi])
    et = torch.empty(ns, dtype=C128, device=dev())
    F = torch.zeros(n_p, dtype=C128, device=dev())
    energies = []
    for r, (lo, hi) in enumerate(bounds):
        Fp = torch.empty(n_p, dtype=C128, device=dev())
        en = torch.empty(1, dtype=C128, device=dev())
        sr.sr_center_force_global(O[lo:hi], e[lo:hi], ns, rows, et[lo:hi], Fp, energy=en,
                                  weights=None if weights is None else weights[lo:hi])
        F += Fp
        energies.append(en)
    torch.cuda.synchronize()
    # every shard computes the same global energy from the same rows
    assert all(torch.equal(x, energies[0]) for x in energies)
    return energies[0].item(), et, F


@pytest.mark.parametrize("parts", [2, 3])
@pytest.mark.parametrize("weighted", [False, True])
def test_sharded_centring_random_with_ill_conditioned_column(sr, parts, weighted):
    rng = np.random.default_rng(parts * 10 + weighted)
    ns, n_p = 1001, 77
    O = rng.standard_normal((ns, n_p)) + 1j * rng.standard_normal((ns, n_p))
    # |<O>|/std ~ 1e9 and ~1e12 (uniform weights: the oracle's mean is a double-double); the
    # weighted oracle accumulates in long double (64-bit mantissa), so there ~1e4 and ~1e6
    big = 1e4 if weighted else 1e9
    O[:, 5] = big * (1 + 2j) + O[:, 5]
    O[:, 6] = big + (1e-2 if weighted else 1e-3) * O[:, 6]
    e = rng.standard_normal(ns) + 1j * rng.standard_normal(ns) + 50.0
    w = None
    if weighted:
        w = rng.random(ns)
        w /= w.sum()
    Od = T(O)
    energy, et, F = sharded_center_force(sr, Od, T(e), parts, None if w is None else T(w))
    A_ref, e_ref = estimators.scaled_centered(O, e, w)
    F_ref = estimators.force(O, e, w)
    E_ref = estimators.energy(e, w)
    assert abs(energy - E_ref) <= 1e-13 * abs(E_ref)
    A = Od.cpu().numpy()
    assert rel(A, A_ref) < 1e-11
    for c in (5, 6):                                    # column by column where it cancels
        assert rel(A[:, c], A_ref[:, c]) < 1e-11, c
    assert rel(et.cpu().numpy(), e_ref) < 1e-11
    assert rel(F.cpu().numpy(), F_ref) < 1e-9
    # and the same as the unsharded kernel on the same data
    O2 = T(O)
    en1 = torch.empty(1, dtype=C128, device=dev())
    et1 = torch.empty(ns, dtype=C128, device=dev())
    F1 = torch.empty(n_p, dtype=C128, device=dev())
    sr.sr_center_force(O2, T(e), en1, et1, F1, weights=None if w is None else T(w))
    assert rel(A, O2.cpu().numpy()) < 1e-13
    assert rel(F.cpu().numpy(), F1.cpu().numpy()) < 1e-12


@pytest.mark.parametrize("cfg,parts", [(0, 2), (0, 3), (1, 2), (1, 3)])
def test_sharded_centring_network_configs(sr, cfg, parts):
    """configs[0] / configs[1]: the GPU's own O and E_loc (stages 1-2), split into 2 or 3 row
    shards, against the oracle's centring of the same O and E_loc."""
    w = workloads.CONFIGS[cfg]
    spins, params = workloads.make_inputs(w)
    ns = w.n_samples
    theta = T(sr.model.pack(params))
    lp = torch.empty(ns, dtype=C128, device=dev())
    O = torch.empty(ns, w.n_params, dtype=C128, device=dev())
    sr.sr_jacobian(w.widths, theta, T(spins), lp, O)
    ij, jj = sr.lattice.for_workload(w)
    e = torch.empty(ns, dtype=C128, device=dev())
    sr.sr_local_energy(w.widths, theta, T(ij), T(jj), T(spins), lp, e)
    O_h, e_h = O.cpu().numpy(), e.cpu().numpy()
    if cfg == 0:   # stages 1-2 themselves against the oracle (small enough here)
        assert rel(O_h, network.jacobian(params, spins)) < 1e-11
        assert rel(e_h, hamiltonian.local_energies(params, spins, hamiltonian.bonds_for(w))) < 1e-10
    energy, et, F = sharded_center_force(sr, O, e, parts)
    A_ref, e_ref = estimators.scaled_centered(O_h, e_h)
    assert abs(energy - estimators.energy(e_h)) <= 1e-13 * abs(estimators.energy(e_h))
    A = O.cpu().numpy()
    assert rel(A, A_ref) < 1e-11
    # per layer block too (the deep blocks are the badly conditioned ones)
    offs = sr.block_offsets(w.widths)
    for b in range(len(offs) - 1):
        assert rel(A[:, offs[b]:offs[b + 1]], A_ref[:, offs[b]:offs[b + 1]]) < 1e-11, b
    assert rel(et.cpu().numpy(), e_ref) < 1e-11
    assert rel(F.cpu().numpy(), estimators.force(O_h, e_h)) < 1e-9


def test_sharded_centring_single_sample_shards(sr):
    """Ragged extreme: 3 samples over 3 shards (one row each)."""
    rng = np.random.default_rng(9)
    ns, n_p = 3, 40
    O = rng.standard_normal((ns, n_p)) + 1j * rng.standard_normal((ns, n_p))
    e = rng.standard_normal(ns) + 1j * rng.standard_normal(ns)
    Od = T(O)
    energy, et, F = sharded_center_force(sr, Od, T(e), 3)
    A_ref, e_ref = estimators.scaled_centered(O, e)
    assert rel(Od.cpu().numpy(), A_ref) < 1e-11
    assert rel(et.cpu().numpy(), e_ref) < 1e-11
    assert rel(F.cpu().numpy(), estimators.force(O, e)) < 1e-9
