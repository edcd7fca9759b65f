"""Seeded synthetic workloads for the block-SR step (shared by oracle/ and the CUDA path).

This module is the ONLY code shared between ``oracle/`` and the product package.
It holds no arithmetic of the method (no network evaluation, no Hamiltonian, no
estimator): only the workload descriptions of BASELINE.json ``configs`` and the
seeded random draws those configurations specify.

Recipe (BASELINE.json ``configs``):

* spins: each sample is a uniformly random permutation of N/2 entries +1 and
  N/2 entries -1, i.e. a uniform draw from the zero-magnetisation sector
  (§2, "a configuration x in {-1,+1}^N"; §3 both models live at S^z=0);
  stored as int8, row-major [N_s, N].
* weights: complex128, real and imaginary parts i.i.d. N(0, sigma^2) with
  sigma = 0.1 / sqrt(fan_in) (BASELINE.json configs: "real and imaginary parts
  N(0, 0.1/sqrt(fan_in))", read as the standard deviation), one (W_l, b_l) pair per
  dense layer, W_l of shape [fan_out, fan_in].

Every draw uses numpy's PCG64 generator seeded with (seed, stream-id) so that the
spin stream and the weight stream are independent and reproducible.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

_STREAM_SPINS = 1
_STREAM_WEIGHTS = 2


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json configuration (lattice, network widths, N_s, lambda)."""

    name: str
    lattice: str                # "chain" or "square"
    extent: Tuple[int, ...]     # (L,) for the chain, (Lx, Ly) for the square lattice
    j1: float
    j2: float
    widths: Tuple[int, ...]     # (N, h_1, ..., h_L): dense layers N->h_1->...->h_L
    n_samples: int
    lam: float = 1e-3
    seed: int = 0
    note: str = ""

    @property
    def n_sites(self) -> int:
        n = 1
        for e in self.extent:
            n *= e
        return n

    @property
    def n_layers(self) -> int:
        return len(self.widths) - 1

    @property
    def layer_sizes(self) -> List[int]:
        """Complex parameter count of each layer block (W_l then b_l)."""
        return [self.widths[l + 1] * (self.widths[l] + 1) for l in range(self.n_layers)]

    @property
    def n_params(self) -> int:
        return sum(self.layer_sizes)

    def with_samples(self, n_samples: int) -> "Workload":
        return Workload(self.name, self.lattice, self.extent, self.j1, self.j2,
                        self.widths, n_samples, self.lam, self.seed, self.note)


# BASELINE.json "configs", in order.
CONFIGS: List[Workload] = [
    Workload("heis_chain_N10", "chain", (10,), 1.0, 0.0, (10, 20, 20), 512,
             note="configs[0]: 1D Heisenberg ring N=10, MLP 10->20->20, 2 blocks, n_p=640"),
    Workload("heis_chain_N40", "chain", (40,), 1.0, 0.0, (40, 80, 80, 80), 4096,
             note="configs[1]: 1D Heisenberg ring N=40, MLP 40->80->80->80, 3 blocks, n_p=16240"),
    Workload("j1j2_6x6", "square", (6, 6), 1.0, 0.5, (36, 144, 144, 144, 144), 16384,
             note="configs[2]: J1-J2 6x6, MLP 36->144x4, 4 blocks, n_p=67968"),
    Workload("j1j2_10x10_w128", "square", (10, 10), 1.0, 0.5, (100,) + (128,) * 6, 32768,
             note="configs[3]: J1-J2 10x10, MLP 100->128 + five 128->128, 6 blocks, n_p=95488"),
    Workload("j1j2_10x10_w160", "square", (10, 10), 1.0, 0.5, (100,) + (160,) * 8, 65536,
             note="configs[4]: J1-J2 10x10, MLP 100->160 + seven 160->160, 8 blocks, n_p=196480"),
]
BY_NAME = {w.name: w for w in CONFIGS}


def _rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([int(seed), int(stream)]))


def draw_spins(n_sites: int, n_samples: int, seed: int) -> np.ndarray:
    """Uniform zero-magnetisation configurations, int8 [n_samples, n_sites] of +-1."""
    if n_sites % 2:
        raise ValueError("zero-magnetisation sector needs an even number of sites")
    rng = _rng(seed, _STREAM_SPINS)
    # argsort of i.i.d. uniforms is a uniformly random permutation of each row;
    # sites holding the first N/2 ranks get +1, so every row has sum 0.
    ranks = np.argsort(rng.random((n_samples, n_sites)), axis=1)
    return np.where(ranks < n_sites // 2, 1, -1).astype(np.int8)


def draw_params(widths, seed: int, scale: float = 0.1) -> List[Tuple[np.ndarray, np.ndarray]]:
    """Complex weights [(W_l [fan_out, fan_in], b_l [fan_out])], re/im ~ N(0,(scale/sqrt(fan_in))^2)."""
    rng = _rng(seed, _STREAM_WEIGHTS)
    params = []
    for l in range(len(widths) - 1):
        fan_in, fan_out = int(widths[l]), int(widths[l + 1])
        sd = scale / np.sqrt(fan_in)
        w = rng.normal(0.0, sd, (fan_out, fan_in)) + 1j * rng.normal(0.0, sd, (fan_out, fan_in))
        b = rng.normal(0.0, sd, fan_out) + 1j * rng.normal(0.0, sd, fan_out)
        params.append((np.ascontiguousarray(w, dtype=np.complex128),
                       np.ascontiguousarray(b, dtype=np.complex128)))
    return params


def draw_complex(shape, seed: int, stream: int = 7) -> np.ndarray:
    """Generic complex128 standard-normal draw (test matrices, right-hand sides)."""
    rng = _rng(seed, stream)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def sector_states(n_sites: int) -> np.ndarray:
    """All zero-magnetisation configurations in ascending basis index (bit i set <=> s_i=+1).

    Used to feed the whole sector (with Born weights) through both sides for the
    exact-enumeration checks of configs[0]."""
    rows = []
    for idx in range(1 << n_sites):
        if bin(idx).count("1") == n_sites // 2:
            rows.append([1 if (idx >> i) & 1 else -1 for i in range(n_sites)])
    return np.asarray(rows, dtype=np.int8)


def make_inputs(w: Workload, n_samples: int | None = None):
    """(spins int8 [N_s, N], params list) for a workload, both seeded by w.seed."""
    ns = w.n_samples if n_samples is None else n_samples
    return draw_spins(w.n_sites, ns, w.seed), draw_params(w.widths, w.seed)
