"""Host-side set-up of the product path against the oracle's independent versions."""
import numpy as np

import workloads
from oracle import hamiltonian, network


def test_lattice_bonds_match_oracle():
    import paper_2510_08430_b200 as sr
    for w in workloads.CONFIGS:
        ij, jj = sr.lattice.for_workload(w)
        mine = {(min(i, j), max(i, j), J) for (i, j), J in zip(ij.tolist(), jj.tolist())}
        ref = {(min(i, j), max(i, j), J) for i, j, J in hamiltonian.bonds_for(w)}
        assert mine == ref and len(ij) == len(ref)
    ij, jj = sr.lattice.bond_arrays(sr.lattice.chain(4), spin_units=True)
    assert np.all(jj == 0.25)


def test_parameter_packing_matches_oracle_order():
    import paper_2510_08430_b200 as sr
    params = workloads.draw_params((10, 20, 20), seed=4)
    assert np.array_equal(sr.model.pack(params), network.flatten(params))
    assert sr.model.widths_of(params) == [10, 20, 20]
    assert sr.block_offsets([10, 20, 20]) == network.layer_offsets(params)
    assert sr.n_params([100] + [128] * 6) == 95488


def test_shard_ranges_and_owners():
    from paper_2510_08430_b200.parallel import block_owner, shard_range
    for n in (1, 7, 4096, 65536):
        for g in (1, 2, 3, 8):
            rs = [shard_range(n, r, g) for r in range(g)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(g - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
    assert [block_owner(b, 8) for b in range(8)] == list(range(8))    # configs[4]: one block per GPU
    from paper_2510_08430_b200.parallel import block_ranges
    sizes4 = [16160] + [25760] * 7
    assert block_ranges(sizes4, 8) == [(b, b + 1) for b in range(8)]
    assert [block_owner(b, 8, sizes4) for b in range(8)] == list(range(8))
    for sizes in ([3280, 6480, 6480], [5328] + [20880] * 3, [12928] + [16512] * 5, [640], sizes4):
        for g in (1, 2, 3, 4, 8):
            rs = block_ranges(sizes, g)
            assert len(rs) == g and rs[0][0] == 0 and rs[-1][1] == len(sizes)
            assert all(rs[i][1] == rs[i + 1][0] for i in range(g - 1))          # contiguous cover
            owned = [hi - lo for lo, hi in rs]
            assert all(o >= 1 for o in owned[:min(g, len(sizes))])             # a block per rank while they last
    assert block_ranges([3280, 6480, 6480], 2) == [(0, 2), (2, 3)]


def test_workload_inputs_are_seeded_and_in_sector():
    s1 = workloads.draw_spins(36, 100, 3)
    s2 = workloads.draw_spins(36, 100, 3)
    assert np.array_equal(s1, s2)
    assert np.all(s1.sum(axis=1) == 0) and set(np.unique(s1)) == {-1, 1}
    p = workloads.draw_params((100, 128), 0)
    sd = 0.1 / np.sqrt(100)
    assert abs(p[0][0].real.std() / sd - 1) < 0.05 and abs(p[0][0].imag.std() / sd - 1) < 0.05


def test_bench_reference_arm_json_contract():
    """bench.py --impl reference (the CPU-oracle arm of this tier) prints one JSON line with
    the keys the driver reads, on the same config as the native arm."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "impl", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["config"]["workload"] == "j1j2_10x10_w128"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1


def test_bench_workload_scaling():
    """bench.py measures configs[3] by default (the largest single-GPU configuration, strong
    scaling over N) and configs[4] with 8192 samples per GPU (weak scaling)."""
    import bench
    assert bench.DEFAULT_WORKLOAD == workloads.CONFIGS[3].name
    for n in (1, 2, 4, 8):
        assert bench.workload_for("j1j2_10x10_w160", n).n_samples == 8192 * n
        assert bench.workload_for("j1j2_10x10_w128", n).n_samples == 32768
    c = bench.config_of(bench.workload_for("j1j2_10x10_w160", 8), 8, "int8", True, "sharded")
    assert c["samples_per_gpu"] == 8192 and c["n_samples"] == 65536 and c["scaling"].startswith("weak")


def test_lncosh_series_constants_and_accuracy():
    """The small-argument lncosh / tanh series of the CUDA kernels (csrc/common.cuh): the
    constants are the Bernoulli-number coefficients c_n = 2^{2n}(2^{2n}-1) B_{2n}/(2n (2n)!)
    (lncosh z = z^2/2 - z^4/12 + ..., tanh z = z - z^3/3 + ...), and 11 terms in float64 are
    within 5e-16 relative of 40-digit log cosh / tanh on |z| <= 1/4."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import lncosh_series as ls
    from fractions import Fraction
    c, t = ls.coefficients()
    assert c[0] == Fraction(1, 2) and c[1] == Fraction(-1, 12) and c[2] == Fraction(1, 45)
    assert t[0] == 1 and t[1] == Fraction(-1, 3) and t[2] == Fraction(2, 15)
    h = ls.header_constants()
    assert h["c"] == [float(x) for x in c] and h["t"] == [float(x) for x in t]
    el, et = ls.max_rel_errors(n=800)
    assert el < 5e-16 and et < 5e-16


def test_bench_config_chunked_and_full_samples():
    """bench.config_of for the sample-chunked configs[4] run (all 65536 samples on one GPU):
    not labelled weak scaling, the resident O is one chunk."""
    import bench
    w = workloads.BY_NAME["j1j2_10x10_w160"]
    c = bench.config_of(w, 1, "int8", False, "chunked", 8192)
    assert c["n_samples"] == 65536 and c["scaling"].startswith("strong")
    assert "25.75 GB resident" in c["l2"] and "206 GB over the chunks" in c["l2"]
    c1 = bench.config_of(bench.workload_for("j1j2_10x10_w160", 1), 1, "int8", False, "per_block")
    assert c1["scaling"].startswith("weak") and c1["n_samples"] == 8192
