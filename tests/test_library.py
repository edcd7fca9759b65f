"""CPU checks of the C ABI boundary: libsrblock.so builds, loads, exports every symbol
include/sr_block.h declares, and the binding covers exactly those symbols.  No compute
call is made (there is no GPU here); only the pure-host queries run."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sr_block.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"SR_API\s+[\w\s\*]+?\b(sr_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    import paper_2510_08430_b200 as sr
    return sr.load()


def test_header_declares_the_north_star_entry_points():
    names = declared_symbols()
    for n in ("sr_jacobian", "sr_local_energy", "sr_block_qgt", "sr_block_solve", "sr_full_qgt_solve",
              "sr_ntk_solve", "sr_center_force", "sr_step", "sr_step_host"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_binding_covers_the_header():
    from paper_2510_08430_b200 import _lib
    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_library_is_sm100a_only():
    import paper_2510_08430_b200 as sr
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump -lelf {sr.LIB_PATH}").read()
    assert "sm_100a" in out and "sm_90" not in out


def test_host_queries(lib):
    import paper_2510_08430_b200 as sr
    assert lib.sr_version() == 100
    w = [40, 80, 80, 80]
    small = sr.sr_step_workspace_bytes(w, 512, 40)
    big = sr.sr_step_workspace_bytes(w, 4096, 40)
    assert 0 < small < big
    # O alone is N_s * n_p complex numbers
    assert big >= 4096 * 16240 * 16
    L, wa = sr._lib._widths(w)
    assert lib.sr_jacobian_workspace_bytes(L, wa, 4096) > 0
    assert lib.sr_block_solve_workspace_bytes(3, sr._lib._offsets(sr.block_offsets(w))) > 0
    # invalid widths are rejected by the queries (0 bytes) without touching a device
    bad, wb = sr._lib._widths([40, 300])
    assert lib.sr_jacobian_workspace_bytes(bad, wb, 10) == 0


def test_invalid_arguments_fail_before_any_device_work(lib):
    import paper_2510_08430_b200 as sr
    L, wa = sr._lib._widths([4, 300])
    rc = lib.sr_jacobian(L, wa, None, None, 1, None, None, 10, None, 0, None)
    assert rc == -1 and b"width" in lib.sr_last_error()
    rc = lib.sr_block_solve(0, None, None, None, 1e-3, None, None, None, 0, None)
    assert rc == -1


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    from paper_2510_08430_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(_lib.SRError):
        _lib.load(build_if_missing=False)


def test_int8_engine_host_side(lib):
    """Engine switch and the int8 Gram's workspace query / argument checks (no device work)."""
    import paper_2510_08430_b200 as sr
    assert lib.sr_get_gram_engine() == sr.GRAM_INT8           # library default
    assert lib.sr_set_gram_engine(7) == -1                    # unknown engine: unchanged
    assert lib.sr_get_gram_engine() == sr.GRAM_INT8
    assert lib.sr_set_gram_engine(sr.GRAM_FP64) == sr.GRAM_INT8
    assert lib.sr_set_gram_engine(sr.GRAM_INT8) == sr.GRAM_FP64
    offs = sr._lib._offsets([0, 3280, 9760, 16240])
    ws = lib.sr_block_qgt_i8_workspace_bytes(4096, 3, offs)
    # 7 digit slices x (Re A, Im A, -Re A) x N_s bytes per parameter, plus column exponents
    assert ws >= 21 * 4096 * 16240
    assert lib.sr_block_qgt_i8_workspace_bytes(8192, 3, offs) > ws
    assert lib.sr_block_qgt_i8_workspace_bytes(-1, 3, offs) == 0
    bad = sr._lib._offsets([0, 10, 5])
    assert lib.sr_block_qgt_i8_workspace_bytes(16, 2, bad) == 0
    rc = lib.sr_block_qgt_i8(16, 2, bad, None, 10, None, None, 0, None)
    assert rc == -1 and b"block_offsets" in lib.sr_last_error()
    rc = lib.sr_block_qgt_i8(16, 3, offs, None, 16240, None, None, 0, None)
    assert rc == -1 and b"null" in lib.sr_last_error()
    rc = lib.sr_block_qgt_i8(16, 3, offs, None, 100, None, None, 0, None)   # lda < n_p
    assert rc == -1


def test_kernel_timer_without_launches(lib):
    import paper_2510_08430_b200 as sr
    sr.sr_kernel_timer(True)
    sr.sr_kernel_timer(False)
    assert sr.sr_kernel_time_ms("gram_i8") == (0.0, 0)


def test_per_block_schedule_workspace(lib):
    """SR_SCHED_PER_BLOCK (sr_set_step_schedule): the step workspace holds one block's factor
    instead of every S_b and its factor copy -- configs[4] at 8192 samples fits one B200."""
    import paper_2510_08430_b200 as sr
    import workloads
    w = workloads.CONFIGS[4]
    ns, nb = 8192, 200
    prev = sr.sr_set_step_schedule(sr.SCHED_PER_BLOCK)
    try:
        assert sr.sr_get_step_schedule() == sr.SCHED_PER_BLOCK
        per_block = sr.sr_step_workspace_bytes(w.widths, ns, nb)
        assert sr.sr_step_s_offset(w.widths, ns, nb) == 2 ** 64 - 1
    finally:
        sr.sr_set_step_schedule(prev)
    batched = sr.sr_step_workspace_bytes(w.widths, ns, nb)
    O = ns * w.n_params * 16
    n_max = max(w.layer_sizes)
    assert per_block < O + 2 * 16 * (n_max + 64) ** 2 + 21 * ns * n_max + (8 << 30)
    assert per_block < 60e9 < 150e9 < batched
    offs = sr._lib._offsets(sr.block_offsets(w.widths))
    assert lib.sr_block_qgt_solve_workspace_bytes(ns, len(w.layer_sizes), offs) >= 16 * n_max ** 2
    assert lib.sr_set_step_schedule(7) == -1 and sr.sr_get_step_schedule() == prev
