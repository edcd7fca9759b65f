"""ctypes binding of libsrblock.so (include/sr_block.h): argument marshalling only.

Every function here has the name of the C entry point it wraps, takes torch tensors
(device memory owned by the caller) and plain Python numbers, checks dtype/device/
shape, allocates the workspace the matching *_workspace_bytes() query asks for when
none is given, and calls the C function on the current CUDA stream.  No arithmetic of
the method happens in Python; there is no CPU fallback: if the library cannot be
loaded, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from . import build as _build

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsrblock.so")
# measurement tools only (tools/gram_energy.py): load a variant build of the same library
_LIB_OVERRIDE = os.environ.get("SR_LIB_VARIANT")

_vp, _i64, _i32, _sz, _dbl = C.c_void_p, C.c_int64, C.c_int, C.c_size_t, C.c_double
_I32P = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)

# name -> (restype, argtypes); mirrors include/sr_block.h
SIGNATURES = {
    "sr_version": (_i32, []),
    "sr_last_error": (C.c_char_p, []),
    "sr_launch_count": (_i64, []),
    "sr_reset_launch_count": (None, []),
    "sr_kernel_timer": (None, [_i32]),
    "sr_kernel_time_ms": (_dbl, [C.c_char_p, _I64P]),
    "sr_kernel_timeline": (C.c_size_t, [C.c_char_p, C.c_size_t]),
    "sr_trace_buffer": (_i32, [C.c_void_p, _i64]),
    "sr_gram_nh": (_i32, [_i64, _i64, _i64, C.c_void_p, _i64, C.c_void_p, _i64, C.c_void_p, _i64, C.c_void_p]),
    "sr_aHv_workspace_bytes": (_sz, [_i64, _i64]),
    "sr_aHv": (_i32, [_i64, _i64, C.c_void_p, _i64, C.c_void_p, _dbl, C.c_void_p, C.c_void_p, _sz, C.c_void_p]),
    "sr_av": (_i32, [_i64, _i64, _vp, _i64, _vp, _dbl, _vp, _vp]),
    "sr_zdotc_workspace_bytes": (_sz, []),
    "sr_zdotc": (_i32, [_i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "sr_cg_axpy": (_i32, [_i64, _vp, _vp, _vp, _vp, _dbl, _vp]),
    "sr_cg_xpby": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp]),
    "sr_gram_tn": (_i32, [_i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp]),
    "sr_gram_nh_sub": (_i32, [_i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp]),
    "sr_cols_i8_workspace_bytes": (_sz, [_i64, _i64]),
    "sr_cols_i8_prepare": (_i32, [_i64, _i64, _vp, _i64, _vp, _sz, _vp]),
    "sr_cols_i8_gram": (_i32, [_i64, _i64, _i64, _i64, _i64, _vp, _i64, _i32, _vp, _sz, _vp]),
    "sr_rows_i8_sub_workspace_bytes": (_sz, [_i64, _i64]),
    "sr_rows_i8_prepare": (_i32, [_i64, _i64, _vp, _i64, _vp, _sz, _vp]),
    "sr_rows_i8_sub": (_i32, [_i64, _i64, _i64, _i64, _i64, _vp, _i64, _vp, _sz, _vp]),
    "sr_chol_inv_workspace_bytes": (_sz, [_i64]),
    "sr_chol_inv": (_i32, [_i64, _vp, _dbl, _vp, _i64, _vp, _i64, _vp, _vp, _sz, _vp]),
    "sr_graph_capture_begin": (_i32, [C.c_void_p]),
    "sr_graph_capture_end": (_i32, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "sr_graph_launch": (_i32, [C.c_void_p, C.c_void_p]),
    "sr_graph_destroy": (_i32, [C.c_void_p]),
    "sr_jacobian_workspace_bytes": (_sz, [_i32, _I32P, _i64]),
    "sr_jacobian": (_i32, [_i32, _I32P, _vp, _vp, _i64, _vp, _vp, _i64, _vp, _sz, _vp]),
    "sr_local_energy_workspace_bytes": (_sz, [_i32, _I32P, _i64, _i64]),
    "sr_local_energy": (_i32, [_i32, _I32P, _vp, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "sr_center_force_workspace_bytes": (_sz, [_i64, _i64]),
    "sr_center_force": (_i32, [_i64, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "sr_column_moments_workspace_bytes": (_sz, [_i64, _i64]),
    "sr_column_moments": (_i32, [_i64, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "sr_center_force_global": (_i32, [_i64, _i64, _i64, _vp, _i64, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _sz,
                                      _vp]),
    "sr_block_qgt_workspace_bytes": (_sz, [_i32, _I64P]),
    "sr_block_qgt": (_i32, [_i64, _i32, _I64P, _vp, _i64, _vp, _vp, _sz, _vp]),
    "sr_block_qgt_i8_workspace_bytes": (_sz, [_i64, _i32, _I64P]),
    "sr_block_qgt_i8": (_i32, [_i64, _i32, _I64P, _vp, _i64, _vp, _vp, _sz, _vp]),
    "sr_block_qgt_i8_acc": (_i32, [_i64, _i32, _I64P, _vp, _i64, _vp, _vp, _sz, _vp]),
    "sr_set_gram_engine": (_i32, [_i32]),
    "sr_get_gram_engine": (_i32, []),
    "sr_block_solve_workspace_bytes": (_sz, [_i32, _I64P]),
    "sr_block_solve": (_i32, [_i32, _I64P, _vp, _vp, _dbl, _vp, _vp, _vp, _sz, _vp]),
    "sr_block_qgt_solve_workspace_bytes": (_sz, [_i64, _i32, _I64P]),
    "sr_block_qgt_solve": (_i32, [_i64, _i32, _I64P, _vp, _i64, _vp, _dbl, _vp, _vp, _vp, _sz, _vp]),
    "sr_set_step_schedule": (_i32, [_i32]),
    "sr_get_step_schedule": (_i32, []),
    "sr_full_qgt_solve_workspace_bytes": (_sz, [_i64, _i64]),
    "sr_full_qgt_solve": (_i32, [_i64, _i64, _vp, _i64, _vp, _dbl, _vp, _vp, _vp, _vp, _sz, _vp]),
    "sr_ntk_solve_workspace_bytes": (_sz, [_i64, _i64]),
    "sr_ntk_solve": (_i32, [_i64, _i64, _vp, _i64, _vp, _dbl, _vp, _vp, _vp, _vp, _sz, _vp]),
    "sr_step_workspace_bytes": (_sz, [_i32, _I32P, _i64, _i64]),
    "sr_step_s_offset": (_sz, [_i32, _I32P, _i64, _i64]),
    "sr_step": (_i32, [_i32, _I32P, _vp, _vp, _i64, _i64, _vp, _vp, _dbl, _vp, _vp, _vp, _sz, _vp]),
    "sr_step_host_extra_bytes": (_sz, [_i32, _I32P, _i64, _i64]),
    "sr_step_host": (_i32, [_i32, _I32P, _vp, _vp, _i64, _i64, _vp, _vp, _dbl, _vp, _vp, _vp, _sz, _vp]),
}


class SRError(RuntimeError):
    pass


_lib = None


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load libsrblock.so (building it in-tree with nvcc if it is missing or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    if _LIB_OVERRIDE:
        lib = C.CDLL(_LIB_OVERRIDE)
    else:
        if build_if_missing and not _build.up_to_date():
            _build.build()
        if not os.path.exists(LIB_PATH):
            raise SRError(f"{LIB_PATH} is missing; run python -m paper_2510_08430_b200.build")
        lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(status: int, name: str):
    if status != 0:
        msg = load().sr_last_error().decode()
        raise SRError(f"{name} failed with status {status}: {msg}")


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dev(t, dtype, name):
    if t is None:
        return
    if not t.is_cuda:
        raise SRError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise SRError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise SRError(f"{name} must be contiguous")


def _widths(widths):
    arr = (C.c_int32 * len(widths))(*[int(w) for w in widths])
    return len(widths) - 1, arr


def _offsets(offs):
    return (C.c_int64 * len(offs))(*[int(o) for o in offs])


def _stream(device=None):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _workspace(nbytes, device, workspace):
    if workspace is not None:
        if workspace.numel() * workspace.element_size() < nbytes:
            raise SRError("workspace too small")
        return workspace
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def _ws_args(ws):
    return C.c_void_p(ws.data_ptr()), C.c_size_t(ws.numel() * ws.element_size())


def n_params(widths):
    return sum(int(widths[l + 1]) * (int(widths[l]) + 1) for l in range(len(widths) - 1))


def block_offsets(widths):
    offs = [0]
    for l in range(len(widths) - 1):
        offs.append(offs[-1] + int(widths[l + 1]) * (int(widths[l]) + 1))
    return offs


# ------------------------------------------------------------------ stage (1)
def sr_jacobian(widths, theta, spins, log_psi, O, workspace=None):
    lib = load()
    L, w = _widths(widths)
    ns = spins.shape[0]
    _dev(theta, torch.complex128, "theta")
    _dev(spins, torch.int8, "spins")
    _dev(log_psi, torch.complex128, "log_psi")
    _dev(O, torch.complex128, "O")
    ws = _workspace(lib.sr_jacobian_workspace_bytes(L, w, ns), spins.device, workspace)
    _check(lib.sr_jacobian(L, w, _ptr(theta), _ptr(spins), ns, _ptr(log_psi), _ptr(O), O.shape[1],
                           *_ws_args(ws), _stream(spins.device)), "sr_jacobian")


# ------------------------------------------------------------------ stage (2)
def sr_local_energy(widths, theta, bonds_ij, bond_j, spins, log_psi, e_loc, workspace=None):
    lib = load()
    L, w = _widths(widths)
    ns, nb = spins.shape[0], bonds_ij.shape[0]
    _dev(bonds_ij, torch.int32, "bonds_ij")
    _dev(bond_j, torch.float64, "bond_j")
    _dev(e_loc, torch.complex128, "e_loc")
    ws = _workspace(lib.sr_local_energy_workspace_bytes(L, w, ns, nb), spins.device, workspace)
    _check(lib.sr_local_energy(L, w, _ptr(theta), nb, _ptr(bonds_ij), _ptr(bond_j), _ptr(spins), ns,
                               _ptr(log_psi), _ptr(e_loc), *_ws_args(ws), _stream(spins.device)),
           "sr_local_energy")


# ------------------------------------------------------------------ stage (3)
def sr_center_force(O, e_loc, energy, e_tilde, F, weights=None, workspace=None):
    lib = load()
    ns, npar = O.shape[0], F.shape[0]
    _dev(O, torch.complex128, "O")
    _dev(weights, torch.float64, "weights")
    ws = _workspace(lib.sr_center_force_workspace_bytes(ns, npar), O.device, workspace)
    _check(lib.sr_center_force(ns, npar, _ptr(O), O.shape[1], _ptr(weights), _ptr(e_loc), _ptr(energy),
                               _ptr(e_tilde), _ptr(F), *_ws_args(ws), _stream(O.device)), "sr_center_force")


def sr_column_moments(O, e_loc, n_total, moments, weights=None, workspace=None):
    """moments: complex [2*n_p + 2] (one row, see include/sr_block.h)."""
    lib = load()
    ns = O.shape[0]
    npar = (moments.shape[-1] - 2) // 2
    ws = _workspace(lib.sr_column_moments_workspace_bytes(ns, npar), O.device, workspace)
    _check(lib.sr_column_moments(ns, n_total, npar, _ptr(O), O.shape[1], _ptr(weights), _ptr(e_loc),
                                 _ptr(moments), *_ws_args(ws), _stream(O.device)), "sr_column_moments")


def sr_center_force_global(O, e_loc, n_total, moments, e_tilde, F_partial, energy=None, weights=None,
                           workspace=None):
    """moments: complex [n_parts, 2*n_p + 2] (all ranks' rows)."""
    lib = load()
    ns, npar = O.shape[0], F_partial.shape[0]
    rows = moments.reshape(-1, 2 * npar + 2)
    ws = _workspace(lib.sr_column_moments_workspace_bytes(ns, npar), O.device, workspace)
    _check(lib.sr_center_force_global(ns, n_total, npar, _ptr(O), O.shape[1], _ptr(weights), _ptr(e_loc),
                                      rows.shape[0], _ptr(rows), _ptr(energy), _ptr(e_tilde), _ptr(F_partial),
                                      *_ws_args(ws), _stream(O.device)), "sr_center_force_global")


# ------------------------------------------------------------------ stage (4)
def _cols(A, name):
    """A CUDA complex128 matrix whose rows are contiguous (a column slice of a wider matrix
    is allowed): returns its leading dimension."""
    if not A.is_cuda or A.dtype != torch.complex128 or A.dim() != 2 or (A.shape[1] > 1 and A.stride(1) != 1):
        raise SRError(f"{name} must be a CUDA complex128 matrix with unit column stride")
    return A.stride(0) if A.shape[0] > 1 else A.shape[1]


def sr_block_qgt(A, offsets, S):
    """Stage (4) on the FP64 DMMA engine.  A may be a column slice (leading dimension = A.stride(0))."""
    lib = load()
    lda = _cols(A, "A")
    _dev(S, torch.complex128, "S")
    nblk = len(offsets) - 1
    need = sum((offsets[b + 1] - offsets[b]) ** 2 for b in range(nblk))
    if S.numel() < need:
        raise SRError("S too small for the packed blocks")
    _check(lib.sr_block_qgt(A.shape[0], nblk, _offsets(offsets), _ptr(A), lda, _ptr(S), None, 0,
                            _stream(A.device)), "sr_block_qgt")


def sr_block_qgt_i8(A, offsets, S, workspace=None):
    """Stage (4) on the int8 tcgen05 tensor cores (digit slices; include/sr_block.h).  A may be
    a column slice (leading dimension = A.stride(0))."""
    lib = load()
    lda = _cols(A, "A")
    _dev(S, torch.complex128, "S")
    nblk = len(offsets) - 1
    need = sum((offsets[b + 1] - offsets[b]) ** 2 for b in range(nblk))
    if S.numel() < need:
        raise SRError("S too small for the packed blocks")
    off = _offsets(offsets)
    ws = _workspace(lib.sr_block_qgt_i8_workspace_bytes(A.shape[0], nblk, off), A.device, workspace)
    _check(lib.sr_block_qgt_i8(A.shape[0], nblk, off, _ptr(A), lda, _ptr(S), *_ws_args(ws),
                               _stream(A.device)), "sr_block_qgt_i8")


def sr_block_qgt_i8_acc(A, offsets, S, workspace=None):
    """S += A_b^H A_b per block (int8 engine; the sample-chunked step)."""
    lib = load()
    lda = _cols(A, "A")
    _dev(S, torch.complex128, "S")
    nblk = len(offsets) - 1
    need = sum((offsets[b + 1] - offsets[b]) ** 2 for b in range(nblk))
    if S.numel() < need:
        raise SRError("S too small for the packed blocks")
    off = _offsets(offsets)
    ws = _workspace(lib.sr_block_qgt_i8_workspace_bytes(A.shape[0], nblk, off), A.device, workspace)
    _check(lib.sr_block_qgt_i8_acc(A.shape[0], nblk, off, _ptr(A), lda, _ptr(S), *_ws_args(ws), _stream(A.device)),
           "sr_block_qgt_i8_acc")


GRAM_FP64, GRAM_INT8 = 0, 1


def sr_set_gram_engine(engine):
    """Engine of sr_step's stage (4): GRAM_FP64 (DMMA) or GRAM_INT8 (tcgen05 digit slices)."""
    prev = int(load().sr_set_gram_engine(int(engine)))
    if prev < 0:
        raise SRError(f"unknown gram engine {engine}")
    return prev


def sr_get_gram_engine():
    return int(load().sr_get_gram_engine())


# ------------------------------------------------------------------ stage (5)
def sr_block_solve(offsets, S, F, lam, dtheta, info=None, workspace=None):
    lib = load()
    nblk = len(offsets) - 1
    off = _offsets(offsets)
    ws = _workspace(lib.sr_block_solve_workspace_bytes(nblk, off), S.device, workspace)
    _check(lib.sr_block_solve(nblk, off, _ptr(S), _ptr(F), float(lam), _ptr(dtheta), _ptr(info),
                              *_ws_args(ws), _stream(S.device)), "sr_block_solve")


def sr_block_qgt_solve(A, offsets, F, lam, dtheta, info=None, workspace=None):
    """Stages (4)+(5) one block at a time (include/sr_block.h): A may be a column slice."""
    lib = load()
    lda = _cols(A, "A")
    nblk = len(offsets) - 1
    off = _offsets(offsets)
    for t, n in ((F, "F"), (dtheta, "dtheta")):
        _dev(t, torch.complex128, n)
        if t.numel() < offsets[-1]:
            raise SRError(f"{n} shorter than n_p")
    ws = _workspace(lib.sr_block_qgt_solve_workspace_bytes(A.shape[0], nblk, off), A.device, workspace)
    _check(lib.sr_block_qgt_solve(A.shape[0], nblk, off, _ptr(A), lda, _ptr(F), float(lam), _ptr(dtheta), _ptr(info),
                                  *_ws_args(ws), _stream(A.device)), "sr_block_qgt_solve")


SCHED_BATCHED, SCHED_PER_BLOCK = 0, 1


def sr_set_step_schedule(schedule):
    """Schedule of sr_step's stages (4)-(5): SCHED_BATCHED or SCHED_PER_BLOCK."""
    prev = int(load().sr_set_step_schedule(int(schedule)))
    if prev < 0:
        raise SRError(f"unknown step schedule {schedule}")
    return prev


def sr_get_step_schedule():
    return int(load().sr_get_step_schedule())


def sr_full_qgt_solve(A, F, lam, dtheta, S_out=None, info=None, workspace=None):
    lib = load()
    ns, npar = A.shape[0], F.shape[0]
    lda = _cols(A, "A")
    ws = _workspace(lib.sr_full_qgt_solve_workspace_bytes(ns, npar), A.device, workspace)
    _check(lib.sr_full_qgt_solve(ns, npar, _ptr(A), lda, _ptr(F), float(lam), _ptr(dtheta),
                                 _ptr(S_out), _ptr(info), *_ws_args(ws), _stream(A.device)),
           "sr_full_qgt_solve")


def sr_ntk_solve(A, e_tilde, lam, dtheta, T_out=None, info=None, workspace=None):
    lib = load()
    ns, npar = A.shape[0], dtheta.shape[0]
    ws = _workspace(lib.sr_ntk_solve_workspace_bytes(ns, npar), A.device, workspace)
    _check(lib.sr_ntk_solve(ns, npar, _ptr(A), A.shape[1], _ptr(e_tilde), float(lam), _ptr(dtheta),
                            _ptr(T_out), _ptr(info), *_ws_args(ws), _stream(A.device)), "sr_ntk_solve")


def sr_gram_nh(A, B, C_out):
    """C_out = A B^H (rows of A against rows of B; A, B may be row slices / column slices)."""
    lda, ldb = _cols(A, "A"), _cols(B, "B")
    ldc = _cols(C_out, "C")
    if A.shape[1] != B.shape[1] or C_out.shape[0] != A.shape[0] or C_out.shape[1] != B.shape[0]:
        raise SRError("sr_gram_nh: shape mismatch")
    _check(load().sr_gram_nh(A.shape[0], B.shape[0], A.shape[1], _ptr(A), lda, _ptr(B), ldb, _ptr(C_out), ldc,
                             _stream(A.device)), "sr_gram_nh")


def sr_aHv(A, v, alpha, out, workspace=None):
    """out = alpha A^H v."""
    lib = load()
    lda = _cols(A, "A")
    _dev(v, torch.complex128, "v")
    _dev(out, torch.complex128, "out")
    ws = _workspace(lib.sr_aHv_workspace_bytes(A.shape[0], A.shape[1]), A.device, workspace)
    _check(lib.sr_aHv(A.shape[0], A.shape[1], _ptr(A), lda, _ptr(v), float(alpha), _ptr(out), *_ws_args(ws),
                      _stream(A.device)), "sr_aHv")


def sr_gram_tn(A, B, C_out):
    """C_out = A^H B (A: k x m, B: k x n; column slices allowed)."""
    lda, ldb, ldc = _cols(A, "A"), _cols(B, "B"), _cols(C_out, "C")
    if A.shape[0] != B.shape[0] or C_out.shape[0] != A.shape[1] or C_out.shape[1] != B.shape[1]:
        raise SRError("sr_gram_tn: shape mismatch")
    _check(load().sr_gram_tn(A.shape[1], B.shape[1], A.shape[0], _ptr(A), lda, _ptr(B), ldb, _ptr(C_out), ldc,
                             _stream(A.device)), "sr_gram_tn")


def sr_gram_nh_sub(A, B, C_out):
    """C_out -= A B^H (rows of A against rows of B; slices allowed)."""
    lda, ldb, ldc = _cols(A, "A"), _cols(B, "B"), _cols(C_out, "C")
    if A.shape[1] != B.shape[1] or C_out.shape[0] != A.shape[0] or C_out.shape[1] != B.shape[0]:
        raise SRError("sr_gram_nh_sub: shape mismatch")
    _check(load().sr_gram_nh_sub(A.shape[0], B.shape[0], A.shape[1], _ptr(A), lda, _ptr(B), ldb, _ptr(C_out), ldc,
                                 _stream(A.device)), "sr_gram_nh_sub")


class ColSlices:
    """Digit slices of all columns of A on the int8 engine (sr_cols_i8_prepare), for
    rectangles of its Gram: C (+)= A[:, row0:row0+m]^H A[:, 0:n] (sr_cols_i8_gram)."""

    def __init__(self, A):
        lib = load()
        self.ns, self.ncols = A.shape
        lda = _cols(A, "A")
        self.ws = _workspace(lib.sr_cols_i8_workspace_bytes(self.ns, self.ncols), A.device, None)
        self.dev = A.device
        _check(lib.sr_cols_i8_prepare(self.ns, self.ncols, _ptr(A), lda, *_ws_args(self.ws), _stream(A.device)),
               "sr_cols_i8_prepare")

    def gram(self, row0, C_out, accumulate=False):
        m, n = C_out.shape
        _check(load().sr_cols_i8_gram(self.ns, self.ncols, int(row0), m, n, _ptr(C_out), _cols(C_out, "C"),
                                      1 if accumulate else 0, *_ws_args(self.ws), _stream(self.dev)), "sr_cols_i8_gram")


class RowSlices:
    """Digit slices of the rows of L (rows x K <= 8192, sr_rows_i8_prepare), for rectangular
    trailing updates C -= L[row0:row0+m] L[0:n]^H (sr_rows_i8_sub)."""

    def __init__(self, L, workspace=None):
        lib = load()
        self.rows, self.K = L.shape
        ldl = _cols(L, "L")
        self.ws = _workspace(lib.sr_rows_i8_sub_workspace_bytes(self.rows, self.K), L.device, workspace)
        self.dev = L.device
        _check(lib.sr_rows_i8_prepare(self.rows, self.K, _ptr(L), ldl, *_ws_args(self.ws), _stream(L.device)),
               "sr_rows_i8_prepare")

    def sub(self, row0, C_out):
        m, n = C_out.shape
        _check(load().sr_rows_i8_sub(self.rows, self.K, int(row0), m, n, _ptr(C_out), _cols(C_out, "C"),
                                     *_ws_args(self.ws), _stream(self.dev)), "sr_rows_i8_sub")


def sr_chol_inv(M, lam, L_out, Linv_out, info=None, workspace=None):
    """M + lam I = L L^H (M contiguous n x n, lower triangle read); L_out, Linv_out = L, L^{-1}."""
    lib = load()
    n = M.shape[0]
    _dev(M, torch.complex128, "M")
    ws = _workspace(lib.sr_chol_inv_workspace_bytes(n), M.device, workspace)
    _check(lib.sr_chol_inv(n, _ptr(M), float(lam), _ptr(L_out), _cols(L_out, "L"), _ptr(Linv_out),
                           _cols(Linv_out, "Linv"), _ptr(info), *_ws_args(ws), _stream(M.device)), "sr_chol_inv")


def sr_av(A, v, alpha, out):
    """out = alpha A v (A may be a column slice)."""
    lda = _cols(A, "A")
    for t, n in ((v, "v"), (out, "out")):
        _dev(t, torch.complex128, n)
    _check(load().sr_av(A.shape[0], A.shape[1], _ptr(A), lda, _ptr(v), float(alpha), _ptr(out), _stream(A.device)),
           "sr_av")


def sr_zdotc(x, y, out, workspace=None):
    """out[0] = sum conj(x) y (device complex scalar)."""
    lib = load()
    ws = _workspace(lib.sr_zdotc_workspace_bytes(), x.device, workspace)
    _check(lib.sr_zdotc(x.numel(), _ptr(x), _ptr(y), _ptr(out), *_ws_args(ws), _stream(x.device)), "sr_zdotc")


def sr_cg_axpy(x, y, num, den, sign):
    """y += sign (num / den) x  (num, den: device complex scalars)."""
    _check(load().sr_cg_axpy(x.numel(), _ptr(x), _ptr(y), _ptr(num), _ptr(den), float(sign), _stream(x.device)),
           "sr_cg_axpy")


def sr_cg_xpby(x, y, num, den):
    """y = x + (num / den) y."""
    _check(load().sr_cg_xpby(x.numel(), _ptr(x), _ptr(y), _ptr(num), _ptr(den), _stream(x.device)), "sr_cg_xpby")


# ------------------------------------------------------------------ full step
def sr_step_workspace_bytes(widths, n_samples, n_bonds):
    L, w = _widths(widths)
    return int(load().sr_step_workspace_bytes(L, w, n_samples, n_bonds))


def sr_step_s_offset(widths, n_samples, n_bonds):
    L, w = _widths(widths)
    return int(load().sr_step_s_offset(L, w, n_samples, n_bonds))


def sr_step_host_extra_bytes(widths, n_samples, n_bonds):
    L, w = _widths(widths)
    return int(load().sr_step_host_extra_bytes(L, w, n_samples, n_bonds))


def sr_step(widths, theta, spins, bonds_ij, bond_j, lam, dtheta, energy, workspace):
    lib = load()
    L, w = _widths(widths)
    _check(lib.sr_step(L, w, _ptr(theta), _ptr(spins), spins.shape[0], bonds_ij.shape[0], _ptr(bonds_ij),
                       _ptr(bond_j), float(lam), _ptr(dtheta), _ptr(energy), *_ws_args(workspace),
                       _stream(workspace.device)), "sr_step")


def sr_step_host(widths, theta_h, spins_h, bonds_ij_h, bond_j_h, lam, dtheta_h, energy_h, workspace):
    """Host tensors in/out (pinned for async copies); synchronises the stream."""
    lib = load()
    L, w = _widths(widths)
    for t, n in ((theta_h, "theta_h"), (spins_h, "spins_h"), (dtheta_h, "dtheta_h")):
        if t.is_cuda or not t.is_contiguous():
            raise SRError(f"{n} must be a contiguous host tensor")
    _check(lib.sr_step_host(L, w, _ptr(theta_h), _ptr(spins_h), spins_h.shape[0], bonds_ij_h.shape[0],
                            _ptr(bonds_ij_h), _ptr(bond_j_h), float(lam), _ptr(dtheta_h), _ptr(energy_h),
                            *_ws_args(workspace), _stream(workspace.device)), "sr_step_host")


def sr_launch_count():
    return int(load().sr_launch_count())


def sr_reset_launch_count():
    load().sr_reset_launch_count()


def sr_kernel_timer(enable):
    load().sr_kernel_timer(1 if enable else 0)


class Graph:
    """A CUDA graph captured through the library (sr_graph_capture_begin/end): per-node
    priorities are kept at instantiation, unlike torch.cuda.CUDAGraph.  Usage:
        g = Graph(device); with g.capture(): <library calls on torch's current stream>
        g.replay()"""

    def __init__(self, device):
        self.device = torch.device(device)
        self.stream = torch.cuda.Stream(self.device)
        self.exec = None

    def capture(self):
        import contextlib

        @contextlib.contextmanager
        def _cap():
            lib = load()
            self.stream.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(self.stream):
                _check(lib.sr_graph_capture_begin(C.c_void_p(self.stream.cuda_stream)), "sr_graph_capture_begin")
                try:
                    yield self
                finally:
                    h = C.c_void_p()
                    _check(lib.sr_graph_capture_end(C.c_void_p(self.stream.cuda_stream), C.byref(h)),
                           "sr_graph_capture_end")
                    self.exec = h
            torch.cuda.current_stream(self.device).wait_stream(self.stream)
        return _cap()

    def replay(self):
        _check(load().sr_graph_launch(self.exec, _stream(self.device)), "sr_graph_launch")

    def __del__(self):
        try:
            if self.exec is not None and _lib is not None:
                _lib.sr_graph_destroy(self.exec)
        except Exception:
            pass


TRACE_KINDS = {1: "diag", 2: "trsm", 3: "skinny_sub", 4: "gram", 5: "trail", 6: "rhs", 7: "back", 8: "back_rest",
               9: "split_rows", 10: "init", 11: "split", 12: "colmax", 13: "output"}


def sr_trace_buffer(records):
    """Install (a zeroed uint8 CUDA tensor of 40-byte records) or remove (None) the device trace."""
    if records is None:
        _check(load().sr_trace_buffer(None, 0), "sr_trace_buffer")
    else:
        _check(load().sr_trace_buffer(_ptr(records), records.numel() // 40), "sr_trace_buffer")


def sr_trace_records(records):
    """Decode a trace buffer: list of (gridid, kind name, tag, sm, t0_ns, t1_ns)."""
    import numpy as np
    raw = records.cpu().numpy().view(np.uint8)
    n = int(raw[:8].view(np.uint64)[0])
    dt = np.dtype([("grid", "<u8"), ("t0", "<u8"), ("t1", "<u8"), ("kind", "<i4"), ("tag", "<i4"), ("sm", "<i4"),
                   ("pad", "<i4")])
    rec = raw[40:40 * (1 + min(n, raw.size // 40 - 1))].view(dt)
    return [(int(r["grid"]), TRACE_KINDS.get(int(r["kind"]), str(r["kind"])), int(r["tag"]), int(r["sm"]),
             int(r["t0"]), int(r["t1"])) for r in rec]


def sr_kernel_timeline():
    """Pending kernel-timer records as (name, stream_index, begin_ms, end_ms) tuples."""
    lib = load()
    n = lib.sr_kernel_timeline(None, 0)
    buf = C.create_string_buffer(n)
    lib.sr_kernel_timeline(buf, n)
    out = []
    for line in buf.value.decode().splitlines():
        name, sid, a, b = line.split()
        out.append((name, int(sid), float(a), float(b)))
    return out


def sr_kernel_time_ms(kernel):
    """(summed ms, launches) of `kernel` since the last read (see include/sr_block.h)."""
    n = C.c_int64(0)
    ms = load().sr_kernel_time_ms(kernel.encode(), C.byref(n))
    return float(ms), int(n.value)
