"""ctypes binding of libslq_b200.so (C ABI in include/slq_b200.h).

There is no fallback: if the library is missing or no CUDA device is present,
every compute entry point raises ``SlqLibraryError``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import SlqLibraryError, TridiagonalEigenError

LIB_PATH = os.environ.get("SLQ_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libslq_b200.so")

SLQ_OK, SLQ_ERR_VALUE, SLQ_ERR_EIGEN, SLQ_ERR_CUDA, SLQ_ERR_NONFINITE, SLQ_ERR_ALLOC = range(6)
LAPLACIAN, NORMALIZED_LAPLACIAN, DENSITY = 0, 1, 2
F64, F32 = 0, 1
FN_HEAT, FN_WAVE_RE, FN_WAVE_IM, FN_XLOGX, FN_IDENTITY = range(5)

# kernel classes as counted by the library (cgs_step = the persistent per-step CGS kernel, or the
# separate update kernels on the fallback path)
KERNEL_CLASSES = ("prepare", "probe", "spmm", "cgs_dot", "cgs_step", "reduce", "eig", "quad",
                  "estimate", "batched")

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_u64 = ctypes.c_uint64
_dbl = ctypes.c_double
_int = ctypes.c_int


class GraphInfo(ctypes.Structure):
    _fields_ = [("n", _i64), ("nnz", _i64), ("trace_l", _dbl), ("max_degree", _dbl),
                ("isolated", _i64), ("unit_weights", _i32), ("ntiles", _i32)]


class Seed(ctypes.Structure):
    """slq_seed: the seed's little-endian uint32 entropy words (numpy SeedSequence, slq.py:63-72)."""
    _fields_ = [("words", ctypes.c_uint32 * 8), ("nwords", ctypes.c_int32)]


def seed_arg(seed) -> "ctypes._Pointer":
    """ctypes pointer to the slq_seed of a non-negative integer seed (< 2^256), split into uint32
    words exactly as numpy's SeedSequence does; negative seeds raise ValueError like numpy."""
    s = int(seed)
    if s < 0:
        raise ValueError("expected non-negative integer")
    words = []
    while True:
        words.append(s & 0xFFFFFFFF)
        s >>= 32
        if not s:
            break
    if len(words) > 8:
        raise ValueError("seeds of more than 256 bits are not supported by the device probe stream")
    out = Seed()
    for i, w in enumerate(words):
        out.words[i] = w
    out.nwords = len(words)
    return ctypes.pointer(out)


_SP = ctypes.POINTER(Seed)

_SIGS = {
    "slq_graph_create": (_int, [_i64, _i64, _vp, _vp, _vp, _vp, ctypes.POINTER(_vp)]),
    "slq_graph_create_host": (_int, [_i64, _i64, _vp, _vp, _vp, _vp, ctypes.POINTER(_vp)]),
    "slq_graph_create_i32": (_int, [_i64, _i64, _vp, _vp, _vp, _vp, ctypes.POINTER(_vp)]),
    "slq_graph_create_rmat": (_int, [_int, _int, _dbl, _dbl, _dbl, _u64, _vp, ctypes.POINTER(_vp)]),
    "slq_rmat_uniform_host": (_int, [_u64, _u64, _int, ctypes.POINTER(_dbl)]),
    "slq_graph_csr": (_int, [_vp, _vp, _vp, _vp]),
    "slq_graph_create_edges": (_int, [_i64, _i64, _vp, _vp, _vp, _vp, ctypes.POINTER(_vp)]),
    "slq_graph_weights": (_int, [_vp, _vp, ctypes.POINTER(_i32), _vp]),
    "slq_trace_squared": (_int, [_vp, _int, ctypes.POINTER(_dbl)]),
    "slq_graph_info": (_int, [_vp, ctypes.POINTER(GraphInfo)]),
    "slq_graph_fold_isolated": (_int, [_vp, _dbl, ctypes.POINTER(_i64)]),
    "slq_graph_destroy": (None, [_vp]),
    "slq_graph_degrees": (_int, [_vp, _vp, _vp]),
    "slq_operator_interval": (_int, [_vp, _int, ctypes.POINTER(_dbl), ctypes.POINTER(_dbl)]),
    "slq_operator_apply": (_int, [_vp, _int, _vp, _vp, _i64, _i64, _vp]),
    "slq_lanczos": (_int, [_vp, _int, _u64, _i64, _i64, _int, _int, _int, _vp, _vp, _vp, _vp]),
    "slq_lanczos_start": (_int, [_vp, _int, _vp, _i64, _i64, _int, _int, _int, _vp, _vp, _vp, _vp]),
    "slq_lanczos_basis": (_int, [_vp, _int, _u64, _i64, _i64, _int, _int, _int, _vp, _vp, _vp, _vp, _vp]),
    "slq_lanczos_start_basis": (_int, [_vp, _int, _vp, _i64, _i64, _int, _int, _int, _vp, _vp, _vp, _vp, _vp]),
    "slq_gauss_rules": (_int, [_vp, _vp, _vp, _i64, _int, _dbl, _dbl, _vp, _vp, _vp, _vp]),
    "slq_quadrature": (_int, [_vp, _vp, _vp, _i64, _int, _vp, _i64, _int, _vp, _vp]),
    "slq_estimate": (_int, [_vp, _i64, _i64, _dbl, _vp, _vp, _vp]),
    "slq_probes": (_int, [_u64, _i64, _i64, _i64, _vp, _i64, _vp]),
    "slq_probe_state": (_int, [_u64, _u64, ctypes.POINTER(_u64)]),
    "slq_rules": (_int, [_vp, _int, _u64, _i64, _i64, _int, _int, _int, _vp, _vp, _vp, _vp, _vp]),
    "slq_integrate": (_int, [_vp, _vp, _vp, _i64, _int, _vp, _i64, _vp, _int, _dbl, _vp, _vp, _vp, _vp, _vp]),
    "slq_signature": (_int, [_vp, _int, _u64, _i64, _int, _int, _int, _vp, _i64, _vp, _int, _vp, _vp, _vp, _vp]),
    "slq_lanczos_batched": (_int, [_vp, _vp, _i64, _int, _u64, _int, _int, _int, _vp, _vp, _vp, _vp, _vp]),
    "slq_integrate_batched": (_int, [_vp, _vp, _vp, _i64, _int, _int, _vp, _vp, _i64, _int, _vp, _vp, _vp, _vp]),
    "slq_graph_second_passes": (_int, [_vp, ctypes.POINTER(_i64)]),
    "slq_lanczos_seeded": (_int, [_vp, _int, _SP, _i64, _i64, _int, _int, _int, _vp, _vp, _vp, _vp]),
    "slq_rules_seeded": (_int, [_vp, _int, _SP, _i64, _i64, _int, _int, _int, _vp, _vp, _vp, _vp, _vp]),
    "slq_rules_pair_seeded": (_int, [_vp, _SP, _i64, _i64, _int, _int, _int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "slq_rules_host": (_int, [_vp, _int, _SP, _i64, _i64, _int, _int, _int, _vp, _vp, _vp]),
    "slq_probes_seeded": (_int, [_SP, _i64, _i64, _i64, _vp, _i64, _vp]),
    "slq_probe_state_seeded": (_int, [_SP, _u64, ctypes.POINTER(_u64)]),
    "slq_lanczos_batched_seeded": (_int, [_vp, _vp, _i64, _int, _SP, _int, _int, _int, _vp, _vp, _vp, _vp, _vp]),
    "slq_trim_pool": (_int, []),
    "slq_l2_limits": (_int, [ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "slq_graph_lanczos_rows": (_int, [_vp, _vp, _i64, ctypes.POINTER(_i64)]),
    "slq_last_error": (ctypes.c_char_p, []),
    "slq_launch_count": (_u64, []),
    "slq_profile_begin": (None, []),
    "slq_profile_end": (_int, [ctypes.POINTER(_dbl), ctypes.POINTER(_i64), _int]),
    "slq_build_info": (ctypes.c_char_p, []),
}

_LIB = None


def load(path: str = LIB_PATH):
    """Load the shared library (no CUDA device needed: loading only resolves symbols)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise SlqLibraryError(
            f"{path} is missing; build it with `python -m paper_2003_01282_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def check(rc: int, alpha=None, beta=None) -> None:
    if rc == SLQ_OK:
        return
    msg = load().slq_last_error().decode(errors="replace")
    if rc in (SLQ_ERR_VALUE, SLQ_ERR_NONFINITE):
        raise ValueError(msg)
    if rc == SLQ_ERR_EIGEN:
        raise TridiagonalEigenError(msg, alpha=alpha, beta=beta)
    if rc == SLQ_ERR_ALLOC:
        raise MemoryError(msg)
    raise SlqLibraryError(msg)


ST_EIGEN, ST_NAN_TRI, ST_NAN_F, ST_BAD_COL = 1, 2, 4, 8


def check_status(status: int, alpha=None, beta=None) -> None:
    """Raise the reference's exception for a device status word of the asynchronous calls."""
    status = int(status)
    if status == 0:
        return
    if status & ST_BAD_COL:
        raise ValueError("column index out of range [0, n)")
    if status & ST_NAN_TRI:
        raise ValueError("array must not contain infs or NaNs")
    if status & ST_EIGEN:
        raise TridiagonalEigenError("tridiagonal eigensolver failed: no convergence", alpha=alpha, beta=beta)
    if status & ST_NAN_F:
        raise ValueError("f returned a non-finite value at quadrature nodes")
    raise SlqLibraryError(f"unknown device status {status}")


def int_array(values) -> ctypes.Array:
    arr = (ctypes.c_int * len(values))(*[int(v) for v in values])
    return arr


def ptr(t) -> int | None:
    """Device/host pointer of a torch tensor or numpy array (None for None)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def stream_handle(device=None) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise SlqLibraryError("no CUDA device visible: the SLQ engine runs only on the GPU (no CPU fallback)")
    load()
    return torch


def trim_pool() -> None:
    """Give the library's cached stream-ordered pool memory on the current device back to the driver."""
    check(load().slq_trim_pool())


def launch_count() -> int:
    return int(load().slq_launch_count())


def profile_begin() -> None:
    load().slq_profile_begin()


def profile_end() -> dict:
    n = len(KERNEL_CLASSES)
    ms = (ctypes.c_double * n)()
    cnt = (ctypes.c_int64 * n)()
    load().slq_profile_end(ms, cnt, n)
    return {k: {"ms": float(ms[i]), "launches": int(cnt[i])} for i, k in enumerate(KERNEL_CLASSES)}
