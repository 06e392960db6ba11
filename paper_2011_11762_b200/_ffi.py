"""ctypes binding of libqmb200.so (include/qmb200.h).

The library is loaded from the package directory (built in-tree by ``_build.build``). There is no
CPU fallback: when the library or a CUDA device is missing, every compute entry point raises
``DeviceUnavailableError``.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import (
    ConfigurationError,
    DeviceUnavailableError,
    DimensionMismatchError,
    QuadmatError,
    StoreCapacityError,
)

LIB_PATH = Path(__file__).resolve().parent / "libqmb200.so"

ABI_VERSION = 2  # include/qmb200.h QM_ABI_VERSION

QM_OK, QM_ERR_INVALID, QM_ERR_CUDA, QM_ERR_WORKSPACE, QM_ERR_UNSUPPORTED = 0, -1, -2, -3, -4

# Every symbol include/qmb200.h declares (tests check the .so exports all of them).
EXPORTS = (
    "qm_abi_version",
    "qm_last_error",
    "qm_launch_count",
    "qm_read_i64",
    "qm_encode_keys",
    "qm_decode_keys",
    "qm_build_workspace_bytes",
    "qm_build_count",
    "qm_build_fill",
    "qm_build_fill_meta",
    "qm_spgemm_workspace_bytes",
    "qm_spgemm_count",
    "qm_spgemm_count_masked",
    "qm_spgemm_count_part",
    "qm_row_index_workspace_bytes",
    "qm_row_index_build",
    "qm_spgemm_count_ix",
    "qm_spgemm_fill_ix",
    "qm_spgemm_fill_workspace_bytes",
    "qm_spgemm_fill",
    "qm_spgemm_fill_keys",
    "qm_spgemm_fill_triples",
    "qm_numeric",
    "qm_numeric_masked",
    "qm_numeric_workspace_bytes",
    "qm_numeric_pools",
    "qm_ipc_export",
    "qm_ipc_open",
    "qm_ipc_close",
    "qm_numeric_pools_ex",
    "qm_stage_plan_workspace_bytes",
    "qm_stage_plan",
    "qm_numeric_path",
    "qm_numeric_kernel",
    "qm_compact_workspace_bytes",
    "qm_compact",
    "qm_block_stats",
    "qm_block_masks",
    "qm_block_meta",
    "qm_gather_blocks",
    "qm_gather_blocks_t",
    "qm_transpose_blocks",
    "qm_axpby_blocks",
    "qm_add_identity_blocks",
    "qm_node_norms_workspace_bytes",
    "qm_node_norms",
    "qm_prune_level_workspace_bytes",
    "qm_prune_level",
    "qm_prune_all_workspace_bytes",
    "qm_prune_all",
    "qm_filter_triples_workspace_bytes",
    "qm_filter_triples",
    "qm_ancestor_norms",
    "qm_filter_triples_norms",
    "qm_generate_blocks",
    "qm_fp64_peak_kernel",
)


class QmLayout(ctypes.Structure):
    _fields_ = [
        ("n_logical", ctypes.c_int64),
        ("leaf_dim", ctypes.c_int32),
        ("depth", ctypes.c_int32),
        ("block_size", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


def make_layout(params, block_size: int) -> QmLayout:
    return QmLayout(params.n_logical, params.leaf_dim, params.depth, block_size, 0)


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_SZ = ctypes.c_size_t
_LP = ctypes.POINTER(QmLayout)

MAX_RANKS = 8  # QM_MAX_RANKS


class QmRowIndex(ctypes.Structure):
    """include/qmb200.h qm_row_index: one operand's row-sorted view (device pointers)."""

    _fields_ = [("rowptr", ctypes.c_void_p), ("row", ctypes.c_void_p), ("col", ctypes.c_void_p),
                ("perm", ctypes.c_void_p), ("mask", ctypes.c_void_p)]


class QmHalo(ctypes.Structure):
    """include/qmb200.h qm_halo: the peer-owned blocks one rank gathers (staged multi-GPU product)."""

    _fields_ = [
        ("world", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("index", ctypes.c_void_p * 2),
        ("count", ctypes.c_int64 * 2),
        ("pool", ctypes.c_void_p * 2),
        ("peer_base", (ctypes.c_uint64 * MAX_RANKS) * 2),
        ("offset", (ctypes.c_int64 * (MAX_RANKS + 1)) * 2),
        ("min_ns", ctypes.c_int64),
    ]

_SIGS = {
    "qm_abi_version": (ctypes.c_int, []),
    "qm_last_error": (ctypes.c_char_p, []),
    "qm_launch_count": (ctypes.c_uint64, []),
    "qm_read_i64": (ctypes.c_int, [_P, _I32, ctypes.POINTER(_I64), _P]),
    "qm_encode_keys": (ctypes.c_int, [_LP, _P, _P, _I64, _P, _P]),
    "qm_decode_keys": (ctypes.c_int, [_LP, _P, _I64, _P, _P, _P]),
    "qm_build_workspace_bytes": (_SZ, [_LP, _I64]),
    "qm_build_count": (ctypes.c_int, [_LP, _P, _P, _I64, _P, _SZ, ctypes.POINTER(_I64),
                                      ctypes.POINTER(_I64), _P]),
    "qm_build_fill": (ctypes.c_int, [_LP, _P, _I64, _P, _SZ, _I64, _P, _P, _P, _P, _P, _P]),
    "qm_build_fill_meta": (ctypes.c_int, [_LP, _P, _I64, _P, _SZ, _I64, _P, _P, _P, _P, _P, _P, _P, _P]),
    "qm_spgemm_workspace_bytes": (_SZ, [_LP, _I64, _I64]),
    "qm_spgemm_count": (ctypes.c_int, [_LP, _P, _I64, _P, _I64, _P, _SZ, ctypes.POINTER(_I64),
                                       ctypes.POINTER(_I64), _P]),
    "qm_spgemm_count_masked": (ctypes.c_int, [_LP, _P, _P, _I64, _P, _P, _I64, _I32, _P, _SZ,
                                             ctypes.POINTER(_I64), ctypes.POINTER(_I64), _P]),
    "qm_spgemm_count_part": (ctypes.c_int, [_LP, _P, _P, _I64, _P, _P, _I64, _I32, _I32, _P, _SZ,
                                            ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I64), _P,
                                            _P]),
    "qm_row_index_workspace_bytes": (_SZ, [_LP, _I64]),
    "qm_row_index_build": (ctypes.c_int, [_LP, _P, _I64, _P, _P, _SZ, _P, _P, _P, _P, _P, _P, _P]),
    "qm_spgemm_count_ix": (ctypes.c_int, [_LP, _P, _I64, _P, _I64, _I32, _I32, _I32, _P, _SZ, ctypes.POINTER(_I64),
                                          ctypes.POINTER(_I64), _P, _P, _P]),
    "qm_spgemm_fill_ix": (ctypes.c_int, [_LP, _P, _I64, _P, _I64, _I64, _I64, _I64, _P, _SZ, _P, _SZ, _P, _P, _P,
                                         _P]),
    "qm_spgemm_fill_workspace_bytes": (_SZ, [_LP, _I64]),
    "qm_spgemm_fill": (ctypes.c_int, [_LP, _I64, _I64, _I64, _I64, _P, _SZ, _P, _SZ, _P, _P, _P, _P]),
    "qm_spgemm_fill_keys": (ctypes.c_int, [_LP, _I64, _I64, _I64, _P, _SZ, _P, _SZ, _P, _P, _P]),
    "qm_spgemm_fill_triples": (ctypes.c_int, [_LP, _I64, _I64, _I64, _P, _SZ, _P, _SZ, _P, _I64, _I64,
                                              _P, _P]),
    "qm_numeric": (ctypes.c_int, [_LP, _P, _P, _I64, _P, _I64, _P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _SZ,
                                  _P]),
    "qm_numeric_masked": (ctypes.c_int, [_LP, _P, _P, _P, _I64, _P, _P, _I64, _I32, _P, _P, _P, _I64, _I64, _P, _P,
                                         _P, _P, _P, _P, _SZ, _P]),
    "qm_numeric_workspace_bytes": (_SZ, [_I32, _I64, _I64]),
    "qm_ipc_export": (ctypes.c_int, [_P, _P, ctypes.POINTER(_I64)]),
    "qm_ipc_open": (ctypes.c_int, [_P, ctypes.POINTER(_P)]),
    "qm_ipc_close": (ctypes.c_int, [_P]),
    "qm_numeric_pools_ex": (ctypes.c_int, [_LP, _P, _P, _I32, _P, _P, _I32, _P, _P, _P, _P, _P, _P, _P, _P,
                                           _I64, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "qm_stage_plan_workspace_bytes": (_SZ, [_I64, _I64, _I64, _I32]),
    "qm_stage_plan": (ctypes.c_int, [_P, _I64, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I32, _P, _SZ, _P, _P,
                                     _P, _P, ctypes.POINTER(_I64), _P]),
    "qm_numeric_pools": (ctypes.c_int, [_LP, _P, _P, _I32, _P, _P, _I32, _P, _P, _I64, _I64, _P, _P, _P, _P,
                                        _P, _SZ, _P]),
    "qm_numeric_path": (ctypes.c_int, [_I32]),
    "qm_numeric_kernel": (ctypes.c_char_p, [_LP, _I64, _I64, _I32, _I32]),
    "qm_compact_workspace_bytes": (_SZ, [_I64]),
    "qm_compact": (ctypes.c_int, [_I32, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "qm_block_stats": (ctypes.c_int, [_I32, _I64, _P, _P, _P, _P]),
    "qm_block_masks": (ctypes.c_int, [_I32, _I64, _P, _P, _P, _P]),
    "qm_block_meta": (ctypes.c_int, [_I32, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "qm_gather_blocks": (ctypes.c_int, [_I32, _P, _P, _I64, _P, _P]),
    "qm_gather_blocks_t": (ctypes.c_int, [_I32, _P, _P, _P, _I64, _P, _P]),
    "qm_transpose_blocks": (ctypes.c_int, [_I32, _P, _I64, _P, _P]),
    "qm_axpby_blocks": (ctypes.c_int, [_I32, _I64, _P, _P, ctypes.c_double, ctypes.c_double, _P, _P, _P, _P,
                                       _P, _P, _P]),
    "qm_add_identity_blocks": (ctypes.c_int, [_I32, _I64, _P, _P, _P, ctypes.c_double, _I64, _P, _P, _P]),
    "qm_node_norms_workspace_bytes": (_SZ, [_I64]),
    "qm_node_norms": (ctypes.c_int, [_LP, _P, _P, _I64, _P, _P, ctypes.POINTER(_I64), _P, _SZ, _P]),
    "qm_prune_level_workspace_bytes": (_SZ, [_I64]),
    "qm_prune_level": (ctypes.c_int, [_LP, _I32, ctypes.c_double, _P, _I64, _P, _P, _I64, _I32, _P, _P, _I64,
                                      _I32, _I32, _I32, _P, _P, ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                                      _P, _SZ, _P]),
    "qm_prune_all_workspace_bytes": (_SZ, [_I64]),
    "qm_prune_all": (ctypes.c_int, [_LP, ctypes.c_double, _P, _P, _I64, _P, _I32, _P, _P, _I64, _P, _I32, _I32,
                                    _I32, _I64, _P, _P, _I64, _P, _P, _SZ, _P]),
    "qm_filter_triples_workspace_bytes": (_SZ, [_I64, _I64]),
    "qm_filter_triples": (ctypes.c_int, [_LP, _P, _P, _I32, _P, _P, _P, _I64, _I64, _P, _I64, _P, _P, _P,
                                         ctypes.POINTER(_I64), ctypes.POINTER(_I64), _P, _SZ, _P]),
    "qm_ancestor_norms": (ctypes.c_int, [_LP, _P, _I64, _P, _P, _I64, _P, _I32, _P, _P]),
    "qm_filter_triples_norms": (ctypes.c_int, [_LP, ctypes.c_double, _P, _P, _P, _I64, _I64, _P, _I64, _P, _I64,
                                               _P, _P, _P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), _P, _SZ,
                                               _P]),
    "qm_generate_blocks": (ctypes.c_int, [_LP, _P, _I64, ctypes.c_uint64, ctypes.c_uint32, _I32,
                                          _I64, _P, _P, _P]),
    "qm_fp64_peak_kernel": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _I64, _P,
                                           ctypes.POINTER(ctypes.c_double), _P]),
}

_lib = None
_lock = threading.Lock()


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load (once) and type the library. Raises DeviceUnavailableError if it is not built."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        # QM_LIB_PATH: an experimental build of the same library (A/B kernel variants); default in-tree
        p = Path(path) if path else Path(os.environ.get("QM_LIB_PATH") or LIB_PATH)
        if not p.exists():
            raise DeviceUnavailableError(
                f"{p} is not built; run paper_2011_11762_b200._build.build() (nvcc, sm_100a)"
            )
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.qm_abi_version() != ABI_VERSION:
            raise ConfigurationError(f"libqmb200 ABI {lib.qm_abi_version()} != {ABI_VERSION} (rebuild: "
                                     "paper_2011_11762_b200._build.build())")
        if path is None:
            _lib = lib
        return lib


def last_error() -> str:
    """The calling thread's last libqmb200 error message."""
    return (load().qm_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str) -> None:
    """Map a qm_status onto the reference's exception types."""
    if rc == QM_OK:
        return
    msg = (load().qm_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}"
    if rc == QM_ERR_INVALID:
        if "dimension" in msg or "conform" in msg:
            raise DimensionMismatchError(text)
        raise ConfigurationError(text)
    if rc == QM_ERR_UNSUPPORTED:
        raise ConfigurationError(text)
    if rc == QM_ERR_CUDA and ("out of memory" in msg or "memory allocation" in msg):
        raise StoreCapacityError(text)
    raise QuadmatError(f"{text} (status {rc})")


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return 0 if t is None else int(t.data_ptr())


def stream_handle(stream) -> int:
    return 0 if stream is None else int(stream.cuda_stream)


def read_i64s(t, n: int, stream=None) -> list[int]:
    """The first n (<= 8) int64 values of a device tensor, one synchronisation (qm_read_i64)."""
    import torch  # noqa: PLC0415

    out = (ctypes.c_int64 * n)()
    st = stream if stream is not None else torch.cuda.current_stream(t.device)
    check(load().qm_read_i64(ptr(t), n, out, stream_handle(st)), "qm_read_i64")
    return [int(x) for x in out]


def read_i64(t, stream=None) -> int:
    """One int64 device value to the host without a copy engine (qm_read_i64)."""
    import torch  # noqa: PLC0415

    out = ctypes.c_int64(0)
    st = stream if stream is not None else torch.cuda.current_stream(t.device)
    check(load().qm_read_i64(ptr(t), 1, ctypes.byref(out), stream_handle(st)), "qm_read_i64")
    return int(out.value)
