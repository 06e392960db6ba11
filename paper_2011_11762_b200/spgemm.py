"""C = A*B on device block sets through libqmb200 (the hot path).

Pipeline, all stream-ordered on one CUDA stream:

    qm_spgemm_count  -> (nC, nT)        symbolic phase: row indexes, per-row C/triple counts
    qm_spgemm_fill   -> c_keys, c_tptr, tri
    qm_numeric       -> c_blocks, c_sumsq, c_nonzero, zero_count
    qm_compact       (only when some C block is exactly zero, _set_block's np.any drop)

This is what the reference's task graph computes for the regular variant: _multiply_body's
recursion (ops.py:197-241) enumerates the same triples, BlockSparseLeaf.multiply/add
(block_sparse.py:112-152) sums them, and _put_leaf (ops.py:119-122) drops exactly-zero blocks.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import torch

from . import _ffi
from .blocks import BlockSet
from .errors import ConfigurationError, DeviceUnavailableError, StoreCapacityError


@dataclass
class SymbolicPlan:
    """Output of the symbolic phase for one product (reusable for repeated numeric passes)."""

    n_c: int
    n_triples: int
    c_keys: torch.Tensor
    c_tptr: torch.Tensor
    tri: torch.Tensor  # int32 [2*nT]: (a_index, b_index) pairs


@dataclass
class MultiplyStats:
    n_a: int = 0
    n_b: int = 0
    n_c_symbolic: int = 0
    n_c: int = 0
    n_triples: int = 0
    zero_blocks: int = 0
    flops: int = 0  # leaf-GEMM flops 2*bs^3*T
    launches: int = 0
    extra: dict = field(default_factory=dict)


def _require_cuda(t: torch.Tensor):
    if t.device.type != "cuda":
        raise DeviceUnavailableError(
            "the multiply runs only on the CUDA path (libqmb200 on a B200); operands are on "
            f"{t.device}. There is no CPU fallback."
        )


def _alloc(shape, dtype, device):
    try:
        return torch.empty(shape, dtype=dtype, device=device)
    except torch.cuda.OutOfMemoryError as e:  # device OOM maps to the store's capacity error
        raise StoreCapacityError(f"device memory exhausted allocating {shape} {dtype}: {e}") from e


def symbolic(layout, a: BlockSet, b: BlockSet, stream=None) -> SymbolicPlan:
    lib = _ffi.load()
    dev = a.device
    sh = _ffi.stream_handle(stream)
    lp = ctypes.byref(layout)
    ws_bytes = lib.qm_spgemm_workspace_bytes(lp, a.n, b.n)
    ws = _alloc(max(ws_bytes, 1), torch.uint8, dev)
    n_c = ctypes.c_int64(0)
    n_t = ctypes.c_int64(0)
    _ffi.check(
        lib.qm_spgemm_count(lp, _ffi.ptr(a.keys), a.n, _ffi.ptr(b.keys), b.n, _ffi.ptr(ws), ws_bytes,
                            ctypes.byref(n_c), ctypes.byref(n_t), sh),
        "qm_spgemm_count",
    )
    nc, nt = int(n_c.value), int(n_t.value)
    c_keys = _alloc(nc, torch.int64, dev)
    c_tptr = _alloc(nc + 1, torch.int64, dev)
    tri = _alloc(2 * nt, torch.int32, dev)
    fill_bytes = lib.qm_spgemm_fill_workspace_bytes(lp, nc)
    fws = _alloc(max(fill_bytes, 1), torch.uint8, dev)
    _ffi.check(
        lib.qm_spgemm_fill(lp, _ffi.ptr(a.keys), a.n, _ffi.ptr(b.keys), b.n, _ffi.ptr(ws), ws_bytes,
                           _ffi.ptr(fws), fill_bytes, _ffi.ptr(c_keys), _ffi.ptr(c_tptr),
                           _ffi.ptr(tri), sh),
        "qm_spgemm_fill",
    )
    return SymbolicPlan(nc, nt, c_keys, c_tptr, tri)


def numeric(layout, a: BlockSet, b: BlockSet, plan: SymbolicPlan, stream=None,
            out: BlockSet | None = None):
    """Runs the numeric kernel; returns (blockset before compaction, nonzero flags, zero counter)."""
    lib = _ffi.load()
    bs = layout.block_size
    dev = a.device
    nc = plan.n_c
    if out is None:
        out = BlockSet(plan.c_keys, _alloc((nc, bs, bs), torch.float64, dev),
                       _alloc(nc, torch.float64, dev))
    nz = _alloc(nc, torch.uint8, dev)
    zc = torch.zeros(1, dtype=torch.int64, device=dev)
    _ffi.check(
        lib.qm_numeric(ctypes.byref(layout), _ffi.ptr(a.blocks), a.n, _ffi.ptr(b.blocks), b.n,
                       _ffi.ptr(plan.tri), _ffi.ptr(plan.c_tptr), nc, _ffi.ptr(out.blocks),
                       _ffi.ptr(out.sumsq), _ffi.ptr(nz), _ffi.ptr(zc), _ffi.stream_handle(stream)),
        "qm_numeric",
    )
    return out, nz, zc


def compact(bs: int, c: BlockSet, nz: torch.Tensor, n_zero: int, stream=None) -> BlockSet:
    """Drops exactly-zero C blocks (order preserved)."""
    if n_zero == 0:
        return c
    lib = _ffi.load()
    keep = c.n - n_zero
    dev = c.device
    out = BlockSet(_alloc(keep, torch.int64, dev), _alloc((keep, bs, bs), torch.float64, dev),
                   _alloc(keep, torch.float64, dev))
    if keep == 0:
        return out
    wb = lib.qm_compact_workspace_bytes(c.n)
    ws = _alloc(max(wb, 1), torch.uint8, dev)
    _ffi.check(
        lib.qm_compact(bs, c.n, _ffi.ptr(nz), _ffi.ptr(c.keys), _ffi.ptr(c.blocks),
                       _ffi.ptr(c.sumsq), _ffi.ptr(out.keys), _ffi.ptr(out.blocks),
                       _ffi.ptr(out.sumsq), _ffi.ptr(ws), wb, _ffi.stream_handle(stream)),
        "qm_compact",
    )
    return out


def multiply_blocks(layout, a: BlockSet, b: BlockSet, stream=None,
                    stats: MultiplyStats | None = None, events: dict | None = None) -> BlockSet:
    """Full regular product of two conformant block sets on their CUDA device.

    ``events`` (optional): CUDA events recorded on the stream around the phases, keys
    "symbolic", "numeric", "end" -- used by bench.py to time the numeric kernel alone."""
    _require_cuda(a.blocks)
    _require_cuda(b.blocks)
    if a.device != b.device:
        raise ConfigurationError(f"operands live on different devices: {a.device} vs {b.device}")
    bs = layout.block_size
    if a.n and a.bs != bs or b.n and b.bs != bs:
        raise ConfigurationError("operands must share leaf kind and block size")
    lib = _ffi.load()
    l0 = lib.qm_launch_count()
    if stream is None:
        stream = torch.cuda.current_stream(a.device)
    if a.n == 0 or b.n == 0:
        return BlockSet.empty(bs, a.device)
    if events is not None:
        events["symbolic"].record(stream)
    plan = symbolic(layout, a, b, stream)
    if stats is not None:
        stats.n_a, stats.n_b = a.n, b.n
        stats.n_c_symbolic, stats.n_triples = plan.n_c, plan.n_triples
        stats.flops = 2 * bs ** 3 * plan.n_triples
    if plan.n_c == 0:
        return BlockSet.empty(bs, a.device)
    if events is not None:
        events["numeric"].record(stream)
    c, nz, zc = numeric(layout, a, b, plan, stream)
    if events is not None:
        events["end"].record(stream)
    n_zero = _sync_item(zc, stream)
    c = compact(bs, c, nz, n_zero, stream)
    if stats is not None:
        stats.zero_blocks = n_zero
        stats.n_c = c.n
        stats.launches = int(lib.qm_launch_count() - l0)
    return c


def _sync_item(t: torch.Tensor, stream) -> int:
    stream.synchronize()
    return int(t.item())
