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
import os
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


class SymbolicState:
    """Workspaces of one symbolic phase (row indexes, fill scratch) kept between its steps."""

    def __init__(self, layout, a_keys: torch.Tensor, n_a: int, b_keys: torch.Tensor, n_b: int, stream=None,
                 a_cmask: torch.Tensor | None = None, b_rmask: torch.Tensor | None = None, upper: bool = False,
                 part: tuple[int, int] | None = None, ix=None):
        """part = (world, rank): the rank's share of a multi-GPU product (qm_spgemm_count_part) --
        only the C blocks of its own key range (self.key_range) are counted and emitted.
        ix = (qm_row_index of A, of B): the operands' cached row indexes (BlockSet.row_index); the
        count / fill calls then use them instead of indexing the keys themselves."""
        self.lib = _ffi.load()
        self.ix = ix
        self.layout = layout
        self.lp = ctypes.byref(layout)
        self.n_a, self.n_b = n_a, n_b
        self.dev = a_keys.device
        self.sh = _ffi.stream_handle(stream)
        self.ws_bytes = self.lib.qm_spgemm_workspace_bytes(self.lp, n_a, n_b)
        self.ws = _alloc(max(self.ws_bytes, 1), torch.uint8, self.dev)
        n_c = ctypes.c_int64(0)
        n_t = ctypes.c_int64(0)
        self.key_range, self.tile_work, self.key_cuts = None, 0, None
        if ix is not None:
            world, rank = part if part is not None else (0, 0)
            po = (ctypes.c_int64 * 3)()
            if part is not None:
                self.key_cuts = _alloc(world + 1, torch.int64, self.dev)
            _ffi.check(
                self.lib.qm_spgemm_count_ix(self.lp, ctypes.byref(ix[0]), n_a, ctypes.byref(ix[1]), n_b,
                                            1 if upper else 0, world, rank, _ffi.ptr(self.ws), self.ws_bytes,
                                            ctypes.byref(n_c), ctypes.byref(n_t), po if part is not None else None,
                                            _ffi.ptr(self.key_cuts), self.sh),
                "qm_spgemm_count_ix",
            )
            if part is not None:
                self.key_range = (int(po[0]) & (2**64 - 1), int(po[1]) & (2**64 - 1))
                self.tile_work = int(po[2])
        elif part is not None:
            world, rank = part
            po = (ctypes.c_int64 * 3)()
            self.key_cuts = _alloc(world + 1, torch.int64, self.dev)
            _ffi.check(
                self.lib.qm_spgemm_count_part(self.lp, _ffi.ptr(a_keys), _ffi.ptr(a_cmask), n_a, _ffi.ptr(b_keys),
                                              _ffi.ptr(b_rmask), n_b, world, rank, _ffi.ptr(self.ws), self.ws_bytes,
                                              ctypes.byref(n_c), ctypes.byref(n_t), po, _ffi.ptr(self.key_cuts),
                                              self.sh),
                "qm_spgemm_count_part",
            )
            self.key_range = (int(po[0]) & (2**64 - 1), int(po[1]) & (2**64 - 1))
            self.tile_work = int(po[2])
        else:
            _ffi.check(  # support masks (None = full support): pairs whose product is exactly zero are skipped
                self.lib.qm_spgemm_count_masked(self.lp, _ffi.ptr(a_keys), _ffi.ptr(a_cmask), n_a, _ffi.ptr(b_keys),
                                                _ffi.ptr(b_rmask), n_b, 1 if upper else 0, _ffi.ptr(self.ws),
                                                self.ws_bytes, ctypes.byref(n_c), ctypes.byref(n_t), self.sh),
                "qm_spgemm_count_masked",
            )
        self.n_c, self.n_t = int(n_c.value), int(n_t.value)
        self.fill_bytes = self.lib.qm_spgemm_fill_workspace_bytes(self.lp, self.n_c)
        self.fws = _alloc(max(self.fill_bytes, 1), torch.uint8, self.dev)

    def keys(self):
        """C keys (quadtree order) and triple offsets c_tptr[nC+1]."""
        c_keys = _alloc(self.n_c, torch.int64, self.dev)
        c_tptr = _alloc(self.n_c + 1, torch.int64, self.dev)
        if self.ix is not None:
            self.fill_ix(c_keys, c_tptr, None, 0, 0)
            return c_keys, c_tptr
        _ffi.check(
            self.lib.qm_spgemm_fill_keys(self.lp, self.n_a, self.n_b, self.n_c, _ffi.ptr(self.ws),
                                         self.ws_bytes, _ffi.ptr(self.fws), self.fill_bytes,
                                         _ffi.ptr(c_keys), _ffi.ptr(c_tptr), self.sh),
            "qm_spgemm_fill_keys",
        )
        return c_keys, c_tptr

    def triples(self, c_tptr: torch.Tensor, t_lo: int = 0, t_hi: int | None = None) -> torch.Tensor:
        """(a_index, b_index) int32 pairs of triples [t_lo, t_hi)."""
        t_hi = self.n_t if t_hi is None else t_hi
        tri = _alloc(2 * max(t_hi - t_lo, 0), torch.int32, self.dev)
        if self.ix is not None:
            self.fill_ix(None, c_tptr, tri, t_lo, t_hi)
            return tri
        _ffi.check(
            self.lib.qm_spgemm_fill_triples(self.lp, self.n_a, self.n_b, self.n_c, _ffi.ptr(self.ws),
                                            self.ws_bytes, _ffi.ptr(self.fws), self.fill_bytes,
                                            _ffi.ptr(c_tptr), t_lo, t_hi, _ffi.ptr(tri), self.sh),
            "qm_spgemm_fill_triples",
        )
        return tri


    def fill_ix(self, c_keys, c_tptr, tri, t_lo: int, t_hi: int):
        """qm_spgemm_fill_ix: C keys + c_tptr (c_keys given) and / or triples [t_lo, t_hi)."""
        _ffi.check(
            self.lib.qm_spgemm_fill_ix(self.lp, ctypes.byref(self.ix[0]), self.n_a, ctypes.byref(self.ix[1]), self.n_b,
                                       self.n_c, t_lo, t_hi, _ffi.ptr(self.ws), self.ws_bytes, _ffi.ptr(self.fws),
                                       self.fill_bytes, _ffi.ptr(c_keys), _ffi.ptr(c_tptr), _ffi.ptr(tri), self.sh),
            "qm_spgemm_fill_ix",
        )


def support_filter_enabled() -> bool:
    """QM_SUPPORT_FILTER=0 disables the exact-zero product filter (A/B measurements, tests)."""
    return os.environ.get("QM_SUPPORT_FILTER", "1") != "0"


def row_index_enabled() -> bool:
    """QM_ROW_INDEX=0: the symbolic phase indexes the operands' keys itself on every product."""
    return os.environ.get("QM_ROW_INDEX", "1") != "0"


def _use_masks(a: BlockSet, b: BlockSet, stream=None) -> bool:
    """Support masks matter unless A's blocks all have full column support or B's all have full row
    support (dense blocks: every pair and every k panel contributes, so filtering is skipped)."""
    if not support_filter_enabled():
        return False
    a.support_masks(stream)
    b.support_masks(stream)
    return not (a.masks_full[1] or b.masks_full[0])


def symbolic(layout, a: BlockSet, b: BlockSet, stream=None, upper: bool = False) -> SymbolicPlan:
    """Triples of C = A*B. Block pairs whose support masks do not meet (A(i,k)'s nonzero columns vs
    B(k,j)'s nonzero rows) multiply to an exactly-zero block and yield no triple; a C block left
    without triples is an exact-zero block the reference computes and then drops (_set_block,
    block_sparse.py:37-41), so the product is unchanged."""
    a_cm = b_rm = None
    use = _use_masks(a, b, stream)
    if use:
        a_cm, b_rm = a.masks[1], b.masks[0]
    ix = None
    if row_index_enabled() and type(a) is BlockSet and type(b) is BlockSet:  # (views index their entries)
        ia, ib = a.row_index(layout, stream), b.row_index(layout, stream)
        ix = (BlockSet.ix_struct(ia, "a" if use else None), BlockSet.ix_struct(ib, "b" if use else None))
    st = SymbolicState(layout, a.keys, a.n, b.keys, b.n, stream, a_cm, b_rm, upper, ix=ix)
    c_keys = _alloc(st.n_c, torch.int64, st.dev)
    c_tptr = _alloc(st.n_c + 1, torch.int64, st.dev)
    tri = _alloc(2 * st.n_t, torch.int32, st.dev)
    if ix is not None:
        st.fill_ix(c_keys, c_tptr, tri, 0, st.n_t)
    else:
        _ffi.check(  # C keys, c_tptr and every triple in one call (keys() + triples() of SymbolicState)
            st.lib.qm_spgemm_fill(st.lp, st.n_a, st.n_b, st.n_c, st.n_t, _ffi.ptr(st.ws), st.ws_bytes,
                                  _ffi.ptr(st.fws), st.fill_bytes, _ffi.ptr(c_keys), _ffi.ptr(c_tptr),
                                  _ffi.ptr(tri), st.sh),
            "qm_spgemm_fill",
        )
    return SymbolicPlan(st.n_c, st.n_t, c_keys, c_tptr, tri)


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
    zc = _alloc(2, torch.int64, dev)  # [exact-zero C blocks, k panels executed]: set by the library
    wb = lib.qm_numeric_workspace_bytes(bs, nc, plan.n_triples)
    ws = _alloc(wb, torch.uint8, dev) if wb else None
    use_masks = _use_masks(a, b, stream)
    tri, flags = plan.tri, 0
    pa, pb = getattr(a, "pool", None), getattr(b, "pool", None)
    if pa is not None or pb is not None:  # virtual transposes: view indices -> stored block | bit 31
        t2 = plan.tri.view(-1, 2)
        tri = torch.stack([a.src[t2[:, 0].long()] if pa is not None else t2[:, 0],
                           b.src[t2[:, 1].long()] if pb is not None else t2[:, 1]], dim=1).reshape(-1).contiguous()
        flags = 1  # QM_NUMERIC_TRANSPOSED_REFS
    sa, sb = pa if pa is not None else a, pb if pb is not None else b  # the stored pools
    am = sa.support_masks(stream) if use_masks else None
    bm = sb.support_masks(stream) if use_masks else None
    _ffi.check(
        lib.qm_numeric_masked(ctypes.byref(layout), _ffi.ptr(a.keys), _ffi.ptr(sa.blocks), _ffi.ptr(am), sa.n,
                              _ffi.ptr(sb.blocks), _ffi.ptr(bm), sb.n, flags, _ffi.ptr(tri), _ffi.ptr(plan.c_tptr),
                              _ffi.ptr(plan.c_keys), nc, plan.n_triples, _ffi.ptr(out.blocks),
                              _ffi.ptr(out.sumsq), _ffi.ptr(nz), _ffi.ptr(zc), _ffi.ptr(zc[1:]), _ffi.ptr(ws), wb,
                              _ffi.stream_handle(stream)),
        "qm_numeric_masked",
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
                    stats: MultiplyStats | None = None, events: dict | None = None,
                    plan_filter=None, upper: bool = False) -> BlockSet:
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
    plan = symbolic(layout, a, b, stream, upper)  # upper: only C blocks of leaves li <= lj
    if plan_filter is not None:  # e.g. the approximate variant's pruned triples (approximate.py)
        plan = plan_filter(plan)
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
    n_zero, panels = _ffi.read_i64s(zc, 2, stream)
    c = compact(bs, c, nz, n_zero, stream)
    if stats is not None:
        stats.zero_blocks = n_zero
        if panels >= 0:  # k depth executed over all triples (k panels where the supports miss are skipped)
            stats.extra["k_rows"] = panels
            stats.flops = 2 * bs * bs * panels
        stats.n_c = c.n
        stats.launches = int(lib.qm_launch_count() - l0)
    return c


def _sync_item(t: torch.Tensor, stream) -> int:
    """Device int64 -> host via a mapped buffer (qm_read_i64): unlike .item(), it does not queue
    behind large D2H copies of earlier products on the copy engine."""
    return _ffi.read_i64(t, stream)
