"""Multiply variants of the reference (ops.py:47-76, 582-608) on device block sets.

The reference never materialises a transpose: tasks carry ta/tb flags and `_virtual_child`
(ops.py:100-116) maps quadrants, and symmetric matrices store only the upper triangle at leaf
granularity (SW quadrant of every diagonal-path node is nil and implied by NE^T; diagonal leaves
hold full blocks, session.py:93-100). `upper` (symmetric_square, rank_k) makes every diagonal-path
node skip its SW quadrant (ops.py:214-216) while leaf products stay full, so the result holds
exactly the blocks of leaves (li, lj) with li <= lj.

On the GPU the same algebra is expressed on flat block sets:
  * transpose(X):        keys (bi,bj) -> (bj,bi) re-sorted, blocks transposed (qm_transpose_blocks);
  * expand_symmetric(S): S plus transposed copies of the blocks of strictly-upper leaves;
  * upper(C):            only the blocks of leaves with li <= lj.
then the regular product runs unchanged:
  regular/symmetric  C = expand(A) * expand(B)                      (a_sym / b_sym flags)
  symmetric_square   C = upper(expand(A) * expand(A))               result symmetric
  rank_k             C = upper(A * transpose(A))                    result symmetric
where upper(.) is not a filter on the result: the symbolic phase enumerates only the C blocks of
upper leaves (qm_spgemm_count_masked with QM_SPGEMM_UPPER), so the dropped half is never computed.
"""

from __future__ import annotations

import torch

from . import _ffi
from .blocks import BlockSet
from .layout import Geometry


def _decode(geom: Geometry, keys: torch.Tensor):
    lib = _ffi.load()
    n = int(keys.shape[0])
    bi = torch.empty(n, dtype=torch.int32, device=keys.device)
    bj = torch.empty(n, dtype=torch.int32, device=keys.device)
    lay = _ffi.make_layout(geom.params, geom.bs)
    import ctypes

    _ffi.check(lib.qm_decode_keys(ctypes.byref(lay), _ffi.ptr(keys), n, _ffi.ptr(bi), _ffi.ptr(bj),
                                  _ffi.stream_handle(torch.cuda.current_stream(keys.device))),
               "qm_decode_keys")
    return bi, bj


def _encode(geom: Geometry, bi: torch.Tensor, bj: torch.Tensor) -> torch.Tensor:
    import ctypes

    lib = _ffi.load()
    n = int(bi.shape[0])
    keys = torch.empty(n, dtype=torch.int64, device=bi.device)
    lay = _ffi.make_layout(geom.params, geom.bs)
    _ffi.check(lib.qm_encode_keys(ctypes.byref(lay), _ffi.ptr(bi.contiguous()), _ffi.ptr(bj.contiguous()),
                                  n, _ffi.ptr(keys), _ffi.stream_handle(torch.cuda.current_stream(bi.device))),
               "qm_encode_keys")
    return keys


def _gather(bset_blocks: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    lib = _ffi.load()
    n = int(idx.shape[0])
    bs = int(bset_blocks.shape[1])
    out = torch.empty((n, bs, bs), dtype=torch.float64, device=bset_blocks.device)
    if n:
        _ffi.check(lib.qm_gather_blocks(bs, _ffi.ptr(bset_blocks), _ffi.ptr(idx.contiguous()), n, _ffi.ptr(out),
                                        _ffi.stream_handle(torch.cuda.current_stream(idx.device))),
                   "qm_gather_blocks")
    return out


def _transposed_blocks(blocks: torch.Tensor) -> torch.Tensor:
    lib = _ffi.load()
    n = int(blocks.shape[0])
    bs = int(blocks.shape[1])
    out = torch.empty_like(blocks)
    if n:
        _ffi.check(lib.qm_transpose_blocks(bs, _ffi.ptr(blocks), n, _ffi.ptr(out),
                                           _ffi.stream_handle(torch.cuda.current_stream(blocks.device))),
                   "qm_transpose_blocks")
    return out


def _sorted(keys: torch.Tensor, blocks: torch.Tensor, sumsq: torch.Tensor, masks=None,
            masks_full=(False, False)) -> BlockSet:
    order = torch.argsort(keys, stable=True)
    out = BlockSet(keys[order].contiguous(), _gather(blocks, order), sumsq[order].contiguous())
    if masks is not None:  # support masks follow their blocks (no mask pass on the derived set)
        out.masks, out.masks_full = masks[:, order].contiguous(), masks_full
    return out


class BlockView(BlockSet):
    """A virtual block set over a stored pool: entry m is the pool's block src[m] & 0x7fffffff,
    transposed when bit 31 of src[m] is set (src: int32). Keys, norms and support masks are the
    view's own; `blocks` is the pool's tensor (never indexed by view position on the host). The
    numeric kernel reads transposed entries through a transposed TMA box / fragment addressing
    (qm_numeric_masked with QM_NUMERIC_TRANSPOSED_REFS) -- the reference's virtual transposes
    (`_virtual_child`, ops.py:100-116), never materialised."""

    def __init__(self, keys, pool: BlockSet, src: torch.Tensor, sumsq: torch.Tensor, tsel: torch.Tensor):
        super().__init__(keys, pool.blocks, sumsq)
        self.pool, self.src, self._tsel = pool, src, tsel  # tsel: bool[n], entry is transposed
        self._any_t = True  # some entry is transposed (every view built here has one)

    def support_masks(self, stream=None) -> torch.Tensor:
        if self.masks is None:
            pm = self.pool.support_masks(stream)
            idx = (self.src.long() & 0x7FFFFFFF)
            rows, cols = pm[0][idx], pm[1][idx]
            self.masks = torch.stack([torch.where(self._tsel, cols, rows), torch.where(self._tsel, rows, cols),
                                      pm[2][idx]])
            fr, fc = self.pool.masks_full
            both = fr and fc
            self.masks_full = (both, both) if self._any_t else (fr, fc)
        return self.masks


def _src32(idx: torch.Tensor, tsel: torch.Tensor) -> torch.Tensor:
    """int32 view entries: stored index, bit 31 set for a transposed use (two's complement)."""
    return torch.where(tsel, idx - (1 << 31), idx).to(torch.int32)


def virtual_ok(bs: int) -> bool:
    """Transposes stay virtual when the bs 32/64/128 TMA kernel runs the product
    (QM_VIRTUAL_TRANSPOSE=0 materialises them, for A/B comparisons)."""
    import os  # noqa: PLC0415

    return bs in (32, 64, 128) and _ffi.load().qm_numeric_path(bs) == 2 and \
        os.environ.get("QM_VIRTUAL_TRANSPOSE", "1") != "0"


def transpose_view(geom: Geometry, x: BlockSet) -> BlockSet:
    """X^T as a view of X's blocks (keys swapped and re-sorted, every entry's transpose flag
    toggled; X may itself be a view)."""
    if x.n == 0:
        return x
    bi, bj = _decode(geom, x.keys)
    keys = _encode(geom, bj, bi)
    order = torch.argsort(keys, stable=True)
    if isinstance(x, BlockView):
        pool, idx, tsel = x.pool, (x.src.long() & 0x7FFFFFFF)[order], ~x._tsel[order]
    else:
        pool, idx, tsel = x, order, torch.ones(x.n, dtype=torch.bool, device=keys.device)
    return BlockView(keys[order].contiguous(), pool, _src32(idx, tsel), x.sumsq[order].contiguous(), tsel)


def expand_symmetric_view(geom: Geometry, s: BlockSet) -> BlockSet:
    """expand_symmetric as a view: the stored blocks plus transposed references for the blocks of
    strictly-upper leaves, no block copied."""
    if s.n == 0:
        return s
    bi, bj = _decode(geom, s.keys)
    off = (bi // geom.nbl) < (bj // geom.nbl)
    # the count through mapped memory (torch.nonzero's own read-back would use a copy engine)
    n_off = _ffi.read_i64s(off.sum().reshape(1).to(torch.int64), 1)[0]
    if n_off == 0:
        return s
    idx = torch.nonzero_static(off, size=n_off).flatten()
    tk = _encode(geom, bj[idx], bi[idx])
    keys = torch.cat([s.keys, tk])
    order = torch.argsort(keys, stable=True)
    src = torch.cat([torch.arange(s.n, dtype=torch.int64, device=keys.device), idx])[order]
    tsel = order >= s.n
    view = BlockView(keys[order].contiguous(), s, _src32(src, tsel), s.sumsq[src].contiguous(), tsel)
    view._any_t = True
    return view


def transpose(geom: Geometry, x: BlockSet) -> BlockSet:
    """X^T as a block set (the virtual transpose of op_view / tb=True, materialised)."""
    if x.n == 0:
        return x
    bi, bj = _decode(geom, x.keys)
    keys = _encode(geom, bj, bi)
    m = x.masks[[1, 0, 2]] if x.masks is not None else None  # a transposed block swaps row / column supports
    return _sorted(keys, _transposed_blocks(x.blocks), x.sumsq, m, (x.masks_full[1], x.masks_full[0]))


def expand_symmetric(geom: Geometry, s: BlockSet) -> BlockSet:
    """Full matrix of an upper-stored symmetric block set: adds B(bj,bi) = B(bi,bj)^T for every
    block of a strictly-upper leaf (diagonal leaves already hold both triangles)."""
    if s.n == 0:
        return s
    bi, bj = _decode(geom, s.keys)
    nbl = geom.nbl
    off = (bi // nbl) < (bj // nbl)
    idx = torch.nonzero(off).flatten()
    if idx.numel() == 0:
        return s
    tk = _encode(geom, bj[idx], bi[idx])
    keys = torch.cat([s.keys, tk])
    order = torch.argsort(keys, stable=True)
    src = torch.cat([torch.arange(s.n, dtype=torch.int64, device=keys.device), idx])[order].contiguous()
    tflag = (order >= s.n).to(torch.uint8)  # the appended entries are the transposed copies
    n = int(order.shape[0])
    blocks = torch.empty((n, s.bs, s.bs), dtype=torch.float64, device=keys.device)
    _ffi.check(_ffi.load().qm_gather_blocks_t(s.bs, _ffi.ptr(s.blocks), _ffi.ptr(src), _ffi.ptr(tflag), n,
                                              _ffi.ptr(blocks),
                                              _ffi.stream_handle(torch.cuda.current_stream(keys.device))),
               "qm_gather_blocks_t")
    out = BlockSet(keys[order].contiguous(), blocks, s.sumsq[src].contiguous())
    if s.masks is not None:  # copies swap row / column supports
        m = torch.cat([s.masks, s.masks[[1, 0, 2]][:, idx]], dim=1)
        both = s.masks_full[0] and s.masks_full[1]
        out.masks, out.masks_full = m[:, order].contiguous(), (both, both)
    return out

