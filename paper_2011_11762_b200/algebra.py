"""The step after a product: add, scale, add_scaled_identity, truncate on device
block sets, with the reference's exact semantics.

Reference: session.py:148-185; ops.py:147-190 (add / scale with their nil fallbacks), 253-345
(add_scaled_identity), 388-454 + 637-650 (two-pass global truncation: census of block norms,
greedy ascending-norm drop plan, rewrite); leaves/block_sparse.py:134-224.

Block arithmetic runs in libqmb200 (qm_axpby_blocks, qm_add_identity_blocks) with exact IEEE
products and sums (no FMA contraction), so results are bit-identical to numpy's; exact-zero blocks
are dropped (_set_block). Key merging and the truncation ordering use torch on the device; the
greedy prefix sum of the truncation plan runs sequentially on the host (np.cumsum), as the
reference's loop does, so the drop decision at the threshold matches.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _ffi
from .blocks import BlockSet
from .layout import Geometry


def _stream(dev):
    return _ffi.stream_handle(torch.cuda.current_stream(dev))


def _drop_zero_blocks(bs: int, c: BlockSet, nz: torch.Tensor | None = None,
                      zero_count: torch.Tensor | None = None) -> BlockSet:
    """Drops exactly-zero blocks (_set_block). `nz`/`zero_count` come fused from qm_axpby_blocks;
    otherwise qm_block_stats computes them (and c.sumsq)."""
    from .spgemm import compact

    if c.n == 0:
        return c
    lib = _ffi.load()
    if nz is None:
        nz = torch.empty(c.n, dtype=torch.uint8, device=c.device)
        _ffi.check(lib.qm_block_stats(bs, c.n, _ffi.ptr(c.blocks), _ffi.ptr(c.sumsq), _ffi.ptr(nz),
                                      _stream(c.device)), "qm_block_stats")
        zero_count = (nz == 0).sum().reshape(1).to(torch.int64)
    n_zero = _ffi.read_i64(zero_count)
    return compact(bs, c, nz, n_zero)


def _leaf_ids(geom: Geometry, keys: torch.Tensor) -> torch.Tensor:
    return keys >> (2 * geom.lbits)


def _member(sorted_vals: torch.Tensor, q: torch.Tensor) -> torch.Tensor:
    if sorted_vals.numel() == 0:
        return torch.zeros_like(q, dtype=torch.bool)
    pos = torch.searchsorted(sorted_vals, q).clamp(max=sorted_vals.numel() - 1)
    return sorted_vals[pos] == q


def _axpby(bs, ia, ib, alpha, beta, A, B, out_keys) -> BlockSet:
    """alpha*A[ia] + beta*B[ib] with the output's norms and zero flags fused; exact-zero blocks
    dropped."""
    lib = _ffi.load()
    n = int(ia.shape[0])
    dev = out_keys.device
    out = torch.empty((n, bs, bs), dtype=torch.float64, device=dev)
    sumsq = torch.empty(n, dtype=torch.float64, device=dev)
    nz = torch.empty(n, dtype=torch.uint8, device=dev)
    zc = torch.zeros(1, dtype=torch.int64, device=dev)
    _ffi.check(lib.qm_axpby_blocks(bs, n, _ffi.ptr(ia.contiguous()), _ffi.ptr(ib.contiguous()), alpha,
                                   beta, _ffi.ptr(A), _ffi.ptr(B), _ffi.ptr(out), _ffi.ptr(sumsq),
                                   _ffi.ptr(nz), _ffi.ptr(zc), _stream(dev)),
               "qm_axpby_blocks")
    return _drop_zero_blocks(bs, BlockSet(out_keys.contiguous(), out, sumsq), nz, zc)


def add(geom: Geometry, a: BlockSet, b: BlockSet, alpha: float, beta: float) -> BlockSet:
    """alpha*A + beta*B for two non-empty block sets (nil operands are handled by the caller,
    as _add_fallback does)."""
    bs = geom.bs
    if alpha == 1.0 and beta == 0.0:  # BlockSparseLeaf.add returns self; B-only leaves scale to nil
        return a
    keys = torch.unique(torch.cat([a.keys, b.keys]))
    n = int(keys.shape[0])
    dev = keys.device
    ia = torch.full((n,), -1, dtype=torch.int64, device=dev)
    ib = torch.full((n,), -1, dtype=torch.int64, device=dev)
    ia[torch.searchsorted(keys, a.keys)] = torch.arange(a.n, device=dev)
    ib[torch.searchsorted(keys, b.keys)] = torch.arange(b.n, device=dev)
    if alpha == 0.0 or beta == 0.0:
        # a leaf present in only one operand takes the fallback path: scale by 0 gives nil
        lk = _leaf_ids(geom, keys)
        la, lb = torch.unique(_leaf_ids(geom, a.keys)), torch.unique(_leaf_ids(geom, b.keys))
        keep = torch.ones(n, dtype=torch.bool, device=dev)
        if alpha == 0.0:
            keep &= ~(_member(la, lk) & ~_member(lb, lk))
        if beta == 0.0:
            keep &= ~(_member(lb, lk) & ~_member(la, lk))
        keys, ia, ib = keys[keep], ia[keep], ib[keep]
    return _axpby(bs, ia, ib, alpha, beta, a.blocks, b.blocks, keys)


def scale(geom: Geometry, a: BlockSet, alpha: float) -> BlockSet:
    """alpha*A (alpha not in {0, 1}; those are identity / nil at the caller, ops.py:172-185)."""
    ia = torch.arange(a.n, device=a.device)
    ib = torch.full_like(ia, -1)
    return _axpby(geom.bs, ia, ib, alpha, 0.0, a.blocks, a.blocks, a.keys)


def add_scaled_identity(geom: Geometry, a: BlockSet | None, c: float, device) -> BlockSet:
    """A + c*I on the logical diagonal (ops.py:253-345). `a` may be None (nil)."""
    from .variants import _encode

    bs, nbl = geom.bs, geom.nbl
    p = geom.params
    dev = torch.device(device)
    nbd = -(-p.n_logical // bs)  # diagonal blocks touching the logical range
    bi = torch.arange(nbd, dtype=torch.int64, device=dev)
    dkeys = _encode(geom, bi.to(torch.int32), bi.to(torch.int32))
    li = bi // nbl
    full_leaf = (li + 1) * p.leaf_dim <= p.n_logical
    if a is not None and a.n:
        leaves = torch.unique(_leaf_ids(geom, a.keys))
        present = _member(leaves, _leaf_ids(geom, dkeys))
        pos = torch.searchsorted(a.keys, dkeys).clamp(max=a.n - 1)
        ia = torch.where(a.keys[pos] == dkeys, pos, torch.full_like(pos, -1))
        blocks_a = a.blocks
    else:
        present = torch.zeros(nbd, dtype=torch.bool, device=dev)
        ia = torch.full((nbd,), -1, dtype=torch.int64, device=dev)
        blocks_a = torch.empty((1, bs, bs), dtype=torch.float64, device=dev)
    mode = torch.where(present & full_leaf, 0, 1).to(torch.int8)
    lib = _ffi.load()
    diag = torch.empty((nbd, bs, bs), dtype=torch.float64, device=dev)
    _ffi.check(lib.qm_add_identity_blocks(bs, nbd, _ffi.ptr(ia.contiguous()), _ffi.ptr(bi), _ffi.ptr(mode.contiguous()),
                                          float(c), p.n_logical, _ffi.ptr(blocks_a), _ffi.ptr(diag),
                                          _stream(dev)), "qm_add_identity_blocks")
    new = _drop_zero_blocks(bs, BlockSet(dkeys, diag, torch.empty(nbd, dtype=torch.float64, device=dev)))
    if a is None or a.n == 0:
        return new
    rest = ~_member(dkeys.sort().values, a.keys)
    keys = torch.cat([a.keys[rest], new.keys])
    order = torch.argsort(keys)
    blocks = torch.cat([a.blocks[rest], new.blocks])[order].contiguous()
    sumsq = torch.cat([a.sumsq[rest], new.sumsq])[order].contiguous()
    return BlockSet(keys[order].contiguous(), blocks, sumsq)


def _repr_rank(nbl: int) -> np.ndarray:
    """Rank of repr((bi, bj)) in string order for local keys (the reference sorts census items by
    (norm, path, repr(key)), ops.py:637-650)."""
    keys = [(i, j) for i in range(nbl) for j in range(nbl)]
    order = sorted(range(len(keys)), key=lambda t: repr(keys[t]))
    rank = np.empty(len(keys), dtype=np.int64)
    rank[order] = np.arange(len(keys))
    return rank


def truncate(geom: Geometry, a: BlockSet, tau: float, symmetric: bool) -> tuple[BlockSet, float]:
    """Two-pass global truncation (session.py:173-185): census of block norms, greedy ascending-norm
    prefix whose sum of squares stays <= tau^2, drop. Returns (kept blocks, removed norm)."""
    from .variants import _decode, _gather

    dev = a.device
    nbl = geom.nbl
    bi, bj = _decode(geom, a.keys)
    bi, bj = bi.to(torch.int64), bj.to(torch.int64)
    li, lj = bi // nbl, bj // nbl
    norm = torch.sqrt(a.sumsq)
    leaf = _leaf_ids(geom, a.keys)
    lbi, lbj = bi - li * nbl, bj - lj * nbl
    rank = torch.as_tensor(_repr_rank(nbl), device=dev)
    if symmetric:
        # ops.py:388-401: diagonal leaves -> sym_block_items (mirror pairs (lo, hi) combined as
        # sqrt(a*a + b*b), block_sparse.py:205-217); other leaves -> block norm * sqrt(2)
        diag = li == lj
        lo, hi = torch.minimum(lbi, lbj), torch.maximum(lbi, lbj)
        item_local = torch.where(diag, lo * nbl + hi, lbi * nbl + lbj)
        item = leaf * (nbl * nbl) + item_local
        uitem, inv = torch.unique(item, return_inverse=True)
        ni = uitem.shape[0]
        na = torch.zeros(ni, dtype=torch.float64, device=dev)  # norm of (lo, hi)
        nb = torch.zeros(ni, dtype=torch.float64, device=dev)  # norm of (hi, lo)
        upper_blk = (lbi <= lbj) | ~diag
        na[inv[upper_blk]] = norm[upper_blk]
        low = ~upper_blk
        nb[inv[low]] = norm[low]
        idiag = torch.zeros(ni, dtype=torch.bool, device=dev)
        idiag[inv[diag]] = True
        inorm = torch.where(idiag, torch.sqrt(na * na + nb * nb), na * math.sqrt(2.0))
        ileaf = uitem // (nbl * nbl)
        ilocal = uitem % (nbl * nbl)
    else:
        uitem = leaf * (nbl * nbl) + lbi * nbl + lbj
        inv = torch.arange(a.n, device=dev)
        inorm, ileaf, ilocal = norm, leaf, lbi * nbl + lbj
    # order: (norm, path, repr(key)); path order == leaf Morton order
    o = torch.argsort(rank[ilocal], stable=True)
    o = o[torch.argsort(ileaf[o], stable=True)]
    o = o[torch.argsort(inorm[o], stable=True)]
    sq_sorted = (inorm[o] * inorm[o]).cpu().numpy()
    csum = np.cumsum(sq_sorted)  # sequential, as the reference's loop
    budget = tau * tau
    n_drop = int(np.searchsorted(csum > budget, True)) if csum.size else 0
    if n_drop == 0:
        return a, 0.0
    removed = math.sqrt(float(csum[n_drop - 1]))
    dropped_items = o[:n_drop]
    drop_item = torch.zeros(uitem.shape[0], dtype=torch.bool, device=dev)
    drop_item[dropped_items] = True
    keep = ~drop_item[inv]
    idx = torch.nonzero(keep).flatten()
    out = BlockSet(a.keys[idx].contiguous(), _gather(a.blocks, idx), a.sumsq[idx].contiguous())
    return out, removed
