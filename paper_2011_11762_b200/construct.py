"""Host-side construction of block sets (the caller side of the path).

``blocks_from_triplets`` reproduces the reference's normalised build bit for bit:
quadtree.build_from_triplets (quadtree.py:90-142) partitions entries by quadrant, keeping their
input order, and BlockSparseLeaf.from_triplets (leaves/block_sparse.py:47-68) stable-sorts a leaf's
entries by block and sums duplicates with ``np.add.at`` into a zero block, dropping blocks that are
exactly zero (``np.any``, :37-41). A single stable sort by quadtree key yields the same per-block
entry order, so duplicate sums are identical; the result is the stored block set in key order.
"""

from __future__ import annotations

import numpy as np

from .errors import ContractViolationError, OutOfRangeError
from .layout import Geometry


def _check_range(n_logical: int, rows: np.ndarray, cols: np.ndarray):
    if rows.size and (
        rows.min() < 0 or rows.max() >= n_logical or cols.min() < 0 or cols.max() >= n_logical
    ):
        raise OutOfRangeError(f"entry index outside [0, {n_logical})")


def mirror_symmetric(rows, cols, vals, leaf_dim: int):
    """session.py:88-100: symmetric input is upper-triangle triplets; entries inside a diagonal
    leaf tile are mirrored so diagonal leaves hold full blocks."""
    if np.any(rows > cols):
        raise ContractViolationError("symmetric matrices are built from upper-triangle triplets")
    mirror = (rows != cols) & (rows // leaf_dim == cols // leaf_dim)
    return (
        np.concatenate([rows, cols[mirror]]),
        np.concatenate([cols, rows[mirror]]),
        np.concatenate([vals, vals[mirror]]),
    )


def blocks_from_triplets(geom: Geometry, rows, cols, vals):
    """Returns (keys int64[n], blocks float64[n,bs,bs]) of the stored (nonzero) blocks."""
    rows = np.asarray(rows, dtype=np.int64).ravel()
    cols = np.asarray(cols, dtype=np.int64).ravel()
    vals = np.asarray(vals, dtype=np.float64).ravel()
    _check_range(geom.params.n_logical, rows, cols)
    bs = geom.bs
    if rows.size == 0:
        return np.zeros(0, np.int64), np.zeros((0, bs, bs))
    bi, lr = np.divmod(rows, bs)
    bj, lc = np.divmod(cols, bs)
    key = geom.qkey(bi, bj)
    order = np.argsort(key, kind="stable")
    ks = key[order]
    starts = np.flatnonzero(np.concatenate([[True], ks[1:] != ks[:-1]]))
    ukeys = ks[starts]
    blk_of = np.repeat(np.arange(starts.size), np.diff(np.append(starts, ks.size)))
    flat = blk_of * (bs * bs) + lr[order] * bs + lc[order]
    buf = np.zeros(starts.size * bs * bs)
    v = vals[order]
    if np.unique(flat).size == flat.size:
        buf[flat] = v + 0.0  # 0.0 + v as np.add.at does (turns -0.0 into +0.0)
    else:
        np.add.at(buf, flat, v)
    blocks = buf.reshape(starts.size, bs, bs)
    keep = np.any(blocks != 0.0, axis=(1, 2)) | np.isnan(blocks).any(axis=(1, 2))
    return ukeys[keep], np.ascontiguousarray(blocks[keep])


def blocks_from_tiles(geom: Geometry, tile_fn, support_fn):
    """quadtree.build_from_tiles (quadtree.py:145-193) for block-sparse leaves: walks the tree,
    skipping subtrees without support, and cuts each leaf tile into blocks (from_dense,
    block_sparse.py:70-83). Returns (keys, blocks) in key order."""
    p = geom.params
    bs, nbl = geom.bs, geom.nbl
    keys, blocks = [], []

    def build(level, r0, c0):
        dim = p.node_dim(level)
        if r0 >= p.n_logical or c0 >= p.n_logical:
            return
        if not support_fn(r0, min(r0 + dim, p.n_logical), c0, min(c0 + dim, p.n_logical)):
            return
        if level == p.depth:
            tile = tile_fn(r0, c0)
            if tile is None or not np.any(tile):
                return
            t = np.asarray(tile, dtype=np.float64).reshape(nbl, bs, nbl, bs).transpose(0, 2, 1, 3)
            for bi in range(nbl):
                for bj in range(nbl):
                    blk = t[bi, bj]
                    if np.any(blk):
                        keys.append(geom.qkey(r0 // bs + bi, c0 // bs + bj))
                        blocks.append(np.ascontiguousarray(blk))
            return
        half = dim // 2
        for dr, dc in ((0, 0), (0, half), (half, 0), (half, half)):
            build(level + 1, r0 + dr, c0 + dc)

    build(0, 0, 0)
    if not keys:
        return np.zeros(0, np.int64), np.zeros((0, bs, bs))
    return np.asarray(keys, dtype=np.int64).ravel(), np.stack(blocks)


def identity_triplets(n: int, c: float):
    """add_scaled_identity on a nil matrix (ops.py:253-270): c on the logical diagonal only."""
    d = np.arange(n, dtype=np.int64)
    return d, d, np.full(n, float(c))


def blocks_from_triplets_device(geom: Geometry, rows, cols, vals, device, stream=None):
    """Device build (libqmb200 qm_build_count / qm_build_fill / qm_compact): the same blocks as
    ``blocks_from_triplets`` bit for bit, as a BlockSet on ``device``."""
    import ctypes

    import torch

    from . import _ffi
    from .blocks import BlockSet

    lib = _ffi.load()
    dev = torch.device(device)
    bs = geom.bs
    r = torch.as_tensor(np.ascontiguousarray(rows, dtype=np.int64).ravel()).to(dev)
    c = torch.as_tensor(np.ascontiguousarray(cols, dtype=np.int64).ravel()).to(dev)
    v = torch.as_tensor(np.ascontiguousarray(vals, dtype=np.float64).ravel()).to(dev)
    n = int(r.shape[0])
    if n == 0:
        return BlockSet.empty(bs, dev)
    layout = _ffi.make_layout(geom.params, bs)
    lp = ctypes.byref(layout)
    with torch.cuda.device(dev):
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        sh = _ffi.stream_handle(st)
        wb = lib.qm_build_workspace_bytes(lp, n)
        ws = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
        nb = ctypes.c_int64(0)
        bad = ctypes.c_int64(0)
        _ffi.check(lib.qm_build_count(lp, _ffi.ptr(r), _ffi.ptr(c), n, _ffi.ptr(ws), wb,
                                      ctypes.byref(nb), ctypes.byref(bad), sh), "qm_build_count")
        if bad.value:
            raise OutOfRangeError(f"entry index outside [0, {geom.params.n_logical})")
        nblk = int(nb.value)
        out = BlockSet(torch.empty(nblk, dtype=torch.int64, device=dev),
                       torch.empty((nblk, bs, bs), dtype=torch.float64, device=dev),
                       torch.empty(nblk, dtype=torch.float64, device=dev))
        nz = torch.empty(nblk, dtype=torch.uint8, device=dev)
        zc = torch.zeros(3, dtype=torch.int64, device=dev)  # [exact-zero blocks, rows not full, cols not full]
        masks = torch.empty((3, nblk), dtype=torch.int64, device=dev)
        # norms, nonzero flags and support masks in one pass over the filled blocks
        _ffi.check(lib.qm_build_fill_meta(lp, _ffi.ptr(v), n, _ffi.ptr(ws), wb, nblk, _ffi.ptr(out.keys),
                                          _ffi.ptr(out.blocks), _ffi.ptr(out.sumsq), _ffi.ptr(nz),
                                          _ffi.ptr(zc), _ffi.ptr(masks), _ffi.ptr(zc[1:]), sh),
                   "qm_build_fill_meta")
        n_zero, nf_r, nf_c = _ffi.read_i64s(zc, 3, st)
        if n_zero:
            from .spgemm import compact  # noqa: PLC0415

            out = compact(bs, out, nz, n_zero, st)  # masks are recomputed on first use
        else:
            out.masks, out.masks_full = masks, (nf_r == 0, nf_c == 0)
    return out
