"""Inspection and wire-format bridge between device block sets and the reference's quadtree.

The reference inspects matrices by walking chunk trees: canonical_bytes (quadtree.py:293-318),
tree_to_dense (:321-345), tree_stats (:255-273), get_elements (:225-252). A block set in quadtree
key order *is* that tree flattened: every subtree is a contiguous key range and a leaf is the run
of keys sharing ``key >> 2*lbits``. These functions rebuild the reference's byte formats
(codec.py:22-50 node header ``<BBI`` + branch ``<4Q4d``; BlockSparseLeaf.encode ``<cIII`` +
per block ``<IId`` + row-major payload, block_sparse.py:226-231) from that flat form, so results
can be compared byte for byte with the reference and handed back to it.
"""

from __future__ import annotations

import math
import struct

import numpy as np

from .errors import OutOfRangeError
from .layout import Geometry, MatrixParams, TreeStats

_HDR = struct.Struct("<BBI")        # codec.py:26  version, node type, level
_BRANCH_BODY = struct.Struct("<4Q4d")
_LEAF_HDR = struct.Struct("<cIII")  # block_sparse.py:18  tag, n, bs, count
_BLK = struct.Struct("<IId")        # block_sparse.py:19  bi, bj, norm
VERSION, BRANCH, LEAF = 1, 1, 2


def leaf_runs(geom: Geometry, keys: np.ndarray):
    """(leaf Morton ids, start offsets, end offsets) of the leaves present in ``keys``."""
    if keys.size == 0:
        z = np.zeros(0, np.int64)
        return z, z, z
    leaf = keys >> np.int64(geom.leaf_key_shift())
    starts = np.flatnonzero(np.concatenate([[True], leaf[1:] != leaf[:-1]]))
    ends = np.append(starts[1:], keys.size)
    return leaf[starts], starts, ends


def encode_leaf(geom: Geometry, keys: np.ndarray, blocks: np.ndarray) -> bytes:
    """BlockSparseLeaf.encode for one leaf's run of blocks (norms via np.linalg.norm, as
    _set_block computes them, so the bytes equal the reference's)."""
    bi, bj = geom.decode(keys)
    nbl = geom.nbl
    parts = [_LEAF_HDR.pack(b"B", geom.params.leaf_dim, geom.bs, int(keys.size))]
    for x in range(keys.size):
        blk = np.ascontiguousarray(blocks[x], dtype=np.float64)
        parts.append(_BLK.pack(int(bi[x] % nbl), int(bj[x] % nbl), float(np.linalg.norm(blk))))
        parts.append(blk.tobytes(order="C"))
    return b"".join(parts)


def _walk(geom: Geometry, leaves: np.ndarray, visit_leaf, visit_branch, visit_nil, explicit_zero=False):
    """Depth-first NW, NE, SW, SE walk over the leaf Morton ids (quadtree.py:125-135)."""
    depth = geom.params.depth

    def rec(level, prefix, lo, hi):
        if lo == hi and not explicit_zero:
            return visit_nil()
        if level == depth:
            return visit_leaf(level, prefix, lo, hi)
        shift = 2 * (depth - level - 1)
        bounds = [lo]
        for q in range(1, 4):
            bounds.append(int(np.searchsorted(leaves[lo:hi], (prefix * 4 + q) << shift)) + lo)
        bounds.append(hi)
        kids = [rec(level + 1, prefix * 4 + q, bounds[q], bounds[q + 1]) for q in range(4)]
        return visit_branch(level, kids)

    return rec(0, 0, 0, leaves.size)


def canonical_bytes(geom: Geometry, keys: np.ndarray, blocks: np.ndarray, explicit_zero=False) -> bytes:
    """quadtree.canonical_bytes (quadtree.py:293-318) of the matrix held as a flat block set.

    Block norms are computed with single-threaded BLAS: np.linalg.norm is a ddot, which OpenBLAS
    threads (changing the summation order) above ~10^4 elements. The reference's bench and golden
    runs hold BLAS at one thread (bench.py:117 threadpool_limits(1)); so does this bridge.
    """
    from threadpoolctl import threadpool_limits  # noqa: PLC0415

    with threadpool_limits(limits=1, user_api="blas"):
        return _canonical_bytes(geom, keys, blocks, explicit_zero)


def _canonical_bytes(geom: Geometry, keys: np.ndarray, blocks: np.ndarray, explicit_zero=False) -> bytes:
    leaves, starts, ends = leaf_runs(geom, keys)
    parts: list[bytes] = []
    empty_leaf = _LEAF_HDR.pack(b"B", geom.params.leaf_dim, geom.bs, 0)
    depth = geom.params.depth

    def walk(level, prefix, lo, hi):
        if lo == hi and not explicit_zero:
            parts.append(b"N")
            return
        if level == depth:
            parts.append(b"L")
            parts.append(level.to_bytes(4, "little"))
            if lo == hi:
                parts.append(empty_leaf)
            else:
                s, e = starts[lo], ends[lo]
                parts.append(encode_leaf(geom, keys[s:e], blocks[s:e]))
            return
        parts.append(b"B")
        parts.append(level.to_bytes(4, "little"))
        shift = 2 * (depth - level - 1)
        bounds = [lo]
        for q in range(1, 4):
            bounds.append(int(np.searchsorted(leaves[lo:hi], (prefix * 4 + q) << shift)) + lo)
        bounds.append(hi)
        for q in range(4):
            walk(level + 1, prefix * 4 + q, bounds[q], bounds[q + 1])

    walk(0, 0, 0, leaves.size)
    return b"".join(parts)


def tree_stats(geom: Geometry, keys: np.ndarray, blocks: np.ndarray, explicit_zero=False) -> TreeStats:
    """quadtree.tree_stats (quadtree.py:255-273): chunk counts, encoded bytes, nonzeros."""
    stats = TreeStats()
    leaves, starts, ends = leaf_runs(geom, keys)
    bs2 = geom.bs * geom.bs

    def on_leaf(level, prefix, lo, hi):
        stats.n_leaf_chunks += 1
        count = 0 if lo == hi else int(ends[lo] - starts[lo])
        stats.stored_bytes += _HDR.size + _LEAF_HDR.size + count * (_BLK.size + 8 * bs2)
        return True

    def on_branch(level, kids):
        if not any(kids) and not explicit_zero:
            return False
        stats.n_branch_chunks += 1
        stats.stored_bytes += _HDR.size + _BRANCH_BODY.size
        return True

    _walk(geom, leaves, on_leaf, on_branch, lambda: False, explicit_zero)
    stats.nnz = int(np.count_nonzero(blocks)) if blocks.size else 0
    return stats


def tree_norm(geom: Geometry, keys: np.ndarray, sumsq: np.ndarray) -> float:
    """Root norm as the store carries it: leaf = sqrt(fsum(block norm^2)), branch =
    sqrt(fsum(child norm^2)) (quadtree.py:124,138-140; block_sparse.py:91-92)."""
    leaves, starts, ends = leaf_runs(geom, keys)
    bn = np.sqrt(np.asarray(sumsq, dtype=np.float64))

    def on_leaf(level, prefix, lo, hi):
        s, e = starts[lo], ends[lo]
        return math.sqrt(math.fsum(float(v) * float(v) for v in bn[s:e]))

    def on_branch(level, kids):
        return math.sqrt(math.fsum(x * x for x in kids))

    if leaves.size == 0:
        return 0.0
    return _walk(geom, leaves, on_leaf, on_branch, lambda: 0.0)


def to_dense(geom: Geometry, keys: np.ndarray, blocks: np.ndarray, symmetric: bool = False) -> np.ndarray:
    """quadtree.tree_to_dense (quadtree.py:321-345)."""
    p: MatrixParams = geom.params
    bs = geom.bs
    out = np.zeros((p.n_padded, p.n_padded))
    if keys.size:
        bi, bj = geom.decode(keys)
        view = out.reshape(p.n_padded // bs, bs, p.n_padded // bs, bs)
        view[bi, :, bj, :] = blocks
    out = out[: p.n_logical, : p.n_logical]
    if symmetric:
        out = np.triu(out) + np.triu(out, 1).T
    return np.ascontiguousarray(out)


def get_elements(geom: Geometry, keys: np.ndarray, blocks: np.ndarray, rows, cols) -> np.ndarray:
    """quadtree.get_elements (quadtree.py:225-252)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    n = geom.params.n_logical
    if rows.size and (rows.min() < 0 or rows.max() >= n or cols.min() < 0 or cols.max() >= n):
        raise OutOfRangeError(f"probe index outside [0, {n})")
    out = np.zeros(rows.shape[0])
    if keys.size == 0 or rows.size == 0:
        return out
    bs = geom.bs
    want = geom.qkey(rows // bs, cols // bs)
    pos = np.searchsorted(keys, want)
    pos_c = np.minimum(pos, keys.size - 1)
    hit = keys[pos_c] == want
    out[hit] = blocks[pos_c[hit], rows[hit] % bs, cols[hit] % bs]
    return out


# ---- interop with a live reference quadmat session (test / integration helper) ----------------

def from_reference_store(geom: Geometry, store, root) -> tuple[np.ndarray, np.ndarray]:
    """Reads a reference quadtree (chunk ids in ``store``) into (keys, blocks) in key order."""
    from quadmat import codec  # noqa: PLC0415  (reference package; only in this container)

    keys, blocks = [], []
    nbl, bs = geom.nbl, geom.bs
    depth = geom.params.depth

    def walk(cid, level, li, lj):
        if cid.is_nil:
            return
        node = codec.decode_node(store.peek(cid))
        if node[0] == "leaf":
            leaf = node[2]
            for (bi, bj) in sorted(leaf.blocks):
                keys.append(int(geom.qkey(li * nbl + bi, lj * nbl + bj)))
                blocks.append(leaf.blocks[(bi, bj)])
            return
        for q, child in enumerate(node[2]):
            walk(child, level + 1, 2 * li + (q >> 1), 2 * lj + (q & 1))

    walk(root, 0, 0, 0)
    _ = depth
    if not keys:
        return np.zeros(0, np.int64), np.zeros((0, bs, bs))
    return np.asarray(keys, dtype=np.int64), np.stack(blocks)


def to_reference_store(geom: Geometry, store, keys: np.ndarray, blocks: np.ndarray, owner: int = 0):
    """Registers a block set as a normalised reference quadtree; returns the root ChunkId."""
    from quadmat import NIL, codec  # noqa: PLC0415
    from quadmat.leaves import BlockSparseLeaf  # noqa: PLC0415

    leaves, starts, ends = leaf_runs(geom, keys)
    nbl = geom.nbl

    def on_leaf(level, prefix, lo, hi):
        s, e = starts[lo], ends[lo]
        bi, bj = geom.decode(keys[s:e])
        leaf = BlockSparseLeaf(geom.params.leaf_dim, geom.bs)
        for x in range(e - s):
            leaf._set_block((int(bi[x] % nbl), int(bj[x] % nbl)), blocks[s + x])
        payload = codec.encode_leaf_node(level, leaf)
        return store.register(payload, owner, leaf.norm_frobenius())

    def on_branch(level, kids):
        if all(k.is_nil for k in kids):
            return NIL
        norms = [store.norm_of(k) for k in kids]
        payload = codec.encode_branch(level, kids, norms)
        return store.register(payload, owner, math.sqrt(math.fsum(x * x for x in norms)))

    if leaves.size == 0:
        return NIL
    return _walk(geom, leaves, on_leaf, on_branch, lambda: NIL)
