"""CPU oracle of the block-sparse quadtree multiply -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs may
import this module, and only as the checker or the timed CPU baseline. The product path
(paper_2011_11762_b200) never calls it; without libqmb200 on a GPU the product path raises.

This is a plain-numpy restatement of the reference's regular multiply (arXiv 2011.11762 Python
package ``quadmat``), following:

  * ops.py:197-241 ``_multiply_body``: for each non-nil (A-node, B-node) pair at a level,
    C_ij = add(A_i0*B_0j, A_i1*B_1j); nil operands yield nil (``_multiply_fallback`` :244-245).
    The surviving leaf-level products are the block triples (i, k, j); the sum over the leaf
    k-range is a balanced binary tree over the quadtree halves with absent terms passed through
    (``_add_fallback`` ops.py:162-169).
  * leaves/block_sparse.py:112-132 ``BlockSparseLeaf.multiply``: inside one leaf, for each (i, j)
    the k loop runs ascending with ``acc = prod if acc is None else acc + prod`` and
    ``prod = a @ b`` (numpy matmul -> OpenBLAS dgemm; this oracle calls the same numpy).
  * leaves/block_sparse.py:134-152 ``add`` with alpha = beta = 1.0 (``1.0*a + 1.0*b`` == a + b),
    and :37-41 ``_set_block``: a block that is exactly zero (``not np.any``) is not stored; an
    all-zero leaf is nil (ops.py:119-122).

Parity pin: tests/test_oracle_pin.py checks this restatement against outputs of the reference
itself (tests/golden/*.npz, made by tests/golden/make_golden.py by importing the reference in the
build container): bitwise on the reference's order (same numpy dgemm), and the C block sets exactly.
"""

from __future__ import annotations

import concurrent.futures as cf
import os

import numpy as np


# ---- quadtree key (same definition as paper_2011_11762_b200/layout.py; restated here so the
# ---- oracle does not depend on the product package) ---------------------------------------------

def _spread(x):
    v = np.asarray(x).astype(np.uint64)
    for s, m in ((16, 0x0000FFFF0000FFFF), (8, 0x00FF00FF00FF00FF), (4, 0x0F0F0F0F0F0F0F0F),
                 (2, 0x3333333333333333), (1, 0x5555555555555555)):
        v = (v | (v << np.uint64(s))) & np.uint64(m)
    return v


def _compact(v):
    v = np.asarray(v).astype(np.uint64) & np.uint64(0x5555555555555555)
    for s, m in ((1, 0x3333333333333333), (2, 0x0F0F0F0F0F0F0F0F), (4, 0x00FF00FF00FF00FF),
                 (8, 0x0000FFFF0000FFFF), (16, 0x00000000FFFFFFFF)):
        v = (v | (v >> np.uint64(s))) & np.uint64(m)
    return v


def qkey(bi, bj, nbl: int, lbits: int):
    """Depth-first NW, NE, SW, SE order of leaves (quadtree.py:125-135) then sorted (bi, bj) inside
    a leaf (block_sparse.py:228)."""
    bi = np.asarray(bi, dtype=np.int64)
    bj = np.asarray(bj, dtype=np.int64)
    li, ri = np.divmod(bi, nbl)
    lj, rj = np.divmod(bj, nbl)
    m = (_spread(li) << np.uint64(1)) | _spread(lj)
    return ((m << np.uint64(2 * lbits)) | (ri.astype(np.uint64) << np.uint64(lbits))
            | rj.astype(np.uint64)).astype(np.int64)


def qkey_decode(keys, nbl: int, lbits: int):
    k = np.asarray(keys, dtype=np.int64).astype(np.uint64)
    local = k & np.uint64((1 << (2 * lbits)) - 1)
    ri = (local >> np.uint64(lbits)).astype(np.int64)
    rj = (local & np.uint64((1 << lbits) - 1)).astype(np.int64)
    m = k >> np.uint64(2 * lbits)
    return (_compact(m >> np.uint64(1)).astype(np.int64) * nbl + ri,
            _compact(m).astype(np.int64) * nbl + rj)


class Geom:
    """(leaf_dim, depth, bs) -> nbl, lbits; MatrixParams.create (quadtree.py:30-37)."""

    def __init__(self, n_logical: int, leaf_dim: int, bs: int):
        depth = 0
        while leaf_dim * (1 << depth) < n_logical:
            depth += 1
        self.n_logical, self.leaf_dim, self.depth, self.bs = n_logical, leaf_dim, depth, bs
        self.nbl = leaf_dim // bs
        self.lbits = (self.nbl - 1).bit_length()

    def key(self, bi, bj):
        return qkey(bi, bj, self.nbl, self.lbits)

    def decode(self, keys):
        return qkey_decode(keys, self.nbl, self.lbits)


# ---- symbolic phase -----------------------------------------------------------------------------

def symbolic(geom: Geom, a_keys, b_keys):
    """All block triples of C = A*B grouped by C block (ascending key), k ascending per group.

    Returns (c_keys, c_ptr, tri_a, tri_b, tri_k): C block g owns triples [c_ptr[g], c_ptr[g+1]).
    These are the non-nil leaf-level "multiply" tasks of ops.py:197-241.
    """
    a_keys = np.asarray(a_keys, dtype=np.int64)
    b_keys = np.asarray(b_keys, dtype=np.int64)
    ai, ak = geom.decode(a_keys)
    bk, bj = geom.decode(b_keys)
    border = np.lexsort((bj, bk))  # B rows, columns ascending
    bk_s, bj_s = bk[border], bj[border]
    nb = geom.nbl << geom.depth
    b_rp = np.searchsorted(bk_s, np.arange(nb + 1))
    cnt = b_rp[ak + 1] - b_rp[ak]
    tot = int(cnt.sum())
    if tot == 0:
        z = np.zeros(0, np.int64)
        return z, np.zeros(1, np.int64), z, z, z
    a_rep = np.repeat(np.arange(a_keys.size), cnt)
    starts = np.repeat(b_rp[ak], cnt)
    offs = np.arange(tot) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    b_pos = starts + offs
    tri_a = a_rep
    tri_b = border[b_pos]
    tri_k = ak[a_rep]
    ckey = geom.key(ai[a_rep], bj_s[b_pos])
    order = np.lexsort((tri_k, ckey))
    ckey, tri_a, tri_b, tri_k = ckey[order], tri_a[order], tri_b[order], tri_k[order]
    first = np.concatenate([[True], ckey[1:] != ckey[:-1]])
    c_keys = ckey[first]
    c_ptr = np.append(np.flatnonzero(first), ckey.size).astype(np.int64)
    return c_keys, c_ptr, tri_a, tri_b, tri_k


# ---- numeric phase in the reference's summation order -------------------------------------------

def _reduce_reference_order(geom: Geom, ks: np.ndarray, prods: np.ndarray):
    """Sum of the products of one C block in the reference's order; None if it vanishes.

    Leaf level (block_sparse.py:121-131): k ascending inside one leaf k-range, acc = p / acc + p,
    exact-zero result dropped. Above the leaves (ops.py:213-239): balanced binary tree over the
    leaf k index, add(first_half, second_half) with absent terms passed through and exact-zero
    sums dropped (block_sparse.py:141-151, ops.py:119-122).
    """
    lk = ks // geom.nbl
    leaf_part: dict[int, np.ndarray] = {}
    x = 0
    while x < ks.size:
        y = x
        acc = prods[x]
        y += 1
        while y < ks.size and lk[y] == lk[x]:
            acc = acc + prods[y]
            y += 1
        if np.any(acc):
            leaf_part[int(lk[x])] = acc
        x = y
    if not leaf_part:
        return None
    if len(leaf_part) == 1:
        return next(iter(leaf_part.values()))
    return _tree_sparse(leaf_part, geom.depth)


def _tree_sparse(parts: dict, depth: int):
    """Balanced binary-tree sum over present leaf indices (same association as the recursive
    quadtree add, computed bottom-up over the present indices only)."""
    level_parts = dict(parts)
    for _ in range(depth):
        nxt: dict[int, np.ndarray] = {}
        for idx in sorted(level_parts):
            parent = idx >> 1
            if parent in nxt:
                continue
            lo = level_parts.get(parent * 2)
            hi = level_parts.get(parent * 2 + 1)
            if lo is None:
                s = hi
            elif hi is None:
                s = lo
            else:
                s = 1.0 * lo + 1.0 * hi
                if not np.any(s):
                    s = None
            if s is not None:
                nxt[parent] = s
            else:
                nxt.setdefault(parent, None)
        level_parts = {k: v for k, v in nxt.items() if v is not None}
        if not level_parts:
            return None
    return next(iter(level_parts.values()))


def multiply(geom: Geom, a_keys, a_blocks, b_keys, b_blocks, chunk_triples: int = 8192,
             threads: int = 1, c_subset=None):
    """C = A*B. Returns (c_keys, c_blocks, n_triples) with exactly-zero blocks dropped.

    ``c_subset`` (boolean mask over the symbolic C blocks) restricts the numeric work to a sample
    of C blocks (bench cpu_baseline, sampled verification of large configs).
    """
    c_keys, c_ptr, tri_a, tri_b, tri_k = symbolic(geom, a_keys, b_keys)
    return numeric(geom, c_keys, c_ptr, tri_a, tri_b, tri_k, a_blocks, b_blocks, chunk_triples,
                   threads, c_subset)


def numeric(geom: Geom, c_keys, c_ptr, tri_a, tri_b, tri_k, a_blocks, b_blocks,
            chunk_triples: int = 8192, threads: int = 1, c_subset=None):
    groups = np.arange(c_keys.size) if c_subset is None else np.flatnonzero(c_subset)
    # chunks of whole C blocks, ~chunk_triples products each
    bounds = []
    start = 0
    acc = 0
    for gi, g in enumerate(groups):
        acc += int(c_ptr[g + 1] - c_ptr[g])
        if acc >= chunk_triples:
            bounds.append((start, gi + 1))
            start, acc = gi + 1, 0
    if start < groups.size:
        bounds.append((start, groups.size))

    def run(bound):
        lo, hi = bound
        keys_out, blocks_out = [], []
        for g in groups[lo:hi]:
            t0, t1 = int(c_ptr[g]), int(c_ptr[g + 1])
            prods = np.matmul(a_blocks[tri_a[t0:t1]], b_blocks[tri_b[t0:t1]])
            blk = _reduce_reference_order(geom, tri_k[t0:t1], prods)
            if blk is not None:
                keys_out.append(c_keys[g])
                blocks_out.append(blk)
        return keys_out, blocks_out

    if threads > 1:
        # one BLAS thread per worker: the workers already use every core (nested BLAS threading
        # can only oversubscribe them; on the 16-core GPU host both measure 19.0 GFLOP/s)
        from threadpoolctl import threadpool_limits

        with threadpool_limits(limits=1, user_api="blas"), cf.ThreadPoolExecutor(max_workers=threads) as ex:
            parts = list(ex.map(run, bounds))
    else:
        parts = [run(b) for b in bounds]
    keys = [k for p in parts for k in p[0]]
    blocks = [b for p in parts for b in p[1]]
    bs = geom.bs
    if not keys:
        return np.zeros(0, np.int64), np.zeros((0, bs, bs)), int(tri_a.size)
    return np.asarray(keys, dtype=np.int64), np.stack(blocks), int(tri_a.size)


def rel_frobenius(got: np.ndarray, want: np.ndarray) -> float:
    """Relative Frobenius error (tests/oracles.py:151-155 of the reference)."""
    denom = float(np.linalg.norm(want))
    diff = float(np.linalg.norm(np.asarray(got) - np.asarray(want)))
    return diff if denom == 0.0 else diff / denom


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
