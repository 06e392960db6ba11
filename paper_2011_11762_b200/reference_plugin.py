"""Task-plugin seam: a B200 "multiply" task body for the reference's own engine.

The reference binds operations to task types through ``TaskRegistry.register(name, execute,
fallback)`` (engine.py:69-83); "multiply" is bound to ``_multiply_body`` / ``_multiply_fallback``
(ops.py:197-245, 524) with the body signature ``body(ctx, inputs, args) -> ChunkId`` and the
context API ``fetch / put / norm_of / spawn / log_prune`` (engine.py:105-134).

``install(session)`` re-registers "multiply" on a reference ``quadmat.MatrixSession`` so that a
level-0 regular product of block-sparse trees is computed by libqmb200 in one call: the operand
trees are read through ``ctx.fetch`` into quadtree-key block sets, multiplied on the GPU, and the
result is written back through ``ctx.put`` as a normalised reference tree (codec.py / leaf payload
formats, norms as _set_block computes them). Every other case -- deeper levels, transposed or
symmetric operands, tau > 0, other leaf kinds -- is delegated to the reference's own body, so the
engine, its scheduler, transfer accounting and all other operations are untouched.
"""

from __future__ import annotations

import math

import numpy as np

from .layout import Geometry, MatrixParams


def _decode(fetch, cid):
    from quadmat import codec  # noqa: PLC0415  (the reference package)

    return codec.decode_node(fetch(cid))


def infer_geometry(fetch, root) -> Geometry | None:
    """Leaf dimension, block size and depth of a reference tree (first leaf on a left-most path);
    None for a non-block-sparse tree. n_logical is not stored in the tree; padding is implicit,
    so the padded dimension stands in for it (it does not affect the product)."""
    from quadmat.leaves import BlockSparseLeaf  # noqa: PLC0415

    node = _decode(fetch, root)
    while node[0] != "leaf":
        child = next(c for c in node[2] if not c.is_nil)
        node = _decode(fetch, child)
    leaf, level = node[2], node[1]
    if not isinstance(leaf, BlockSparseLeaf):
        return None
    return Geometry(MatrixParams(leaf.n << level, leaf.n, level), leaf.block_size)


def read_blocks(geom: Geometry, fetch, root):
    """Reference tree -> (keys, blocks) in quadtree-key order."""
    keys, blocks = [], []
    nbl = geom.nbl

    def walk(cid, li, lj):
        if cid.is_nil:
            return
        node = _decode(fetch, cid)
        if node[0] == "leaf":
            leaf = node[2]
            for (bi, bj) in sorted(leaf.blocks):
                keys.append(int(geom.qkey(li * nbl + bi, lj * nbl + bj)))
                blocks.append(leaf.blocks[(bi, bj)])
            return
        for q, child in enumerate(node[2]):
            walk(child, 2 * li + (q >> 1), 2 * lj + (q & 1))

    walk(root, 0, 0)
    if not keys:
        return np.zeros(0, np.int64), np.zeros((0, geom.bs, geom.bs))
    return np.asarray(keys, dtype=np.int64), np.stack(blocks)


def write_tree(geom: Geometry, put, norm_of, keys: np.ndarray, blocks: np.ndarray):
    """(keys, blocks) -> a normalised reference tree registered through ``put``; returns its root."""
    from quadmat import NIL, codec  # noqa: PLC0415
    from quadmat.leaves import BlockSparseLeaf  # noqa: PLC0415

    from .bridge import _walk, leaf_runs  # noqa: PLC0415

    leaves, starts, ends = leaf_runs(geom, keys)
    nbl = geom.nbl

    def on_leaf(level, prefix, lo, hi):
        s, e = starts[lo], ends[lo]
        bi, bj = geom.decode(keys[s:e])
        leaf = BlockSparseLeaf(geom.params.leaf_dim, geom.bs)
        for x in range(e - s):
            leaf._set_block((int(bi[x] % nbl), int(bj[x] % nbl)), blocks[s + x])
        if leaf.is_zero():
            return NIL
        return put(codec.encode_leaf_node(level, leaf), leaf.norm_frobenius())

    def on_branch(level, kids):
        if all(k.is_nil for k in kids):
            return NIL
        norms = [norm_of(k) for k in kids]
        return put(codec.encode_branch(level, kids, norms), math.sqrt(math.fsum(x * x for x in norms)))

    if leaves.size == 0:
        return NIL
    return _walk(geom, leaves, on_leaf, on_branch, lambda: NIL)


def gpu_compute(geom: Geometry, ka, ba, kb, bb):
    """The product on the B200 (libqmb200): host block sets in, host block set out."""
    import torch  # noqa: PLC0415

    from . import _ffi, spgemm  # noqa: PLC0415
    from .blocks import BlockSet  # noqa: PLC0415

    dev = torch.device("cuda")
    c = spgemm.multiply_blocks(_ffi.make_layout(geom.params, geom.bs), BlockSet.from_numpy(ka, ba, None, dev),
                               BlockSet.from_numpy(kb, bb, None, dev))
    kc, bc, _ = c.to_host()
    return kc, bc


def make_multiply_body(compute=None):
    """A reference task body for "multiply"; ``compute(geom, ka, ba, kb, bb) -> (kc, bc)``
    defaults to the GPU product."""
    from quadmat import ops as qops  # noqa: PLC0415

    compute = compute or gpu_compute

    def body(ctx, inputs, args):
        special = (args.get("level", 0) != 0 or args.get("ta") or args.get("tb") or args.get("a_sym")
                   or args.get("b_sym") or args.get("upper") or args.get("tau", 0.0) > 0.0)
        if special:
            return qops._multiply_body(ctx, inputs, args)
        a, b = inputs
        ga, gb = infer_geometry(ctx.fetch, a), infer_geometry(ctx.fetch, b)
        if ga is None or gb is None or ga != gb:
            return qops._multiply_body(ctx, inputs, args)  # the reference raises / handles it
        ka, ba = read_blocks(ga, ctx.fetch, a)
        kb, bb = read_blocks(gb, ctx.fetch, b)
        kc, bc = compute(ga, ka, ba, kb, bb)
        return write_tree(ga, ctx.put, ctx.norm_of, kc, bc)

    return body


def install(session, compute=None):
    """Route a reference ``quadmat.MatrixSession``'s level-0 regular products through the B200."""
    from quadmat import ops as qops  # noqa: PLC0415

    session.registry.register("multiply", make_multiply_body(compute), qops._multiply_fallback)
    return session
