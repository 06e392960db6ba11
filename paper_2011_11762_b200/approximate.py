"""Approximate (norm-pruned) multiply: the reference's ``approximate`` variant on the GPU path.

Reference (ops.py:197-204, 232): every multiply task at quadtree level l with non-nil operand
nodes X (rows I, cols K) and Y (rows K, cols J) first checks ``norm(X) * norm(Y) < tau_l`` with
``tau_0 = tau`` and ``tau_{l+1} = tau_l / 8``; a pruned task logs its bound
(``ctx.log_prune``, engine.py:273-275) and returns nil, so its whole subtree of products is
skipped. Node norms are the store's id-carried Frobenius norms (quadtree.py:138-140); for a
symmetric operand they are the norms of the *stored* (upper) chunks, and virtual SW children reuse
the NE chunk (ops.py:100-116).

B200 form: the prune decisions are made level by level on the compressed node structure (torch
on the device): level-l node norms are segment sums of the per-block squared norms over the
quadtree-key order (every node is a contiguous key range); the pairs reached at level l are the
unpruned pairs of level l-1 expanded to their 8 child pairs where both child nodes exist; pruned
pairs go to the log. The surviving leaf pairs then filter the regular symbolic phase's triples,
and the numeric kernel runs unchanged on the kept triples (k order preserved).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from .blocks import BlockSet
from .layout import Geometry


@dataclass
class PruneResult:
    prune_log: list = field(default_factory=list)   # bounds of the pruned tasks (engine.prune_log)
    leaf_pairs: torch.Tensor | None = None           # sorted codes of surviving (li, lk, lj)
    pairs_per_level: list = field(default_factory=list)


def _coords(geom: Geometry, keys: torch.Tensor):
    from .variants import _decode

    bi, bj = _decode(geom, keys)
    return bi.to(torch.int64), bj.to(torch.int64)


class _Nodes:
    """Nodes of one operand at one level: sorted codes r*W + c and norms (stored-chunk norms)."""

    def __init__(self, r, c, sumsq, width, sym: bool):
        code = r * width + c
        order = torch.argsort(code, stable=True)
        code, sq = code[order], sumsq[order]
        uniq, inv = torch.unique_consecutive(code, return_inverse=True)
        acc = torch.zeros(uniq.shape[0], dtype=torch.float64, device=code.device)
        acc.index_add_(0, inv, sq)
        self.width, self.sym = width, sym
        if sym:  # add the virtual lower nodes (r > c) as mirrors of the stored upper ones
            ur, uc = uniq // width, uniq % width
            up = ur < uc
            mcode = uc[up] * width + ur[up]
            allc = torch.cat([uniq, mcode])
            alln = torch.cat([acc, acc[up]])
            o = torch.argsort(allc)
            uniq, acc = allc[o], alln[o]
        self.code = uniq
        self.norm = torch.sqrt(acc)

    def lookup(self, r, c):
        """(exists mask, norms) for node coordinates."""
        q = r * self.width + c
        pos = torch.searchsorted(self.code, q).clamp(max=max(self.code.shape[0] - 1, 0))
        hit = self.code[pos] == q if self.code.shape[0] else torch.zeros_like(q, dtype=torch.bool)
        return hit, torch.where(hit, self.norm[pos], torch.zeros_like(self.norm[pos]))


def prune(geom: Geometry, a: BlockSet, b: BlockSet, tau: float, a_sym: bool = False, b_sym: bool = False,
          b_transposed: bool = False, upper: bool = False) -> PruneResult:
    """Level-by-level prune decisions of the reference's task recursion (regular algebra on the
    logical operands op(A) = A or expand(A), op(B) = B, expand(B) or B^T)."""
    depth = geom.params.depth
    nbl = geom.nbl
    ar, ac = _coords(geom, a.keys)
    br, bc = _coords(geom, b.keys)
    if b_transposed:  # logical B = stored B^T: node (K, J) of B^T is node (J, K) of B
        br, bc = bc, br
    res = PruneResult()
    dev = a.keys.device
    surv = None  # (I, K, J) at the previous level
    for lev in range(depth + 1):
        shift_blocks = nbl << (depth - lev)  # blocks per node side at this level
        width = 1 << lev
        na = _Nodes(ar // shift_blocks, ac // shift_blocks, a.sumsq, width, a_sym)
        nb = _Nodes(br // shift_blocks, bc // shift_blocks, b.sumsq, width, b_sym)
        if lev == 0:
            if na.code.numel() == 0 or nb.code.numel() == 0:
                return res
            I = K = J = torch.zeros(1, dtype=torch.int64, device=dev)
        else:
            d = torch.arange(8, device=dev)
            I = (2 * surv[0][:, None] + (d >> 2)).reshape(-1)
            K = (2 * surv[1][:, None] + ((d >> 1) & 1)).reshape(-1)
            J = (2 * surv[2][:, None] + (d & 1)).reshape(-1)
        ha, nA = na.lookup(I, K)
        hb, nB = nb.lookup(K, J)
        live = ha & hb
        if upper:
            live &= I <= J
        I, K, J, nA, nB = I[live], K[live], J[live], nA[live], nB[live]
        bound = nA * nB
        tau_l = tau / (8.0 ** lev)
        pruned = bound < tau_l
        res.prune_log.extend(bound[pruned].tolist())
        keep = ~pruned
        surv = (I[keep], K[keep], J[keep])
        res.pairs_per_level.append(int(live.sum().item()))
        if surv[0].numel() == 0:
            return res
    w = 1 << depth
    res.leaf_pairs = torch.sort((surv[0] * w + surv[1]) * w + surv[2]).values
    return res


def filter_plan(geom: Geometry, plan, a: BlockSet, b: BlockSet, pr: PruneResult, b_transposed=False):
    """Keeps the triples whose leaf pair survived; rebuilds c_keys / c_tptr (C blocks left with no
    triple vanish, like an all-pruned subtree)."""
    from .spgemm import SymbolicPlan

    dev = plan.c_keys.device
    if pr.leaf_pairs is None or plan.n_triples == 0:
        z = torch.zeros(0, dtype=torch.int64, device=dev)
        return SymbolicPlan(0, 0, z, torch.zeros(1, dtype=torch.int64, device=dev),
                            torch.zeros(0, dtype=torch.int32, device=dev))
    nbl, w = geom.nbl, 1 << geom.params.depth
    tri = plan.tri.view(-1, 2).to(torch.int64)
    ar, ac = _coords(geom, a.keys)
    br, bc = _coords(geom, b.keys)
    li, lk = ar[tri[:, 0]] // nbl, ac[tri[:, 0]] // nbl
    lj = (bc[tri[:, 1]] if not b_transposed else br[tri[:, 1]]) // nbl
    code = (li * w + lk) * w + lj
    pos = torch.searchsorted(pr.leaf_pairs, code).clamp(max=pr.leaf_pairs.shape[0] - 1)
    keep = pr.leaf_pairs[pos] == code
    counts = torch.zeros(plan.n_c, dtype=torch.int64, device=dev)
    grp = torch.repeat_interleave(torch.arange(plan.n_c, device=dev), torch.diff(plan.c_tptr))
    counts.index_add_(0, grp, keep.to(torch.int64))
    alive = counts > 0
    c_keys = plan.c_keys[alive].contiguous()
    cnt = counts[alive]
    c_tptr = torch.zeros(cnt.shape[0] + 1, dtype=torch.int64, device=dev)
    c_tptr[1:] = torch.cumsum(cnt, 0)
    tri_k = plan.tri.view(-1, 2)[keep].reshape(-1).contiguous()
    return SymbolicPlan(int(c_keys.shape[0]), int(tri_k.shape[0] // 2), c_keys, c_tptr, tri_k)
