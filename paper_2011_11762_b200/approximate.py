"""Approximate (norm-pruned) multiply: the reference's ``approximate`` variant on the GPU path.

Reference (ops.py:197-204, 232): every multiply task at quadtree level l with non-nil operand
nodes X (rows I, cols K) and Y (rows K, cols J) first checks ``norm(X) * norm(Y) < tau_l`` with
``tau_0 = tau`` and ``tau_{l+1} = tau_l / 8``; a pruned task logs its bound
(``ctx.log_prune``, engine.py:273-275) and returns nil, so its whole subtree of products is
skipped. Node norms are the store's id-carried Frobenius norms (quadtree.py:138-140); for a
symmetric operand they are the norms of the *stored* (upper) chunks, and virtual SW children reuse
the NE chunk (ops.py:100-116).

B200 form (csrc/qm_prune.cu): qm_node_norms builds every level's node table of an operand
bottom-up from the block sums of squares (nodes are runs of equal Morton codes in quadtree-key
order; sqrt of the compensated sum of the children's squared norms, like the reference's
sqrt(fsum(...))); qm_prune_all runs the whole recursion in one cooperative launch: level l expands
the surviving pairs of level l-1 to their 8 child pairs, looks both operand nodes up (a symmetric
operand's lower nodes read their stored upper mirror), classifies each pair dead / pruned / alive
and appends the alive pairs and the pruned bounds (the log), with a grid-wide barrier between
levels and one host synchronisation for the whole prune (qm_prune_level keeps the level-at-a-time
form). The surviving leaf pairs then filter the regular symbolic phase's triples, and the numeric
kernel runs unchanged on the kept triples (k order preserved).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _ffi
from .blocks import BlockSet
from .layout import Geometry


@dataclass
class PruneResult:
    prune_log: list | torch.Tensor = field(default_factory=list)  # pruned tasks' bounds (engine.prune_log)
    leaf_pairs: torch.Tensor | None = None           # sorted codes of surviving (li, lk, lj)
    pairs_per_level: list = field(default_factory=list)


def _node_tables(geom: Geometry, s: BlockSet, lay):
    """Every level's (Morton codes, norms, count) of one operand (qm_node_norms) -- the quadtree's
    node norms, fixed for an (immutable) block set, so kept with it after the first product."""
    import ctypes

    cached = getattr(s, "_node_tables", None)
    if cached is not None and cached[0] == (geom.params.depth, geom.nbl):
        return cached[1]

    lib = _ffi.load()
    n = s.n
    L = geom.params.depth + 1
    dev = s.keys.device
    codes = torch.empty(max(L * n, 1), dtype=torch.int64, device=dev)
    norms = torch.empty(max(L * n, 1), dtype=torch.float64, device=dev)
    counts = (ctypes.c_int64 * L)()
    wb = lib.qm_node_norms_workspace_bytes(n)
    ws = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
    _ffi.check(lib.qm_node_norms(ctypes.byref(lay), _ffi.ptr(s.keys), _ffi.ptr(s.sumsq), n, _ffi.ptr(codes),
                                 _ffi.ptr(norms), counts, _ffi.ptr(ws), wb,
                                 _ffi.stream_handle(torch.cuda.current_stream(dev))), "qm_node_norms")
    tables = [(codes[l * n:], norms[l * n:], int(counts[l])) for l in range(L)]
    s._node_tables = ((geom.params.depth, geom.nbl), tables)
    return tables


def prune(geom: Geometry, a: BlockSet, b: BlockSet, tau: float, a_sym: bool = False, b_sym: bool = False,
          b_transposed: bool = False, upper: bool = False) -> PruneResult:
    """The prune decisions of the reference's task recursion on the device, every level in one
    launch (qm_prune_all: a grid-wide barrier between levels, one host synchronisation in all), for
    the logical operands op(A) = A or expand(A), op(B) = B, expand(B) or B^T; node norms are those
    of the stored chunks. Capacities start at 32 pairs per leaf node and grow 8x on overflow."""
    import ctypes

    res = PruneResult()
    if a.n == 0 or b.n == 0:
        return res
    lib = _ffi.load()
    depth = geom.params.depth
    dev = a.keys.device
    lay = _ffi.make_layout(geom.params, geom.bs)
    ta = _node_tables(geom, a, lay)
    tb = ta if b is a else _node_tables(geom, b, lay)
    sh = _ffi.stream_handle(torch.cuda.current_stream(dev))
    L = depth + 1
    ac = (ctypes.c_int64 * L)(*[t[2] for t in ta])
    bc = (ctypes.c_int64 * L)(*[t[2] for t in tb])
    cap = max(4096, 32 * max(ta[depth][2], tb[depth][2]))
    while True:
        cap_log = 8 * cap
        leaf = torch.empty(cap, dtype=torch.int64, device=dev)
        log = torch.empty(cap_log, dtype=torch.float64, device=dev)
        wb = lib.qm_prune_all_workspace_bytes(cap)
        ws = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
        counts = (ctypes.c_int64 * (2 * L + 2))()
        _ffi.check(lib.qm_prune_all(ctypes.byref(lay), float(tau), _ffi.ptr(ta[0][0]), _ffi.ptr(ta[0][1]), a.n, ac,
                                    int(a_sym), _ffi.ptr(tb[0][0]), _ffi.ptr(tb[0][1]), b.n, bc, int(b_sym),
                                    int(b_transposed), int(upper), cap, _ffi.ptr(leaf), _ffi.ptr(log), cap_log,
                                    counts, _ffi.ptr(ws), wb, sh), "qm_prune_all")
        if counts[2 * L + 1] == 0:
            break
        cap *= 8  # a level outgrew the buffers: rerun with room (decisions are deterministic)
    levels = [(int(counts[2 * lv]), int(counts[2 * lv + 1])) for lv in range(L)]
    for na, npr in levels:
        res.pairs_per_level.append(na + npr)
        if na == 0:
            break
    n_log = int(counts[2 * L])
    if n_log:
        res.prune_log = log[:n_log]  # device; _EngineInfo converts on first read
    n_leaf = levels[depth][0] if len(res.pairs_per_level) == L else 0
    if n_leaf:
        parents = leaf[:n_leaf]
        w = 1 << depth
        mask = (1 << 21) - 1
        I, K, J = parents >> 42, (parents >> 21) & mask, parents & mask
        res.leaf_pairs = torch.sort((I * w + K) * w + J).values
    return res


def filter_plan(geom: Geometry, plan, a: BlockSet, b: BlockSet, pr: PruneResult, b_transposed=False):
    """Keeps the triples whose leaf pair survived and rebuilds c_keys / c_tptr (qm_filter_triples:
    C blocks left with no triple vanish, like an all-pruned subtree)."""
    import ctypes

    from .spgemm import SymbolicPlan

    dev = plan.c_keys.device
    if pr.leaf_pairs is None or plan.n_triples == 0:
        z = torch.zeros(0, dtype=torch.int64, device=dev)
        return SymbolicPlan(0, 0, z, torch.zeros(1, dtype=torch.int64, device=dev),
                            torch.zeros(0, dtype=torch.int32, device=dev))
    lib = _ffi.load()
    lay = _ffi.make_layout(geom.params, geom.bs)
    nc, nt = plan.n_c, plan.n_triples
    tri = torch.empty(2 * nt, dtype=torch.int32, device=dev)
    c_tptr = torch.empty(nc + 1, dtype=torch.int64, device=dev)
    c_keys = torch.empty(nc, dtype=torch.int64, device=dev)
    wb = lib.qm_filter_triples_workspace_bytes(nc, nt)
    ws = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
    nc2, nt2 = ctypes.c_int64(0), ctypes.c_int64(0)
    pairs = pr.leaf_pairs.contiguous()
    _ffi.check(lib.qm_filter_triples(ctypes.byref(lay), _ffi.ptr(a.keys), _ffi.ptr(b.keys), int(b_transposed),
                                     _ffi.ptr(plan.tri), _ffi.ptr(plan.c_tptr), _ffi.ptr(plan.c_keys), nc, nt,
                                     _ffi.ptr(pairs), int(pairs.shape[0]), _ffi.ptr(tri), _ffi.ptr(c_tptr),
                                     _ffi.ptr(c_keys), ctypes.byref(nc2), ctypes.byref(nt2), _ffi.ptr(ws), wb,
                                     _ffi.stream_handle(torch.cuda.current_stream(dev))), "qm_filter_triples")
    n_c, n_t = int(nc2.value), int(nt2.value)
    return SymbolicPlan(n_c, n_t, c_keys[:n_c], c_tptr[:n_c + 1], tri[:2 * n_t])


class Pruner:
    """The approximate variant on the product's hot path (session.run_spec).

    The prune *decisions* needed for the product reduce to a per-triple test: a leaf product
    survives the reference's pruned recursion iff none of its ancestor tasks was pruned, i.e. at
    every level l, norm(A ancestor) * norm(B ancestor) >= tau / 8^l (ops.py:199-204, 232). So the
    hot path is: ancestor norms of the operands' entries (qm_ancestor_norms; cached on a stored
    block set, recomputed for a per-product view), then one filter pass over the symbolic plan
    (qm_filter_triples_norms) -- no level-by-level recursion, no per-level synchronisation. The
    prune *log* (the bounds of the pruned tasks, engine.prune_log) is computed from the same node
    tables on first access only (qm_prune_all, every level in one launch)."""

    def __init__(self, geom: Geometry, a_src: BlockSet, b_src: BlockSet, tau: float, a_sym: bool = False,
                 b_sym: bool = False, upper: bool = False):
        self.geom, self.tau = geom, float(tau)
        self.a_src, self.b_src = a_src, b_src
        self.a_sym, self.b_sym, self.upper = a_sym, b_sym, upper
        self.lay = _ffi.make_layout(geom.params, geom.bs)
        self.ta = _node_tables(geom, a_src, self.lay)
        self.tb = self.ta if b_src is a_src else _node_tables(geom, b_src, self.lay)
        self._result = None

    def _ancestors(self, x: BlockSet, src: BlockSet, tables, sym: bool) -> torch.Tensor:
        """[(depth+1) * n] ancestor norms of x's entries in src's node tables (cached on x)."""
        import ctypes

        cache = getattr(x, "_anc_cache", None)
        key = (id(src), bool(sym), self.geom.params.depth)
        if cache is not None and key in cache and cache[key][0] is tables:
            return cache[key][1]
        L = self.geom.params.depth + 1
        out = torch.empty(max(L * x.n, 1), dtype=torch.float64, device=x.keys.device)
        counts = (ctypes.c_int64 * L)(*[t[2] for t in tables])
        _ffi.check(_ffi.load().qm_ancestor_norms(ctypes.byref(self.lay), _ffi.ptr(x.keys), x.n, _ffi.ptr(tables[0][0]),
                                                 _ffi.ptr(tables[0][1]), src.n, counts, int(sym), _ffi.ptr(out),
                                                 _ffi.stream_handle(torch.cuda.current_stream(x.keys.device))),
                   "qm_ancestor_norms")
        if cache is None:
            cache = {}
            try:
                x._anc_cache = cache
            except AttributeError:
                pass
        cache[key] = (tables, out)
        return out

    def filter(self, plan, ax: BlockSet, bx: BlockSet):
        """The plan's triples whose ancestor tasks all survive (C blocks left empty vanish)."""
        import ctypes

        from .spgemm import SymbolicPlan

        dev = plan.c_keys.device
        if plan.n_triples == 0:
            return plan
        anc_a = self._ancestors(ax, self.a_src, self.ta, self.a_sym)
        anc_b = self._ancestors(bx, self.b_src, self.tb, self.b_sym)
        lib = _ffi.load()
        nc, nt = plan.n_c, plan.n_triples
        tri = torch.empty(2 * nt, dtype=torch.int32, device=dev)
        c_tptr = torch.empty(nc + 1, dtype=torch.int64, device=dev)
        c_keys = torch.empty(nc, dtype=torch.int64, device=dev)
        wb = lib.qm_filter_triples_workspace_bytes(nc, nt)
        ws = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
        nc2, nt2 = ctypes.c_int64(0), ctypes.c_int64(0)
        _ffi.check(lib.qm_filter_triples_norms(ctypes.byref(self.lay), self.tau, _ffi.ptr(plan.tri),
                                               _ffi.ptr(plan.c_tptr), _ffi.ptr(plan.c_keys), nc, nt, _ffi.ptr(anc_a),
                                               ax.n, _ffi.ptr(anc_b), bx.n, _ffi.ptr(tri), _ffi.ptr(c_tptr),
                                               _ffi.ptr(c_keys), ctypes.byref(nc2), ctypes.byref(nt2), _ffi.ptr(ws),
                                               wb, _ffi.stream_handle(torch.cuda.current_stream(dev))),
                   "qm_filter_triples_norms")
        n_c, n_t = int(nc2.value), int(nt2.value)
        return SymbolicPlan(n_c, n_t, c_keys[:n_c], c_tptr[:n_c + 1], tri[:2 * n_t])

    def result(self) -> PruneResult:
        """The full prune (log and pairs per level), computed on first request."""
        if self._result is None:
            self._result = prune(self.geom, self.a_src, self.b_src, self.tau, a_sym=self.a_sym, b_sym=self.b_sym,
                                 upper=self.upper)
        return self._result
