"""Multi-GPU product C = A*B: one process per GPU, torch.distributed (NCCL over NVLink/NVSwitch).

Reference analogue: chunks are owned round-robin by subtree at a split depth (OwnerPolicy,
quadtree.py:47-63), work is stolen breadth-first (engine.py:286-300) and remote operands are
fetched through the transfer layer whose received bytes are counted per worker
(TransferSim.fetch, chunkstore.py:188-210; WorkerStats.bytes_received :54-63).

B200 design:
  * ownership: each rank holds one contiguous quadtree-key range of A and of B (a union of
    quadtree subtrees -- structure preserving, never a random permutation);
  * structure: the ranks all-gather the operands' keys (8 bytes per block) and run the symbolic
    phase's row indexing and C key pass on the global structure;
  * partition: C's key range is cut into P contiguous ranges of equal triple count (c_tptr is the
    prefix sum of per-C-block work), so every C block's whole k sum lives on one GPU -- no
    reduction, bitwise the same result for any P;
  * exchange: each rank emits only its own triples, derives the A and B blocks it needs, requests
    them from their owners (all-to-all-v of indices) and receives them (all-to-all-v of blocks,
    packed by qm_gather_blocks) -- one halo exchange, no data-path collective besides it;
  * compute: the local numeric kernel over the received pools; C stays distributed.

The collectives go through ``Comm`` so the same code runs over NCCL (product) and gloo (CPU tests
with a test backend); ``LocalComm`` is the single-rank case.
"""

from __future__ import annotations

import atexit
import ctypes
import os
import time
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import spgemm
from .blocks import BlockSet
from .errors import ConfigurationError, ContractViolationError


class Comm:
    """torch.distributed collectives used by the product (process group `group`)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # gloo moves host memory only: device tensors are staged through the host (tests run the
        # CUDA backend with several ranks on one GPU this way, with no cross-rank GPU waits)
        self.stage = dist.get_backend(group) == "gloo"

    def _in(self, t: torch.Tensor) -> torch.Tensor:
        return t.cpu() if self.stage else t

    def _out(self, t: torch.Tensor, device) -> torch.Tensor:
        return t.to(device) if self.stage else t

    def allgather_varlen(self, t: torch.Tensor) -> tuple[torch.Tensor, list[int]]:
        """Concatenation over ranks (rank order) of 1-D tensors of different lengths."""
        dev = t.device
        t = self._in(t)
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        ns = [torch.zeros_like(n) for _ in range(self.world)]
        self.dist.all_gather(ns, n, group=self.group)
        counts = [int(x.item()) for x in ns]
        mx = max(counts) if counts else 0
        pad = torch.zeros(mx, dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        outs = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(outs, pad, group=self.group)
        return self._out(torch.cat([o[:c] for o, c in zip(outs, counts)]), dev), counts

    def gather_known(self, t: torch.Tensor, counts: list) -> torch.Tensor:
        """Concatenation over ranks of 1-D tensors whose lengths `counts` every rank already knows."""
        dev = t.device
        t = self._in(t)
        mx = max(counts) if counts else 0
        pad = torch.zeros(mx, dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        outs = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(outs, pad, group=self.group)
        return self._out(torch.cat([o[:c] for o, c in zip(outs, counts)]), dev)

    def allreduce_max_vec(self, xs: list, device) -> list:
        """Element-wise max over ranks of a few host floats (one collective)."""
        t = torch.tensor(xs, dtype=torch.float64, device="cpu" if self.stage else device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return [float(x) for x in t.cpu().tolist()]

    def allgather_fixed(self, t: torch.Tensor) -> torch.Tensor:
        """[world, *t.shape]: every rank's tensor of the same shape, in rank order."""
        dev = t.device
        t = self._in(t)
        outs = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(outs, t, group=self.group)
        return self._out(torch.stack(outs), dev)

    def alltoallv(self, send: torch.Tensor, send_counts: list[int],
                  recv_counts: list[int] | None = None) -> tuple[torch.Tensor, list[int]]:
        """Rows send[sum(send_counts[:d]) : ...] go to rank d; returns received rows (source rank
        order) and the per-source counts (exchanged first unless the caller knows them)."""
        dev0 = send.device
        send = self._in(send)
        dev = send.device
        if recv_counts is None:
            sc = torch.tensor(send_counts, dtype=torch.int64, device=dev)
            rc = torch.empty_like(sc)
            self.dist.all_to_all_single(rc, sc, group=self.group)
            recv_counts = [int(x) for x in rc.cpu().tolist()]
        inner = 1
        for d in send.shape[1:]:
            inner *= int(d)
        flat = send.reshape(send.shape[0], inner)  # explicit width: a rank may send zero rows
        out = torch.empty((sum(recv_counts), flat.shape[1]), dtype=send.dtype, device=dev)
        self.dist.all_to_all_single(out, flat.contiguous(), recv_counts, send_counts, group=self.group)
        return self._out(out.reshape((out.shape[0],) + tuple(send.shape[1:])), dev0), recv_counts

    def barrier(self):
        self.dist.barrier(group=self.group)

    def allreduce_max(self, x: float, device) -> float:
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if self.stage else device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())


class LocalComm:
    """Single rank: every collective is the identity."""

    rank, world = 0, 1

    def allgather_varlen(self, t):
        return t, [int(t.shape[0])]

    def gather_known(self, t, counts):
        return t

    def allreduce_max_vec(self, xs, device):
        return list(xs)

    def allgather_fixed(self, t):
        return t.unsqueeze(0)

    def alltoallv(self, send, send_counts, recv_counts=None):
        return send, list(send_counts)

    def barrier(self):
        pass

    def allreduce_max(self, x, device):
        return x


class CudaBackend:
    """The product backend: libqmb200 kernels on the rank's GPU."""

    def __init__(self, stream=None):
        self.stream = stream

    def numeric_peer(self, layout, tri, c_tptr, c_keys, rank, a_off, b_off, a_bases, b_bases, a_local,
                     b_local, b_is_a, masks, staged=True, info=None):
        """staged_numeric on this rank's GPU, then the exact-zero drop."""
        from . import _ffi

        stream = self.stream if self.stream is not None else torch.cuda.current_stream(c_keys.device)
        c, nz, zc = staged_numeric(layout, tri, c_tptr, c_keys, rank, a_off, b_off, a_bases, b_bases,
                                   a_local, b_local, b_is_a, masks, stream, staged=staged, info=info)
        n_zero, k_rows = _ffi.read_i64s(zc, 2, stream)
        if info is not None:
            info["k_rows"] = k_rows  # k depth executed (panels skipped by the support masks excluded)
        return spgemm.compact(layout.block_size, c, nz, n_zero, self.stream)

    def symbolic_state(self, layout, a_keys: torch.Tensor, b_keys: torch.Tensor, a_cmask=None, b_rmask=None,
                       part=None, ix=None):
        return spgemm.SymbolicState(layout, a_keys, int(a_keys.shape[0]), b_keys, int(b_keys.shape[0]),
                                    self.stream, a_cmask, b_rmask, part=part, ix=ix)

    def row_indexes(self, layout, ka, kb, ma, mb, fa, fb, b_is_a):
        """Row indexes of the gathered global structure (qm_row_index_build on structure-only block
        sets): ((qm_row_index of A, of B), the tensors they point into)."""
        bs = layout.block_size
        dev = ka.device

        def structure(keys, rows, cols, flags):
            n = int(keys.shape[0])
            s = BlockSet(keys, torch.empty((0, bs, bs), dtype=torch.float64, device=dev),
                         torch.empty(0, dtype=torch.float64, device=dev))
            if cols is not None or rows is not None:
                ones = torch.full((n,), -1, dtype=torch.int64, device=dev)
                s.masks = torch.stack([rows if rows is not None else ones, cols if cols is not None else ones,
                                       flags if flags is not None else torch.zeros_like(ones)]).contiguous()
            return s

        masked = ma is not None
        sa = structure(ka, mb if b_is_a else None, ma, fa)
        sb = sa if b_is_a else structure(kb, mb, None, fb)
        ia, ib = sa.row_index(layout, self.stream), sb.row_index(layout, self.stream)
        structs = (BlockSet.ix_struct(ia, "a" if masked else None), BlockSet.ix_struct(ib, "b" if masked else None))
        return structs, (ia, ib)

    def gather_blocks(self, blocks: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
        import ctypes  # noqa: F401

        from . import _ffi

        n = int(idx.shape[0])
        bs = int(blocks.shape[1])
        out = torch.empty((n, bs, bs), dtype=blocks.dtype, device=blocks.device)
        if n:
            _ffi.check(_ffi.load().qm_gather_blocks(bs, _ffi.ptr(blocks), _ffi.ptr(idx.contiguous()), n,
                                                    _ffi.ptr(out), _ffi.stream_handle(self.stream)),
                       "qm_gather_blocks")
        return out

    def numeric(self, layout, pool_a: BlockSet, pool_b: BlockSet, tri: torch.Tensor,
                c_tptr: torch.Tensor, c_keys: torch.Tensor) -> BlockSet:
        from . import _ffi

        plan = spgemm.SymbolicPlan(int(c_keys.shape[0]), int(tri.shape[0] // 2), c_keys, c_tptr, tri)
        c, nz, zc = spgemm.numeric(layout, pool_a, pool_b, plan, self.stream)
        stream = self.stream if self.stream is not None else torch.cuda.current_stream(c_keys.device)
        n_zero, self.last_k_rows = _ffi.read_i64s(zc, 2, stream)
        return spgemm.compact(layout.block_size, c, nz, n_zero, self.stream)


@dataclass
class DistStats:
    rank: int = 0
    world: int = 1
    n_c_global: int = 0
    n_triples_global: int = 0
    c_range: tuple = (0, 0)   # this rank's C key range [lo, hi) (a union of quadtree subtrees)
    t_range: tuple = (0, 0)   # (0, this rank's triples)
    tile_work: int = 0        # total structural triples of the partition pass
    n_c_local: int = 0
    bytes_received: int = 0
    bytes_sent: int = 0
    blocks_received: int = 0
    mode: str = "exchange"
    phase_s: dict = field(default_factory=dict)
    extra: dict = field(default_factory=dict)
    k_rows: int = -1          # k depth this rank executed (2*bs^2 flops each); -1 = not counted


MAX_TILE_LEVELS = 8  # csrc/qm_symbolic.cu kMaxTileLevels


def _panel_groups(m: np.ndarray) -> np.ndarray:
    """Nonzero 16-bit groups of each mask (csrc k_tile_work's panel_groups)."""
    m = m.astype(np.uint64)
    g = np.zeros(m.shape, dtype=np.int64)
    for s in (0, 16, 32, 48):
        g += ((m >> np.uint64(s)) & np.uint64(0xFFFF)) != 0
    return g


def tile_partition(geom, ka: np.ndarray, kb: np.ndarray, world: int, a_cmask=None, b_rmask=None) -> list[int]:
    """Host statement of qm_spgemm_count_part's partition (its CPU twin and test oracle): C tiles =
    aligned quadtree subtrees at level min(depth, 8) (tile code = C key >> kshift), weighed by their
    work; tiles are cut in Morton order where the exclusive work prefix first reaches r*W // world.
    Work of a block pair A(i,k)*B(k,j): 1 without support masks (structural triples); with masks
    (A's column masks, B's row masks) the number of 16-row k panels where they meet, the depth the
    numeric kernel executes (0 for disjoint supports). Returns the world+1 key bounds; rank r owns
    C keys [bounds[r], bounds[r+1])."""
    import scipy.sparse as sp  # noqa: PLC0415

    depth = geom.params.depth
    tl = min(depth, MAX_TILE_LEVELS)
    kshift = 2 * (depth - tl) + 2 * geom.lbits
    ntiles = 1 << (2 * tl)
    nb = geom.nbg
    ai, ak = geom.decode(np.asarray(ka, dtype=np.int64))
    bk, bj = geom.decode(np.asarray(kb, dtype=np.int64))
    if a_cmask is None and b_rmask is None:
        pa = sp.csr_matrix((np.ones(ai.size, dtype=np.int64), (ai, ak)), shape=(nb, nb))
        pb = sp.csr_matrix((np.ones(bk.size, dtype=np.int64), (bk, bj)), shape=(nb, nb))
        c = (pa @ pb).tocoo()
        tiles = geom.qkey(c.row.astype(np.int64), c.col.astype(np.int64)) >> kshift
        work = np.bincount(tiles, weights=c.data, minlength=ntiles).astype(np.int64)
    else:  # every pair, weighed by its executed k panels
        full = np.full(1, np.iinfo(np.uint64).max, dtype=np.uint64)
        am = np.asarray(a_cmask).view(np.uint64) if a_cmask is not None else np.broadcast_to(full, ai.shape)
        bm = np.asarray(b_rmask).view(np.uint64) if b_rmask is not None else np.broadcast_to(full, bk.shape)
        order = np.argsort(bk, kind="stable")
        bptr = np.searchsorted(bk[order], np.arange(nb + 1))
        cnt = bptr[ak + 1] - bptr[ak]
        a_idx = np.repeat(np.arange(ai.size), cnt)
        start = np.repeat(bptr[ak], cnt)
        within = np.arange(a_idx.size) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        b_idx = order[start + within]
        w = _panel_groups(am[a_idx] & bm[b_idx])
        tiles = geom.qkey(ai[a_idx].astype(np.int64), bj[b_idx].astype(np.int64)) >> kshift
        work = np.bincount(tiles, weights=w, minlength=ntiles).astype(np.int64)
    prefix = np.concatenate([[0], np.cumsum(work)])
    W = int(prefix[-1])
    cuts = [0] + [int(np.searchsorted(prefix[:ntiles], (W * r) // world, side="left")) for r in range(1, world)]
    cuts.append(ntiles)
    return [x << kshift for x in cuts]


def partition(c_tptr: torch.Tensor, world: int) -> tuple[list[int], list[int]]:
    """Contiguous C ranges of (nearly) equal triple count: bounds over C indices and triples."""
    n_c = int(c_tptr.shape[0]) - 1
    n_t = int(c_tptr[-1].item())
    targets = torch.tensor([(r * n_t) // world for r in range(1, world)], dtype=torch.int64,
                           device=c_tptr.device)
    cuts = torch.searchsorted(c_tptr, targets).cpu().tolist() if world > 1 else []
    cb = [0] + [min(max(int(x), 0), n_c) for x in cuts] + [n_c]
    for r in range(1, len(cb)):
        cb[r] = max(cb[r], cb[r - 1])
    tb = c_tptr[torch.tensor(cb, device=c_tptr.device)].cpu().tolist()
    return cb, [int(x) for x in tb]


# CUDA IPC mappings of peer pools, kept across products (opening a handle costs far more than a
# product's bookkeeping): handle bytes -> mapped base address in this process, plus the handles
# each (process group, peer rank) used last, so mappings a peer no longer exports are closed.
_IPC_MAPPED: dict[bytes, int] = {}
_IPC_BY_PEER: dict[tuple, set] = {}
_REC = 88  # per pool record: 64-byte handle, int64 offset, int64 block count, valid flag (+pad)


def release_peer_mappings():
    """Closes every cached peer-pool mapping of this process (call before tearing down the
    process group; also registered atexit)."""
    from . import _ffi

    if not _IPC_MAPPED:
        return
    lib = _ffi.load()
    for base in _IPC_MAPPED.values():
        lib.qm_ipc_close(base)
    _IPC_MAPPED.clear()
    _IPC_BY_PEER.clear()


atexit.register(release_peer_mappings)


class PeerPools:
    """Block pools of every rank, mapped into this GPU's address space for the fused kernel.

    Each rank exports (qm_ipc_export) the CUDA IPC handle of the allocation holding its pool and
    the pool's offset in it; the fixed-size records are all-gathered in one collective and every
    peer handle is opened once per process (qm_ipc_open, peer access over NVLink on a multi-GPU
    node; on a single GPU the "peers" are other processes sharing it) and cached: repeated products
    on the same pools map nothing new. A cached mapping is closed when its peer stops exporting it.

    Failures to export or map (no peer access between two GPUs, IPC unsupported) do not raise:
    they leave ``ok`` False, and ``multiply`` agrees on the mode across ranks before any kernel
    runs (every rank falls back to the exchange when one cannot map its peers)."""

    def __init__(self, comm, pools):
        import ctypes

        from . import _ffi

        lib = _ffi.load()
        self.lib, self.rank = lib, comm.rank
        self.ok, self.error = True, ""
        dev = pools[0].device
        rec = np.zeros((len(pools), _REC), dtype=np.uint8)
        for p_i, t in enumerate(pools):
            if t.numel() == 0:
                continue
            h = ctypes.create_string_buffer(64)
            off = ctypes.c_int64(0)
            if lib.qm_ipc_export(_ffi.ptr(t), h, ctypes.byref(off)) != 0:
                self.ok, self.error = False, _ffi.last_error()
                continue
            rec[p_i, :64] = np.frombuffer(h.raw, dtype=np.uint8)
            rec[p_i, 64:80] = np.array([off.value, t.shape[0]], dtype=np.int64).view(np.uint8)
            rec[p_i, 80] = 1
        every = comm.allgather_fixed(torch.from_numpy(rec.reshape(-1)).to(dev))
        every = every.cpu().numpy().reshape(comm.world, len(pools), _REC)
        self.ptrs = [[0] * comm.world for _ in pools]
        self.counts = [[0] * comm.world for _ in pools]
        bs = int(pools[0].shape[1])
        self._dummy = torch.zeros((1, bs, bs), dtype=torch.float64, device=dev)
        gkey = id(comm.group)
        for r in range(comm.world):
            used = set()
            for p_i in range(len(pools)):
                if r == comm.rank:
                    t = pools[p_i]
                    self.ptrs[p_i][r] = _ffi.ptr(t) if t.numel() else _ffi.ptr(self._dummy)
                    self.counts[p_i][r] = max(int(t.shape[0]), 1)
                    continue
                e = every[r, p_i]
                self.ptrs[p_i][r], self.counts[p_i][r] = _ffi.ptr(self._dummy), 1
                if not e[80]:
                    continue
                handle = e[:64].tobytes()
                off, n = (int(x) for x in e[64:80].view(np.int64))
                base = _IPC_MAPPED.get(handle)
                if base is None:
                    out = ctypes.c_void_p(0)
                    if lib.qm_ipc_open(handle, ctypes.byref(out)) != 0:
                        self.ok, self.error = False, _ffi.last_error()
                        continue
                    base = _IPC_MAPPED[handle] = int(out.value)
                used.add(handle)
                self.ptrs[p_i][r], self.counts[p_i][r] = base + off, n
            if r != comm.rank:
                for h in _IPC_BY_PEER.get((gkey, r), set()) - used:
                    base = _IPC_MAPPED.pop(h, None)
                    if base is not None:
                        lib.qm_ipc_close(base)
                _IPC_BY_PEER[(gkey, r)] = used

    def close(self):
        """Mappings stay cached for the next product (release_peer_mappings closes them)."""


def staged_numeric(layout, tri: torch.Tensor, c_tptr: torch.Tensor, c_keys: torch.Tensor, rank: int,
                   a_off: list, b_off: list, a_bases: list, b_bases: list, a_local: torch.Tensor,
                   b_local: torch.Tensor, b_is_a: bool, masks=None, stream=None, staged: bool = True,
                   info: dict | None = None, emulate_link_gbs: float | None = None):
    """Numeric phase of one rank over the operands of every rank (SURVEY 8(e) "needed A/B subtrees
    fetched over NVLink"), C blocks needing no remote block first.

    tri: int32 [2T] triples (a, b) in global block indices (rank r owns A indices [a_off[r],
    a_off[r+1]), likewise B); a_bases[r] / b_bases[r]: device address of rank r's pool (mapped peer
    memory; ignored for `rank`). staged=True: qm_stage_plan (device) finds the peer-owned blocks,
    re-indexes the triples into [local pool | halo pool] and orders the C blocks needing no halo
    first; k_halo_gather copies each halo block once (bulk copies on a few SMs, reading the peer
    pools over NVLink) while the numeric kernel, launched as its programmatic dependent, computes
    the local-only C blocks; its claims of the other C blocks wait for the gather grid
    (qm_numeric_pools_ex). staged=False ("fused"): the kernel's TMA reads remote blocks from the peer
    pools directly, every reference over NVLink. Per-C-block summation order is the triples' order
    either way: bitwise the single-GPU product.
    masks = (a column masks, b row masks, a flags, b flags) in global indices, or None.
    emulate_link_gbs (measurement only): the gather lasts at least halo bytes / this bandwidth,
    emulating NVLink when the "peers" are slices of pools on this GPU (scaling projection).
    Returns (C BlockSet before compaction, nonzero flags, [zero blocks, k rows] device counters)."""
    from . import _ffi

    lib = _ffi.load()
    bs = layout.block_size
    dev = c_keys.device
    nc, nt = int(c_keys.shape[0]), int(tri.numel()) // 2
    stream = stream if stream is not None else torch.cuda.current_stream(dev)
    sh = _ffi.stream_handle(stream)
    blk = bs * bs * 8
    info = info if info is not None else {}
    world = len(a_off) - 1
    if a_local.shape[0] == 0 or b_local.shape[0] == 0:  # (an empty pool still needs a valid address)
        dummy = torch.zeros((1, bs, bs), dtype=torch.float64, device=dev)
    la = a_local if a_local.shape[0] else dummy
    lb = b_local if b_local.shape[0] else dummy
    na_g, nb_g = a_off[-1], b_off[-1]
    order = halo = None
    gate_units = 0
    keep = []
    # outputs and workspace first: they do not depend on the plan's counts
    out = BlockSet(c_keys, torch.empty((nc, bs, bs), dtype=torch.float64, device=dev),
                   torch.empty(nc, dtype=torch.float64, device=dev))
    nz = torch.empty(nc, dtype=torch.uint8, device=dev)
    zc = torch.empty(2, dtype=torch.int64, device=dev)  # (zeroed by the library)
    wb = lib.qm_numeric_workspace_bytes(bs, nc, nt)
    ws = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
    if staged:
        tri_packed = torch.empty(2 * nt, dtype=torch.int32, device=dev)
        order = torch.empty(max(nc, 1), dtype=torch.int32, device=dev)
        cap_a = max(na_g - (a_off[rank + 1] - a_off[rank]), 1)
        cap_b = max(nb_g - (b_off[rank + 1] - b_off[rank]), 1)
        ha = torch.empty(cap_a, dtype=torch.int32, device=dev)
        hb = ha if b_is_a else torch.empty(cap_b, dtype=torch.int32, device=dev)
        swb = lib.qm_stage_plan_workspace_bytes(na_g, nb_g, nc, 1 if b_is_a else 0)
        sws = torch.empty(max(swb, 1), dtype=torch.uint8, device=dev)
        counts = (ctypes.c_int64 * 3)()
        _ffi.check(lib.qm_stage_plan(_ffi.ptr(tri), nt, _ffi.ptr(c_tptr), nc, a_off[rank], a_off[rank + 1], na_g,
                                     b_off[rank], b_off[rank + 1], nb_g, 1 if b_is_a else 0, _ffi.ptr(sws), swb,
                                     _ffi.ptr(tri_packed), _ffi.ptr(order), _ffi.ptr(ha),
                                     None if b_is_a else _ffi.ptr(hb), counts, sh), "qm_stage_plan")
        n_local, n_ha, n_hb = int(counts[0]), int(counts[1]), int(counts[2])
        pool_a = torch.empty((max(n_ha, 1), bs, bs), dtype=torch.float64, device=dev)
        pool_b = pool_a if b_is_a else torch.empty((max(n_hb, 1), bs, bs), dtype=torch.float64, device=dev)
        halo = _ffi.QmHalo()
        halo.world = world
        halo.index[0], halo.count[0], halo.pool[0] = _ffi.ptr(ha), n_ha, _ffi.ptr(pool_a)
        if not b_is_a:
            halo.index[1], halo.count[1], halo.pool[1] = _ffi.ptr(hb), n_hb, _ffi.ptr(pool_b)
        for o, (bases, off) in enumerate(((a_bases, a_off), (b_bases, b_off))):
            for r in range(world):
                halo.peer_base[o][r] = int(bases[r]) if r != rank else 0
            for r in range(world + 1):
                halo.offset[o][r] = int(off[r])
        n_halo = n_ha + (0 if b_is_a else n_hb)
        if emulate_link_gbs:
            halo.min_ns = int(n_halo * blk / (emulate_link_gbs * 1e9) * 1e9)
        gate_units = n_local * (1 if bs <= 64 else (bs // 64) ** 2)
        info["halo_bytes"] = n_halo * blk
        info["local_c_blocks"], info["c_blocks"] = n_local, nc
        counts_a, counts_b = [int(la.shape[0]), max(n_ha, 1)], [int(lb.shape[0]), max(pool_b.shape[0], 1)]
        ptrs_a, ptrs_b = [_ffi.ptr(la), _ffi.ptr(pool_a)], [_ffi.ptr(lb), _ffi.ptr(pool_b)]
        keep += [pool_a, pool_b, ha, hb, sws, order]
    else:  # fused: every pool is a (mapped) rank pool; index = owner << 28 | local
        offa = torch.tensor(a_off, dtype=torch.int64, device=dev)
        offb = offa if b_is_a else torch.tensor(b_off, dtype=torch.int64, device=dev)
        t2 = tri.view(-1, 2).to(torch.int64)
        ga, gb = t2[:, 0].contiguous(), t2[:, 1].contiguous()
        own_a = torch.searchsorted(offa[1:], ga, right=True)
        own_b = torch.searchsorted(offb[1:], gb, right=True)
        tri_packed = torch.stack([(own_a << 28) | (ga - offa[own_a]), (own_b << 28) | (gb - offb[own_b])],
                                 dim=1).to(torch.int32).reshape(-1).contiguous()
        ptrs_a = [int(a_bases[r]) if r != rank else _ffi.ptr(la) for r in range(world)]
        ptrs_b = [int(b_bases[r]) if r != rank else _ffi.ptr(lb) for r in range(world)]
        counts_a = [max(a_off[r + 1] - a_off[r], 1) for r in range(world)]
        counts_b = [max(b_off[r + 1] - b_off[r], 1) for r in range(world)]
    ma = mb = fa = fb = mask_tri = None
    if masks is not None:  # the kernel reads A's column masks and B's row masks (+ NaN/Inf flags)
        ma, mb, fa, fb = masks
        mask_tri = tri
    arr_p = lambda v: (ctypes.c_void_p * len(v))(*v)  # noqa: E731
    arr_n = lambda v: (ctypes.c_int64 * len(v))(*v)  # noqa: E731
    _ffi.check(lib.qm_numeric_pools_ex(ctypes.byref(layout), arr_p(ptrs_a), arr_n(counts_a), len(ptrs_a),
                                       arr_p(ptrs_b), arr_n(counts_b), len(ptrs_b), _ffi.ptr(tri_packed),
                                       _ffi.ptr(mask_tri), _ffi.ptr(ma), _ffi.ptr(fa), _ffi.ptr(mb), _ffi.ptr(fb),
                                       _ffi.ptr(order),
                                       ctypes.byref(halo) if halo is not None else None, gate_units,
                                       _ffi.ptr(c_tptr), nc, nt, _ffi.ptr(out.blocks), _ffi.ptr(out.sumsq),
                                       _ffi.ptr(nz), _ffi.ptr(zc), _ffi.ptr(zc[1:]), _ffi.ptr(ws), wb, sh),
               "qm_numeric_pools_ex")
    info["_keep"] = keep + [ws, tri_packed]  # alive until the caller synchronises
    return out, nz, zc


def _fetch(comm, backend, local_blocks: torch.Tensor, offsets: list[int], need: torch.Tensor):
    """Request/serve exchange: returns the blocks of the sorted global indices `need`, in order,
    plus (bytes received from peers, bytes sent to peers, blocks received from peers)."""
    dev = need.device
    off = torch.tensor(offsets, dtype=torch.int64, device=dev)
    owner = torch.searchsorted(off[1:], need, right=True)
    req_counts = torch.bincount(owner, minlength=comm.world).cpu().tolist()
    wanted, serve_counts = comm.alltoallv(need, req_counts)  # indices peers want from me
    local_idx = wanted.reshape(-1) - offsets[comm.rank]
    payload = backend.gather_blocks(local_blocks, local_idx)
    # every owner returns exactly the blocks requested from it: the receive counts are known
    blocks, got_counts = comm.alltoallv(payload, serve_counts, recv_counts=req_counts)
    bsz = int(local_blocks.shape[1]) ** 2 * local_blocks.element_size()
    peers_in = sum(c for r, c in enumerate(got_counts) if r != comm.rank)
    peers_out = sum(c for r, c in enumerate(serve_counts) if r != comm.rank)
    return blocks, peers_in * bsz, peers_out * bsz, peers_in


NVLINK_GBS = 770.0   # measured peer copy bandwidth per direction (B200_PROFILING.md)
# auto mode: the fused kernel reads every remote block *reference* over NVLink; it is chosen only
# when those reads are a small share of the compute (banded: < 1 %), else the staged halo (each
# remote block once, overlapped with the local-only blocks; decay at P = 2 moves 98 MB instead of
# 555 MB of references)
FUSED_MAX_SHARE = 0.05
FP64_TFLOPS = 35.0   # sustained numeric-kernel rate used by the mode heuristic


def multiply(comm, layout, a_local: BlockSet, b_local: BlockSet, backend=None, b_is_a: bool = False,
             timer=None, mode: str | None = None):
    """This rank's part of C = A*B. `a_local`/`b_local` are the rank's owned key ranges (ascending
    across ranks). Returns (C blocks of this rank's C key range, DistStats).

    mode "exchange": request/serve halo exchange, then the local numeric kernel.
    mode "fused":    no exchange; the numeric kernel's TMA producer reads remote blocks directly
                     from their owners' pools (PeerPools, CUDA IPC over NVLink), overlapped with
                     the math (qm_numeric_pools_ex).
    mode "staged":   each remote block is gathered once from the peer pools into a local halo
                     pool (bulk copies on a few SMs) while the numeric kernel runs the C blocks
                     whose triples are all local; claims of the others wait for the gather
                     (staged_numeric). No collective for the halo.
    mode None:       $QM_DIST_MODE, default "auto".
    mode "auto":     fused when its estimated NVLink time (every remote block reference is a
                     remote read: peer loads bypass the local L2) stays under 5 % of the
                     estimated compute time, else staged (heavy reuse of remote blocks: decay,
                     random patterns); the exchange when some rank cannot map its peers."""
    backend = backend or CudaBackend()
    mode = mode or os.environ.get("QM_DIST_MODE", "auto")
    if mode not in ("auto", "exchange", "fused", "staged"):
        raise ConfigurationError(f"unknown distributed mode {mode!r} (auto, exchange, fused, staged)")
    stats = DistStats(rank=comm.rank, world=comm.world)
    clock = timer or (lambda: time.perf_counter())
    t0 = clock()
    bs = layout.block_size
    dev = a_local.blocks.device
    empty = BlockSet.empty(bs, dev)
    # Support masks (spgemm.symbolic): gathered with the keys when the operands' blocks have
    # partial supports, so every rank skips the same exactly-zero block pairs and k panels. The
    # filter is needed unless ALL of A's blocks have full column supports or ALL of B's full row
    # supports: one max-reduction of the two "not full" flags over the ranks.
    bl = a_local if b_is_a else b_local
    # One fixed-size header per rank (block counts; whether its blocks have partial supports) is the
    # only host-synchronising collective before the symbolic phase; the payloads (keys, masks) are
    # then gathered with known sizes. Support masks are gathered when the filter matters: unless
    # ALL of A's blocks have full column supports or ALL of B's full row supports.
    masks_on = spgemm.support_filter_enabled() and a_local.blocks.is_cuda
    if masks_on:
        a_local.support_masks()
        if not b_is_a:
            b_local.support_masks()
    # (the last two header fields are the operands' serials: the gathered global structure and its
    # row indexes are metadata of the distributed operands, kept with the local block set and
    # reused while every rank multiplies the same sets)
    # Every rank also reports which structure it has cached, so all ranks agree on reusing it (no
    # rank skips a gather the others perform).
    cached = a_local.__dict__.get("_dist_struct")
    mine = cached[1] if cached is not None and cached[0] == id(getattr(comm, "group", None)) else 0
    hdr = torch.tensor([a_local.n, b_local.n, int(masks_on and not a_local.masks_full[1]),
                        int(masks_on and not bl.masks_full[0]), a_local.serial, bl.serial, mine],
                       dtype=torch.int64, device="cpu" if getattr(comm, "stage", True) else dev)
    allh = comm.allgather_fixed(hdr).reshape(-1, 7).cpu().tolist()
    a_counts = [int(r[0]) for r in allh]
    b_counts = a_counts if b_is_a else [int(r[1]) for r in allh]
    use_masks = any(r[2] for r in allh) and any(r[3] for r in allh)
    skey = hash((comm.world, b_is_a, use_masks, tuple((int(r[4]), int(r[5])) for r in allh),
                 int(layout.n_logical), int(layout.leaf_dim), int(layout.depth), int(layout.block_size))) or 1
    hit = cached[2] if cached is not None and all(int(r[6]) == skey for r in allh) else None
    ix = None
    if hit is not None:
        ka, kb, ma, mb, fa, fb, ix = hit
        bad = torch.zeros((), dtype=torch.bool, device=ka.device)
    else:
        ka = comm.gather_known(a_local.keys, a_counts)
        kb = ka if b_is_a else comm.gather_known(b_local.keys, b_counts)
        ma = mb = fa = fb = None
        if use_masks:
            ma = comm.gather_known(a_local.masks[1].contiguous(), a_counts)
            mb = comm.gather_known(bl.masks[0].contiguous(), b_counts)
            fa = comm.gather_known(a_local.masks[2].contiguous(), a_counts)
            fb = fa if b_is_a else comm.gather_known(bl.masks[2].contiguous(), b_counts)
        # ownership contract (ascending, disjoint key ranges): checked on the device, read after the
        # symbolic phase's own synchronisation
        bad = torch.zeros((), dtype=torch.bool, device=ka.device)
        if ka.shape[0] > 1:
            bad |= (ka[1:] <= ka[:-1]).any()
        if kb.shape[0] > 1 and not b_is_a:
            bad |= (kb[1:] <= kb[:-1]).any()
        if getattr(backend, "row_indexes", None) is not None and ka.is_cuda and ka.shape[0] and kb.shape[0]:
            ix = backend.row_indexes(layout, ka, kb, ma, mb, fa, fb, b_is_a)
    a_off = [0] + list(np.cumsum(a_counts).tolist())
    b_off = [0] + list(np.cumsum(b_counts).tolist())
    if ka.shape[0] == 0 or kb.shape[0] == 0:
        return empty, stats
    t1 = clock()
    # Partitioned symbolic phase (qm_spgemm_count_part): a cheap global pass weighs the C tiles
    # (quadtree subtrees), cuts them into `world` contiguous key ranges of equal work, and this
    # rank counts and emits only the C blocks of its own range (the reference's workers likewise
    # expand only the tasks they execute, ops.py:197-241 / engine.py:286-300).
    if ix is not None:
        st = backend.symbolic_state(layout, ka, kb, a_cmask=ma, b_rmask=mb, part=(comm.world, comm.rank),
                                    ix=ix[0])
    else:
        st = backend.symbolic_state(layout, ka, kb, a_cmask=ma, b_rmask=mb, part=(comm.world, comm.rank))
    if hit is None:
        if bool(bad.item()):
            raise ContractViolationError("distributed operands must own ascending, disjoint key ranges")
        # (one structure per local operand: the latest product's)
        a_local.__dict__["_dist_struct"] = (id(getattr(comm, "group", None)), skey, (ka, kb, ma, mb, fa, fb, ix))
    stats.c_range, stats.tile_work = st.key_range, st.tile_work
    stats.n_c_local, stats.t_range = st.n_c, (0, st.n_t)

    def finish(c):
        """Global totals of the product, gathered once at the end -- the collective is also the
        barrier after which no rank reads another's pools."""
        tot = comm.allgather_fixed(torch.tensor([st.n_c, st.n_t], dtype=torch.int64,
                                                device="cpu" if getattr(comm, "stage", True) else dev))
        tot = tot.reshape(-1, 2).sum(dim=0).tolist()
        stats.n_c_global, stats.n_triples_global = int(tot[0]), int(tot[1])
        return c, stats

    lo, hi = 0, st.n_t
    if st.n_c:  # (a rank with an empty range still takes part in every collective below)
        c_keys, c_tptr = st.keys()
        tri = st.triples(c_tptr, lo, hi).view(-1, 2).to(torch.int64)
    else:
        c_keys = torch.zeros(0, dtype=torch.int64, device=dev)
        c_tptr = torch.zeros(1, dtype=torch.int64, device=dev)
        tri = torch.zeros((0, 2), dtype=torch.int64, device=dev)
    t2 = clock()
    peer_ok = (comm.world > 1 and mode != "exchange" and hasattr(backend, "numeric_peer")
               and layout.block_size in (32, 64, 128) and comm.world <= 8)
    if peer_ok:
        offa = torch.tensor(a_off, dtype=torch.int64, device=dev)
        offb = offa if b_is_a else torch.tensor(b_off, dtype=torch.int64, device=dev)
        own_a = torch.searchsorted(offa[1:], tri[:, 0].contiguous(), right=True)
        own_b = torch.searchsorted(offb[1:], tri[:, 1].contiguous(), right=True)
        blk_bytes = bs * bs * 8
        remote_refs = int(((own_a != comm.rank).sum() + (own_b != comm.rank).sum()).item()) if hi > lo else 0
        fused_s = remote_refs * blk_bytes / (NVLINK_GBS * 1e9)
        compute_s = 2.0 * bs ** 3 * (hi - lo) / (FP64_TFLOPS * 1e12)
        # 0 = fused (the kernel's TMA reads remote blocks in place: few remote references),
        # 1 = staged (copy engines pull the halo once while local-only C blocks compute);
        # every rank must take the same path (the peer mappings are collective)
        want = (0.0 if mode == "fused" else 1.0 if mode == "staged"
                else (0.0 if fused_s <= FUSED_MAX_SHARE * compute_s else 1.0))
        if dev.type == "cuda":
            torch.cuda.synchronize(dev)  # this rank's pools are written (any stream) before it
        # exports them; the records' all-gather inside PeerPools completes only once every rank has
        # done the same, so it is also the barrier before anyone reads a peer's pool
        pools = PeerPools(comm, [a_local.blocks] if b_is_a else [a_local.blocks, b_local.blocks])
        want, not_ok = comm.allreduce_max_vec([want, 0.0 if pools.ok else 1.0], dev)
        if not_ok > 0.0:
            # some rank cannot map its peers' pools: every rank takes the exchange path
            if not pools.ok:
                warnings.warn(f"rank {comm.rank}: peer pools unavailable ({pools.error}); "
                              "using the halo exchange", RuntimeWarning, stacklevel=2)
            pools.close()
            comm.barrier()
            pools = None
        if pools is not None:
            info = {}
            masks = (ma, mb, fa, fb) if ma is not None else None
            try:
                tri32 = tri.to(torch.int32).reshape(-1).contiguous()
                c = (backend.numeric_peer(layout, tri32, c_tptr, c_keys, comm.rank, a_off, b_off, pools.ptrs[0],
                                          pools.ptrs[-1], a_local.blocks, bl.blocks, b_is_a, masks,
                                          staged=want > 0.0, info=info) if hi > lo else empty)
                torch.cuda.synchronize(dev)
            finally:
                pools.close()
            t4 = clock()
            stats.n_c_local = c.n
            stats.mode = "staged" if want > 0.0 else "fused"
            # NVLink bytes: the staged halo (each remote block once), or every remote reference (fused)
            stats.bytes_received = info.get("halo_bytes", remote_refs * blk_bytes)
            stats.blocks_received = stats.bytes_received // blk_bytes
            stats.phase_s = {"structure": t1 - t0, "symbolic": t2 - t1, "exchange": 0.0,
                             "numeric": t4 - t2}
            stats.extra = {k: v for k, v in info.items() if not k.startswith("_")}
            stats.k_rows = int(info.get("k_rows", -1)) if hi > lo else 0
            return finish(c)  # (its collective: every rank has finished reading the others' pools)
    need_a = torch.unique(tri[:, 0]) if hi > lo else tri.new_zeros(0)
    need_b = torch.unique(tri[:, 1]) if hi > lo else tri.new_zeros(0)
    pool_a, ra, sa, na = _fetch(comm, backend, a_local.blocks, a_off, need_a)
    if b_is_a:
        pool_b, rb, sb, nb = _fetch(comm, backend, a_local.blocks, a_off, need_b)
    else:
        pool_b, rb, sb, nb = _fetch(comm, backend, b_local.blocks, b_off, need_b)
    stats.bytes_received, stats.bytes_sent, stats.blocks_received = ra + rb, sa + sb, na + nb
    t3 = clock()
    if hi == lo:
        stats.k_rows = 0
        return finish(empty)
    la = torch.searchsorted(need_a, tri[:, 0].contiguous())
    lb = torch.searchsorted(need_b, tri[:, 1].contiguous())
    tri_local = torch.stack([la, lb], dim=1).to(torch.int32).reshape(-1).contiguous()
    dummy_a = torch.empty(0, dtype=torch.float64, device=dev)
    # pool keys are the blocks' quadtree keys (the bs-16 grouping and claim orders decode them)
    pk_a, pk_b = ka[need_a], kb[need_b]
    if ma is not None:  # the pools' masks are the gathered ones (A columns, B rows, flags), not recomputed
        none_a = torch.full((need_a.shape[0],), -1, dtype=torch.int64, device=dev)
        none_b = torch.full((need_b.shape[0],), -1, dtype=torch.int64, device=dev)
        pa = BlockSet(pk_a, pool_a, dummy_a, torch.stack([none_a, ma[need_a], fa[need_a]]), (False, False))
        pb = BlockSet(pk_b, pool_b, dummy_a, torch.stack([mb[need_b], none_b, fb[need_b]]), (False, False))
    else:  # full supports (or filter off): nothing to skip, and no per-product mask pass
        pa = BlockSet(pk_a, pool_a, dummy_a, masks_full=(True, True))
        pb = BlockSet(pk_b, pool_b, dummy_a, masks_full=(True, True))
        pa.masks = pb.masks = torch.empty((3, 0), dtype=torch.int64, device=dev)
    c = backend.numeric(layout, pa, pb, tri_local, c_tptr, c_keys)
    stats.k_rows = int(getattr(backend, "last_k_rows", -1))
    t4 = clock()
    stats.n_c_local = c.n
    stats.mode = "exchange"
    stats.phase_s = {"structure": t1 - t0, "symbolic": t2 - t1, "exchange": t3 - t2, "numeric": t4 - t3}
    return finish(c)


def owned_range(keys_sorted: np.ndarray, bounds: list[int], rank: int) -> np.ndarray:
    """Keys of rank `rank` when the key space is cut at `bounds` (key values, len world+1)."""
    lo = np.searchsorted(keys_sorted, bounds[rank], side="left")
    hi = np.searchsorted(keys_sorted, bounds[rank + 1], side="left")
    return keys_sorted[lo:hi]
