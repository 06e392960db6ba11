"""Multi-rank product path on CPU: world_size 2 and 3 over gloo, with the oracle as the compute
backend and the product's own partition / request-serve exchange code (distributed.py).

Checks: the union of the ranks' C ranges equals the single-process product bit for bit (same
summation order per C block), the partition balances triples, and halo bytes are reported.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import spgemm_oracle as O
from paper_2011_11762_b200 import distributed as D
from paper_2011_11762_b200 import generators as G
from paper_2011_11762_b200._ffi import make_layout
from paper_2011_11762_b200.blocks import BlockSet


class OracleBackend:
    """Test backend: oracle symbolic/numeric on the CPU; same interface as D.CudaBackend."""

    def __init__(self, geom):
        self.geom = geom
        self.og = O.Geom(geom.params.n_logical, geom.params.leaf_dim, geom.bs)

    def symbolic_state(self, layout, a_keys, b_keys, a_cmask=None, b_rmask=None, part=None):
        """The oracle's symbolic product restricted, like qm_spgemm_count_part, to this rank's C key
        range from the tile partition (D.tile_partition, the host statement of the device cut)."""
        outer = self
        self.ka = a_keys.numpy()
        kc, cptr, ta, tb, tk = O.symbolic(self.og, a_keys.numpy(), b_keys.numpy())
        key_range = None
        if part is not None:
            world, rank = part
            bounds = D.tile_partition(self.geom, a_keys.numpy(), b_keys.numpy(), world)
            key_range = (bounds[rank], bounds[rank + 1])
            sel = (kc >= key_range[0]) & (kc < key_range[1])
            c0, c1 = int(np.argmax(sel)) if sel.any() else 0, int(sel.sum())
            t0, t1 = int(cptr[c0]), int(cptr[c0 + c1])
            kc, cptr = kc[c0:c0 + c1], cptr[c0:c0 + c1 + 1] - t0
            ta, tb = ta[t0:t1], tb[t0:t1]

        class St:
            n_c, n_t = int(kc.size), int(ta.size)
            tile_work = 0

            def keys(self):
                return torch.from_numpy(kc), torch.from_numpy(cptr)

            def triples(self, c_tptr, lo, hi):
                return torch.from_numpy(np.stack([ta[lo:hi], tb[lo:hi]], 1).astype(np.int32).reshape(-1))

        St.key_range = key_range
        _ = outer
        return St()

    def gather_blocks(self, blocks, idx):
        return blocks.index_select(0, idx)

    def numeric(self, layout, pa, pb, tri, c_tptr, c_keys):
        t = tri.view(-1, 2).numpy().astype(np.int64)
        _, k = self.og.decode(pa.keys.numpy()[t[:, 0]])  # pool keys are the blocks' quadtree keys
        kc, bc, _ = O.numeric(self.og, c_keys.numpy(), c_tptr.numpy(), t[:, 0], t[:, 1], k,
                              pa.blocks.numpy(), pb.blocks.numpy())
        return BlockSet(torch.from_numpy(kc), torch.from_numpy(bc), torch.from_numpy(np.einsum("nij,nij->n", bc, bc)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = {
    "banded": G.BaselineConfig("t-band", "banded", 2048, 32, half_bw=100),
    "random": G.BaselineConfig("t-rand", "random", 2048, 32, per_row=4),
    # edge cases: fewer C tiles than ranks (ragged n = 96 -> 3x3 blocks in a 4x4 grid), and a
    # sparse random pattern with empty block rows/columns (per_row = 1)
    "tiny": G.BaselineConfig("t-tiny", "banded", 96, 32, half_bw=20),
    "sparse": G.BaselineConfig("t-sparse", "random", 512, 32, per_row=1),
}


class NoPoolsBackend(OracleBackend):
    """Offers the peer paths (fused / staged), which must not run: on a host without peer-mappable
    device memory PeerPools cannot export, and every rank has to agree on the exchange instead."""

    def numeric_peer(self, *args, **kwargs):
        raise AssertionError("peer-pool kernel launched although a rank could not map its peers")


def _worker(rank, world, port, case, outdir, mode="auto"):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    cfg = CASES[case]
    geom, (ka, ba), (kb, bb) = G.config_operands_host(cfg)
    # ownership: contiguous key ranges with uneven cut points (ownership need not match C's cut)
    qa = np.r_[0, np.sort(np.random.default_rng(5).choice(ka.size, world - 1, replace=False)), ka.size]
    qb = np.r_[0, np.sort(np.random.default_rng(6).choice(kb.size, world - 1, replace=False)), kb.size]
    la = BlockSet(torch.from_numpy(ka[qa[rank]:qa[rank + 1]]), torch.from_numpy(ba[qa[rank]:qa[rank + 1]]),
                  torch.zeros(0))
    lb = BlockSet(torch.from_numpy(kb[qb[rank]:qb[rank + 1]]), torch.from_numpy(bb[qb[rank]:qb[rank + 1]]),
                  torch.zeros(0))
    comm = D.Comm()
    backend = NoPoolsBackend(geom) if mode in ("fused", "staged") else OracleBackend(geom)
    if mode in ("fused", "staged"):
        import warnings

        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            c, st = D.multiply(comm, make_layout(geom.params, geom.bs), la, lb, backend=backend, mode=mode)
        assert st.mode == "exchange"
        assert any("peer pools unavailable" in str(x.message) for x in w)
    else:
        c, st = D.multiply(comm, make_layout(geom.params, geom.bs), la, lb, backend=backend)
    keys, _ = comm.allgather_varlen(c.keys)
    flat, _ = comm.allgather_varlen(c.blocks.reshape(-1))
    recv = torch.tensor([st.bytes_received, st.t_range[1] - st.t_range[0]], dtype=torch.int64)
    allr = [torch.zeros_like(recv) for _ in range(world)]
    dist.all_gather(allr, recv)
    if rank == 0:
        np.savez(os.path.join(outdir, "out.npz"), keys=keys.numpy(), blocks=flat.numpy(),
                 recv=torch.stack(allr).numpy(), nt=st.n_triples_global)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", ["banded", "random"])
def test_distributed_product_equals_single_process(tmp_path, world, case):
    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    out = np.load(tmp_path / "out.npz")
    cfg = CASES[case]
    geom, (ka, ba), (kb, bb) = G.config_operands_host(cfg)
    kc, bc, T = O.multiply(O.Geom(cfg.n, cfg.bs, cfg.bs), ka, ba, kb, bb)
    np.testing.assert_array_equal(out["keys"], kc)  # same C block set, in key order across ranks
    np.testing.assert_array_equal(out["blocks"].reshape(bc.shape), bc)  # bitwise: same order per block
    per_rank_triples = out["recv"][:, 1]
    assert per_rank_triples.sum() == T == int(out["nt"])
    assert per_rank_triples.max() - per_rank_triples.min() <= 2 * 32  # balanced by triples (+- one C row of work)
    assert out["recv"][:, 0].sum() > 0  # halo blocks crossed ranks


@pytest.mark.parametrize("world,case", [(3, "tiny"), (4, "tiny"), (3, "sparse")])
def test_distributed_edge_cases_equal_single_process(tmp_path, world, case):
    """Ranks left without C blocks (or without owned blocks) still take part in every collective,
    and the union of the ranks' products is the single-process product bit for bit."""
    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    out = np.load(tmp_path / "out.npz")
    cfg = CASES[case]
    geom, (ka, ba), (kb, bb) = G.config_operands_host(cfg)
    kc, bc, T = O.multiply(O.Geom(cfg.n, cfg.bs, cfg.bs), ka, ba, kb, bb)
    np.testing.assert_array_equal(out["keys"], kc)
    np.testing.assert_array_equal(out["blocks"].reshape(bc.shape), bc)
    assert out["recv"][:, 1].sum() == T == int(out["nt"])


@pytest.mark.parametrize("mode", ["fused", "staged"])
def test_peer_modes_fall_back_on_every_rank_when_pools_cannot_be_mapped(tmp_path, mode):
    mp.spawn(_worker, args=(2, _free_port(), "banded", str(tmp_path), mode), nprocs=2, join=True)
    out = np.load(tmp_path / "out.npz")
    cfg = CASES["banded"]
    geom, (ka, ba), (kb, bb) = G.config_operands_host(cfg)
    kc, bc, _ = O.multiply(O.Geom(cfg.n, cfg.bs, cfg.bs), ka, ba, kb, bb)
    np.testing.assert_array_equal(out["keys"], kc)
    np.testing.assert_array_equal(out["blocks"].reshape(bc.shape), bc)


@pytest.mark.parametrize("name,world", [("C1", 2), ("C1", 8), ("C2-16384", 4), ("C3", 8), ("C5-64", 8)])
def test_tile_partition_is_balanced_and_covers_the_key_space(name, world):
    """tile_partition (host twin of qm_spgemm_count_part's cut): world+1 monotone key bounds from
    0 to the end of the key space, each range a union of whole tiles, and balanced: every rank's
    structural triples are within one tile's work of W/world."""
    cfg = G.CONFIGS[name]
    geom = cfg.geometry
    ka, kb = G.config_keys(cfg, 0), G.config_keys(cfg, 1)
    bounds = D.tile_partition(geom, ka, kb, world)
    depth = geom.params.depth
    tl = min(depth, D.MAX_TILE_LEVELS)
    kshift = 2 * (depth - tl) + 2 * geom.lbits
    assert bounds[0] == 0 and bounds[-1] == 1 << (2 * depth + 2 * geom.lbits)
    assert all(x <= y for x, y in zip(bounds, bounds[1:])) and all(b % (1 << kshift) == 0 for b in bounds)
    import scipy.sparse as sp

    nb = geom.nbg
    ai, ak = geom.decode(ka)
    bk, bj = geom.decode(kb)
    c = (sp.csr_matrix((np.ones(ai.size), (ai, ak)), shape=(nb, nb)) @
         sp.csr_matrix((np.ones(bk.size), (bk, bj)), shape=(nb, nb))).tocoo()
    keys = geom.qkey(c.row.astype(np.int64), c.col.astype(np.int64))
    share = np.array([c.data[(keys >= bounds[r]) & (keys < bounds[r + 1])].sum() for r in range(world)])
    tile_work = np.bincount(keys >> kshift, weights=c.data)
    assert share.sum() == c.data.sum()
    assert np.abs(share - c.data.sum() / world).max() <= tile_work.max() + 1


def test_partition_bounds_are_balanced_and_monotone():
    tptr = torch.tensor(np.r_[0, np.cumsum(np.random.default_rng(0).integers(1, 20, 1000))])
    for world in (1, 2, 3, 8):
        cb, tb = D.partition(tptr, world)
        assert cb[0] == 0 and cb[-1] == 1000 and all(x <= y for x, y in zip(cb, cb[1:]))
        share = np.diff(tb)
        assert share.max() - share.min() <= 2 * 20


def test_local_comm_is_identity():
    c = D.LocalComm()
    t = torch.arange(5)
    assert torch.equal(c.allgather_varlen(t)[0], t)
    assert torch.equal(c.alltoallv(t, [5])[0], t)


def _locality_worker(rank, world, port, outdir):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    cfg = G.BaselineConfig(f"loc{world}", "banded", 1024 * world, 64, half_bw=64)
    geom, (ka, ba), (kb, bb) = G.config_operands_host(cfg)
    qa = (np.arange(world + 1) * ka.size) // world
    qb = (np.arange(world + 1) * kb.size) // world
    la = BlockSet(torch.from_numpy(ka[qa[rank]:qa[rank + 1]]), torch.from_numpy(ba[qa[rank]:qa[rank + 1]]),
                  torch.zeros(0))
    lb = BlockSet(torch.from_numpy(kb[qb[rank]:qb[rank + 1]]), torch.from_numpy(bb[qb[rank]:qb[rank + 1]]),
                  torch.zeros(0))
    _, st = D.multiply(D.Comm(), make_layout(geom.params, geom.bs), la, lb, backend=OracleBackend(geom),
                       mode="exchange")
    got = torch.tensor([st.bytes_received], dtype=torch.int64)
    allv = [torch.zeros_like(got) for _ in range(world)]
    dist.all_gather(allv, got)
    if rank == 0:
        np.save(os.path.join(outdir, f"bytes_{world}.npy"), torch.cat(allv).numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_weak_scaling_locality(tmp_path):
    """Mirror of the reference's test_weak_scaling_locality (test_acceptance.py:333-347): banded
    matrices with n growing with the rank count; doubling the ranks may grow the mean bytes each
    rank receives by at most 1.5x (the key-range partition keeps the halo to the band)."""
    means = {}
    for world in (2, 4, 8):
        mp.spawn(_locality_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
        means[world] = float(np.load(tmp_path / f"bytes_{world}.npy").mean())
    assert means[2] > 0
    for low, high in ((2, 4), (4, 8)):
        assert means[high] / means[low] <= 1.5, (low, high, means)


def test_tile_partition_with_masks_weighs_executed_panels():
    """The masked host twin (k_tile_work's weights): every block pair adds the number of 16-row k
    panels where A's column mask and B's row mask meet (0: an exactly-zero product) to its C tile;
    checked against a pair-by-pair loop on a small random structure, and the cut is monotone."""
    from paper_2011_11762_b200.layout import Geometry, MatrixParams

    rng = np.random.default_rng(11)
    n, bs, leaf = 2048, 64, 64
    geom = Geometry(MatrixParams.create(n, leaf), bs)
    nb = geom.nbg
    pa = np.unique(rng.integers(0, nb, (300, 2)), axis=0)
    pb = np.unique(rng.integers(0, nb, (300, 2)), axis=0)
    ka = np.sort(geom.qkey(pa[:, 0], pa[:, 1]))
    kb = np.sort(geom.qkey(pb[:, 0], pb[:, 1]))
    am = rng.integers(0, 2**63, ka.size, dtype=np.int64) & rng.integers(0, 2**63, ka.size, dtype=np.int64)
    bm = rng.integers(0, 2**63, kb.size, dtype=np.int64) & rng.integers(0, 2**63, kb.size, dtype=np.int64)
    world = 4
    bounds = D.tile_partition(geom, ka, kb, world, am, bm)
    assert bounds[0] == 0 and all(x <= y for x, y in zip(bounds, bounds[1:]))
    depth = geom.params.depth
    tl = min(depth, D.MAX_TILE_LEVELS)
    kshift = 2 * (depth - tl) + 2 * geom.lbits
    ai, ak = geom.decode(ka)
    bk, bj = geom.decode(kb)
    work = {}
    for x in range(ka.size):
        for y in np.nonzero(bk == ak[x])[0]:
            m = int(am[x]) & int(bm[y])
            w = sum(((m >> s) & 0xFFFF) != 0 for s in (0, 16, 32, 48))
            t = int(geom.qkey(np.array([ai[x]]), np.array([bj[y]]))[0]) >> kshift
            work[t] = work.get(t, 0) + w
    tiles = np.zeros(1 << (2 * tl), dtype=np.int64)
    for t, w in work.items():
        tiles[t] = w
    prefix = np.concatenate([[0], np.cumsum(tiles)])
    W = int(prefix[-1])
    cuts = [0] + [int(np.searchsorted(prefix[:tiles.size], (W * r) // world, side="left")) for r in range(1, world)]
    cuts.append(tiles.size)
    assert bounds == [c << kshift for c in cuts]


def _cache_worker(rank, world, port, outdir):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    cfg = CASES["banded"]
    geom, (ka, ba), (kb, bb) = G.config_operands_host(cfg)
    qa = [(ka.size * r) // world for r in range(world + 1)]
    qb = [(kb.size * r) // world for r in range(world + 1)]
    la = BlockSet(torch.from_numpy(ka[qa[rank]:qa[rank + 1]]), torch.from_numpy(ba[qa[rank]:qa[rank + 1]]),
                  torch.zeros(0))

    def blocks_b():
        return BlockSet(torch.from_numpy(kb[qb[rank]:qb[rank + 1]]), torch.from_numpy(bb[qb[rank]:qb[rank + 1]]),
                        torch.zeros(0))

    lb = blocks_b()
    comm = D.Comm()
    lay = make_layout(geom.params, geom.bs)
    outs = []
    for step in range(3):
        if step == 2 and rank == 1:
            lb = blocks_b()  # one rank multiplies a new (equal) block set: every rank must re-gather
        c, st = D.multiply(comm, lay, la, lb, backend=OracleBackend(geom))
        keys, _ = comm.allgather_varlen(c.keys)
        flat, _ = comm.allgather_varlen(c.blocks.reshape(-1))
        outs.append((keys.numpy(), flat.numpy()))
    if rank == 0:
        np.savez(os.path.join(outdir, "out.npz"), k0=outs[0][0], b0=outs[0][1], k1=outs[1][0], b1=outs[1][1],
                 k2=outs[2][0], b2=outs[2][1])
    dist.barrier()
    dist.destroy_process_group()


def test_structure_cache_is_agreed_by_every_rank(tmp_path):
    """The gathered global structure is reused only when every rank multiplies the same block sets
    as last time (serials in the header): a repeated product reuses it, a product where one rank
    changed its operand re-gathers on all ranks (no rank skips a collective) -- same result each time."""
    mp.spawn(_cache_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    out = np.load(tmp_path / "out.npz")
    for i in (1, 2):
        np.testing.assert_array_equal(out[f"k{i}"], out["k0"])
        np.testing.assert_array_equal(out[f"b{i}"], out["b0"])
