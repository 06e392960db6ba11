"""The partitioned symbolic phase of the multi-GPU product (qm_spgemm_count_part) on one B200: each
simulated rank counts and emits only its own C key range. Checks, for several world sizes, that
  * the device cut equals the host statement (distributed.tile_partition) bound for bound;
  * the ranks' C keys, in rank order, are exactly the single-GPU product's C keys, and each rank's
    triples are exactly the single-GPU triples of its C blocks (same k order);
  * the ranks' numeric results, concatenated, are bitwise the single-GPU product."""

import numpy as np
import pytest
import torch

from paper_2011_11762_b200 import MatrixSession, _ffi, spgemm
from paper_2011_11762_b200 import distributed as D
from paper_2011_11762_b200 import generators as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda:0")


EXTRA = {  # the staged path at the other TMA block sizes (bs 128: 4 work units per C block)
    "banded-bs32": G.BaselineConfig("t32", "banded", 8192, 32, half_bw=256),
    "banded-bs128": G.BaselineConfig("t128", "banded", 16384, 128, half_bw=512),
    # more ranks than C tiles and than owned blocks (ragged n = 96: 3x3 blocks of a 4x4 grid)
    "tiny": G.BaselineConfig("t-tiny", "banded", 96, 32, half_bw=20),
}


@pytest.mark.parametrize("name", ["C1", "C2-16384", "C3", "C4", "tiny"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_ranks_partition_the_product_exactly(dev, name, world):
    cfg = EXTRA[name] if name in EXTRA else G.CONFIGS[name]
    geom, a, b = G.config_operands_device(cfg, dev)
    if cfg.same_operand:
        b = a
    lay = _ffi.make_layout(geom.params, geom.bs)
    use = spgemm._use_masks(a, b)
    am, bm = (a.masks[1], b.masks[0]) if use else (None, None)
    full = spgemm.symbolic(lay, a, b)
    ref_keys = full.c_keys.cpu().numpy()
    ref_tptr = full.c_tptr.cpu().numpy()
    ref_tri = full.tri.view(-1, 2).cpu().numpy()
    bounds = D.tile_partition(geom, a.keys.cpu().numpy(), b.keys.cpu().numpy(), world,
                              am.cpu().numpy() if use else None, bm.cpu().numpy() if use else None)
    keys, tris, blocks = [], [], []
    c_full = spgemm.multiply_blocks(lay, a, b)
    for r in range(world):
        st = spgemm.SymbolicState(lay, a.keys, a.n, b.keys, b.n, None, am, bm, part=(world, r))
        assert st.key_range == (bounds[r], bounds[r + 1])
        assert st.key_cuts.cpu().tolist() == [x if x < 2**63 else x - 2**64 for x in bounds]
        if st.n_c == 0:
            continue
        ck, ct = st.keys()
        tri = st.triples(ct)
        k = ck.cpu().numpy()
        assert k.min() >= bounds[r] and k.max() < bounds[r + 1]
        lo, hi = np.searchsorted(ref_keys, [k[0], k[-1] + 1])
        np.testing.assert_array_equal(k, ref_keys[lo:hi])
        np.testing.assert_array_equal(tri.view(-1, 2).cpu().numpy(), ref_tri[ref_tptr[lo]:ref_tptr[hi]])
        plan = spgemm.SymbolicPlan(st.n_c, st.n_t, ck, ct, tri)
        c, nz, zc = spgemm.numeric(lay, a, b, plan)
        n_zero = _ffi.read_i64(zc)
        c = spgemm.compact(geom.bs, c, nz, n_zero)
        keys.append(c.keys)
        blocks.append(c.blocks)
        tris.append(st.n_t)
    assert sum(tris) == full.n_triples
    assert torch.equal(torch.cat(keys), c_full.keys)
    assert torch.equal(torch.cat(blocks), c_full.blocks)  # bitwise: same triples, same order per block
    # balance: every rank's triples within one tile's work of the mean (structural counts; C4's
    # masked counts follow them closely)
    if not use:
        assert max(tris) - min(tris) <= max(1, full.n_triples // 64)


def test_partitioned_distributed_path_single_rank_session(dev):
    """The distributed path at world 1 (LocalComm): the whole key space, the single-GPU result."""
    ses = MatrixSession(device=dev)
    cfg = G.CONFIGS["C2-16384"]
    geom, a, b = G.config_operands_device(cfg, dev)
    c1 = ses.multiply(ses.matrix_from_blockset(geom, a), ses.matrix_from_blockset(geom, b)).root.blockset
    c2, st = D.multiply(D.LocalComm(), _ffi.make_layout(geom.params, geom.bs), a, b)
    assert st.c_range == (0, 1 << (2 * geom.params.depth + 2 * geom.lbits))
    assert torch.equal(c1.keys, c2.keys) and torch.equal(c1.blocks, c2.blocks)


def _in_process_peers(t: torch.Tensor, off: list) -> list:
    """Device addresses of every rank's pool when all of them are slices of one tensor (the one-GPU
    stand-in for CUDA-IPC-mapped peer pools)."""
    blk = t.shape[1] * t.shape[2] * t.element_size()
    return [t.data_ptr() + off[r] * blk for r in range(len(off) - 1)]


@pytest.mark.parametrize("name,world,staged", [("C4", 4, True), ("C4", 8, True), ("C2-16384", 3, True),
                                               ("C3", 2, True), ("C4", 4, False), ("banded-bs32", 3, True),
                                               ("banded-bs128", 3, True), ("banded-bs128", 2, False),
                                               ("tiny", 8, True), ("tiny", 8, False)])
def test_staged_and_fused_rank_numeric_equal_single_gpu(dev, name, world, staged):
    """staged_numeric for every rank, the operands' other ranks being slices of the same pools:
    staged (halo gathered by k_halo_gather while the numeric kernel -- its programmatic dependent --
    runs the local-only C blocks, the rest waiting for the gather) and fused (TMA reads of the peer
    pools) give each rank's C blocks bitwise as the single-GPU product; the halo holds each remote
    block once (halo_bytes = unique remote blocks). Also with an emulated slow link (the gather
    lasts >= halo bytes / 20 GB/s), so the gated claims really wait."""
    cfg = EXTRA[name] if name in EXTRA else G.CONFIGS[name]
    geom, a, b = G.config_operands_device(cfg, dev)
    b_is_a = cfg.same_operand
    if b_is_a:
        b = a
    lay = _ffi.make_layout(geom.params, geom.bs)
    use = spgemm._use_masks(a, b)
    am, bm = (a.masks[1], b.masks[0]) if use else (None, None)
    c_full = spgemm.multiply_blocks(lay, a, b)
    a_off = [(a.n * r) // world for r in range(world + 1)]
    b_off = a_off if b_is_a else [(b.n * r) // world for r in range(world + 1)]
    masks = (a.masks[1], b.masks[0], a.masks[2], b.masks[2]) if use else None
    keys, blocks = [], []
    for r in range(world):
        st = spgemm.SymbolicState(lay, a.keys, a.n, b.keys, b.n, None, am, bm, part=(world, r))
        if st.n_c == 0:
            continue
        ck, ct = st.keys()
        tri32 = st.triples(ct)
        tri = tri32.view(-1, 2).to(torch.int64)
        info = {}
        c, nz, zc = D.staged_numeric(lay, tri32, ct, ck, r, a_off, b_off, _in_process_peers(a.blocks, a_off),
                                           _in_process_peers(b.blocks, b_off), a.blocks[a_off[r]:a_off[r + 1]],
                                           b.blocks[b_off[r]:b_off[r + 1]], b_is_a, masks, staged=staged,
                                           info=info, emulate_link_gbs=20.0 if r == 1 else None)
        torch.cuda.synchronize()
        if staged:
            t = tri
            ra = (t[:, 0] < a_off[r]) | (t[:, 0] >= a_off[r + 1])
            rb = (t[:, 1] < b_off[r]) | (t[:, 1] >= b_off[r + 1])
            uniq = (torch.unique(torch.cat([t[:, 0][ra], t[:, 1][rb]])).numel() if b_is_a else
                    torch.unique(t[:, 0][ra]).numel() + torch.unique(t[:, 1][rb]).numel())
            assert info["halo_bytes"] == uniq * geom.bs ** 2 * 8
            assert 0 <= info["local_c_blocks"] <= st.n_c
        c = spgemm.compact(geom.bs, c, nz, _ffi.read_i64(zc))
        keys.append(c.keys)
        blocks.append(c.blocks)
    assert torch.equal(torch.cat(keys), c_full.keys)
    assert torch.equal(torch.cat(blocks), c_full.blocks)
