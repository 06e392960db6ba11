"""GPU parity: libqmb200 through the drop-in API against the reference's outputs and the oracle.

Bar (BASELINE.json north_star): the set of nonzero C blocks bit-exact; values within relative
Frobenius error 1e-12 in float64 (TOL below); integer-valued products bit-exact (canonical bytes).
"""

import numpy as np
import pytest
import torch

import helpers
from oracle import spgemm_oracle as O
from paper_2011_11762_b200 import (
    ConfigurationError,
    ContractViolationError,
    DimensionMismatchError,
    MatrixSession,
    _ffi,
    bridge,
    spgemm,
)
from paper_2011_11762_b200 import generators as G
from paper_2011_11762_b200.blocks import BlockSet
from paper_2011_11762_b200.layout import Geometry, MatrixParams

pytestmark = pytest.mark.gpu
TOL = 1e-12  # north_star: relative Frobenius error in float64


@pytest.fixture(scope="module")
def ses():
    return helpers.gpu_session()


def _host(m):
    return m.root.blockset.to_host() if not m.root.is_nil else (np.zeros(0, np.int64), None, None)


def test_native_library_is_the_path(ses):
    lib = _ffi.load()
    before = lib.qm_launch_count()
    a = helpers.build(ses, helpers.random_sparse(128, 0.05, 1), 64, 64)
    c = ses.multiply(a, a)
    assert lib.qm_launch_count() > before  # the product ran in libqmb200 kernels
    assert c.root.blockset.blocks.is_cuda
    # bs 16 reports the TMA path (grouped leaf-row kernel); one-block-per-leaf layouts fall back to
    # cp.async inside qm_numeric
    assert lib.qm_numeric_path(64) == 2 and lib.qm_numeric_path(16) == 2 and lib.qm_numeric_path(12) == 0


@pytest.mark.parametrize("ci", range(12))
def test_small_cases_match_reference(ses, ci):
    g, cases = helpers.small_cases()
    n, leaf, bs, da_, db_, sa, sb = cases[ci]
    da, db = helpers.random_sparse(n, da_, sa), helpers.random_sparse(n, db_, sb)
    c = ses.multiply(helpers.build(ses, da, leaf, bs), helpers.build(ses, db, leaf, bs))
    kc, bc, _ = _host(c)
    np.testing.assert_array_equal(kc, g[f"c{ci}_keys"])  # C block set bit-exact
    assert helpers.rel(bc, g[f"c{ci}_blocks"]) <= TOL
    assert helpers.rel(ses.to_dense(c), da @ db) <= TOL


def test_integer_product_is_bit_exact(ses):
    """The reference's schedule-independence case (test_acceptance.py:315-325): canonical bytes of
    C = A*A on the value-1.0 band equal the reference's, and sum(C) = flop_count_exact / 2."""
    g = helpers.load("band_ones")
    case = G.ExperimentCase("banded", 8192, 64)
    a = G.generate(ses.store, case, 128, "block_sparse", 32)
    c = ses.multiply(a, a)
    assert helpers.sha(ses.canonical(c)) == bytes(g["sha"])
    assert c.root.blockset.blocks.sum().item() == G.flop_count_exact(case) // 2


@pytest.mark.parametrize("case,leaf,bs", [
    (("banded", 3000, 37, 0, 0, 0), 64, 16),
    (("growing_block", 2048, 20, 300, 0, 0), 128, 32),
    (("random_blocks", 4096, 16, 200, 6, 3), 128, 64),
    (("random_blocks", 1500, 8, 100, 4, 9), 96, 32),
])
def test_generated_families_sum_to_half_the_flop_count(ses, case, leaf, bs):
    """Known-answer test (generators.py:134-138, oracles.py:106-109): on the
    reference's value-1.0 families, every C entry counts scalar products, so sum(C) is exactly
    flop_count_exact / 2 and every C value is an integer."""
    c_ = G.ExperimentCase(*case)
    a = G.generate(ses.store, c_, leaf, "block_sparse", bs)
    c = ses.multiply(a, a)
    blocks = c.root.blockset.blocks
    assert blocks.sum().item() == G.flop_count_exact(c_) // 2
    assert torch.equal(blocks, blocks.round())


@pytest.mark.parametrize("name", ["C1", "C3s", "C4s", "C2-16384"])
def test_configs_match_reference(ses, name):
    g = helpers.load(name)
    cfg = G.CONFIGS.get(name) or {
        "C3s": G.BaselineConfig("C3s", "random", 8192, 64, per_row=8),
        "C4s": G.BaselineConfig("C4s", "decay", 4096, 64, same_operand=True),
    }[name]
    geom, a, b = G.config_operands_device(cfg, ses.device)
    ma = ses.matrix_from_blockset(geom, a)
    mb = ma if cfg.same_operand else ses.matrix_from_blockset(geom, b)
    c = ses.multiply(ma, mb)
    kc, bc, sq = _host(c)
    np.testing.assert_array_equal(kc, g["c_keys"])
    norms = np.array([np.linalg.norm(x) for x in bc])
    assert np.max(np.abs(norms - g["c_norms"]) / g["c_norms"]) <= TOL
    np.testing.assert_allclose(np.sqrt(sq), g["c_norms"], rtol=TOL)  # fused epilogue norms
    checks = np.einsum("nij,ij->n", bc, helpers.check_weights(cfg.bs))
    assert helpers.rel(checks, g["c_checks"]) <= TOL
    assert helpers.rel(bc[g["sample_idx"]], g["sample_blocks"]) <= TOL
    assert abs(np.linalg.norm(bc) - g["c_frob"][0]) <= TOL * g["c_frob"][0]


@pytest.mark.parametrize("name", ["C1", "C3s"])
def test_full_product_vs_oracle(ses, name):
    cfg = G.CONFIGS.get(name) or G.BaselineConfig("C3s", "random", 8192, 64, per_row=8)
    geom, (ka, ba), (kb, bb) = G.config_operands_host(cfg)
    kc, bc, _ = O.multiply(O.Geom(cfg.n, cfg.bs, cfg.bs), ka, ba, kb, bb)
    c = ses.multiply(ses.matrix_from_blocks(geom, ka, ba), ses.matrix_from_blocks(geom, kb, bb))
    k2, b2, _ = _host(c)
    np.testing.assert_array_equal(k2, kc)
    assert helpers.rel(b2, bc) <= TOL


@pytest.mark.parametrize("bs,n,pattern", [(64, 4096, 1), (32, 1000, 1), (128, 1024, 0), (16, 300, 0), (12, 96, 1)])
def test_device_generator_matches_numpy_streams(bs, n, pattern):
    geom = Geometry(MatrixParams.create(n, bs), bs)
    keys = G.banded_block_keys(geom, 100)
    dev = G.device_blocks(geom, keys, seed=7, matrix_id=1, pattern=pattern, half_bw=100, device="cuda:0")
    host = G.host_blocks(geom, keys, 7, 1, pattern, 100)
    np.testing.assert_array_equal(dev.blocks.cpu().numpy(), host)  # bit-identical PCG64 streams
    np.testing.assert_allclose(dev.sumsq.cpu().numpy(), np.einsum("nij,nij->n", host, host), rtol=1e-14)


@pytest.mark.parametrize("kind,n,bs,per_row", [
    ("banded", 4096, 64, 0), ("random", 8192, 64, 8), ("random", 1 << 17, 16, 8), ("banded", 3000, 8, 0),
    ("random", 1 << 17, 16, 64)])
def test_symbolic_phase_matches_oracle_exactly(ses, monkeypatch, kind, n, bs, per_row):
    """Triples, their grouping and k order (block_sparse.py:121-129) equal the oracle's; the
    random 8192-wide grid exercises the multi-window accumulator (window 4096 columns), rows with
    more than 32 A entries the grouped triple emission (32 A entries per group). Structure only
    (the blocks are placeholders), so without the support-mask filter."""
    monkeypatch.setenv("QM_SUPPORT_FILTER", "0")
    cfg = G.BaselineConfig("t", kind, n, bs, half_bw=300, per_row=per_row)
    geom = cfg.geometry
    ka, kb = G.config_keys(cfg, 0), G.config_keys(cfg, 1)
    dev = ses.device
    a = G.BlockSet(torch.from_numpy(ka).to(dev), torch.empty((ka.size, 1, 1), dtype=torch.float64, device=dev),
                   torch.empty(ka.size, dtype=torch.float64, device=dev))
    b = G.BlockSet(torch.from_numpy(kb).to(dev), torch.empty((kb.size, 1, 1), dtype=torch.float64, device=dev),
                   torch.empty(kb.size, dtype=torch.float64, device=dev))
    layout = _ffi.make_layout(geom.params, bs)
    plan = spgemm.symbolic(layout, a, b)
    kc, cptr, ta, tb, _ = O.symbolic(O.Geom(n, bs, bs), ka, kb)
    np.testing.assert_array_equal(plan.c_keys.cpu().numpy(), kc)
    np.testing.assert_array_equal(plan.c_tptr.cpu().numpy(), cptr)
    tri = plan.tri.cpu().numpy().view(np.uint32).reshape(-1, 2).astype(np.int64)
    np.testing.assert_array_equal(tri[:, 0], ta)
    np.testing.assert_array_equal(tri[:, 1], tb)


@pytest.mark.parametrize("case", ["a_empty", "b_empty", "no_match"])
def test_symbolic_c_abi_degenerate_operands(ses, case):
    """qm_spgemm_count straight through the C ABI: an empty operand, or operands whose inner
    indices never meet, give nC = nT = 0 (the nil product, ops.py:244-245)."""
    import ctypes

    lib = _ffi.load()
    geom = Geometry(MatrixParams.create(4096, 64), 64)
    layout = _ffi.make_layout(geom.params, 64)
    enc = lambda bi, bj: torch.from_numpy(geom.qkey(np.array(list(bi)), np.array(list(bj))))
    if case == "no_match":  # A uses inner columns 0..3, B only inner rows 10..13
        ka, kb = enc(range(4), range(4)), enc(range(10, 14), range(4))
    else:
        ka, kb = enc(range(8), range(8)), enc(range(8), range(8))
        if case == "a_empty":
            ka = ka[:0]
        else:
            kb = kb[:0]
    ka, kb = ka.sort().values.to(ses.device), kb.sort().values.to(ses.device)
    ws_n = lib.qm_spgemm_workspace_bytes(ctypes.byref(layout), ka.numel(), kb.numel())
    ws = torch.empty(max(ws_n, 1), dtype=torch.uint8, device=ses.device)
    nc, nt = ctypes.c_int64(-1), ctypes.c_int64(-1)
    st = torch.cuda.current_stream().cuda_stream
    rc = lib.qm_spgemm_count(ctypes.byref(layout), ka.data_ptr(), ka.numel(), kb.data_ptr(), kb.numel(),
                             ws.data_ptr(), ws_n, ctypes.byref(nc), ctypes.byref(nt), st)
    assert rc == 0, _ffi.last_error()
    assert nc.value == 0 and nt.value == 0


def test_identity_multiply_is_bit_exact(ses):
    """test_ops.py:118-126."""
    da = helpers.random_sparse(256, 0.05, 13)
    for leaf, bs in ((64, 64), (64, 16), (32, 8)):
        a = helpers.build(ses, da, leaf, bs)
        eye = ses.identity(256, leaf_dim=leaf, block_size=bs)
        assert ses.canonical(ses.multiply(eye, a)) == ses.canonical(a)
        assert ses.canonical(ses.multiply(a, eye)) == ses.canonical(a)


def test_nil_and_explicit_zero_operands(ses):
    """test_ops.py:129-134, test_acceptance.py:381-430."""
    a = helpers.build(ses, helpers.random_sparse(64, 0.2, 14), 16, 8)
    z = ses.zeros(64, leaf_dim=16, block_size=8)
    ze = ses.zeros(64, leaf_dim=16, block_size=8, explicit=True)
    for x, y in ((a, z), (z, a), (a, ze), (ze, a), (z, z)):
        assert ses.multiply(x, y).root.is_nil


def test_exactly_zero_blocks_are_dropped(ses):
    """An exactly cancelling C block is not stored (_set_block np.any, block_sparse.py:37-41)."""
    bs, n = 64, 256
    rng = np.random.default_rng(3)
    x = rng.integers(-3, 4, (bs, bs)).astype(float)
    y = rng.integers(-3, 4, (bs, bs)).astype(float)
    da = np.zeros((n, n))
    db = np.zeros((n, n))
    da[0:bs, 0:bs] = x
    da[0:bs, bs:2 * bs] = x
    db[0:bs, 0:bs] = y
    db[bs:2 * bs, 0:bs] = -y          # C(0,0) = xy - xy = 0 exactly
    db[bs:2 * bs, 3 * bs:4 * bs] = y  # C(0,3) = xy survives
    c = ses.multiply(helpers.build(ses, da, bs, bs), helpers.build(ses, db, bs, bs))
    kc, bc, _ = _host(c)
    geom = Geometry(MatrixParams.create(n, bs), bs)
    assert list(kc) == list(geom.qkey(np.array([0]), np.array([3])))
    np.testing.assert_array_equal(bc[0], x @ y)


@pytest.mark.parametrize("leaf,bs", [(4, 2), (8, 4), (24, 8), (48, 12), (32, 16), (96, 32), (64, 64), (256, 128), (128, 64)])
def test_block_size_variants_vs_dense(ses, leaf, bs):
    n = 3 * leaf + 5  # padded, multi-level tree
    da, db = helpers.random_sparse(n, 0.05, leaf), helpers.random_sparse(n, 0.05, bs + 100)
    c = ses.multiply(helpers.build(ses, da, leaf, bs), helpers.build(ses, db, leaf, bs))
    assert helpers.rel(ses.to_dense(c), da @ db) <= TOL
    host = MatrixSession(device="cpu")
    ka, ba, _ = helpers.build(host, da, leaf, bs).root.blockset.to_host()
    kb, bb, _ = helpers.build(host, db, leaf, bs).root.blockset.to_host()
    # block set = symbolic product minus exactly-zero blocks (tiny sparse blocks do cancel)
    kc, bc, _ = O.multiply(O.Geom(n, leaf, bs), ka, ba, kb, bb)
    np.testing.assert_array_equal(c.root.blockset.keys.cpu().numpy(), kc)
    assert helpers.rel(c.root.blockset.blocks.cpu().numpy(), bc) <= TOL


def test_conformance_errors(ses):
    a = helpers.build(ses, helpers.random_sparse(64, 0.1, 1), 16, 8)
    b = helpers.build(ses, helpers.random_sparse(128, 0.1, 2), 16, 8)
    c = helpers.build(ses, helpers.random_sparse(64, 0.1, 3), 16, 4)
    with pytest.raises(DimensionMismatchError):
        ses.multiply(a, b)
    with pytest.raises(ConfigurationError):
        ses.multiply(a, c)
    with pytest.raises(ContractViolationError):
        ses.multiply(a)
    with pytest.raises(ContractViolationError):
        ses.multiply(a, variant="symmetric_square")  # needs a symmetric operand (ops.py:590-591)
    with pytest.raises(ConfigurationError):
        ses.multiply(a, a, variant="approximate", tau=-1.0)


def test_c2_131072_sampled_blocks_and_counts(ses):
    """Full-size C2 (BASELINE configs[1] largest): symbolic counts equal SURVEY.md 8(d) and
    sampled C block rows equal the oracle's on regenerated operand blocks."""
    cfg = G.CONFIGS["C2-131072"]
    geom, a, b = G.config_operands_device(cfg, ses.device)
    c = ses.multiply(ses.matrix_from_blockset(geom, a), ses.matrix_from_blockset(geom, b))
    st = ses.last_multiply
    assert (st.n_c, st.n_triples) == (67312, 589832)
    rows = np.r_[0, np.random.default_rng(0).choice(geom.nbg, 12, replace=False), geom.nbg - 1]
    kc, bc = helpers.oracle_rows(cfg, rows)
    keys_all = c.root.blockset.keys.cpu().numpy()
    np.testing.assert_array_equal(keys_all, helpers.structural_c_keys(geom, G.config_keys(cfg, 0),
                                                                      G.config_keys(cfg, 1)))
    got = helpers.lookup(keys_all, c.root.blockset.blocks, kc)
    assert helpers.rel(got, bc) <= TOL


@pytest.mark.parametrize("name,counts", [("C2-16384", (8176, 71944)), ("C2-32768", (16624, 145928)),
                                         ("C2-65536", (33520, 293896))])
def test_c2_sequence_block_set_and_sampled_values(ses, name, counts):
    """BASELINE configs[1] at every N of its sequence: the ENTIRE C block set equals the host
    structural set (scipy, SURVEY 8(d) counts) key for key, and sampled C block rows (first, last,
    random) equal the oracle's on regenerated operand blocks."""
    cfg = G.CONFIGS[name]
    geom, a, b = G.config_operands_device(cfg, ses.device)
    c = ses.multiply(ses.matrix_from_blockset(geom, a), ses.matrix_from_blockset(geom, b))
    assert (ses.last_multiply.n_c, ses.last_multiply.n_triples) == counts
    keys_all = c.root.blockset.keys.cpu().numpy()
    np.testing.assert_array_equal(keys_all, helpers.structural_c_keys(geom, G.config_keys(cfg, 0),
                                                                      G.config_keys(cfg, 1)))
    rows = np.r_[0, np.random.default_rng(7).choice(geom.nbg, 8, replace=False), geom.nbg - 1]
    kc, bc = helpers.oracle_rows(cfg, rows)
    assert helpers.rel(helpers.lookup(keys_all, c.root.blockset.blocks, kc), bc) <= TOL


@pytest.mark.parametrize("impl", ["tma", "cpasync"])
@pytest.mark.parametrize("bs", [16, 32, 64, 128])
def test_both_numeric_kernels_match_oracle(ses, monkeypatch, impl, bs):
    """The TMA/mbarrier kernel (default) and the cp.async kernel (QM_NUMERIC=cpasync) on the
    same product: exact block set, values within TOL of the oracle."""
    monkeypatch.setenv("QM_NUMERIC", impl)
    lib = _ffi.load()
    assert lib.qm_numeric_path(bs) == (2 if impl == "tma" else 1)
    cfg = G.BaselineConfig("k", "banded", 24 * bs, bs, half_bw=3 * bs)
    geom, (ka, ba), (kb, bb) = G.config_operands_host(cfg)
    kc, bc, _ = O.multiply(O.Geom(cfg.n, bs, bs), ka, ba, kb, bb)
    c = ses.multiply(ses.matrix_from_blocks(geom, ka, ba), ses.matrix_from_blocks(geom, kb, bb))
    k2, b2, s2 = _host(c)
    np.testing.assert_array_equal(k2, kc)
    assert helpers.rel(b2, bc) <= TOL
    np.testing.assert_allclose(s2, np.einsum("nij,nij->n", bc, bc), rtol=1e-12)


def test_distributed_path_single_rank_matches(ses):
    """The multi-GPU code path (structure gather, partition, request/serve exchange, remapped
    numeric) on one rank -- LocalComm and a real NCCL process group of size 1 -- equals the
    single-GPU product bit for bit."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2011_11762_b200 import distributed as D

    cfg = G.CONFIGS["C2-16384"]
    geom, a, b = G.config_operands_device(cfg, ses.device)
    layout = _ffi.make_layout(geom.params, geom.bs)
    ref = spgemm.multiply_blocks(layout, a, b)
    c, st = D.multiply(D.LocalComm(), layout, a, b)
    assert torch.equal(c.keys, ref.keys) and torch.equal(c.blocks, ref.blocks)
    assert st.bytes_received == 0 and st.t_range == (0, st.n_triples_global)
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=ses.device)
    try:
        c2, _ = D.multiply(D.Comm(), layout, a, b)
        assert torch.equal(c2.keys, ref.keys) and torch.equal(c2.blocks, ref.blocks)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("bs", [16, 32, 64, 128])
def test_numeric_kernel_is_deterministic_under_repetition(ses, bs):
    """Regression test for a stage-release race: the fixed summation order
    makes every repetition bitwise identical; 60 back-to-back launches must agree exactly."""
    cfg = G.BaselineConfig("rep", "banded", 256 * bs, bs, half_bw=8 * bs)
    geom, a, b = G.config_operands_device(cfg, ses.device)
    layout = _ffi.make_layout(geom.params, bs)
    plan = spgemm.symbolic(layout, a, b)
    first, _, _ = spgemm.numeric(layout, a, b, plan)
    bad = 0
    for _ in range(60):
        c, _, _ = spgemm.numeric(layout, a, b, plan)
        bad += int(not torch.equal(c.blocks, first.blocks))
    torch.cuda.synchronize()
    assert bad == 0


@pytest.mark.parametrize("bs,leaf", [(16, 128), (16, 256), (32, 64)])
def test_grouped_kernels_are_deterministic_under_repetition(ses, monkeypatch, bs, leaf):
    """The grouped kernels (bs 16 groups with the producer's inline merge, leaf 128: row pairs, leaf
    256: single rows; bs 32 quads with 2x2 blocks per leaf) release a stage once its fragments are
    in registers, like k_numeric_tma: 60 back-to-back launches of a banded product agree bitwise."""
    monkeypatch.setenv("QM_G16_GROUPS", "1")
    monkeypatch.setenv("QM_QUAD32", "1")
    n, hb = 256 * bs, 8 * bs
    d = np.arange(-hb, hb + 1)
    rows = np.repeat(np.arange(n), d.size)
    cols = rows + np.tile(d, n)
    keep = (cols >= 0) & (cols < n)
    rows, cols = rows[keep], cols[keep]
    vals = np.random.default_rng(bs + leaf).uniform(-1, 1, rows.size)
    a = ses.matrix_from_triplets(n, rows, cols, vals, leaf_dim=leaf, block_size=bs)
    x = a.root.blockset
    layout = _ffi.make_layout(a.geometry.params, bs)
    lib = _ffi.load()
    plan = spgemm.symbolic(layout, x, x)
    import ctypes

    want = "k_numeric_group16" if bs == 16 else "k_numeric_quad32"
    assert lib.qm_numeric_kernel(ctypes.byref(layout), plan.n_c, plan.n_triples, 0, 0).decode() == want
    first, _, _ = spgemm.numeric(layout, x, x, plan)
    bad = 0
    for _ in range(60):
        c, _, _ = spgemm.numeric(layout, x, x, plan)
        bad += int(not (torch.equal(c.blocks, first.blocks) and torch.equal(c.sumsq, first.sumsq)))
    torch.cuda.synchronize()
    assert bad == 0


@pytest.mark.parametrize("n,leaf,bs", [(13, 4, 2), (100, 16, 4), (37, 12, 4), (300, 64, 16), (1000, 64, 64), (777, 96, 32)])
def test_device_construction_is_bit_identical_to_host(ses, n, leaf, bs):
    """qm_build_* (GPU construction) == the host build == the reference's build:
    duplicate sums in input order (np.add.at), -0.0 -> +0.0, exactly-cancelling blocks dropped."""
    from paper_2011_11762_b200 import construct

    rng = np.random.default_rng(n + bs)
    m = max(4, n * n // 20)
    r = rng.integers(0, n, m)
    c = rng.integers(0, n, m)
    v = rng.standard_normal(m)
    # duplicates, a negative zero, and one block whose entries cancel exactly
    r = np.concatenate([r, r[:50], [0], [n - 1, n - 1]])
    c = np.concatenate([c, c[:50], [n - 1], [0, 0]])
    v = np.concatenate([v, 0.5 * v[:50], [-0.0], [3.0, -3.0]])
    geom = Geometry(MatrixParams.create(n, leaf), bs)
    kh, bh = construct.blocks_from_triplets(geom, r, c, v)
    dev = construct.blocks_from_triplets_device(geom, r, c, v, ses.device)
    np.testing.assert_array_equal(dev.keys.cpu().numpy(), kh)
    np.testing.assert_array_equal(dev.blocks.cpu().numpy(), bh)  # bitwise (incl. signs of zeros)
    assert not np.any(np.signbit(dev.blocks.cpu().numpy()) & (dev.blocks.cpu().numpy() == 0))


def test_device_construction_errors_and_empty(ses):
    from paper_2011_11762_b200 import OutOfRangeError, construct

    geom = Geometry(MatrixParams.create(64, 16), 8)
    with pytest.raises(OutOfRangeError):
        construct.blocks_from_triplets_device(geom, [0, 64], [0, 1], [1.0, 2.0], ses.device)
    assert construct.blocks_from_triplets_device(geom, [], [], [], ses.device).n == 0
    z = construct.blocks_from_triplets_device(geom, [1, 1], [2, 2], [1.5, -1.5], ses.device)
    assert z.n == 0  # the only block sums to exactly zero and is dropped
    m = ses.matrix_from_triplets(64, [1, 1], [2, 2], [1.5, -1.5], leaf_dim=16, block_size=8)
    assert m.root.is_nil


@pytest.mark.parametrize("ci", range(6))
def test_multiply_variants_match_reference(ses, ci):
    """symmetric / symmetric_square / rank_k (ops.py:582-608, virtual children ops.py:100-116):
    same C block set as the reference, values within TOL, result symmetry flag, dense value."""
    g = helpers.load("variants")
    tag = str(g["tags"][ci])
    _, n, leaf, bs, dens, seed = g["cases"][ci]
    n, leaf, bs, seed = int(n), int(leaf), int(bs), int(seed)
    m = helpers.random_sparse(n, float(dens), seed)
    sym = np.triu(m + m.T)
    rs, cs = np.nonzero(sym)
    a_sym = ses.matrix_from_triplets(n, rs, cs, sym[rs, cs], leaf_dim=leaf, block_size=bs, symmetric=True)
    a_gen = helpers.build(ses, m, leaf, bs)
    if tag == "symmetric":
        c = ses.multiply(a_sym, a_gen, variant="symmetric")
        want = (m + m.T) @ m
    elif tag == "symmetric_square":
        c = ses.multiply(a_sym, variant="symmetric_square")
        want = (m + m.T) @ (m + m.T)
    else:
        c = ses.multiply(a_gen, variant="rank_k")
        want = m @ m.T
    kc, bc, _ = _host(c)
    np.testing.assert_array_equal(kc, g[f"c{ci}_keys"])
    assert helpers.rel(bc, g[f"c{ci}_blocks"]) <= TOL
    assert c.symmetric == bool(g[f"c{ci}_symmetric"][0])
    assert helpers.rel(ses.to_dense(c), want) <= TOL
    assert helpers.rel(ses.to_dense(c), g[f"c{ci}_dense"]) <= TOL


@pytest.mark.parametrize("ci", range(16))
def test_approximate_multiply_matches_reference(ses, ci):
    """Norm-pruned multiply (ops.py:197-204, tau/8 per level): same surviving C blocks and the same
    prune log as the reference; the error is bounded by the log and the log by tau
    (test_acceptance.py:278-300)."""
    g = helpers.load("approximate")
    tag = str(g["tags"][ci])
    n, leaf, bs, scale, sa, sb, tau = g["cases"][ci]
    n, leaf, bs, sa, sb = int(n), int(leaf), int(bs), int(sa), int(sb)
    da, db = helpers.decay_sparse(n, sa, scale=scale), helpers.decay_sparse(n, sb, scale=scale)
    if tag == "approximate":
        c = ses.multiply(helpers.build(ses, da, leaf, bs), helpers.build(ses, db, leaf, bs),
                         variant="approximate", tau=tau)
        exact = da @ db
    elif tag == "symmetric_square":
        sym = np.triu(da + da.T)
        r, cc = np.nonzero(sym)
        a = ses.matrix_from_triplets(n, r, cc, sym[r, cc], leaf_dim=leaf, block_size=bs, symmetric=True)
        c = ses.multiply(a, variant="symmetric_square", tau=tau)
        exact = (da + da.T) @ (da + da.T)
    else:
        c = ses.multiply(helpers.build(ses, da, leaf, bs), variant="rank_k", tau=tau)
        exact = da @ da.T
    kc, bc, _ = _host(c)
    np.testing.assert_array_equal(kc, g[f"c{ci}_keys"])
    if kc.size:
        assert helpers.rel(bc, g[f"c{ci}_blocks"]) <= TOL
    log = np.sort(np.array(ses.last_engine.prune_log))
    ref_log = g[f"c{ci}_log"]
    assert log.size == ref_log.size
    np.testing.assert_allclose(log, ref_log, rtol=1e-12)
    skipped = float(np.sum(log))
    diff = np.linalg.norm(ses.to_dense(c) - exact)
    assert diff <= skipped + 1e-12 and skipped <= tau + 1e-12


@pytest.mark.parametrize("variant", ["approximate", "symmetric_square", "rank_k"])
@pytest.mark.parametrize("n,leaf,bs,rel", [(512, 64, 16, 1e-4), (1024, 64, 64, 1e-6), (1000, 128, 32, 1e-3),
                                           (2048, 256, 64, 1e-8)])
def test_ancestor_norm_filter_equals_the_level_recursion(ses, monkeypatch, variant, n, leaf, bs, rel):
    """The product's approximate filter (ancestor norms >= tau/8^l at every level, one pass over the
    triples) keeps exactly the triples of the level-by-level pruned recursion (qm_prune_all's
    surviving leaf pairs, filtered by qm_filter_triples), for general, symmetric and transposed
    (rank_k) operands -- same triples in the same order, so bitwise the same product."""
    from paper_2011_11762_b200 import approximate, variants

    da = helpers.decay_sparse(n, n + bs, scale=3.0)
    if variant == "symmetric_square":
        sym = np.triu(da + da.T)
        r, cc = np.nonzero(sym)
        m = ses.matrix_from_triplets(n, r, cc, sym[r, cc], leaf_dim=leaf, block_size=bs, symmetric=True)
    else:
        m = helpers.build(ses, da, leaf, bs)
    s = m.root.require()
    geom = m.geometry
    tau = rel * float(s.sumsq.sum().item())
    lay = _ffi.make_layout(geom.params, bs)
    a_sym = variant == "symmetric_square"
    ax = variants.expand_symmetric_view(geom, s) if a_sym and variants.virtual_ok(bs) else (
        variants.expand_symmetric(geom, s) if a_sym else s)
    if variant == "rank_k":
        bx = variants.transpose_view(geom, s) if variants.virtual_ok(bs) else variants.transpose(geom, s)
        b_src, b_sym = bx, False
    else:
        bx, b_src, b_sym = ax, s, a_sym
    upper = variant != "approximate"
    plan = spgemm.symbolic(lay, ax, bx, upper=upper)
    pruner = approximate.Pruner(geom, s, b_src, tau, a_sym=a_sym, b_sym=b_sym, upper=upper)
    fast = pruner.filter(plan, ax, bx)
    slow = approximate.filter_plan(geom, plan, ax, bx, pruner.result())
    assert fast.n_triples < plan.n_triples or rel < 1e-7  # something was pruned (most cases)
    assert (fast.n_c, fast.n_triples) == (slow.n_c, slow.n_triples)
    assert torch.equal(fast.c_keys, slow.c_keys) and torch.equal(fast.c_tptr, slow.c_tptr)
    assert torch.equal(fast.tri, slow.tri)


@pytest.mark.parametrize("n,leaf,bs", [(512, 64, 16), (1000, 32, 32), (4096, 256, 64)])
def test_node_norms_follow_the_reference_recursion(ses, n, leaf, bs):
    """qm_node_norms: every level's nodes are the non-nil quadtree nodes, and each norm is
    sqrt(fsum(child_norm^2)) of the level below, down to sqrt(fsum(block_norm^2)) per leaf
    (quadtree.py:138-140, block_sparse.py:91-92) -- here with math.fsum on the host."""
    import math

    from paper_2011_11762_b200 import approximate

    da = helpers.random_sparse(n, 0.01, 7)
    m = helpers.build(ses, da, leaf, bs)
    s = m.root.require()
    geom = m.geometry
    lay = _ffi.make_layout(geom.params, bs)
    tables = approximate._node_tables(geom, s, lay)
    keys = s.keys.cpu().numpy().astype(np.uint64)
    vals = np.sqrt(s.sumsq.cpu().numpy())
    codes = keys >> np.uint64(2 * geom.lbits)
    depth = geom.params.depth
    for lev in range(depth, -1, -1):
        uniq, start = np.unique(codes, return_index=True)
        bounds = list(start) + [codes.size]
        want = np.array([math.sqrt(math.fsum(float(v) * float(v) for v in vals[bounds[i]:bounds[i + 1]]))
                         for i in range(uniq.size)])
        c, nrm, cnt = tables[lev]
        assert cnt == uniq.size
        np.testing.assert_array_equal(c[:cnt].cpu().numpy().astype(np.uint64), uniq)
        np.testing.assert_allclose(nrm[:cnt].cpu().numpy(), want, rtol=2e-16, atol=0)
        codes, vals = uniq >> np.uint64(2), want


def test_approximate_with_zero_tau_is_the_exact_product(ses):
    """test_ops.py:190-197: tau = 0 gives the exact product bit for bit."""
    da = helpers.decay_sparse(64, 77, scale=2.0)
    a = helpers.build(ses, da, 16, 8)
    assert ses.canonical(ses.multiply(a, a, variant="approximate", tau=0.0)) == ses.canonical(ses.multiply(a, a))


@pytest.mark.parametrize("ci", range(15))
def test_add_scale_identity_truncate_match_reference(ses, ci):
    """SURVEY 8(f) #3 on the device: add / scale / add_scaled_identity are bit-identical to the
    reference (canonical bytes); truncation drops the same blocks and removes the same norm."""
    g = helpers.load("algebra")
    op = str(g["ops"][ci])
    n, leaf, bs, seed, p1, p2 = g["cases"][ci]
    n, leaf, bs, seed = int(n), int(leaf), int(bs), int(seed)
    da, db = helpers.random_sparse(n, 0.2, seed), helpers.random_sparse(n, 0.25, seed + 1000)
    a, b = helpers.build(ses, da, leaf, bs), helpers.build(ses, db, leaf, bs)
    removed = 0.0
    if op == "add":
        c = ses.add(a, b, p1, p2)
    elif op == "cancel":
        c = ses.add(a, a, p1, p2)
    elif op == "scale":
        c = ses.scale(a, p1)
    elif op == "asi":
        c = ses.add_scaled_identity(a, p1)
    elif op == "asi_nil":
        c = ses.add_scaled_identity(ses.zeros(n, leaf_dim=leaf, block_size=bs), p1)
    elif op == "truncate":
        c, removed = ses.truncate(a, p1 * np.linalg.norm(da))
    else:
        sym = np.triu(da + da.T)
        r, cc = np.nonzero(sym)
        s_ = ses.matrix_from_triplets(n, r, cc, sym[r, cc], leaf_dim=leaf, block_size=bs, symmetric=True)
        c, removed = ses.truncate(s_, p1 * np.linalg.norm(da + da.T))
    assert c.root.is_nil == bool(g[f"c{ci}_nil"][0])
    assert helpers.sha(ses.canonical(c)) == bytes(g[f"c{ci}_sha"])
    np.testing.assert_array_equal(ses.to_dense(c), g[f"c{ci}_dense"])
    assert abs(removed - g[f"c{ci}_removed"][0]) <= 1e-12 * max(1.0, removed)


def test_add_nil_fallbacks_share_the_survivor(ses):
    """test_ops.py:41-52: adding nil returns the surviving chunk itself when its coefficient is 1."""
    a = helpers.build(ses, helpers.random_sparse(16, 0.4, 3), 4, 2)
    z = ses.zeros(16, leaf_dim=4, block_size=2)
    assert ses.add(a, z).root == a.root
    np.testing.assert_allclose(ses.to_dense(ses.add(z, a, alpha=1.0, beta=2.0)), 2.0 * ses.to_dense(a), atol=1e-15)
    assert ses.add(z, z).root.is_nil
    assert ses.scale(a, 1.0).root == a.root and ses.scale(a, 0.0).root.is_nil
    assert ses.add_scaled_identity(a, 0.0).root == a.root


@pytest.mark.parametrize("n,leaf,bs", [(1, 1, 1), (2, 1, 1), (3, 2, 1), (5, 4, 1), (9, 4, 4), (64, 64, 64), (1000, 2, 1)])
def test_tiny_and_degenerate_shapes(ses, n, leaf, bs):
    """n = 1, bs = 1 (generic SIMT path), one-leaf trees, deep trees of tiny leaves."""
    da, db = helpers.random_sparse(n, 0.5, n), helpers.random_sparse(n, 0.5, n + 7)
    c = ses.multiply(helpers.build(ses, da, leaf, bs), helpers.build(ses, db, leaf, bs))
    assert helpers.rel(ses.to_dense(c), da @ db) <= TOL


def test_products_without_matching_inner_indices_are_nil(ses):
    """No k with A(i,k) and B(k,j): the symbolic phase finds no triple and C is nil."""
    n, bs = 256, 64
    da = np.zeros((n, n))
    db = np.zeros((n, n))
    da[:bs, :bs] = 1.0        # A only touches k in block 0
    db[bs:2 * bs, :bs] = 2.0  # B only has k in block 1
    c = ses.multiply(helpers.build(ses, da, bs, bs), helpers.build(ses, db, bs, bs))
    assert c.root.is_nil and ses.last_multiply.n_triples == 0


def test_very_sparse_with_empty_rows(ses):
    da, db = helpers.random_sparse(777, 0.0005, 1), helpers.random_sparse(777, 0.0005, 2)
    c = ses.multiply(helpers.build(ses, da, 16, 8), helpers.build(ses, db, 16, 8))
    assert helpers.rel(ses.to_dense(c), da @ db) <= TOL


@pytest.mark.parametrize("name,counts", [
    ("C5-64", (1063904, 17827216)), ("C5-128", (270064, 2365448)), ("C5-32", (4222912, 138330400))])
def test_c5_full_size_sampled_rows(ses, name, counts):
    """BASELINE configs[4] at full size (N = 2^20, up to 70 GB on the device): C block and triple
    counts equal SURVEY.md 8(d), sampled C block rows equal the oracle on regenerated blocks, and
    the fused norms match the blocks."""
    cfg = G.CONFIGS[name]
    geom, a, b = G.config_operands_device(cfg, ses.device)
    layout = _ffi.make_layout(geom.params, geom.bs)
    st = spgemm.MultiplyStats()
    c = spgemm.multiply_blocks(layout, a, b, stats=st)
    del a, b
    assert (st.n_c, st.n_triples) == counts
    rows = np.r_[0, np.random.default_rng(1).choice(geom.nbg, 6, replace=False), geom.nbg - 1]
    kc, bc = helpers.oracle_rows(cfg, rows)
    keys_all = c.keys.cpu().numpy()
    # the entire C block set, key for key (host structural product, scipy)
    np.testing.assert_array_equal(keys_all, helpers.structural_c_keys(geom, G.config_keys(cfg, 0),
                                                                      G.config_keys(cfg, 1)))
    got = helpers.lookup(keys_all, c.blocks, kc)
    assert helpers.rel(got, bc) <= TOL
    pos = torch.from_numpy(np.searchsorted(keys_all, kc)).to(c.sumsq.device)
    np.testing.assert_allclose(c.sumsq.index_select(0, pos).cpu().numpy(), np.einsum("nij,nij->n", bc, bc),
                               rtol=1e-12)
    del c
    torch.cuda.empty_cache()


def test_c4_full_size_sampled_rows(ses):
    """BASELINE configs[3] (decay, C = A*A) at full size: sampled C block rows vs the oracle."""
    cfg = G.CONFIGS["C4"]
    geom, (ka, ba), _ = G.config_operands_host(cfg)
    c = ses.multiply(*(2 * [ses.matrix_from_blocks(geom, ka, ba)]))
    # 735,716 block triples; 485,208 of them have meeting supports -- the rest multiply
    # to exact zeros and are skipped, so the 59,678 exact-zero C blocks are never created
    assert ses.last_multiply.n_triples == 485208 and ses.last_multiply.n_c == 60824
    assert ses.last_multiply.zero_blocks == 0
    # the entire nonzero C block set: pairs whose supports meet (host masks, numpy) -- A's entries
    # are positive (exp(-r^2/2)), so no C block cancels to zero otherwise
    rm, cm = helpers.support_masks_np(ba)
    np.testing.assert_array_equal(c.root.blockset.keys.cpu().numpy(), helpers.structural_c_keys(geom, ka, ka, cm, rm))
    assert helpers.structural_c_keys(geom, ka, ka).size == 120502  # structural
    ai, ak = geom.decode(ka)
    rows = np.r_[0, np.random.default_rng(2).choice(geom.nbg, 6, replace=False), geom.nbg - 1]
    sel = np.isin(ai, rows)
    need_k = np.unique(ak[sel])
    sel_b = np.isin(ai, need_k)  # B = A: rows k of A
    kc, bc, _ = O.multiply(O.Geom(cfg.n, cfg.bs, cfg.bs), ka[sel], ba[sel], ka[sel_b], ba[sel_b])
    got = helpers.lookup(c.root.blockset.keys.cpu().numpy(), c.root.blockset.blocks, kc)
    assert helpers.rel(got, bc) <= TOL


def test_c3_full_size_sampled_rows_and_block_set(ses):
    """BASELINE configs[2] (random, no locality) at full size: the exact C block set (host
    symbolic of the oracle) and sampled C block rows against the oracle."""
    cfg = G.CONFIGS["C3"]
    geom, (ka, ba), (kb, bb) = G.config_operands_host(cfg)
    c = ses.multiply(ses.matrix_from_blocks(geom, ka, ba), ses.matrix_from_blocks(geom, kb, bb))
    assert ses.last_multiply.n_triples == 65536  # 1024 block rows x 8 x 8
    kc_all, _, _, _, _ = O.symbolic(O.Geom(cfg.n, cfg.bs, cfg.bs), ka, kb)
    keys = c.root.blockset.keys.cpu().numpy()
    np.testing.assert_array_equal(keys, kc_all)  # no exact-zero products with random values
    ai, _ = geom.decode(ka)
    rows = np.r_[0, np.random.default_rng(3).choice(geom.nbg, 10, replace=False), geom.nbg - 1]
    sel = np.isin(ai, rows)
    kc, bc, _ = O.multiply(O.Geom(cfg.n, cfg.bs, cfg.bs), ka[sel], ba[sel], kb, bb)
    got = helpers.lookup(keys, c.root.blockset.blocks, kc)
    assert helpers.rel(got, bc) <= TOL


@pytest.mark.parametrize("bs", [16, 32, 64, 128])
def test_special_values_subnormal_nan_inf(ses, bs):
    """IEEE edge cases through the DMMA kernels: subnormal operands and products that underflow
    into the subnormal range are kept (no flush-to-zero, so the exact-zero drop of _set_block
    sees what numpy sees), NaN and Inf propagate inside their stored blocks only (block-sparse
    semantics: absent blocks are never touched). One triple per C block, so bitwise vs numpy."""
    n = 4 * bs
    rng = np.random.default_rng(bs)
    da, db = np.zeros((n, n)), np.zeros((n, n))
    da[:bs, :bs] = rng.uniform(-1, 1, (bs, bs)) * 1e-310
    db[:bs, :bs] = rng.uniform(-1, 1, (bs, bs))
    da[bs:2 * bs, bs:2 * bs] = 1e-160
    db[bs:2 * bs, bs:2 * bs] = 1e-160
    da[2 * bs, 2 * bs], db[2 * bs, 2 * bs] = np.nan, 1.0
    da[3 * bs, 3 * bs], db[3 * bs, 3 * bs] = np.inf, 2.0
    a = helpers.build(ses, da, bs, bs)
    b = helpers.build(ses, db, bs, bs)
    got = ses.to_dense(ses.multiply(a, b))
    want = np.zeros((n, n))
    with np.errstate(invalid="ignore", over="ignore", under="ignore"):
        for q in range(4):
            sl = slice(q * bs, (q + 1) * bs)
            want[sl, sl] = da[sl, sl] @ db[sl, sl]
    assert np.array_equal(got, want, equal_nan=True)
    assert np.count_nonzero(got[:bs, :bs]) == bs * bs  # subnormal results survive


@pytest.mark.parametrize("n,leaf,dens", [(1000, 128, 0.02), (700, 64, 0.05), (500, 48, 0.05), (1500, 256, 0.01),
                                         (2048, 128, 0.3)])
def test_bs16_grouped_kernel_vs_oracle(ses, monkeypatch, n, leaf, dens):
    """bs 16 with several blocks per leaf side runs k_numeric_group16 (the C blocks of a leaf row
    segment share their A blocks): exact C block set and values within TOL of the oracle, which
    sums each block's own triples k-ascending -- members missing a k must not see its products.
    Includes 3 and 16 blocks per leaf side (partial and split groups) and a nearly dense case.
    (QM_G16_GROUPS=1: groups whatever the k-list length; by default products with fewer than 4
    triples per C block -- these random patterns -- take the per-block kernel.)"""
    monkeypatch.setenv("QM_G16_GROUPS", "1")
    lib = _ffi.load()
    assert lib.qm_numeric_path(16) == 2
    da, db = helpers.random_sparse(n, dens, n + 1), helpers.random_sparse(n, dens, n + 2)
    c = ses.multiply(helpers.build(ses, da, leaf, 16), helpers.build(ses, db, leaf, 16))
    host = MatrixSession(device="cpu")
    ka, ba, _ = helpers.build(host, da, leaf, 16).root.blockset.to_host()
    kb, bb, _ = helpers.build(host, db, leaf, 16).root.blockset.to_host()
    kc, bc, _ = O.multiply(O.Geom(n, leaf, 16), ka, ba, kb, bb)
    np.testing.assert_array_equal(c.root.blockset.keys.cpu().numpy(), kc)
    assert helpers.rel(c.root.blockset.blocks.cpu().numpy(), bc) <= TOL
    np.testing.assert_allclose(c.root.blockset.sumsq.cpu().numpy(), np.einsum("nij,nij->n", bc, bc), rtol=1e-12)
    assert helpers.rel(ses.to_dense(c), da @ db) <= TOL


@pytest.mark.parametrize("n,leaf,dens", [(1000, 128, 0.02), (500, 48, 0.05), (2048, 128, 0.3), (600, 32, 0.1)])
def test_bs16_row_pair_groups_bitwise_equal_single_row(ses, monkeypatch, n, leaf, dens):
    """Leaf row pairs (R = 2 groups: each B block feeds both rows) change only which products share
    a pipeline stage; every C block still sums its own triples k-ascending with the same fragment
    order, so the result is bitwise the single-row grouping's (QM_GROUP_ROWS=1)."""
    monkeypatch.setenv("QM_G16_GROUPS", "1")
    da, db = helpers.random_sparse(n, dens, n + 5), helpers.random_sparse(n, dens, n + 6)
    a, b = helpers.build(ses, da, leaf, 16), helpers.build(ses, db, leaf, 16)
    c2 = ses.multiply(a, b).root.blockset
    monkeypatch.setenv("QM_GROUP_ROWS", "1")
    c1 = ses.multiply(a, b).root.blockset
    assert torch.equal(c1.keys, c2.keys)
    assert torch.equal(c1.blocks, c2.blocks) and torch.equal(c1.sumsq, c2.sumsq)
    assert helpers.rel(ses.to_dense(ses.multiply(a, b)), da @ db) <= TOL


@pytest.mark.parametrize("n,leaf,dens", [(1000, 128, 0.02), (500, 48, 0.05), (2048, 128, 0.3), (600, 32, 0.1),
                                         (4096, 256, 0.01)])
def test_bs16_inline_merge_bitwise_equal_merge_pass(ses, monkeypatch, n, leaf, dens):
    """The bs 16 grouped kernel's producer merges the members' k-ascending triple lists itself, one
    entry per pipeline stage (default); QM_G16_MERGE=kernel runs the separate merge pass
    (k_group_merge + entries array) instead. Same entries in the same order, so the C blocks, norms
    and exact-zero drops are bitwise identical, for row-pair (leaf <= 128) and single-row groups."""
    monkeypatch.setenv("QM_G16_GROUPS", "1")
    da, db = helpers.random_sparse(n, dens, n + 15), helpers.random_sparse(n, dens, n + 16)
    a, b = helpers.build(ses, da, leaf, 16), helpers.build(ses, db, leaf, 16)
    c2 = ses.multiply(a, b).root.blockset
    monkeypatch.setenv("QM_G16_MERGE", "kernel")
    c1 = ses.multiply(a, b).root.blockset
    assert torch.equal(c1.keys, c2.keys)
    assert torch.equal(c1.blocks, c2.blocks) and torch.equal(c1.sumsq, c2.sumsq)
    monkeypatch.delenv("QM_G16_MERGE")
    assert helpers.rel(ses.to_dense(ses.multiply(a, b)), da @ db) <= TOL


@pytest.mark.parametrize("bs,leaf", [(16, 128), (32, 32)])
def test_grouped_kernels_are_gated_on_k_list_length(ses, monkeypatch, bs, leaf):
    """Groups / quads of C blocks share a pipeline stage per k, which pays when members share k's
    (long k lists: banded); a random pattern with about one triple per C block takes the per-block
    kernel by default (2-3x faster there), and the forced grouped run gives bitwise the same product."""
    nb = 96
    n = nb * bs
    rng = np.random.default_rng(bs)
    pa, pb = np.zeros((nb, nb), bool), np.zeros((nb, nb), bool)
    pa[np.repeat(np.arange(nb), 3), rng.integers(0, nb, 3 * nb)] = True
    pb[np.repeat(np.arange(nb), 3), rng.integers(0, nb, 3 * nb)] = True
    da = np.kron(pa, np.ones((bs, bs))) * rng.uniform(-1, 1, (n, n))
    db = np.kron(pb, np.ones((bs, bs))) * rng.uniform(-1, 1, (n, n))
    a, b = helpers.build(ses, da, leaf, bs), helpers.build(ses, db, leaf, bs)
    lib = _ffi.load()
    ses.multiply(a, b)
    l0 = lib.qm_launch_count()
    c0 = ses.multiply(a, b).root.blockset
    n0 = lib.qm_launch_count() - l0
    st = ses.last_multiply
    assert st.n_triples < 4 * st.n_c_symbolic
    monkeypatch.setenv("QM_G16_GROUPS", "1")
    monkeypatch.setenv("QM_QUAD32", "1")
    l0 = lib.qm_launch_count()
    c1 = ses.multiply(a, b).root.blockset
    assert torch.equal(c0.keys, c1.keys)
    if bs == 32:  # per-block TMA kernel (+ k_combine_tiles) vs quads: same DMMA order, bitwise equal
        assert lib.qm_launch_count() - l0 == n0 - 1
        assert torch.equal(c0.blocks, c1.blocks) and torch.equal(c0.sumsq, c1.sumsq)
    else:         # cp.async per-block kernel vs groups: same k order, another fragment order
        assert helpers.rel(c0.blocks.cpu().numpy(), c1.blocks.cpu().numpy()) <= TOL
    assert helpers.rel(ses.to_dense(ses.multiply(a, b)), da @ db) <= TOL


@pytest.mark.parametrize("bs,leaf", [(16, 128), (16, 32), (16, 256), (32, 32), (32, 64)])
def test_grouped_kernels_on_adversarial_block_patterns(ses, monkeypatch, bs, leaf):
    """Block patterns chosen against the grouped kernels' producer (inline merge of the members'
    triple lists, chunk claims): single-member groups, members whose k ranges do not overlap, one
    member with a k list 20x longer than its neighbours', groups straddling chunk boundaries, a last
    chunk with one C block. Block set exact, values within TOL of the oracle; the bs 32 quad kernel
    is bitwise the per-block kernel's."""
    monkeypatch.setenv("QM_G16_GROUPS", "1")
    nb = 40  # blocks per side
    n = nb * bs
    rng = np.random.default_rng(bs * 1000 + leaf)
    pa, pb = np.zeros((nb, nb), bool), np.zeros((nb, nb), bool)
    pa[0, :] = True                      # one dense block row of A ...
    pb[:, 3] = True                      # ... against one dense block column of B: C(0,3) sums nb triples
    pa[5, 0:3] = True                    # members with disjoint k ranges in one group
    pa[4, 20:23] = True
    pb[0:3, 8] = pb[20:23, 9] = True
    pb[0:3, 9] = True
    for i in range(8, nb, 3):            # scattered single blocks: single-member groups
        pa[i, (7 * i) % nb] = True
        pb[(7 * i) % nb, (11 * i) % nb] = True
    pa[nb - 1, nb - 1] = pb[nb - 1, nb - 1] = True  # the last C block sits alone in its chunk
    da = np.kron(pa, np.ones((bs, bs))) * rng.uniform(-1, 1, (n, n))
    db = np.kron(pb, np.ones((bs, bs))) * rng.uniform(-1, 1, (n, n))
    if bs == 32:
        monkeypatch.setenv("QM_QUAD32", "1")
    a, b = helpers.build(ses, da, leaf, bs), helpers.build(ses, db, leaf, bs)
    c = ses.multiply(a, b).root.blockset
    host = MatrixSession(device="cpu")
    ka, ba, _ = helpers.build(host, da, leaf, bs).root.blockset.to_host()
    kb, bb, _ = helpers.build(host, db, leaf, bs).root.blockset.to_host()
    kc, bc, _ = O.multiply(O.Geom(n, leaf, bs), ka, ba, kb, bb)
    np.testing.assert_array_equal(c.keys.cpu().numpy(), kc)
    assert helpers.rel(c.blocks.cpu().numpy(), bc) <= TOL
    np.testing.assert_allclose(c.sumsq.cpu().numpy(), np.einsum("nij,nij->n", bc, bc), rtol=1e-12)
    monkeypatch.setenv("QM_QUAD32", "0")
    monkeypatch.setenv("QM_G16_MERGE", "kernel")
    c0 = ses.multiply(a, b).root.blockset
    assert torch.equal(c0.blocks, c.blocks) and torch.equal(c0.sumsq, c.sumsq)


@pytest.mark.parametrize("cfg", [G.BaselineConfig("q", "banded", 8192, 32, half_bw=256),
                                 G.BaselineConfig("q", "random", 16384, 32, per_row=8),
                                 G.BaselineConfig("q", "banded", 2048 + 32, 32, half_bw=96)])
def test_bs32_quad_kernel_bitwise_equal_per_block_kernel(ses, monkeypatch, cfg):
    """bs 32 products run quads of C blocks per work unit (k_numeric_quad32: the four blocks
    (2r..2r+1, 2c..2c+1) share one pipeline stage per k, merged by the producer warp); QM_QUAD32=0
    runs one C block per unit (k_numeric_tma). Every block sums its own triples in ascending k with
    the same DMMA order, and the norms are accumulated in the per-block kernel's order: blocks,
    norms and exact-zero drops are bitwise identical (odd block counts: quads with missing members)."""
    geom, a, b = G.config_operands_device(cfg, ses.device)
    ma, mb = ses.matrix_from_blockset(geom, a), ses.matrix_from_blockset(geom, b)
    lib = _ffi.load()
    ses.multiply(ma, mb)  # (builds the operands' cached row indexes: launch counts below are steady-state)
    monkeypatch.setenv("QM_QUAD32", "1")  # (1 = quads whatever the k-list length; default: >= 8 triples per C block)
    l0 = lib.qm_launch_count()
    c1 = ses.multiply(ma, mb).root.blockset
    n1 = lib.qm_launch_count() - l0
    monkeypatch.setenv("QM_QUAD32", "0")
    l0 = lib.qm_launch_count()
    c0 = ses.multiply(ma, mb).root.blockset
    assert lib.qm_launch_count() - l0 == n1 + 1  # the per-block path adds k_combine_tiles: two different kernels ran
    assert torch.equal(c0.keys, c1.keys)
    assert torch.equal(c0.blocks, c1.blocks) and torch.equal(c0.sumsq, c1.sumsq)


@pytest.mark.parametrize("n,leaf,dens", [(700, 64, 0.05), (1500, 32, 0.02), (2048, 64, 0.3)])
def test_bs32_quad_kernel_matches_oracle(ses, monkeypatch, n, leaf, dens):
    """Quads on ragged random patterns, leaf = one block (quad = Morton neighbours) and leaf = 2x2
    blocks (quad = the leaf): block set exact, values within TOL of the oracle, and bitwise the
    per-block kernel's; cancelling blocks are dropped alike."""
    da, db = helpers.random_sparse(n, dens, n + 21), helpers.random_sparse(n, dens, n + 22)
    a, b = helpers.build(ses, da, leaf, 32), helpers.build(ses, db, leaf, 32)
    monkeypatch.setenv("QM_QUAD32", "1")
    c = ses.multiply(a, b)
    host = MatrixSession(device="cpu")
    ka, ba, _ = helpers.build(host, da, leaf, 32).root.blockset.to_host()
    kb, bb, _ = helpers.build(host, db, leaf, 32).root.blockset.to_host()
    kc, bc, _ = O.multiply(O.Geom(n, leaf, 32), ka, ba, kb, bb)
    np.testing.assert_array_equal(c.root.blockset.keys.cpu().numpy(), kc)
    assert helpers.rel(c.root.blockset.blocks.cpu().numpy(), bc) <= TOL
    monkeypatch.setenv("QM_QUAD32", "0")
    c0 = ses.multiply(a, b).root.blockset
    assert torch.equal(c0.blocks, c.root.blockset.blocks) and torch.equal(c0.sumsq, c.root.blockset.sumsq)


@pytest.mark.parametrize("bs,n", [(64, 65536), (32, 16384), (128, 32768), (64, 8192)])
def test_claim_order_is_bitwise_neutral(ses, monkeypatch, bs, n):
    """Claim orders of the numeric kernel: QM_UNIT_ORDER=k (by the k of each C block's first triple:
    A(., k) and B(k, .) reused from L2 on random patterns, C3's shape) and lpt (longest k list first),
    at bs 32/64 and bs 128's 4-tile
    blocks. Only the processing order changes: the result is bitwise the key-order product's, and
    the C3-sized case also matches the oracle on sampled block rows."""
    cfg = G.BaselineConfig("t", "random", n, bs, per_row=8)
    geom, a, b = G.config_operands_device(cfg, ses.device)
    ma, mb = ses.matrix_from_blockset(geom, a), ses.matrix_from_blockset(geom, b)
    monkeypatch.setenv("QM_UNIT_ORDER", "key")
    c0 = ses.multiply(ma, mb).root.blockset
    for kind in ("k", "lpt"):
        monkeypatch.setenv("QM_UNIT_ORDER", kind)
        c1 = ses.multiply(ma, mb).root.blockset
        assert torch.equal(c0.keys, c1.keys)
        assert torch.equal(c0.blocks, c1.blocks) and torch.equal(c0.sumsq, c1.sumsq)
    if n == 65536:
        _, (ka, ba), (kb, bb) = G.config_operands_host(cfg)
        ai, _ = geom.decode(ka)
        rows = np.r_[0, np.random.default_rng(5).choice(geom.nbg, 6, replace=False), geom.nbg - 1]
        sel = np.isin(ai, rows)
        kc, bc, _ = O.multiply(O.Geom(cfg.n, cfg.bs, cfg.bs), ka[sel], ba[sel], kb, bb)
        got = helpers.lookup(c1.keys.cpu().numpy(), c1.blocks, kc)
        assert helpers.rel(got, bc) <= TOL


@pytest.mark.parametrize("bs", [16, 32, 64, 128])
def test_block_support_masks_match_numpy(ses, bs):
    """qm_block_masks: nonzero-row / nonzero-column bit masks per block (coarse bits above 64), full
    masks for blocks holding NaN or Inf."""
    rng = np.random.default_rng(bs)
    blocks = np.where(rng.random((40, bs, bs)) < 0.02, rng.standard_normal((40, bs, bs)), 0.0)
    blocks[3] = 0.0
    blocks[5, 7, 9] = np.nan
    blocks[6, 1, 2] = np.inf
    blocks[7, bs - 1, :] = 1.0
    bset = BlockSet.from_numpy(np.arange(40), blocks, None, ses.device)
    sumsq_stats = bset.sumsq.clone()
    m = bset.support_masks().cpu().numpy().view(np.uint64)
    want_r, want_c, want_f = helpers.support_masks_np(blocks, with_flags=True)
    np.testing.assert_array_equal(m[0], want_r)
    np.testing.assert_array_equal(m[1], want_c)
    np.testing.assert_array_equal(m[2], want_f)
    assert bset.masks_full == (False, False)
    # qm_block_meta: norms + masks in one pass; its sums of squares are bit-identical to
    # qm_block_stats' (the order every fused statistics pass reproduces)
    lib = _ffi.load()
    st = torch.empty(40, dtype=torch.float64, device=ses.device)
    ref = torch.empty(40, dtype=torch.float64, device=ses.device)
    mm = torch.empty((3, 40), dtype=torch.int64, device=ses.device)
    nf = torch.zeros(2, dtype=torch.int64, device=ses.device)
    _ffi.check(lib.qm_block_meta(bs, 40, _ffi.ptr(bset.blocks), _ffi.ptr(st), 0, 0, _ffi.ptr(mm), _ffi.ptr(nf), 0),
               "qm_block_meta")
    _ffi.check(lib.qm_block_stats(bs, 40, _ffi.ptr(bset.blocks), _ffi.ptr(ref), 0, 0), "qm_block_stats")
    torch.cuda.synchronize()
    assert torch.equal(mm, bset.masks)
    assert torch.equal(st.view(torch.int64), ref.view(torch.int64))
    assert nf.cpu().tolist() == [1, 1]
    dense = np.ones((4, bs, bs))
    full = BlockSet.from_numpy(np.arange(4), dense, None, ses.device).compute_meta()
    assert full.masks_full == (True, True)


@pytest.mark.parametrize("n,bw,leaf,bs", [(1024, 20, 64, 64), (768, 10, 32, 32), (512, 5, 128, 16),
                                          (1024, 40, 128, 128), (600, 6, 48, 16)])
def test_support_filter_skips_exact_zero_products(ses, monkeypatch, n, bw, leaf, bs):
    """Block pairs whose supports do not meet are skipped: the executed triples are exactly the
    oracle's triples with meeting masks, the C block set equals the oracle's after its exact-zero
    drop (no zero block is ever created, so nothing is compacted), and the values are bitwise those
    of the unfiltered product (QM_SUPPORT_FILTER=0: the skipped products only add +0)."""
    da = helpers.banded_support_decay(n, bw, n)
    db = helpers.banded_support_decay(n, bw, n + 1)
    a, b = helpers.build(ses, da, leaf, bs), helpers.build(ses, db, leaf, bs)
    c = ses.multiply(a, b)
    st = ses.last_multiply
    host = MatrixSession(device="cpu")
    ka, ba, _ = helpers.build(host, da, leaf, bs).root.blockset.to_host()
    kb, bb, _ = helpers.build(host, db, leaf, bs).root.blockset.to_host()
    g = O.Geom(n, leaf, bs)
    kc, bc, _ = O.multiply(g, ka, ba, kb, bb)
    np.testing.assert_array_equal(c.root.blockset.keys.cpu().numpy(), kc)
    assert helpers.rel(c.root.blockset.blocks.cpu().numpy(), bc) <= TOL
    _, _, ta, tb, _ = O.symbolic(g, ka, kb)
    _, cmask = helpers.support_masks_np(ba)
    rmask, _ = helpers.support_masks_np(bb)
    meet = (cmask[ta] & rmask[tb]) != 0
    assert st.n_triples == int(meet.sum()) and st.n_triples < ta.size  # some products were skipped
    assert st.zero_blocks == 0
    if bs >= 32:  # k panels (16 deep at bs 32/64, 32 deep at bs 128) of the surviving triples where the supports meet
        kp = 16 if bs <= 64 else 32
        npan, w = bs // kp, 64 * kp // max(bs, 64)
        ov = (cmask[ta] & rmask[tb])[meet]
        live = sum(((ov >> np.uint64(p * w)) & np.uint64((1 << w) - 1)) != 0 for p in range(npan))
        want_rows = kp * int(np.maximum(live, 1).sum()) if npan > 1 else bs * int(meet.sum())
        assert st.extra["k_rows"] == want_rows and st.flops == 2 * bs * bs * want_rows
    c2 = ses.multiply(c, c)  # chained product: C's masks computed on first use
    assert c.root.blockset.masks is not None
    assert helpers.rel(ses.to_dense(c2), ses.to_dense(c) @ ses.to_dense(c)) <= TOL
    monkeypatch.setenv("QM_SUPPORT_FILTER", "0")
    c0 = ses.multiply(a, b)
    assert ses.last_multiply.n_triples == ta.size and ses.last_multiply.zero_blocks > 0
    assert torch.equal(c0.root.blockset.keys, c.root.blockset.keys)
    assert torch.equal(c0.root.blockset.blocks, c.root.blockset.blocks)


def test_support_filter_keeps_nan_inf_products(ses):
    """0 * Inf is NaN: a block holding Inf/NaN is never filtered, so its NaN products reach C as in
    the reference (A's only nonzero column is 5, B's Inf sits in row 7: disjoint supports)."""
    bs = 16
    da, db = np.zeros((32, 32)), np.zeros((32, 32))
    da[0:bs, 5] = 1.0
    db[7, 0] = np.inf
    c = ses.to_dense(ses.multiply(helpers.build(ses, da, bs, bs), helpers.build(ses, db, bs, bs)))
    with np.errstate(invalid="ignore"):
        want = da[:bs, :bs] @ db[:bs, :bs]  # the only stored pair of blocks
    assert np.array_equal(c[:bs, :bs], want, equal_nan=True)
    assert np.isnan(c[0, 0]) and not c[bs:].any() and not c[:, bs:].any()


@pytest.mark.parametrize("bs", [32, 64, 128])
def test_panel_skip_keeps_nan_inf_products(ses, bs):
    """The masked TMA kernels (Tma32k16 / Tma64k16 / Tma128) skip k panels where A's columns and B's
    rows do not meet -- but never for a block holding NaN/Inf (masks' flags row): A(0,0)'s only
    nonzero column is 5 (first panel), B(0,0)'s row 5 is nonzero and its Inf sits in row bs-7, the
    last panel, where A(0,0) is zero: 0 * Inf = NaN must reach C like numpy's dgemm.
    Other blocks have partial supports, so the filters are active."""
    n = 2 * bs
    da, db = np.zeros((n, n)), np.zeros((n, n))
    da[:bs, 5] = 1.0
    da[:bs, bs + 3] = 2.0                   # A(0,1): column 3 only
    da[bs + 1, bs:] = 1.0                   # A(1,1): row 1 only
    db[5, :bs] = 1.0
    db[bs - 7, 0] = np.inf                  # B(0,0)
    db[bs + 3, 2] = 3.0                     # B(1,0): row 3 only
    db[bs + 9, bs + 4] = -1.0               # B(1,1): row 9 only (A(0,1)'s column 3 misses it)
    a, b = helpers.build(ses, da, bs, bs), helpers.build(ses, db, bs, bs)
    c = ses.multiply(a, b).root.blockset
    assert ses.last_multiply.n_triples == 4  # of 5 structural: A(0,1)*B(1,1) filtered, masks in use
    host = MatrixSession(device="cpu")
    ka, ba, _ = helpers.build(host, da, bs, bs).root.blockset.to_host()
    kb, bb, _ = helpers.build(host, db, bs, bs).root.blockset.to_host()
    with np.errstate(invalid="ignore"):
        kc, bc, _ = O.multiply(O.Geom(n, bs, bs), ka, ba, kb, bb)  # the reference's stored-block products
    np.testing.assert_array_equal(c.keys.cpu().numpy(), kc)
    got = c.blocks.cpu().numpy()
    assert np.array_equal(got, bc, equal_nan=True)
    assert np.isnan(got[0][:, 0]).all()  # C(0,0)'s column 0: A(0,0)[:, bs-7] = 0 times Inf


@pytest.mark.parametrize("bs,leaf", [(64, 64), (32, 64), (128, 128), (64, 128)])
def test_virtual_transposes_bitwise_equal_materialised(ses, monkeypatch, bs, leaf):
    """symmetric_square / rank_k / symmetric products read stored blocks transposed inside the
    numeric kernel (QM_NUMERIC_TRANSPOSED_REFS: transposed TMA box + fragment addressing) instead of
    materialising the transposes: the result is bitwise the materialised path's
    (QM_VIRTUAL_TRANSPOSE=0) -- the same products summed in the same order -- and matches dense."""
    n = 6 * leaf
    rng = np.random.default_rng(bs + leaf)
    d = np.where(rng.random((n, n)) < 0.15, rng.standard_normal((n, n)), 0.0)
    d = d + d.T
    a = helpers.build(ses, d, leaf, bs)
    up = ses.matrix_from_triplets(n, *helpers.triplets_of(np.triu(d)), leaf_dim=leaf,
                                  block_size=bs, symmetric=True)
    e = helpers.build(ses, rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.2), leaf, bs)
    cases = [("rank_k", lambda: ses.multiply(e, None, "rank_k")),
             ("symmetric_square", lambda: ses.multiply(up, None, "symmetric_square")),
             ("symmetric", lambda: ses.multiply(up, a, "symmetric"))]
    for name, run in cases:
        monkeypatch.setenv("QM_VIRTUAL_TRANSPOSE", "1")
        cv = run().root.blockset
        monkeypatch.setenv("QM_VIRTUAL_TRANSPOSE", "0")
        cm = run().root.blockset
        assert torch.equal(cv.keys, cm.keys), name
        assert torch.equal(cv.blocks, cm.blocks), name


@pytest.mark.parametrize("bs", [32, 64, 128])
def test_masked_and_transposed_kernels_deterministic_under_repetition(ses, bs):
    """The panel-skipping (masked) and transposed-reference instantiations of the numeric kernel use
    the same stage-release protocol as the dense one: 30 repetitions are bitwise identical."""
    n = 8 * bs
    m = helpers.banded_support_decay(n, max(2, bs // 3), bs)
    a = helpers.build(ses, m, bs, bs)
    s = ses.matrix_from_triplets(n, *helpers.triplets_of(np.triu(m + m.T)), leaf_dim=bs, block_size=bs,
                                 symmetric=True)
    for run in (lambda: ses.multiply(a, a), lambda: ses.multiply(s, None, "symmetric_square")):
        first = run().root.blockset.blocks.clone()
        bad = sum(int(not torch.equal(run().root.blockset.blocks, first)) for _ in range(30))
        assert bad == 0


def test_support_filter_multi_window_rows(ses):
    """The support filter in the windowed accumulator: rows spanning more than one 4096-column window
    (8192 block columns, bs 4), blocks with partial supports. Executed triples equal the oracle's
    triples with meeting masks, the C block set equals the oracle's after its exact-zero drop."""
    bs, nbg = 4, 8192
    n = bs * nbg
    rng = np.random.default_rng(11)
    rows, cols, vals = [], [], []
    for bi in range(0, nbg, 37):  # a few block rows reaching across the whole width
        for bj in rng.choice(nbg, 24, replace=False):
            r = bi * bs + rng.integers(0, bs, 2)
            c = bj * bs + rng.integers(0, bs, 2)
            rows += list(r)
            cols += list(c)
            vals += list(rng.uniform(0.5, 1.5, 2))
    for bk in range(nbg):  # B-side rows: one partial block per block row
        bj = rng.integers(0, nbg)
        rows.append(bk * bs + int(rng.integers(0, bs)))
        cols.append(int(bj) * bs + int(rng.integers(0, bs)))
        vals.append(1.0)
    rows, cols, vals = np.array(rows), np.array(cols), np.array(vals)
    a = ses.matrix_from_triplets(n, rows, cols, vals, leaf_dim=bs, block_size=bs)
    c = ses.multiply(a, a)
    st = ses.last_multiply
    host = MatrixSession(device="cpu")
    ka, ba, _ = host.matrix_from_triplets(n, rows, cols, vals, leaf_dim=bs, block_size=bs).root.blockset.to_host()
    g = O.Geom(n, bs, bs)
    kc, bc, _ = O.multiply(g, ka, ba, ka, ba)
    np.testing.assert_array_equal(c.root.blockset.keys.cpu().numpy(), kc)
    assert helpers.rel(c.root.blockset.blocks.cpu().numpy(), bc) <= TOL
    _, _, ta, tb, _ = O.symbolic(g, ka, ka)
    rm, cm = helpers.support_masks_np(ba)
    assert st.n_triples == int(((cm[ta] & rm[tb]) != 0).sum()) < ta.size


@pytest.mark.parametrize("name", ["C1", "C2-16384", "C3", "C4"])
def test_cached_row_index_symbolic_equals_keys_path(ses, monkeypatch, name):
    """The symbolic phase over the operands' cached row indexes (qm_row_index_build +
    qm_spgemm_count_ix / fill_ix) gives the same C keys, c_tptr and triples, in the same order, as
    the path that indexes the keys itself (QM_ROW_INDEX=0); masked (C4) and unmasked."""
    cfg = G.CONFIGS[name]
    geom, a, b = G.config_operands_device(cfg, ses.device)
    if cfg.same_operand:
        b = a
    lay = _ffi.make_layout(geom.params, geom.bs)
    monkeypatch.setenv("QM_ROW_INDEX", "1")
    p1 = spgemm.symbolic(lay, a, b)
    assert "_row_index" in a.__dict__
    monkeypatch.setenv("QM_ROW_INDEX", "0")
    p0 = spgemm.symbolic(lay, a, b)
    assert (p1.n_c, p1.n_triples) == (p0.n_c, p0.n_triples)
    assert torch.equal(p1.c_keys, p0.c_keys) and torch.equal(p1.c_tptr, p0.c_tptr) and torch.equal(p1.tri, p0.tri)


@pytest.mark.parametrize("cfg", [G.CONFIGS["C1"], G.BaselineConfig("t", "random", 2048, 64, per_row=8),
                                 G.BaselineConfig("t", "banded", 12288, 64, half_bw=512)])
def test_single_cta_sort_equals_device_sort(ses, monkeypatch, cfg):
    """Products with at most 8,192 C blocks order their keys in one launch of one CTA (k_sort_small)
    instead of the device-wide radix sort's ten launches (QM_SMALL_SORT=0): same C keys, c_tptr and
    triples, in the same order."""
    geom, a, b = G.config_operands_device(cfg, ses.device)
    lay = _ffi.make_layout(geom.params, geom.bs)
    monkeypatch.setenv("QM_RANK_ORDER", "0")  # (else 2,048 < nC <= 8,192 and QM_SMALL_SORT=0 take the rank ordering)
    monkeypatch.setenv("QM_SMALL_SORT", "1")
    p1 = spgemm.symbolic(lay, a, b)
    assert 0 < p1.n_c <= 8192
    monkeypatch.setenv("QM_SMALL_SORT", "0")
    p0 = spgemm.symbolic(lay, a, b)
    assert (p1.n_c, p1.n_triples) == (p0.n_c, p0.n_triples)
    assert torch.equal(p1.c_keys, p0.c_keys) and torch.equal(p1.c_tptr, p0.c_tptr) and torch.equal(p1.tri, p0.tri)


@pytest.mark.parametrize("name", ["C1", "C2-16384", "C3", "C4"])
def test_rank_ordering_equals_sorted_keys(ses, monkeypatch, name):
    """Products whose key space is small order their C keys by rank in a bitmap of the key space
    (k_rank_scan / k_rank_place: the keys are distinct, so the order is their rank) instead of a
    radix sort (QM_RANK_ORDER=0): same C keys, c_tptr and triples, in the same order; masked (C4)
    and unmasked, with the single-CTA sort switched off so that C1 takes the rank path too."""
    cfg = G.CONFIGS[name]
    geom, a, b = G.config_operands_device(cfg, ses.device)
    if cfg.same_operand:
        b = a
    lay = _ffi.make_layout(geom.params, geom.bs)
    monkeypatch.setenv("QM_SMALL_SORT", "0")
    lib = _ffi.load()
    spgemm.symbolic(lay, a, b)
    l0 = lib.qm_launch_count()
    p1 = spgemm.symbolic(lay, a, b)
    n1 = lib.qm_launch_count() - l0
    monkeypatch.setenv("QM_RANK_ORDER", "0")
    l0 = lib.qm_launch_count()
    p0 = spgemm.symbolic(lay, a, b)
    assert lib.qm_launch_count() - l0 != n1  # (the sort path launches other kernels)
    assert (p1.n_c, p1.n_triples) == (p0.n_c, p0.n_triples)
    assert torch.equal(p1.c_keys, p0.c_keys) and torch.equal(p1.c_tptr, p0.c_tptr) and torch.equal(p1.tri, p0.tri)


def test_cached_row_index_on_wide_rows(ses, monkeypatch):
    """Rows spanning several 4096-column windows of the count accumulator (as
    test_support_filter_multi_window_rows): the row-index path equals the keys path."""
    n, bs = 16384 * 2, 4
    rng = np.random.default_rng(3)
    rows = np.repeat(np.arange(0, n, 97), 40)
    cols = rng.integers(0, n, rows.size)
    vals = rng.uniform(-1, 1, rows.size)
    a = ses.matrix_from_triplets(n, rows, cols, vals, leaf_dim=64, block_size=bs)
    sa = a.root.blockset
    lay = _ffi.make_layout(a.geometry.params, bs)
    monkeypatch.setenv("QM_ROW_INDEX", "1")
    p1 = spgemm.symbolic(lay, sa, sa)
    monkeypatch.setenv("QM_ROW_INDEX", "0")
    p0 = spgemm.symbolic(lay, sa, sa)
    assert torch.equal(p1.c_keys, p0.c_keys) and torch.equal(p1.tri, p0.tri)
