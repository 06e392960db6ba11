"""Host-side logic of the drop-in API: keys, construction, inspection, validation, generators.

Where the reference package is importable (the build container) the host construction and the
inspection methods are compared with it byte for byte; elsewhere those tests skip.
"""

import dataclasses
import math
import sys
from pathlib import Path

import numpy as np
import pytest

import helpers
from paper_2011_11762_b200 import (
    ConfigurationError,
    ContractViolationError,
    DeviceUnavailableError,
    DimensionMismatchError,
    MatrixSession,
    MultiplyVariant,
    OutOfRangeError,
)
from paper_2011_11762_b200 import generators as G
from paper_2011_11762_b200.layout import Geometry, MatrixParams, qkey, qkey_decode

REF = Path("/root/reference/pkg/src")


@pytest.fixture(scope="module")
def quadmat():
    if not REF.exists():
        pytest.skip("reference package not present (only in the build container)")
    sys.path.insert(0, str(REF))
    import quadmat as q

    return q


@pytest.mark.parametrize("nbl", [1, 2, 3, 4, 5, 8])
def test_qkey_roundtrip_and_monotone(nbl):
    lbits = (nbl - 1).bit_length()
    rng = np.random.default_rng(nbl)
    bi = rng.integers(0, 64 * nbl, 2000)
    bj = rng.integers(0, 64 * nbl, 2000)
    k = qkey(bi, bj, nbl, lbits)
    r, c = qkey_decode(k, nbl, lbits)
    np.testing.assert_array_equal(r, bi)
    np.testing.assert_array_equal(c, bj)
    # monotone in the column for a fixed row (what the GPU row index relies on) and vice versa
    row = np.full(500, 17)
    cols = np.arange(500)
    assert np.all(np.diff(qkey(row, cols, nbl, lbits)) > 0)
    assert np.all(np.diff(qkey(cols, row, nbl, lbits)) > 0)


@pytest.mark.parametrize("n,leaf,bs", [(13, 4, 2), (24, 4, 2), (100, 16, 4), (37, 12, 4), (64, 8, 8), (300, 64, 16)])
def test_construction_and_inspection_match_reference(quadmat, n, leaf, bs):
    d = helpers.random_sparse(n, 0.2, n)
    r, c, v = helpers.triplets_of(d)
    # duplicates (summed in input order) and a negative zero
    r = np.concatenate([r, r[:7], [0]])
    c = np.concatenate([c, c[:7], [n - 1]])
    v = np.concatenate([v, -0.25 * v[:7], [-0.0]])
    ref = quadmat.MatrixSession()
    ses = MatrixSession(device="cpu")
    a = ref.matrix_from_triplets(n, r, c, v, leaf_dim=leaf, block_size=bs)
    b = ses.matrix_from_triplets(n, r, c, v, leaf_dim=leaf, block_size=bs)
    assert ref.canonical(a) == ses.canonical(b)
    np.testing.assert_array_equal(ref.to_dense(a), ses.to_dense(b))
    assert dataclasses.asdict(ref.tree_stats(a)) == dataclasses.asdict(ses.tree_stats(b))
    assert math.isclose(ref.norm(a), ses.norm(b), rel_tol=1e-15)
    rr = np.random.default_rng(1).integers(0, n, 64)
    cc = np.random.default_rng(2).integers(0, n, 64)
    np.testing.assert_array_equal(ref.get_elements(a, rr, cc), ses.get_elements(b, rr, cc))


def test_symmetric_identity_and_explicit_zeros_match_reference(quadmat):
    ref = quadmat.MatrixSession()
    ses = MatrixSession(device="cpu")
    d = helpers.random_sparse(40, 0.2, 5)
    s = np.triu(d + d.T)
    r, c, v = helpers.triplets_of(s)
    a = ref.matrix_from_triplets(40, r, c, v, leaf_dim=8, block_size=4, symmetric=True)
    b = ses.matrix_from_triplets(40, r, c, v, leaf_dim=8, block_size=4, symmetric=True)
    assert ref.canonical(a) == ses.canonical(b)
    np.testing.assert_array_equal(ref.to_dense(a), ses.to_dense(b))
    for n in (8, 13, 16):
        assert ref.canonical(ref.identity(n, c=2.0, leaf_dim=4, block_size=2)) == \
            ses.canonical(ses.identity(n, c=2.0, leaf_dim=4, block_size=2))
    ze_r = ref.zeros(16, leaf_dim=4, block_size=2, explicit=True)
    ze_s = ses.zeros(16, leaf_dim=4, block_size=2, explicit=True)
    assert ref.canonical(ze_r) == ses.canonical(ze_s)
    assert dataclasses.asdict(ref.tree_stats(ze_r)) == dataclasses.asdict(ses.tree_stats(ze_s))


def test_generate_matches_reference_generate(quadmat):
    from quadmat import generators as qg

    for case in (G.ExperimentCase("banded", 300, 7), G.ExperimentCase("growing_block", 256, 5, 40),
                 G.ExperimentCase("random_blocks", 512, 3, 30, 4, seed=2)):
        ref = quadmat.MatrixSession()
        ses = MatrixSession(device="cpu")
        qc = qg.ExperimentCase(case.family, case.n, case.b, case.s, case.n_blocks, case.seed)
        a = qg.generate(ref.store, qc, 64, "block_sparse", 16)
        b = G.generate(ses.store, case, 64, "block_sparse", 16)
        assert ref.canonical(a) == ses.canonical(b)
        assert qg.flop_count_exact(qc) == G.flop_count_exact(case)


def test_session_validation():
    with pytest.raises(ConfigurationError):
        MatrixSession(mode="bogus", device="cpu")
    with pytest.raises(ConfigurationError):
        MatrixSession(n_workers=0, device="cpu")
    ses = MatrixSession(device="cpu")
    with pytest.raises(ConfigurationError):
        ses.matrix_from_triplets(8, [0], [0], [1.0], leaf_dim=4, block_size=3)
    with pytest.raises(ConfigurationError):
        ses.matrix_from_triplets(8, [0], [0], [1.0], leaf_dim=4, block_size=2, leaf_kind="dense")
    with pytest.raises(OutOfRangeError):
        ses.matrix_from_triplets(8, [8], [0], [1.0], leaf_dim=4, block_size=2)
    with pytest.raises(ContractViolationError):
        ses.matrix_from_triplets(8, [3], [1], [1.0], leaf_dim=4, block_size=2, symmetric=True)
    with pytest.raises(ConfigurationError):
        MultiplyVariant("bogus")
    with pytest.raises(ConfigurationError):
        MultiplyVariant("approximate", -1.0)
    a = ses.matrix_from_triplets(16, [0, 5], [1, 9], [1.0, 2.0], leaf_dim=4, block_size=2)
    b = ses.matrix_from_triplets(32, [0], [1], [1.0], leaf_dim=4, block_size=2)
    with pytest.raises(DimensionMismatchError):
        ses.multiply(a, b)
    with pytest.raises(ContractViolationError):
        ses.multiply(a)


def test_no_cpu_fallback():
    ses = MatrixSession(device="cpu")
    a = ses.matrix_from_triplets(16, [0, 5], [1, 9], [1.0, 2.0], leaf_dim=4, block_size=2)
    with pytest.raises(DeviceUnavailableError):
        ses.multiply(a, a)


@pytest.mark.parametrize("n,bs,hb", [(4096, 64, 256), (1000, 32, 100), (777, 16, 0), (512, 128, 1024)])
def test_banded_block_keys_equal_brute_force(n, bs, hb):
    geom = Geometry(MatrixParams.create(n, bs), bs)
    keys = G.banded_block_keys(geom, hb)
    i = np.arange(n)
    mask = np.abs(i[:, None] - i[None, :]) <= hb
    nb = -(-n // bs)
    pad = np.zeros((nb * bs, nb * bs), bool)
    pad[:n, :n] = mask
    occ = pad.reshape(nb, bs, nb, bs).any(axis=(1, 3))
    bi, bj = np.nonzero(occ)
    np.testing.assert_array_equal(keys, np.sort(geom.qkey(bi, bj)))


def test_config_counts_match_survey():
    assert G.config_keys(G.CONFIGS["C1"], 0).size == 556
    assert G.config_keys(G.CONFIGS["C2-16384"], 1).size == 4280
    assert G.config_keys(G.CONFIGS["C2-131072"], 0).size == 34744
    assert G.config_keys(G.CONFIGS["C3"], 0).size == 8192
    assert G.config_keys(G.CONFIGS["C5-64"], 0).size == 540400
    assert G.config_keys(G.CONFIGS["C5-32"], 0).size == 2128864


def test_host_block_is_the_numpy_stream():
    blk = G.host_block(3, 1, 5, 7, 8, G.PATTERN_DENSE, 0, 1 << 20)
    np.testing.assert_array_equal(blk, np.random.default_rng([3, 1, 5, 7]).uniform(-1, 1, (8, 8)))


@pytest.mark.parametrize("n,b", [(50, 0), (64, 3), (100, 99)])
def test_flop_oracle_matches_brute_force(n, b):
    i = np.arange(n)
    p = (np.abs(i[:, None] - i[None, :]) <= b).astype(np.int64)
    assert G.flop_count_exact(G.ExperimentCase("banded", n, b)) == 2 * int(p.sum(0) @ p.sum(1))
