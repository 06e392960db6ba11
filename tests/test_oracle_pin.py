"""Pins the CPU oracle (oracle/spgemm_oracle.py) to outputs of the reference itself.

The fixtures in tests/golden/ were produced by running the reference's MatrixSession.multiply
(tests/golden/make_golden.py). The oracle uses the same numpy dgemm and the reference's summation
order, so it must reproduce the reference's canonical bytes bit for bit; for the BASELINE configs it
must reproduce the exact C block set and the per-block norms/checksums.
"""

import numpy as np
import pytest

import helpers
from oracle import spgemm_oracle as O
from paper_2011_11762_b200 import MatrixSession, bridge
from paper_2011_11762_b200 import generators as G
from paper_2011_11762_b200.layout import Geometry, MatrixParams


def _host_operands(n, leaf, bs, da_, db_, sa, sb):
    ses = MatrixSession(device="cpu")
    a = helpers.build(ses, helpers.random_sparse(n, da_, sa), leaf, bs)
    b = helpers.build(ses, helpers.random_sparse(n, db_, sb), leaf, bs)
    return ses, a, b


@pytest.mark.parametrize("ci", range(12))
def test_oracle_matches_reference_canonical_bytes(ci):
    g, cases = helpers.small_cases()
    n, leaf, bs, da_, db_, sa, sb = cases[ci]
    ses, a, b = _host_operands(n, leaf, bs, da_, db_, sa, sb)
    geom = Geometry(MatrixParams.create(n, leaf), bs)
    og = O.Geom(n, leaf, bs)
    ka, ba, _ = a.root.blockset.to_host()
    kb, bb, _ = b.root.blockset.to_host()
    kc, bc, _ = O.multiply(og, ka, ba, kb, bb)
    np.testing.assert_array_equal(kc, g[f"c{ci}_keys"])
    np.testing.assert_array_equal(bc, g[f"c{ci}_blocks"])  # bitwise
    assert helpers.sha(bridge.canonical_bytes(geom, kc, bc)) == bytes(g[f"c{ci}_sha"])


@pytest.mark.parametrize("name", ["C1", "C3s", "C4s", "C2-16384"])
def test_oracle_matches_reference_on_configs(name):
    g = helpers.load(name)
    cfg = G.CONFIGS.get(name) or {
        "C3s": G.BaselineConfig("C3s", "random", 8192, 64, per_row=8),
        "C4s": G.BaselineConfig("C4s", "decay", 4096, 64, same_operand=True),
    }[name]
    geom, (ka, ba), (kb, bb) = G.config_operands_host(cfg)
    og = O.Geom(cfg.n, cfg.bs, cfg.bs)
    kc, bc, _ = O.multiply(og, ka, ba, kb, bb)
    np.testing.assert_array_equal(kc, g["c_keys"])  # exact block set
    np.testing.assert_array_equal(np.array([np.linalg.norm(x) for x in bc]), g["c_norms"])
    np.testing.assert_array_equal(np.einsum("nij,ij->n", bc, helpers.check_weights(cfg.bs)), g["c_checks"])
    np.testing.assert_array_equal(bc[g["sample_idx"]], g["sample_blocks"])


def test_oracle_symbolic_counts_match_scipy():
    import scipy.sparse as sp

    cfg = G.CONFIGS["C2-16384"]
    geom = cfg.geometry
    ka, kb = G.config_keys(cfg, 0), G.config_keys(cfg, 1)
    og = O.Geom(cfg.n, cfg.bs, cfg.bs)
    kc, cptr, ta, tb, tk = O.symbolic(og, ka, kb)
    nb = geom.nbg
    ai, ak = geom.decode(ka)
    bk, bj = geom.decode(kb)
    A = sp.csr_matrix((np.ones(ai.size), (ai, ak)), shape=(nb, nb))
    B = sp.csr_matrix((np.ones(bk.size), (bk, bj)), shape=(nb, nb))
    C = (A @ B).tocoo()
    assert C.nnz == kc.size == 8176  # SURVEY.md 8(d) C2@16384
    assert int(C.sum()) == ta.size == 71944
    # triples are grouped by C block, k ascending inside a group
    grp = np.repeat(np.arange(kc.size), np.diff(cptr))
    assert np.all((np.diff(tk) > 0) | (np.diff(grp) != 0))


def test_band_ones_oracle_bit_exact_and_flop_identity():
    g = helpers.load("band_ones")
    geom = Geometry(MatrixParams.create(8192, 128), 32)
    keys = G.banded_block_keys(geom, 64)
    blocks = G.host_blocks(geom, keys, 0, 0, G.PATTERN_BAND_ONES, 64)
    kc, bc, _ = O.multiply(O.Geom(8192, 128, 32), keys, blocks, keys, blocks)
    assert helpers.sha(bridge.canonical_bytes(geom, kc, bc)) == bytes(g["sha"])
    # C is integer valued: sum(C) equals the pattern flop count / 2 exactly (generators.py:134-138)
    assert bc.sum() == g["c_sum"][0] == G.flop_count_exact(G.ExperimentCase("banded", 8192, 64)) // 2
