"""Property-based checks of the host-side invariants (hypothesis)."""

import numpy as np
import torch
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import spgemm_oracle as O
from paper_2011_11762_b200 import construct
from paper_2011_11762_b200 import distributed as D
from paper_2011_11762_b200.layout import Geometry, MatrixParams, qkey, qkey_decode


@settings(max_examples=60, deadline=None)
@given(nbl=st.integers(1, 9), depth=st.integers(0, 8), seed=st.integers(0, 2**31 - 1))
def test_qkey_is_a_bijection_ordered_like_the_quadtree(nbl, depth, seed):
    lbits = (nbl - 1).bit_length()
    nb = nbl << depth
    rng = np.random.default_rng(seed)
    bi, bj = rng.integers(0, nb, 300), rng.integers(0, nb, 300)
    k = qkey(bi, bj, nbl, lbits)
    r, c = qkey_decode(k, nbl, lbits)
    assert np.array_equal(r, bi) and np.array_equal(c, bj)
    # every quadtree node (leaf-grid prefix) is a contiguous key range: sorting by key never
    # interleaves two leaves
    order = np.argsort(k)
    leaf = (bi // nbl) * (1 << 20) + (bj // nbl)
    seen, prev = set(), None
    for x in leaf[order]:
        if x != prev:
            assert x not in seen
            seen.add(x)
            prev = x


@settings(max_examples=40, deadline=None)
@given(n=st.integers(1, 60), leaf=st.sampled_from([2, 4, 6, 8, 12]), seed=st.integers(0, 2**31 - 1))
def test_construction_sums_duplicates_in_input_order(n, leaf, seed):
    bs = [d for d in (1, 2, 3, 4, 6) if leaf % d == 0][-1]
    geom = Geometry(MatrixParams.create(n, leaf), bs)
    rng = np.random.default_rng(seed)
    m = int(rng.integers(1, 3 * n + 2))
    r, c = rng.integers(0, n, m), rng.integers(0, n, m)
    v = rng.standard_normal(m)
    keys, blocks = construct.blocks_from_triplets(geom, r, c, v)
    dense = np.zeros((n, n))
    for x in range(m):  # sequential, input order: np.add.at's definition
        dense[r[x], c[x]] += v[x]
    from paper_2011_11762_b200 import bridge

    assert np.array_equal(bridge.to_dense(geom, keys, blocks), dense)
    assert np.all(np.diff(keys) > 0)
    assert all(np.any(b != 0) for b in blocks)


@settings(max_examples=60, deadline=None)
@given(counts=st.lists(st.integers(1, 40), min_size=1, max_size=300), world=st.integers(1, 8))
def test_partition_is_monotone_covering_and_balanced(counts, world):
    tptr = torch.tensor(np.r_[0, np.cumsum(counts)])
    cb, tb = D.partition(tptr, world)
    assert cb[0] == 0 and cb[-1] == len(counts) and all(x <= y for x, y in zip(cb, cb[1:]))
    assert tb[0] == 0 and tb[-1] == sum(counts)
    share = np.diff(tb)
    assert share.max() - sum(counts) / world <= max(counts)


@settings(max_examples=30, deadline=None)
@given(nb=st.integers(1, 40), da=st.floats(0.05, 0.6), db=st.floats(0.05, 0.6), seed=st.integers(0, 2**31 - 1))
def test_oracle_symbolic_equals_boolean_product(nb, da, db, seed):
    rng = np.random.default_rng(seed)
    pa, pb = rng.random((nb, nb)) < da, rng.random((nb, nb)) < db
    g = O.Geom(nb * 2, 2, 2)
    ka = g.key(*np.nonzero(pa))
    kb = g.key(*np.nonzero(pb))
    kc, cptr, _, _, _ = O.symbolic(g, np.sort(ka), np.sort(kb))
    prod = pa.astype(int) @ pb.astype(int)
    i, j = np.nonzero(prod)
    assert np.array_equal(np.sort(g.key(i, j)), kc)
    assert cptr[-1] == prod.sum()
