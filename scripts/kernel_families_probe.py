"""Small products through every kernel family, each checked against dense numpy (compute-sanitizer
is not available on the GPU pool, so this is the bounds/values smoke of the new paths):
dense-support bs 16/32/64/128, masked (partial supports) bs 32/64/128 with panel skipping,
virtual transposes (symmetric_square, rank_k), approximate, bs 16 row-pair groups, generic bs."""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import torch

import helpers
from paper_2011_11762_b200 import MatrixSession

ses = MatrixSession(device="cuda:0")
rng = np.random.default_rng(0)
for leaf, bs, n in ((64, 64, 512), (64, 32, 384), (128, 128, 512), (128, 16, 512), (48, 12, 240)):
    d = helpers.random_sparse(n, 0.05, bs)
    a = helpers.build(ses, d, leaf, bs)
    c = ses.multiply(a, a)
    assert helpers.rel(ses.to_dense(c), d @ d) <= 1e-12
    m = helpers.banded_support_decay(n, max(2, bs // 3), bs)
    am = helpers.build(ses, m, leaf, bs)
    cm = ses.multiply(am, am)
    assert helpers.rel(ses.to_dense(cm), m @ m) <= 1e-12
    s = np.triu(d + d.T)
    sym = ses.matrix_from_triplets(n, *helpers.triplets_of(s), leaf_dim=leaf, block_size=bs, symmetric=True)
    full = s + np.triu(s, 1).T
    cs = ses.multiply(sym, None, "symmetric_square")  # symmetric result: to_dense mirrors the upper leaves
    assert helpers.rel(ses.to_dense(cs), full @ full) <= 1e-12
    cr = ses.multiply(a, None, "rank_k")
    assert helpers.rel(ses.to_dense(cr), d @ d.T) <= 1e-12
    ca = ses.multiply(sym, None, "symmetric_square", tau=1e-3)
    torch.cuda.synchronize()
    print(f"leaf {leaf} bs {bs}: ok", flush=True)
print("kernel families probe done")
