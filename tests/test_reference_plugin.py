"""The task-plugin seam against the real reference engine (the reference package installed under
baseline/_ref, or the build container's reference tree). The compute function is the oracle here,
so the plugged engine must produce the reference's own canonical bytes bit for bit -- proving that
reading the operand trees through ctx.fetch and writing the product back through ctx.put is exact,
for every engine mode and worker count. tests/test_reference_dropin.py runs the same body with
gpu_compute (libqmb200) on a B200."""

import numpy as np
import pytest

import helpers
from oracle import spgemm_oracle as O

pytestmark = pytest.mark.skipif(helpers.reference_src() is None, reason="reference package not present")


def _oracle_compute(geom, ka, ba, kb, bb):
    kc, bc, _ = O.multiply(O.Geom(geom.params.n_logical, geom.params.leaf_dim, geom.bs), ka, ba, kb, bb)
    return kc, bc


@pytest.mark.parametrize("mode,workers", [("simulate", 1), ("simulate", 3), ("threaded", 2)])
@pytest.mark.parametrize("n,leaf,bs", [(24, 4, 2), (100, 16, 8), (37, 12, 4), (256, 64, 64)])
def test_plugged_engine_reproduces_reference_products(mode, workers, n, leaf, bs):
    quadmat = helpers.import_reference()

    from paper_2011_11762_b200 import reference_plugin

    da, db = helpers.random_sparse(n, 0.2, n), helpers.random_sparse(n, 0.25, n + 1)
    plain = quadmat.MatrixSession(n_workers=workers, mode=mode)
    plugged = reference_plugin.install(quadmat.MatrixSession(n_workers=workers, mode=mode), _oracle_compute)
    outs = []
    for ses in (plain, plugged):
        a = ses.matrix_from_triplets(n, *np.nonzero(da), da[np.nonzero(da)], leaf_dim=leaf, block_size=bs)
        b = ses.matrix_from_triplets(n, *np.nonzero(db), db[np.nonzero(db)], leaf_dim=leaf, block_size=bs)
        outs.append(ses.canonical(ses.multiply(a, b)))
    assert outs[0] == outs[1]
    # variants and non-block-sparse leaves still go through the reference's own body
    a = plugged.matrix_from_triplets(n, *np.nonzero(da), da[np.nonzero(da)], leaf_dim=leaf, block_size=bs)
    np.testing.assert_allclose(plugged.to_dense(plugged.multiply(a, variant="rank_k")), np.triu(da @ da.T) +
                               np.triu(da @ da.T, 1).T, atol=1e-12)
