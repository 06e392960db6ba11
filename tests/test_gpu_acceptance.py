"""Randomised operation suite against dense numpy, in the shape of the reference's release gate
(pkg/tests/test_acceptance.py:104-220: log-uniform sizes up to 512, leaf/block sizes that force a
multi-level tree, densities 0.02-0.25; TOL_EXACT 1e-15 for add/build, TOL_FLOAT 1e-12 for
everything that multiplies)."""

import numpy as np
import pytest

import helpers

pytestmark = pytest.mark.gpu
N_INSTANCES = 60
TOL_EXACT = 1e-15
TOL_FLOAT = 1e-12


def _shape(rng):
    n = max(8, min(512, int(round(2 ** float(rng.uniform(3.0, 9.0))))))
    padded = 1 << (n - 1).bit_length()
    leaf_dim = max(4, padded // 4)
    return n, leaf_dim, max(2, leaf_dim // 4)


def _rel(got, want):
    return np.linalg.norm(got - want) / max(1.0, np.linalg.norm(want))


@pytest.fixture(scope="module")
def ses():
    return helpers.gpu_session()


@pytest.mark.parametrize("op", ["multiply", "symmetric_square", "rank_k", "add", "build", "truncate"])
def test_randomised_operation_suite(ses, op):
    rng = np.random.default_rng([20_000, ["multiply", "symmetric_square", "rank_k", "add", "build", "truncate"].index(op)])
    for i in range(N_INSTANCES):
        n, leaf, bs = _shape(rng)
        density = float(rng.uniform(0.02, 0.25))
        kw = dict(leaf_dim=leaf, block_size=bs)
        da = helpers.random_sparse(n, density, int(rng.integers(1 << 30)))
        db = helpers.random_sparse(n, density, int(rng.integers(1 << 30)))
        try:
            if op == "multiply":
                c = ses.multiply(helpers.build(ses, da, **kw), helpers.build(ses, db, **kw))
                assert _rel(ses.to_dense(c), da @ db) <= TOL_FLOAT
            elif op == "symmetric_square":
                s = (da + da.T) / 2
                r, cc = np.nonzero(np.triu(s))
                a = ses.matrix_from_triplets(n, r, cc, s[r, cc], symmetric=True, **kw)
                c = ses.multiply(a, variant="symmetric_square")
                assert _rel(ses.to_dense(c), s @ s) <= TOL_FLOAT
            elif op == "rank_k":
                c = ses.multiply(helpers.build(ses, da, **kw), variant="rank_k")
                assert _rel(ses.to_dense(c), da @ da.T) <= TOL_FLOAT
            elif op == "add":
                alpha, beta = float(rng.uniform(-2, 2)), float(rng.uniform(-2, 2))
                c = ses.add(helpers.build(ses, da, **kw), helpers.build(ses, db, **kw), alpha, beta)
                assert _rel(ses.to_dense(c), alpha * da + beta * db) <= TOL_EXACT
            elif op == "build":
                a = helpers.build(ses, da, **kw)
                assert _rel(ses.to_dense(a), da) <= TOL_EXACT
                rows, cols = rng.integers(0, n, 3 * n), rng.integers(0, n, 3 * n)
                got = ses.get_elements(a, rows, cols)
                assert np.max(np.abs(got - da[rows, cols])) <= TOL_EXACT * max(1.0, np.abs(da).max())
            else:
                tau = float(rng.uniform(0.0, 1.1)) * np.linalg.norm(da)
                out, removed = ses.truncate(helpers.build(ses, da, **kw), tau)
                diff = np.linalg.norm(ses.to_dense(out) - da)
                assert diff <= tau or diff <= removed * (1 + 1e-12)
                assert abs(diff - removed) <= 1e-12 * max(1.0, removed)
        except AssertionError as exc:
            raise AssertionError(f"{op} instance {i} (n={n}, leaf={leaf}, bs={bs}): {exc}") from exc
