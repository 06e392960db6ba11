"""The drop-in boundary exercised by the reference's OWN code (SURVEY.md 8(b) seams 1-3).

* seam (2), the bench seam: the reference harness ``quadmat/bench.py`` (run_bench, bench.py:93-141:
  session, ``generate``, ``multiply_spec``, ``run_spec``, ``last_stats``) is executed from its
  installed source with only its imports redirected to this package -- nothing else changed;
* seam (3), the task plugin: the reference engine with "multiply" re-registered to run
  ``reference_plugin.gpu_compute`` (libqmb200) reproduces the reference's own products.

The reference package comes from baseline/_ref (the offline install that travels with the repo
snapshot) or the build container's reference tree; these tests skip when neither is present.
Test infrastructure only: the product path never imports the reference.
"""

import re
import sys
import types

import numpy as np
import pytest

import helpers

REF = helpers.reference_src()
needs_ref = pytest.mark.skipif(REF is None, reason="reference package (baseline/_ref) not present")


def test_ops_module_is_the_reference_ops_surface():
    """`from .ops import MultiplyVariant, multiply_spec` (reference bench.py:24) resolves here."""
    from paper_2011_11762_b200 import ops
    from paper_2011_11762_b200.errors import ConfigurationError

    assert ops.MultiplyVariant.regular().tag == "regular"
    assert ops.MultiplyVariant.approximate(0.5).tau == 0.5
    assert ops._VARIANTS == ("regular", "symmetric", "symmetric_square", "rank_k", "approximate")
    with pytest.raises(ConfigurationError):
        ops.MultiplyVariant("nope")
    with pytest.raises(ConfigurationError):
        ops.TruncationSpec(-1.0)


def _reference_bench_module():
    """The reference's bench.py, its relative imports pointed at paper_2011_11762_b200."""
    src = (REF / "quadmat" / "bench.py").read_text()
    src2, n = re.subn(r"^from \.(\w+) import", r"from paper_2011_11762_b200.\1 import", src, flags=re.M)
    assert n >= 4 and "from ." not in src2  # errors, generators, ops, session
    mod = types.ModuleType("quadmat_bench_on_b200")
    sys.modules[mod.__name__] = mod  # dataclasses resolve their module through sys.modules
    exec(compile(src2, "quadmat/bench.py (imports -> paper_2011_11762_b200)", "exec"), mod.__dict__)
    return mod


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("family,n,b,leaf,bs", [("banded", 4096, 64, 256, 64), ("banded", 2048, 200, 128, 16),
                                                ("growing_block", 1024, 32, 128, 32)])
def test_reference_run_bench_runs_on_the_dropin(family, n, b, leaf, bs):
    """run_bench (reference bench.py:93-141) with only the imports changed: every repeat times a
    B200 product of the generated case; the oracle flop count and per-worker stats are populated."""
    bench = _reference_bench_module()
    from paper_2011_11762_b200 import generators as G

    kw = {"s": 64} if family != "banded" else {}
    case = bench.ExperimentCase(family, n, b, **kw)
    cfg = bench.BenchConfig(case=case, n_workers=1, leaf_dim=leaf, block_size=bs, mode="shared_memory",
                            repeats=2)
    recs = bench.run_bench(cfg)
    assert len(recs) == 2 and all(r.wall_seconds > 0 for r in recs)
    assert all(r.flops == G.flop_count_exact(case) for r in recs)
    assert all(r.tasks_min > 0 and r.bytes_min == 0 for r in recs)  # one GPU: block triples, no halo


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("family,n,b,leaf,bs", [("banded", 2048, 64, 256, 64), ("banded", 1000, 30, 128, 16),
                                                ("growing_block", 1024, 32, 128, 32)])
def test_generated_products_equal_the_reference_bitwise(family, n, b, leaf, bs):
    """The same run_bench flow on both packages (generate -> multiply_spec -> run_spec): the
    generators emit 1.0-valued patterns, so the products are integer-valued and the C trees'
    canonical bytes must be identical (quadtree.py:293-318)."""
    quadmat = helpers.import_reference()
    from quadmat import generators as RG
    from quadmat import ops as rops

    from paper_2011_11762_b200 import MatrixSession
    from paper_2011_11762_b200 import generators as G
    from paper_2011_11762_b200 import ops

    kw = {"s": 64} if family != "banded" else {}
    rses = quadmat.MatrixSession(n_workers=1, mode="threaded")
    rm = RG.generate(rses.store, RG.ExperimentCase(family, n, b, **kw), leaf, "block_sparse", bs, rses.owner_policy)
    rspec, _ = rops.multiply_spec(rm, rm, rops.MultiplyVariant.regular())
    rc = rses.run_spec(rspec)
    ses = MatrixSession(n_workers=1, mode="threaded")
    m = G.generate(ses.store, G.ExperimentCase(family, n, b, **kw), leaf, "block_sparse", bs, ses.owner_policy)
    spec, _ = ops.multiply_spec(m, m, ops.MultiplyVariant.regular())
    c = ses.run_spec(spec)
    want = rses.canonical(quadmat.Matrix(rc, rm.params, rm.leaf_kind, rm.block_size, False))
    got = ses.canonical(type(m)(c, m.params, m.leaf_kind, m.block_size, False))
    assert got == want
    assert ses.last_stats[0].tasks_executed > 0


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("mode,workers", [("simulate", 1), ("simulate", 3), ("threaded", 2)])
@pytest.mark.parametrize("n,leaf,bs", [(256, 64, 64), (512, 128, 32), (300, 64, 16), (1024, 256, 128)])
def test_plugged_reference_engine_runs_the_gpu_kernels(mode, workers, n, leaf, bs):
    """reference_plugin.install(session) with its default compute (libqmb200 on the B200): the
    reference engine's level-0 regular products come from the GPU. Integer-valued operands give
    exact products, so the canonical bytes equal the unplugged reference's; random values agree
    within the north-star tolerance (relative Frobenius 1e-12)."""
    quadmat = helpers.import_reference()
    from paper_2011_11762_b200 import _ffi, reference_plugin

    lib = _ffi.load()
    rng = np.random.default_rng(n + bs)
    ints = np.where(rng.random((n, n)) < 0.1, rng.integers(-3, 4, (n, n)), 0).astype(float)
    flts = np.where(rng.random((n, n)) < 0.1, rng.standard_normal((n, n)), 0.0)
    for d, exact in ((ints, True), (flts, False)):
        plain = quadmat.MatrixSession(n_workers=workers, mode=mode)
        plugged = reference_plugin.install(quadmat.MatrixSession(n_workers=workers, mode=mode))
        outs = []
        for s in (plain, plugged):
            a = s.matrix_from_triplets(n, *np.nonzero(d), d[np.nonzero(d)], leaf_dim=leaf, block_size=bs)
            l0 = lib.qm_launch_count()
            c = s.multiply(a, a)
            outs.append((s, c, lib.qm_launch_count() - l0))
        assert outs[0][2] == 0 and outs[1][2] > 0  # only the plugged engine launched libqmb200 kernels
        if exact:
            assert outs[0][0].canonical(outs[0][1]) == outs[1][0].canonical(outs[1][1])
        else:
            assert helpers.rel(outs[1][0].to_dense(outs[1][1]), outs[0][0].to_dense(outs[0][1])) <= 1e-12
