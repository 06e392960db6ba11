"""Shared test helpers: seeded inputs, golden fixture loading, GPU session factory."""

from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
CHECK_SEED = 12345


def random_sparse(n: int, density: float, seed: int) -> np.ndarray:
    """Random sparse support with standard-normal values (the reference test oracle's recipe,
    pkg/tests/oracles.py:112-119)."""
    rng = np.random.default_rng(seed)
    k = max(1, int(n * n * density))
    idx = rng.choice(n * n, size=k, replace=False)
    out = np.zeros((n, n))
    out[np.divmod(idx, n)] = rng.standard_normal(k)
    return out


def triplets_of(dense: np.ndarray):
    rows, cols = np.nonzero(dense)
    return rows, cols, dense[rows, cols]


def build(session, dense, leaf_dim, block_size, **kw):
    n = dense.shape[0]
    r, c, v = triplets_of(dense)
    return session.matrix_from_triplets(n, r, c, v, leaf_dim=leaf_dim, block_size=block_size, **kw)


def load(name: str):
    return np.load(GOLDEN / f"{name}.npz")


def sha(b: bytes) -> bytes:
    return hashlib.sha256(b).digest()


def check_weights(bs: int) -> np.ndarray:
    return np.random.default_rng(CHECK_SEED).uniform(-1.0, 1.0, (bs, bs))


def small_cases():
    g = load("small_cases")
    cases = [tuple(int(x) if i < 3 or i > 4 else float(x) for i, x in enumerate(row)) for row in g["cases"]]
    return g, cases


def gpu_session(**kw):
    import torch

    from paper_2011_11762_b200 import MatrixSession

    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return MatrixSession(device="cuda:0", **kw)


def reference_src():
    """Directory holding the reference package ``quadmat`` (pkg/src): the offline install under
    baseline/_ref (it travels to the GPU box with the repo snapshot), else the read-only reference
    tree of the build container; None when neither exists. Test infrastructure only."""
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    for cand in (root / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (cand / "quadmat" / "__init__.py").exists():
            return cand
    return None


def import_reference():
    """The reference package ``quadmat`` (sys.path gets reference_src())."""
    import sys

    src = reference_src()
    if src is None:
        return None
    if str(src) not in sys.path:
        sys.path.insert(0, str(src))
    import quadmat

    return quadmat


def rel(got, want) -> float:
    den = float(np.linalg.norm(want))
    d = float(np.linalg.norm(np.asarray(got) - np.asarray(want)))
    return d if den == 0 else d / den


def oracle_rows(cfg, rows):
    """Oracle C blocks of the given C block rows of a banded/random BASELINE config, computed on
    the host from regenerated operand blocks (block-keyed streams)."""
    from oracle import spgemm_oracle as O
    from paper_2011_11762_b200 import generators as G

    geom = cfg.geometry
    pat = G.config_pattern(cfg)
    ka, kb = G.config_keys(cfg, 0), G.config_keys(cfg, 1)
    ai, ak = geom.decode(ka)
    sel = np.isin(ai, rows)
    ka_s = ka[sel]
    bk, _ = geom.decode(kb)
    kb_s = kb[np.isin(bk, np.unique(ak[sel]))]
    ba = G.host_blocks(geom, ka_s, cfg.seed, 0, pat, cfg.half_bw)
    bb = G.host_blocks(geom, kb_s, cfg.seed, 1, pat, cfg.half_bw)
    kc, bc, _ = O.multiply(O.Geom(cfg.n, cfg.bs, cfg.bs), ka_s, ba, kb_s, bb)
    return kc, bc


def structural_c_keys(geom, ka: np.ndarray, kb: np.ndarray, a_cmask=None, b_rmask=None) -> np.ndarray:
    """The exact C block set of A*B on the host, sorted quadtree keys: every (i, j) with some k such
    that A(i,k) and B(k,j) are stored (the non-nil multiply tasks of ops.py:197-241). With the
    operands' support masks (a_cmask[t] = A block t's nonzero columns, b_rmask[t] = B block t's
    nonzero rows) only pairs whose supports meet count -- the others multiply to exactly zero, and
    a C block made only of such pairs is the exact-zero block _set_block drops
    (block_sparse.py:37-41). Operands with uniform random values (no cancellation) or positive
    values (C4) have exactly this nonzero C block set."""
    import scipy.sparse as sp

    nb = geom.nbg
    ai, ak = geom.decode(ka)
    bk, bj = geom.decode(kb)
    if a_cmask is None:
        pa = sp.csr_matrix((np.ones(ka.size, dtype=np.int64), (ai, ak)), shape=(nb, nb))
        pb = sp.csr_matrix((np.ones(kb.size, dtype=np.int64), (bk, bj)), shape=(nb, nb))
        c = (pa @ pb).tocoo()
        return np.sort(geom.qkey(c.row.astype(np.int64), c.col.astype(np.int64)))
    # masked: expand the (A block, B block) pairs per k, keep those whose supports meet
    order_b = np.argsort(bk, kind="stable")
    bk_s = bk[order_b]
    lo = np.searchsorted(bk_s, ak, side="left")
    hi = np.searchsorted(bk_s, ak, side="right")
    cnt = hi - lo
    ia = np.repeat(np.arange(ka.size), cnt)
    off = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    ib = order_b[np.repeat(lo, cnt) + off]
    meet = (a_cmask[ia] & b_rmask[ib]) != 0
    keys = geom.qkey(ai[ia[meet]].astype(np.int64), bj[ib[meet]].astype(np.int64))
    return np.unique(keys)


def lookup(keys_all: np.ndarray, blocks_dev, want: np.ndarray):
    """Copies the device blocks with the given keys to the host (keys must be present)."""
    import torch

    pos = np.searchsorted(keys_all, want)
    assert np.all(pos < keys_all.size) and np.array_equal(keys_all[pos], want), "missing C blocks"
    idx = torch.from_numpy(pos).to(blocks_dev.device)
    return blocks_dev.index_select(0, idx).cpu().numpy()


def decay_sparse(n: int, seed: int, width=None, scale: float = 4.0) -> np.ndarray:
    """Banded support with decaying magnitudes (pkg/tests/oracles.py:122-132 recipe)."""
    rng = np.random.default_rng(seed)
    width = width or max(4, n // 4)
    i = np.arange(n)
    dist = np.abs(i[:, None] - i[None, :])
    return np.exp(-dist / scale) * (dist <= width) * rng.standard_normal((n, n))


def support_masks_np(blocks: np.ndarray, with_flags: bool = False):
    """numpy statement of qm_block_meta's masks: bit r (r*64//bs above 64) of the row / column mask
    is set when that row / column of the block holds a nonzero; a NaN/Inf block gets full masks
    (bs bits, or all 64 from bs 64 up) and flag bit 0."""
    n, bs, _ = blocks.shape
    nz = blocks != 0
    bit = np.arange(bs) if bs <= 64 else (np.arange(bs) * 64) // bs
    w = (np.uint64(1) << bit.astype(np.uint64))
    rows = np.bitwise_or.reduce(np.where(nz.any(axis=2), w[None, :], np.uint64(0)), axis=1)
    cols = np.bitwise_or.reduce(np.where(nz.any(axis=1), w[None, :], np.uint64(0)), axis=1)
    bad = ~np.isfinite(blocks).all(axis=(1, 2))
    full = np.uint64(0xFFFFFFFFFFFFFFFF if bs >= 64 else (1 << bs) - 1)
    r = np.where(bad, full, rows).astype(np.uint64)
    c = np.where(bad, full, cols).astype(np.uint64)
    if with_flags:
        return r, c, bad.astype(np.uint64)
    return r, c


def banded_support_decay(n: int, bw: int, seed: int) -> np.ndarray:
    """Element-level band |i-j| <= bw with positive decaying values: blocks near the band edge are
    partly empty, so many block pairs multiply to exact zeros (the C4 decay situation)."""
    rng = np.random.default_rng(seed)
    i = np.arange(n)
    dist = np.abs(i[:, None] - i[None, :])
    return np.where(dist <= bw, np.exp(-dist / 8.0) * rng.uniform(0.5, 1.5, (n, n)), 0.0)
