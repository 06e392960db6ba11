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
