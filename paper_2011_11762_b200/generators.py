"""Workload generators.

Two families:

1. The reference's own experiment families (generators.py:29-270 of the reference): banded,
   growing_block and random_blocks patterns with value 1.0, the closed-form flop oracle
   ``flop_count_exact`` and ``generate(store, case, ...)`` with the reference signature. C is
   integer-valued for these, so the GPU product must match bit for bit.

2. The BASELINE.json configurations with block-keyed uniform values:
   block (bi, bj) of matrix m holds np.random.default_rng([seed, m, bi, bj]).uniform(-1, 1, (bs, bs))
   masked by the element pattern. The device generator (qm_generate_blocks) reproduces those
   streams bit for bit, so the host oracle can regenerate any block of any size of problem.

   C1  banded N=4096, |i-j| <= 256, bs 64                   (parity config, CPU-runnable)
   C2  banded N in {16384, 32768, 65536, 131072}, hb 512, bs 64
   C3  random: 1024 x 1024 block grid, 8 distinct block columns per block row, bs 64
   C4  decay: 65536 points in a cube at 0.1/A^3, RCB order, exp(-r^2/2) > 1e-10, bs 64, C = A*A
   C5  banded N = 2^20, hb 1024, bs in {32, 64, 128}
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _ffi, construct
from .blocks import BlockSet
from .errors import ConfigurationError, PlacementError
from .layout import Geometry, MatrixParams, resolve_leaf_kind, LeafKind

FAMILIES = ("banded", "growing_block", "random_blocks")

# ---------------------------------------------------------------------------------------------
# 1. Reference experiment families (value 1.0)
# ---------------------------------------------------------------------------------------------


@dataclass(frozen=True)
class ExperimentCase:
    """generators.py:32-56 of the reference."""

    family: str
    n: int
    b: int
    s: int = 0
    n_blocks: int = 0
    seed: int = 0

    def __post_init__(self):
        if self.family not in FAMILIES:
            raise ConfigurationError(f"unknown family {self.family!r}")
        if self.n < 1:
            raise ConfigurationError("n must be positive")
        if self.b < 0:
            raise ConfigurationError("half-bandwidth b must be >= 0")
        if self.s < 0 or self.s > self.n:
            raise ConfigurationError("block size s must be in [0, n]")
        if self.family == "random_blocks":
            if self.n_blocks < 0:
                raise ConfigurationError("n_blocks must be >= 0")
            if self.n_blocks * self.s > self.n:
                raise PlacementError(
                    f"{self.n_blocks} blocks of size {self.s} cannot fit in n={self.n}"
                )


def block_positions(case: ExperimentCase, max_tries: int = 1000) -> list[int]:
    """generators.py:64-96: seeded non-overlapping diagonal block offsets, ascending."""
    if case.family == "banded" or case.s == 0:
        return []
    if case.family == "growing_block":
        return [0]
    n, s, b = case.n, case.s, case.b
    count = case.n_blocks
    if count == 0:
        return []
    lo, hi = b, n - s - b
    if lo > hi:
        lo, hi = 0, n - s
    rng = np.random.default_rng(case.seed)
    placed: list[int] = []
    tries = 0
    budget = max_tries * count
    while len(placed) < count:
        if tries >= budget:
            raise PlacementError(
                f"could not place {count} non-overlapping blocks of size {s} in [{lo}, {hi}] "
                f"after {budget} tries"
            )
        tries += 1
        p = int(rng.integers(lo, hi + 1))
        if all(abs(p - q) >= s for q in placed):
            placed.append(p)
    return sorted(placed)


def _banded_widths(n: int, b: int) -> np.ndarray:
    k = np.arange(n, dtype=np.int64)
    return np.minimum(k + b, n - 1) - np.maximum(k - b, 0) + 1


def _block_corrections(n, b, s, positions, squared: bool) -> int:
    total = 0
    for p in positions:
        k = np.arange(p, p + s, dtype=np.int64)
        wu = np.minimum(np.maximum(k + b, p + s - 1), n - 1) - np.maximum(np.minimum(k - b, p), 0) + 1
        wb = np.minimum(k + b, n - 1) - np.maximum(k - b, 0) + 1
        if squared:
            total += int(np.sum(wu * wu - wb * wb, dtype=np.int64))
        else:
            total += int(np.sum(wu - wb, dtype=np.int64))
    return total


def pattern_nnz(case: ExperimentCase) -> int:
    """generators.py:128-131."""
    w = _banded_widths(case.n, case.b)
    return int(np.sum(w, dtype=np.int64)) + _block_corrections(
        case.n, case.b, case.s, block_positions(case), False)


def flop_count_exact(case: ExperimentCase) -> int:
    """generators.py:134-138: 2 * |{(i,j,k): P(i,k) and P(k,j)}| (scalar pattern flops)."""
    w = _banded_widths(case.n, case.b)
    base = int(np.sum(w * w, dtype=np.int64))
    corr = _block_corrections(case.n, case.b, case.s, block_positions(case), True)
    return 2 * (base + corr)


def _case_tile_fns(case: ExperimentCase, leaf_dim: int):
    positions = block_positions(case)
    n, b, s = case.n, case.b, case.s

    def support(r0, r1, c0, c1):
        if c0 - r1 + 1 <= b and r0 - c1 + 1 <= b:
            return True
        return any(p < r1 and r0 < p + s and p < c1 and c0 < p + s for p in positions)

    def tile(r0, c0):
        i = r0 + np.arange(leaf_dim)
        j = c0 + np.arange(leaf_dim)
        mask = np.abs(i[:, None] - j[None, :]) <= b
        for p in positions:
            if p < r0 + leaf_dim and r0 < p + s and p < c0 + leaf_dim and c0 < p + s:
                ri0, ri1 = max(p - r0, 0), min(p + s - r0, leaf_dim)
                ci0, ci1 = max(p - c0, 0), min(p + s - c0, leaf_dim)
                mask[ri0:ri1, ci0:ci1] = True
            elif p >= r0 + leaf_dim and p >= c0 + leaf_dim:
                break
        mask &= (i[:, None] < n) & (j[None, :] < n)
        if not mask.any():
            return None
        return mask.astype(np.float64)

    return tile, support


def generate(store, case: ExperimentCase, leaf_dim: int = 128, leaf_kind=LeafKind.BLOCK_SPARSE,
             block_size: int = 16, owner_policy=None):
    """generators.generate (reference generators.py:231-270), same signature; ``store`` is a
    session's DeviceStore. Pure-band cases are generated on the device (pattern 2 of
    qm_generate_blocks); cases with dense diagonal blocks are cut from host tiles."""
    from .session import Matrix  # noqa: PLC0415  (cycle)

    kind = resolve_leaf_kind(leaf_kind)
    if kind is not LeafKind.BLOCK_SPARSE:
        raise ConfigurationError(f"leaf kind {kind.value!r} is outside the B200 path")
    params = MatrixParams.create(case.n, leaf_dim)
    geom = Geometry(params, block_size)
    if not block_positions(case) and store.device.type == "cuda":
        keys = banded_block_keys(geom, case.b)
        bset = device_blocks(geom, keys, seed=0, matrix_id=0, pattern=2, half_bw=case.b,
                             device=store.device)
    else:
        tile, support = _case_tile_fns(case, leaf_dim)
        keys, blocks = construct.blocks_from_tiles(geom, tile, support)
        bset = BlockSet.from_numpy(keys, blocks, None, store.device)
    return Matrix(store.register(bset), params, kind, block_size, False)


# ---------------------------------------------------------------------------------------------
# 2. BASELINE configurations (block-keyed uniform values)
# ---------------------------------------------------------------------------------------------

PATTERN_DENSE, PATTERN_BAND, PATTERN_BAND_ONES = 0, 1, 2


def banded_block_keys(geom: Geometry, half_bw: int) -> np.ndarray:
    """Sorted quadtree keys of the blocks that intersect the band |i - j| <= half_bw inside
    [0, n_logical)^2 (the support test of generators.py:246-249 at block granularity)."""
    n = geom.params.n_logical
    bs = geom.bs
    nb = -(-n // bs)
    w = (half_bw + bs - 1) // bs + 1
    bi = np.repeat(np.arange(nb, dtype=np.int64), 2 * w + 1)
    bj = bi + np.tile(np.arange(-w, w + 1, dtype=np.int64), nb)
    ok = (bj >= 0) & (bj < nb)
    bi, bj = bi[ok], bj[ok]
    # minimum |i - j| between row range [bi*bs, bi*bs+bs-1] and column range of bj (clipped to n)
    r0, r1 = bi * bs, np.minimum(bi * bs + bs, n) - 1
    c0, c1 = bj * bs, np.minimum(bj * bs + bs, n) - 1
    gap = np.maximum(0, np.maximum(c0 - r1, r0 - c1))
    keep = gap <= half_bw
    keys = geom.qkey(bi[keep], bj[keep])
    keys.sort()
    return keys


def random_block_keys(geom: Geometry, per_row: int, seed: int, matrix_id: int) -> np.ndarray:
    """C3 pattern: each block row has ``per_row`` distinct block columns,
    default_rng([seed, m, 0xB10C]).choice(nbg, per_row, replace=False) per row in order."""
    nb = -(-geom.params.n_logical // geom.bs)
    rng = np.random.default_rng([seed, matrix_id, 0xB10C])
    bi = np.repeat(np.arange(nb, dtype=np.int64), per_row)
    bj = np.concatenate([np.sort(rng.choice(nb, per_row, replace=False)) for _ in range(nb)])
    keys = geom.qkey(bi, bj.astype(np.int64))
    keys.sort()
    return keys


def host_block(seed: int, matrix_id: int, bi: int, bj: int, bs: int, pattern: int, half_bw: int,
               n_logical: int) -> np.ndarray:
    """The block-keyed value stream on the host (numpy): what qm_generate_blocks reproduces."""
    i = bi * bs + np.arange(bs)[:, None]
    j = bj * bs + np.arange(bs)[None, :]
    mask = (i < n_logical) & (j < n_logical)
    if pattern != PATTERN_DENSE:
        mask &= np.abs(i - j) <= half_bw
    if pattern == PATTERN_BAND_ONES:
        return mask.astype(np.float64)
    vals = np.random.default_rng([seed, matrix_id, int(bi), int(bj)]).uniform(-1.0, 1.0, (bs, bs))
    return np.where(mask, vals, 0.0)


def host_blocks(geom: Geometry, keys: np.ndarray, seed: int, matrix_id: int, pattern: int,
                half_bw: int = 0) -> np.ndarray:
    bi, bj = geom.decode(keys)
    out = np.empty((keys.size, geom.bs, geom.bs))
    for x in range(keys.size):
        out[x] = host_block(seed, matrix_id, int(bi[x]), int(bj[x]), geom.bs, pattern, half_bw,
                            geom.params.n_logical)
    return out


def device_blocks(geom: Geometry, keys: np.ndarray | torch.Tensor, seed: int, matrix_id: int,
                  pattern: int, half_bw: int = 0, device=None, stream=None) -> BlockSet:
    """Block-keyed values generated on the device (libqmb200 qm_generate_blocks)."""
    lib = _ffi.load()
    dev = torch.device(device) if device is not None else torch.device("cuda")
    if dev.type != "cuda":
        raise ConfigurationError("device_blocks needs a CUDA device")
    k = keys if isinstance(keys, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(keys))
    k = k.to(dev)
    n = int(k.shape[0])
    bs = geom.bs
    blocks = torch.empty((n, bs, bs), dtype=torch.float64, device=dev)
    sumsq = torch.empty(n, dtype=torch.float64, device=dev)
    layout = _ffi.make_layout(geom.params, bs)
    with torch.cuda.device(dev):
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        _ffi.check(lib.qm_generate_blocks(ctypes.byref(layout), _ffi.ptr(k), n, seed, matrix_id,
                                          pattern, half_bw, _ffi.ptr(blocks), 0, _ffi.stream_handle(st)),
                   "qm_generate_blocks")
        # operand metadata (norms + support masks + NaN/Inf flags) in one read of the new blocks
        return BlockSet(k, blocks, sumsq).compute_meta(st)


# ---- C4: decay matrix ---------------------------------------------------------------------------

def rcb_order(points: np.ndarray) -> np.ndarray:
    """Recursive coordinate bisection: split at the median of the axis of largest extent (stable
    argsort), recurse down to single points; returns the visiting order."""
    out = np.empty(points.shape[0], dtype=np.int64)
    pos = 0
    stack = [np.arange(points.shape[0])]
    # explicit stack, left part first
    while stack:
        idx = stack.pop()
        if idx.size == 1:
            out[pos] = idx[0]
            pos += 1
            continue
        p = points[idx]
        axis = int(np.argmax(p.max(axis=0) - p.min(axis=0)))
        order = idx[np.argsort(p[:, axis], kind="stable")]
        half = idx.size // 2
        stack.append(order[half:])
        stack.append(order[:half])
    return out


def decay_triplets(n_points: int = 65536, density: float = 0.1, seed: int = 0,
                   cutoff: float = 1e-10):
    """C4 element list: points uniform in a cube of side (n/density)^(1/3), RCB-ordered,
    a_ij = exp(-0.5 r^2) kept where >= cutoff, no periodic images."""
    from scipy.spatial import cKDTree  # noqa: PLC0415

    side = (n_points / density) ** (1.0 / 3.0)
    pts = np.random.default_rng(seed).uniform(0.0, side, (n_points, 3))
    pts = pts[rcb_order(pts)]
    rc = math.sqrt(-2.0 * math.log(cutoff))
    pairs = cKDTree(pts).query_pairs(rc, output_type="ndarray")
    d2 = np.sum((pts[pairs[:, 0]] - pts[pairs[:, 1]]) ** 2, axis=1)
    v = np.exp(-0.5 * d2)
    keep = v >= cutoff
    i, j, v = pairs[keep, 0], pairs[keep, 1], v[keep]
    diag = np.arange(n_points)
    rows = np.concatenate([diag, i, j])
    cols = np.concatenate([diag, j, i])
    vals = np.concatenate([np.ones(n_points), v, v])
    return n_points, rows.astype(np.int64), cols.astype(np.int64), vals


# ---- named BASELINE configurations ---------------------------------------------------------------

@dataclass(frozen=True)
class BaselineConfig:
    name: str
    kind: str          # "banded" | "random" | "decay"
    n: int
    bs: int
    half_bw: int = 0
    per_row: int = 0
    seed: int = 0
    same_operand: bool = False  # C = A*A

    @property
    def geometry(self) -> Geometry:
        return Geometry(MatrixParams.create(self.n, self.bs), self.bs)  # L64 layout: leaf = block


CONFIGS = {
    "C1": BaselineConfig("C1", "banded", 4096, 64, half_bw=256),
    "C2-16384": BaselineConfig("C2-16384", "banded", 16384, 64, half_bw=512),
    "C2-32768": BaselineConfig("C2-32768", "banded", 32768, 64, half_bw=512),
    "C2-65536": BaselineConfig("C2-65536", "banded", 65536, 64, half_bw=512),
    "C2-131072": BaselineConfig("C2-131072", "banded", 131072, 64, half_bw=512),
    "C3": BaselineConfig("C3", "random", 65536, 64, per_row=8),
    "C4": BaselineConfig("C4", "decay", 65536, 64, same_operand=True),
    "C5-32": BaselineConfig("C5-32", "banded", 1 << 20, 32, half_bw=1024),
    "C5-64": BaselineConfig("C5-64", "banded", 1 << 20, 64, half_bw=1024),
    "C5-128": BaselineConfig("C5-128", "banded", 1 << 20, 128, half_bw=1024),
}


def config_keys(cfg: BaselineConfig, matrix_id: int) -> np.ndarray:
    geom = cfg.geometry
    if cfg.kind == "banded":
        return banded_block_keys(geom, cfg.half_bw)
    if cfg.kind == "random":
        return random_block_keys(geom, cfg.per_row, cfg.seed, matrix_id)
    raise ConfigurationError(f"{cfg.name}: keys of a {cfg.kind} config come from its triplets")


def config_pattern(cfg: BaselineConfig) -> int:
    return PATTERN_BAND if cfg.kind == "banded" else PATTERN_DENSE


def config_operands_host(cfg: BaselineConfig):
    """(geom, (keysA, blocksA), (keysB, blocksB)) on the host (numpy streams)."""
    geom = cfg.geometry
    if cfg.kind == "decay":
        n, r, c, v = decay_triplets(cfg.n, seed=cfg.seed)
        ka, ba = construct.blocks_from_triplets(geom, r, c, v)
        return geom, (ka, ba), (ka, ba)
    out = []
    for m in (0, 1):
        keys = config_keys(cfg, m)
        out.append((keys, host_blocks(geom, keys, cfg.seed, m, config_pattern(cfg), cfg.half_bw)))
    return geom, out[0], out[1]


def config_operands_device(cfg: BaselineConfig, device) -> tuple[Geometry, BlockSet, BlockSet]:
    """Operands resident on ``device``; uniform-value configs are generated on the device."""
    geom = cfg.geometry
    if cfg.kind == "decay":
        _, (ka, ba), _ = config_operands_host(cfg)
        a = BlockSet.from_numpy(ka, ba, None, device)
        if a.device.type == "cuda":
            a.compute_meta()  # input metadata, like the block norms (one pass: norms + masks)
        return geom, a, a
    sets = []
    for m in (0, 1):
        keys = config_keys(cfg, m)
        sets.append(device_blocks(geom, keys, cfg.seed, m, config_pattern(cfg), cfg.half_bw, device))
    return geom, sets[0], sets[1]


def structure_counts(cfg: BaselineConfig) -> dict:
    """Block-level structure of a configuration's product, on the host (numpy/scipy, no device):
    nnzb(A), nnzb(B), the structural C block count and triple count T (every (A block, B block)
    pair with a matching k, as BlockSparseLeaf.multiply enumerates them). Both
    bench arms report these as the workload definition."""
    import scipy.sparse as sp  # noqa: PLC0415

    geom = cfg.geometry
    if cfg.kind == "decay":
        _, (ka, _), (kb, _) = config_operands_host(cfg)
    else:
        ka, kb = config_keys(cfg, 0), config_keys(cfg, 1)
    nb = geom.nbg

    def occ(keys):
        bi, bj = geom.decode(keys)
        return sp.csr_matrix((np.ones(keys.size, dtype=np.int64), (bi, bj)), shape=(nb, nb))

    pa, pb = occ(ka), occ(kb)
    c = pa @ pb
    return {"nnzb_a": int(ka.size), "nnzb_b": int(kb.size), "nnzb_c_structural": int(c.nnz),
            "triples_structural": int(c.sum())}
