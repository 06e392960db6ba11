"""Matrix geometry and the quadtree block key.

``MatrixParams``, ``OwnerPolicy`` and ``TreeStats`` keep the reference's fields and semantics
(pkg/src/quadmat/quadtree.py:24-71). The quadtree itself is not materialised: a matrix is the set
of its stored ``bs x bs`` blocks ordered by the quadtree key

    qkey(bi, bj) = morton(bi // nbl, bj // nbl) << 2*lbits | (bi % nbl) << lbits | (bj % nbl)

(nbl = leaf_dim // bs, lbits = ceil(log2 nbl), Morton with the row bit high). Ascending qkey is the
reference's depth-first NW, NE, SW, SE walk (quadtree.py:125-135, canonical_bytes :293-318) down
to the leaves, then BlockSparseLeaf.encode's sorted (bi, bj) order inside a leaf
(leaves/block_sparse.py:226-231), so every subtree is one contiguous key range. The device
library uses the same function (csrc/qm_common.cuh: qkey).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError


class LeafKind(enum.Enum):
    """Leaf representations of the reference (leaves/base.py:22-25). The B200 path stores
    ``BLOCK_SPARSE`` leaves; the other kinds are outside the hot path."""

    DENSE = "dense"
    BLOCK_SPARSE = "block_sparse"
    HIERARCHICAL = "hierarchical"


def resolve_leaf_kind(kind) -> LeafKind:
    if isinstance(kind, LeafKind):
        return kind
    if isinstance(kind, str):
        try:
            return LeafKind(kind)
        except ValueError:
            raise ConfigurationError(f"unknown leaf kind {kind!r}") from None
    value = getattr(kind, "value", None)  # a reference quadmat.LeafKind
    if isinstance(value, str):
        return resolve_leaf_kind(value)
    raise ConfigurationError(f"unknown leaf kind {kind!r}")


@dataclass(frozen=True)
class MatrixParams:
    """quadtree.py:24-44: logical dimension, leaf dimension and minimal tree depth."""

    n_logical: int
    leaf_dim: int
    depth: int

    @classmethod
    def create(cls, n_logical: int, leaf_dim: int) -> "MatrixParams":
        if n_logical < 1 or leaf_dim < 1:
            raise ConfigurationError("matrix and leaf dimensions must be positive")
        depth = 0
        while leaf_dim * (1 << depth) < n_logical:
            depth += 1
        return cls(int(n_logical), int(leaf_dim), depth)

    @property
    def n_padded(self) -> int:
        return self.leaf_dim * (1 << self.depth)

    def node_dim(self, level: int) -> int:
        return self.leaf_dim * (1 << (self.depth - level))


@dataclass(frozen=True)
class OwnerPolicy:
    """quadtree.py:47-63: round-robin ownership over the subtree index at a split depth. Kept for
    API compatibility; the multi-GPU partition (distributed.py) uses work-balanced key ranges."""

    n_workers: int = 1
    split_depth: int | None = None

    def resolve_split(self, depth: int) -> int:
        if self.split_depth is not None:
            return min(self.split_depth, depth)
        d = 0
        while (1 << (2 * d)) < self.n_workers:
            d += 1
        return min(d, depth)

    def owner_of(self, subtree_index: int) -> int:
        return subtree_index % self.n_workers


@dataclass
class TreeStats:
    """quadtree.py:66-71."""

    n_leaf_chunks: int = 0
    n_branch_chunks: int = 0
    stored_bytes: int = 0
    nnz: int = 0


@dataclass(frozen=True)
class Geometry:
    """Block geometry of (params, block_size); mirrors qm::Geometry in csrc/qm_common.cuh."""

    params: MatrixParams
    bs: int

    def __post_init__(self):
        if self.bs < 1 or self.params.leaf_dim % self.bs != 0:
            raise ConfigurationError(
                f"block size {self.bs} must divide leaf dimension {self.params.leaf_dim}"
            )

    @property
    def nbl(self) -> int:
        return self.params.leaf_dim // self.bs

    @property
    def lbits(self) -> int:
        return (self.nbl - 1).bit_length()

    @property
    def nbg(self) -> int:
        return self.nbl << self.params.depth

    @property
    def key_bits(self) -> int:
        return 2 * (self.params.depth + self.lbits)

    def qkey(self, bi, bj) -> np.ndarray:
        return qkey(bi, bj, self.nbl, self.lbits)

    def decode(self, keys) -> tuple[np.ndarray, np.ndarray]:
        return qkey_decode(keys, self.nbl, self.lbits)

    def leaf_key_shift(self) -> int:
        """Right shift that maps a block qkey to its leaf's Morton index."""
        return 2 * self.lbits


def _spread(x: np.ndarray) -> np.ndarray:
    v = x.astype(np.uint64)
    v = (v | (v << np.uint64(16))) & np.uint64(0x0000FFFF0000FFFF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x00FF00FF00FF00FF)
    v = (v | (v << np.uint64(4))) & np.uint64(0x0F0F0F0F0F0F0F0F)
    v = (v | (v << np.uint64(2))) & np.uint64(0x3333333333333333)
    v = (v | (v << np.uint64(1))) & np.uint64(0x5555555555555555)
    return v


def _compact(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.uint64) & np.uint64(0x5555555555555555)
    v = (v | (v >> np.uint64(1))) & np.uint64(0x3333333333333333)
    v = (v | (v >> np.uint64(2))) & np.uint64(0x0F0F0F0F0F0F0F0F)
    v = (v | (v >> np.uint64(4))) & np.uint64(0x00FF00FF00FF00FF)
    v = (v | (v >> np.uint64(8))) & np.uint64(0x0000FFFF0000FFFF)
    v = (v | (v >> np.uint64(16))) & np.uint64(0x00000000FFFFFFFF)
    return v


def qkey(bi, bj, nbl: int, lbits: int) -> np.ndarray:
    """Vectorised quadtree key (int64; keys stay below 2**62)."""
    bi = np.asarray(bi, dtype=np.int64)
    bj = np.asarray(bj, dtype=np.int64)
    li, ri = np.divmod(bi, nbl)
    lj, rj = np.divmod(bj, nbl)
    m = (_spread(li) << np.uint64(1)) | _spread(lj)
    key = (m << np.uint64(2 * lbits)) | (ri.astype(np.uint64) << np.uint64(lbits)) | rj.astype(np.uint64)
    return key.astype(np.int64)


def qkey_decode(keys, nbl: int, lbits: int) -> tuple[np.ndarray, np.ndarray]:
    k = np.asarray(keys, dtype=np.int64).astype(np.uint64)
    local = k & np.uint64((1 << (2 * lbits)) - 1)
    ri = (local >> np.uint64(lbits)).astype(np.int64)
    rj = (local & np.uint64((1 << lbits) - 1)).astype(np.int64)
    m = k >> np.uint64(2 * lbits)
    li = _compact(m >> np.uint64(1)).astype(np.int64)
    lj = _compact(m).astype(np.int64)
    return li * nbl + ri, lj * nbl + rj
