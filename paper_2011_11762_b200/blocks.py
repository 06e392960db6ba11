"""Device-resident block storage: the B200 replacement of the chunk store for this path.

The reference keeps every quadtree node as an immutable encoded chunk in a ChunkStore
(chunkstore.py:66-138; leaf payload = BlockSparseLeaf.encode, block_sparse.py:226-231). Here a
matrix is one ``BlockSet``: three torch tensors on one device --

    keys   int64[n]        ascending quadtree keys (layout.qkey)
    blocks float64[n,bs,bs] row-major block payloads (the leaf payload's block bytes)
    sumsq  float64[n]      squared Frobenius norm per block (block_norms, block_sparse.py:41)

``QuadChunk`` stands in for ``ChunkId`` as ``Matrix.root`` (``is_nil``, identity equality), and
``DeviceStore`` keeps the reference's byte budget (StoreCapacityError, chunkstore.py:86-90).
Memory is owned by PyTorch; libqmb200 only ever sees raw pointers.
"""

from __future__ import annotations

import ctypes
import itertools
import math
import threading
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from .errors import ContractViolationError, StoreCapacityError


_SERIALS = itertools.count(1)


@dataclass
class BlockSet:
    keys: torch.Tensor
    blocks: torch.Tensor
    sumsq: torch.Tensor
    # int64[3, n] support masks (row 0: nonzero rows, row 1: nonzero columns, row 2: flags, bit 0 =
    # the block holds a NaN/Inf; qm_block_meta), computed with the norms by the block set's producer
    # (device generator / builder) or on first use by a product, and kept with the (immutable) set.
    masks: torch.Tensor | None = None
    # (every block has all rows nonzero, every block has all columns nonzero): set with `masks`
    masks_full: tuple[bool, bool] = (False, False)

    def support_masks(self, stream=None) -> torch.Tensor:
        """Per-block nonzero-row / nonzero-column bit masks (device). A product skips block pairs
        whose masks do not meet: their product is exactly zero (spgemm.multiply_blocks)."""
        if self.masks is None:
            self.compute_meta(stream, sumsq=False)
        return self.masks

    def compute_meta(self, stream=None, sumsq: bool = True) -> "BlockSet":
        """Norms (sumsq) and support masks of every block in one read of the blocks (qm_block_meta);
        the all-full flags are read back through mapped memory (a copy-engine read would queue behind
        bulk D2H copies in flight, e.g. a pipelined serving loop's result copies)."""
        from . import _ffi  # noqa: PLC0415

        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        m = torch.empty((3, self.n), dtype=torch.int64, device=self.device)
        if self.n:
            nf = torch.zeros(2, dtype=torch.int64, device=self.device)
            _ffi.check(_ffi.load().qm_block_meta(self.bs, self.n, _ffi.ptr(self.blocks),
                                                 _ffi.ptr(self.sumsq) if sumsq else 0, 0, 0, _ffi.ptr(m),
                                                 _ffi.ptr(nf), _ffi.stream_handle(st)),
                       "qm_block_meta")
            f0, f1 = _ffi.read_i64s(nf, 2, st)
            self.masks_full = (f0 == 0, f1 == 0)
        else:
            self.masks_full = (True, True)
        self.masks = m
        return self

    def row_index(self, layout, stream=None) -> dict:
        """The block set's row-sorted view (qm_row_index_build): operand metadata like the norms and
        masks, built once per (block set, layout) and kept with the immutable set, so a product's
        symbolic phase skips its own row indexing. Tensors: rowptr, row, col, perm (int32) and the
        column / row masks in row-sorted order (int64; when the set has masks)."""
        from . import _ffi  # noqa: PLC0415

        key = (int(layout.n_logical), int(layout.leaf_dim), int(layout.depth), int(layout.block_size))
        cache = self.__dict__.setdefault("_row_index", {})
        got = cache.get(key)
        if got is not None and (got["cmask"] is not None or self.masks is None):
            return got
        lib = _ffi.load()
        dev = self.device
        n = self.n
        nbg = (layout.leaf_dim // layout.block_size) << layout.depth
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        ix = {t: torch.empty(max(n, 1), dtype=torch.int32, device=dev) for t in ("row", "col", "perm")}
        ix["rowptr"] = torch.empty(nbg + 1, dtype=torch.int32, device=dev)
        has_m = self.masks is not None and n > 0
        ix["cmask"] = torch.empty(max(n, 1), dtype=torch.int64, device=dev) if has_m else None
        ix["rmask"] = torch.empty(max(n, 1), dtype=torch.int64, device=dev) if has_m else None
        wb = lib.qm_row_index_workspace_bytes(ctypes.byref(layout), n)
        ws = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
        _ffi.check(lib.qm_row_index_build(ctypes.byref(layout), _ffi.ptr(self.keys), n,
                                          _ffi.ptr(self.masks) if has_m else 0, _ffi.ptr(ws), wb,
                                          _ffi.ptr(ix["rowptr"]), _ffi.ptr(ix["row"]), _ffi.ptr(ix["col"]),
                                          _ffi.ptr(ix["perm"]), _ffi.ptr(ix["cmask"]), _ffi.ptr(ix["rmask"]),
                                          _ffi.stream_handle(st)), "qm_row_index_build")
        cache[key] = ix
        return ix

    @staticmethod
    def ix_struct(ix: dict, role: str | None):
        """qm_row_index of a row index as the left (role "a": column masks) or right ("b": row
        masks) operand; role None: no masks."""
        from . import _ffi  # noqa: PLC0415

        mask = None if role is None else ix["cmask"] if role == "a" else ix["rmask"]
        return _ffi.QmRowIndex(_ffi.ptr(ix["rowptr"]), _ffi.ptr(ix["row"]), _ffi.ptr(ix["col"]), _ffi.ptr(ix["perm"]),
                               _ffi.ptr(mask))

    @property
    def serial(self) -> int:
        """A process-unique id of this (immutable) block set: tags metadata derived from it and
        its peers' sets in a multi-GPU product (distributed.multiply's structure cache)."""
        sid = self.__dict__.get("_serial")
        if sid is None:
            sid = self.__dict__["_serial"] = next(_SERIALS)
        return sid

    @property
    def n(self) -> int:
        return int(self.keys.shape[0])

    @property
    def bs(self) -> int:
        return int(self.blocks.shape[1])

    @property
    def device(self) -> torch.device:
        return self.blocks.device

    @property
    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.keys, self.blocks, self.sumsq))

    @staticmethod
    def empty(bs: int, device) -> "BlockSet":
        return BlockSet(
            torch.empty(0, dtype=torch.int64, device=device),
            torch.empty((0, bs, bs), dtype=torch.float64, device=device),
            torch.empty(0, dtype=torch.float64, device=device),
        )

    @staticmethod
    def from_numpy(keys: np.ndarray, blocks: np.ndarray, sumsq: np.ndarray | None, device,
                   pin: bool = False) -> "BlockSet":
        if sumsq is None:
            sumsq = np.einsum("nij,nij->n", blocks, blocks) if blocks.size else np.zeros(0)
        k = torch.from_numpy(np.ascontiguousarray(keys, dtype=np.int64))
        b = torch.from_numpy(np.ascontiguousarray(blocks, dtype=np.float64))
        s = torch.from_numpy(np.ascontiguousarray(sumsq, dtype=np.float64))
        dev = torch.device(device)
        if dev.type == "cpu":
            return BlockSet(k, b, s)
        return BlockSet(k.to(dev, non_blocking=pin), b.to(dev, non_blocking=pin),
                        s.to(dev, non_blocking=pin))

    def to_host(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        return (self.keys.cpu().numpy(), self.blocks.cpu().numpy(), self.sumsq.cpu().numpy())


class QuadChunk:
    """Root handle of a matrix value (replaces ``ChunkId``; chunkstore.py:27-41)."""

    __slots__ = ("id", "blockset", "explicit_zero", "__weakref__")

    def __init__(self, cid: int, blockset: BlockSet | None, explicit_zero: bool = False):
        self.id = cid
        self.blockset = blockset
        self.explicit_zero = explicit_zero

    @property
    def is_nil(self) -> bool:
        return self.id == 0

    @property
    def n_blocks(self) -> int:
        return 0 if self.blockset is None else self.blockset.n

    def require(self) -> BlockSet:
        if self.blockset is None:
            raise ContractViolationError("nil chunk id cannot be dereferenced")
        return self.blockset

    def __eq__(self, other):
        return isinstance(other, QuadChunk) and other.id == self.id

    def __hash__(self):
        return hash(self.id)

    def __repr__(self):
        return "NIL" if self.id == 0 else f"QuadChunk({self.id}, blocks={self.n_blocks})"


NIL = QuadChunk(0, None)


class DeviceStore:
    """Byte-budgeted registry of matrix values on one device.

    Unlike the reference store (which never frees) a value's memory is released
    when the last Python reference to its ``QuadChunk`` goes away; the budget counts live bytes.
    """

    def __init__(self, device, max_bytes: int | None = None):
        self.device = torch.device(device)
        self._max_bytes = max_bytes
        self._live = 0
        self._ids = itertools.count(1)
        self._lock = threading.Lock()
        self.n_registered = 0

    def _release(self, nbytes: int):
        with self._lock:
            self._live -= nbytes

    def register(self, blockset: BlockSet, explicit_zero: bool = False) -> QuadChunk:
        if blockset.n == 0 and not explicit_zero:
            return NIL
        size = blockset.nbytes
        with self._lock:
            if self._max_bytes is not None and self._live + size > self._max_bytes:
                raise StoreCapacityError(
                    f"store capacity exhausted: {self._live} + {size} > {self._max_bytes} bytes"
                )
            self._live += size
            self.n_registered += 1
            cid = next(self._ids)
        chunk = QuadChunk(cid, blockset, explicit_zero)
        weakref.finalize(chunk, self._release, size)
        return chunk

    def check_room(self, extra_bytes: int):
        if self._max_bytes is not None and self._live + extra_bytes > self._max_bytes:
            raise StoreCapacityError(
                f"store capacity exhausted: {self._live} + {extra_bytes} > {self._max_bytes} bytes"
            )

    @property
    def total_bytes(self) -> int:
        return self._live

    def norm_of(self, chunk: QuadChunk) -> float:
        if chunk.is_nil or chunk.blockset is None or chunk.blockset.n == 0:
            return 0.0
        return math.sqrt(float(chunk.blockset.sumsq.sum().item()))
