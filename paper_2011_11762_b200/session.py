"""Drop-in driver API: ``MatrixSession`` with the reference's construction, multiply and inspection
entry points (pkg/src/quadmat/session.py:20-238), executing the multiply on a B200.

Scripts written against ``quadmat`` run with only the import changed:

    from paper_2011_11762_b200 import MatrixSession      # was: from quadmat import MatrixSession
    ses = MatrixSession(n_workers=1, mode="threaded")
    a = ses.matrix_from_triplets(n, rows, cols, vals, leaf_dim=64, block_size=64)
    c = ses.multiply(a, a)
    ses.to_dense(c); ses.canonical(c); ses.tree_stats(c); ses.norm(c)

``mode`` names the reference's CPU scheduler ("simulate" | "threaded"); both are accepted and the
work runs on the GPU ("gpu" is the native name). ``n_workers`` > 1 inside a torch.distributed job
selects the multi-GPU partition (distributed.py). Matrices live on the session's device as
``BlockSet`` tensors; the inspection methods copy to the host.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import bridge, construct, spgemm
from ._ffi import make_layout
from .blocks import NIL, BlockSet, DeviceStore, QuadChunk
from .errors import (
    ConfigurationError,
    ContractViolationError,
    DeviceUnavailableError,
    DimensionMismatchError,
)
from .layout import Geometry, LeafKind, MatrixParams, OwnerPolicy, TreeStats, resolve_leaf_kind

_MODES = ("gpu", "simulate", "threaded")
_VARIANTS = ("regular", "symmetric", "symmetric_square", "rank_k", "approximate")


@dataclass(frozen=True)
class Matrix:
    """A matrix value (quadtree.py:74-82): root handle plus what is needed to interpret it."""

    root: QuadChunk
    params: MatrixParams
    leaf_kind: LeafKind
    block_size: int
    symmetric: bool = False

    @property
    def geometry(self) -> Geometry:
        return Geometry(self.params, self.block_size)


@dataclass(frozen=True)
class MultiplyVariant:
    """ops.py:47-76 (same tags and validation)."""

    tag: str = "regular"
    tau: float = 0.0

    def __post_init__(self):
        if self.tag not in _VARIANTS:
            raise ConfigurationError(f"unknown multiply variant {self.tag!r}")
        if self.tau < 0:
            raise ConfigurationError("approximate multiply needs tau >= 0")

    @classmethod
    def regular(cls):
        return cls("regular")

    @classmethod
    def symmetric(cls):
        return cls("symmetric")

    @classmethod
    def symmetric_square(cls):
        return cls("symmetric_square")

    @classmethod
    def rank_k(cls):
        return cls("rank_k")

    @classmethod
    def approximate(cls, tau: float):
        return cls("approximate", tau)


@dataclass(frozen=True)
class TruncationSpec:
    """ops.py:79-88."""

    tau: float
    mode: str = "global_frobenius"

    def __post_init__(self):
        if self.tau < 0:
            raise ConfigurationError("truncation needs tau >= 0")
        if self.mode != "global_frobenius":
            raise ConfigurationError(f"unknown truncation mode {self.mode!r}")


@dataclass
class TaskSpec:
    """engine.py:42-49. ``run_spec`` executes a level-0 "multiply" spec as one GPU product."""

    task_type: str
    inputs: list
    args: dict = field(default_factory=dict)
    depth: int = 0
    parent: int | None = None


@dataclass
class WorkerStats:
    """chunkstore.py:54-63, one record per GPU: tasks_executed = block triples computed,
    bytes_received = block bytes fetched from peers in the halo exchange."""

    worker: int
    tasks_executed: int = 0
    steals: int = 0
    bytes_received: int = 0
    cache_hits: int = 0
    cache_misses: int = 0


def _check_conformant(a: Matrix, b: Matrix):
    """ops.py:541-547."""
    if a.params != b.params:
        raise DimensionMismatchError(f"operand params differ: {a.params} vs {b.params}")
    if a.leaf_kind != b.leaf_kind or a.block_size != b.block_size:
        raise ConfigurationError("operands must share leaf kind and block size")


def multiply_spec(a: Matrix, b: Matrix | None, variant: MultiplyVariant) -> tuple[TaskSpec, bool]:
    """ops.multiply_spec (ops.py:582-608): same validation, same (spec, result_is_symmetric)."""
    tag = variant.tag
    if tag in ("symmetric_square", "rank_k"):
        if b is not None and b.root != a.root:
            raise ContractViolationError(f"{tag} takes a single operand")
        b = a
    if b is None:
        raise ContractViolationError(f"variant {tag} needs two operands")
    _check_conformant(a, b)
    if tag == "symmetric_square" and not a.symmetric:
        raise ContractViolationError("symmetric_square needs a symmetric operand")
    if tag == "symmetric" and not (a.symmetric or b.symmetric):
        raise ContractViolationError("symmetric variant needs a symmetric operand")
    if tag == "rank_k" and a.symmetric:
        raise ContractViolationError("rank_k takes a general operand")
    upper = tag in ("symmetric_square", "rank_k")
    args = {
        "level": 0,
        "ta": False,
        "tb": tag == "rank_k",
        "a_sym": a.symmetric,
        "b_sym": b.symmetric,
        "upper": upper,
        "tau": float(variant.tau),
        "geometry": a.geometry,
    }
    return TaskSpec("multiply", [a.root, b.root], args), upper


def _default_device():
    if torch.cuda.is_available():
        return torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
    return torch.device("cpu")


class MatrixSession:
    """Owns a device store and runs each product on the GPU (session.py:20-64)."""

    def __init__(
        self,
        n_workers: int = 1,
        mode: str = "gpu",
        cache_capacity_bytes: int = 64 << 20,
        seed: int = 0,
        store_capacity_bytes: int | None = None,
        record_events: bool = False,
        device=None,
    ):
        if mode not in _MODES:
            raise ConfigurationError(f"mode must be one of {_MODES}, got {mode!r}")
        if n_workers < 1:
            raise ConfigurationError("n_workers must be >= 1")
        if cache_capacity_bytes <= 0:
            raise ConfigurationError("cache capacity must be positive")
        self.device = torch.device(device) if device is not None else _default_device()
        self.store = DeviceStore(self.device, store_capacity_bytes)
        self.n_workers = n_workers
        self.mode = mode
        self.seed = seed
        self.record_events = record_events
        self.cache_capacity_bytes = cache_capacity_bytes
        self.last_stats: list[WorkerStats] | None = None
        self.last_multiply: spgemm.MultiplyStats | None = None
        self.last_engine = None
        # n_workers > 1 inside a torch.distributed job of that size = one rank per GPU with the
        # work-balanced key-range partition. Outside such a job the reference's workers are a CPU
        # scheduling detail and the product runs on this process's GPU.
        self.comm = None
        if n_workers > 1:
            import torch.distributed as dist  # noqa: PLC0415

            if dist.is_available() and dist.is_initialized():
                if dist.get_world_size() != n_workers:
                    raise ConfigurationError(
                        f"n_workers={n_workers} but the process group has {dist.get_world_size()} ranks"
                    )
                from .distributed import Comm  # noqa: PLC0415

                self.comm = Comm()

    # -- engine plumbing ------------------------------------------------------------------------

    def run_spec(self, spec: TaskSpec) -> QuadChunk:
        """Executes a level-0 "multiply" TaskSpec (the bench seam, reference bench.py:114-120)."""
        if spec.task_type != "multiply":
            raise ConfigurationError(
                f"task type {spec.task_type!r} is outside the B200 hot path (only 'multiply')"
            )
        args = spec.args
        tau = float(args.get("tau", 0.0))
        if args.get("ta"):
            raise ConfigurationError("a transposed left operand is not a level-0 multiply spec")
        a_root, b_root = spec.inputs
        geom: Geometry = args["geometry"]
        stats = spgemm.MultiplyStats()
        self.last_multiply = stats
        if a_root.is_nil or b_root.is_nil or a_root.n_blocks == 0 or b_root.n_blocks == 0:
            self.last_stats = [WorkerStats(0)]
            return NIL  # _multiply_fallback (ops.py:244-245): a nil operand gives nil
        a, b = a_root.require(), b_root.require()
        layout = make_layout(geom.params, geom.bs)
        plain = not (args.get("tb") or args.get("upper") or args.get("a_sym") or args.get("b_sym")
                     or tau > 0.0)
        if self.comm is not None:
            if not plain:
                raise ConfigurationError("multi-GPU products run the regular variant on general operands")
            return self._run_distributed(layout, a, b, a_root is b_root, stats)
        spgemm._require_cuda(a.blocks)
        with torch.cuda.device(a.device):
            plan_filter = None
            if not plain:  # variants: materialise the reference's virtual transposes (variants.py)
                from . import variants  # noqa: PLC0415

                same = a_root is b_root
                a_stored, b_stored = a, b
                if spgemm.support_filter_enabled():  # on the stored sets (kept), carried through
                    a.support_masks()                # the transposes / expansions below
                    b.support_masks()
                virt = variants.virtual_ok(geom.bs)  # transposes as TMA / fragment addressing
                expand = variants.expand_symmetric_view if virt else variants.expand_symmetric
                if args.get("a_sym"):
                    a = expand(geom, a)
                if args.get("b_sym"):
                    b = a if (same and args.get("a_sym")) else expand(geom, b)
                if args.get("tb"):
                    b = (variants.transpose_view if virt else variants.transpose)(geom, b)
                if tau > 0.0:  # approximate: prune decisions on stored-chunk norms (approximate.py)
                    from . import approximate  # noqa: PLC0415

                    b_norms, b_sym = (b, False) if args.get("tb") else (b_stored, bool(args.get("b_sym")))
                    pruner = approximate.Pruner(geom, a_stored, b_norms, tau, a_sym=bool(args.get("a_sym")),
                                                b_sym=b_sym, upper=bool(args.get("upper")))
                    self.last_engine = _EngineInfo(pruner)  # the prune log is computed on first read
                    ax, bx = a, b
                    plan_filter = lambda plan: pruner.filter(plan, ax, bx)  # noqa: E731
            # upper variants: the symbolic phase enumerates only the kept (upper-leaf) C blocks
            c = spgemm.multiply_blocks(layout, a, b, stats=stats, plan_filter=plan_filter,
                                       upper=bool(args.get("upper")))
        self.last_stats = [WorkerStats(0, tasks_executed=stats.n_triples)]
        return self.store.register(c)

    def _run_distributed(self, layout, a, b, same, stats):
        from . import distributed  # noqa: PLC0415

        spgemm._require_cuda(a.blocks)
        c, ds = distributed.multiply(self.comm, layout, a, b, b_is_a=same)
        stats.n_c = c.n
        stats.n_triples = ds.n_triples_global
        stats.flops = 2 * layout.block_size ** 3 * ds.n_triples_global
        mine = torch.tensor([ds.t_range[1] - ds.t_range[0], ds.bytes_received], dtype=torch.int64,
                            device="cpu" if self.comm.stage else a.device)
        allv = [torch.zeros_like(mine) for _ in range(self.comm.world)]
        self.comm.dist.all_gather(allv, mine)
        self.last_stats = [WorkerStats(r, tasks_executed=int(v[0]), bytes_received=int(v[1]))
                           for r, v in enumerate(allv)]
        self.last_distributed = ds
        return self.store.register(c)

    def _distribute(self, bset: BlockSet) -> BlockSet:
        """Keeps this rank's contiguous key range (equal block counts per rank)."""
        if self.comm is None:
            return bset
        n, w, r = bset.n, self.comm.world, self.comm.rank
        lo, hi = (n * r) // w, (n * (r + 1)) // w
        return BlockSet(bset.keys[lo:hi].contiguous(), bset.blocks[lo:hi].contiguous(),
                        bset.sumsq[lo:hi].contiguous())

    def _gathered(self, bset: BlockSet) -> BlockSet:
        """All ranks' parts of a distributed matrix, in key order (inspection only)."""
        if self.comm is None:
            return bset
        k, _ = self.comm.allgather_varlen(bset.keys)
        b, _ = self.comm.allgather_varlen(bset.blocks.reshape(-1))
        s, _ = self.comm.allgather_varlen(bset.sumsq)
        return BlockSet(k, b.reshape(-1, bset.bs, bset.bs), s)

    @property
    def owner_policy(self) -> OwnerPolicy:
        return OwnerPolicy(self.n_workers)

    # -- construction ---------------------------------------------------------------------------

    def _geometry(self, n: int, leaf_dim: int, leaf_kind, block_size: int) -> tuple[Geometry, LeafKind]:
        kind = resolve_leaf_kind(leaf_kind)
        if kind is not LeafKind.BLOCK_SPARSE:
            raise ConfigurationError(
                f"leaf kind {kind.value!r} is outside the B200 path; use 'block_sparse'"
            )
        return Geometry(MatrixParams.create(n, leaf_dim), int(block_size)), kind

    def matrix_from_blocks(self, geom: Geometry, keys: np.ndarray, blocks: np.ndarray,
                           symmetric: bool = False, sumsq: np.ndarray | None = None) -> Matrix:
        """Registers an already-normalised block set (keys ascending, no zero blocks)."""
        bset = self._distribute(BlockSet.from_numpy(keys, blocks, sumsq, self.device))
        root = self.store.register(bset)
        return Matrix(root, geom.params, LeafKind.BLOCK_SPARSE, geom.bs, symmetric)

    def matrix_from_blockset(self, geom: Geometry, bset: BlockSet, symmetric: bool = False) -> Matrix:
        return Matrix(self.store.register(bset), geom.params, LeafKind.BLOCK_SPARSE, geom.bs, symmetric)

    def matrix_from_triplets(self, n: int, rows, cols, vals, leaf_dim: int = 128,
                             leaf_kind=LeafKind.BLOCK_SPARSE, block_size: int = 16,
                             symmetric: bool = False) -> Matrix:
        """session.py:72-104."""
        geom, _ = self._geometry(n, leaf_dim, leaf_kind, block_size)
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.float64)
        if symmetric:
            rows, cols, vals = construct.mirror_symmetric(rows, cols, vals, leaf_dim)
        if self.device.type == "cuda":  # device build (qm_build_*), bit-identical to the host one
            bset = construct.blocks_from_triplets_device(geom, rows, cols, vals, self.device)
            return Matrix(self.store.register(self._distribute(bset)), geom.params,
                          LeafKind.BLOCK_SPARSE, geom.bs, symmetric)
        keys, blocks = construct.blocks_from_triplets(geom, rows, cols, vals)
        return self.matrix_from_blocks(geom, keys, blocks, symmetric)

    def zeros(self, n: int, leaf_dim: int = 128, leaf_kind=LeafKind.BLOCK_SPARSE,
              block_size: int = 16, symmetric: bool = False, explicit: bool = False) -> Matrix:
        """session.py:106-124. ``explicit`` keeps a non-nil root with no stored blocks."""
        geom, kind = self._geometry(n, leaf_dim, leaf_kind, block_size)
        if explicit:
            root = self.store.register(BlockSet.empty(geom.bs, self.device), explicit_zero=True)
        else:
            root = NIL
        return Matrix(root, geom.params, kind, geom.bs, symmetric)

    def identity(self, n: int, c: float = 1.0, leaf_dim: int = 128,
                 leaf_kind=LeafKind.BLOCK_SPARSE, block_size: int = 16,
                 symmetric: bool = False) -> Matrix:
        """session.py:126-137 (c on the logical diagonal)."""
        r, cc, v = construct.identity_triplets(n, c)
        m = self.matrix_from_triplets(n, r, cc, v, leaf_dim, leaf_kind, block_size)
        return Matrix(m.root, m.params, m.leaf_kind, m.block_size, symmetric)

    def assign_from_triplets(self, n, rows, cols, vals, leaf_dim: int = 128,
                             leaf_kind="block_sparse", block_size: int = 16) -> Matrix:
        """session.py:191-198 (the task-built variant of matrix_from_triplets; same result)."""
        return self.matrix_from_triplets(n, rows, cols, vals, leaf_dim, leaf_kind, block_size)

    def load_coordinate(self, path, leaf_dim: int = 128, leaf_kind="block_sparse",
                        block_size: int = 16, symmetric: bool = False) -> Matrix:
        """session.py:139-144 (1-based coordinate text)."""
        n, rows, cols, vals = _read_coordinate_text(path)
        return self.matrix_from_triplets(n, rows, cols, vals, leaf_dim, leaf_kind, block_size, symmetric)

    # -- operations -----------------------------------------------------------------------------

    def multiply(self, a: Matrix, b: Matrix | None = None,
                 variant: MultiplyVariant | str = "regular", tau: float = 0.0) -> Matrix:
        """session.py:160-171."""
        if isinstance(variant, str):
            variant = MultiplyVariant(variant, tau)
        spec, upper = multiply_spec(a, b, variant)
        root = self.run_spec(spec)
        return Matrix(root, a.params, a.leaf_kind, a.block_size, upper)

    def _wrap(self, bset, like: Matrix, symmetric=None) -> Matrix:
        sym = like.symmetric if symmetric is None else symmetric
        return Matrix(self.store.register(bset), like.params, like.leaf_kind, like.block_size, sym)

    def _local_only(self, what: str):
        if self.comm is not None:
            raise ConfigurationError(f"{what} runs on one GPU; multi-GPU sessions only multiply")

    def add(self, a: Matrix, b: Matrix, alpha: float = 1.0, beta: float = 1.0) -> Matrix:
        """session.py:148-150 / ops.add_spec + _add_body/_add_fallback (ops.py:147-169)."""
        from . import algebra  # noqa: PLC0415

        _check_conformant(a, b)
        if a.symmetric != b.symmetric:
            raise ContractViolationError("add needs both operands general or both symmetric")
        self._local_only("add")
        a_nil = a.root.is_nil or a.root.n_blocks == 0
        b_nil = b.root.is_nil or b.root.n_blocks == 0
        if a_nil and b_nil:
            return Matrix(NIL, a.params, a.leaf_kind, a.block_size, a.symmetric)
        if a_nil or b_nil:  # _add_fallback: the survivor, scaled by its coefficient
            survivor, coeff = (b, beta) if a_nil else (a, alpha)
            return self.scale(survivor, coeff)
        return self._wrap(algebra.add(a.geometry, a.root.require(), b.root.require(), float(alpha),
                                      float(beta)), a)

    def scale(self, a: Matrix, alpha: float) -> Matrix:
        """session.py:152-154 / _scale_body (ops.py:172-185): 1.0 shares the chunk, 0.0 is nil."""
        from . import algebra  # noqa: PLC0415

        if alpha == 1.0:
            return a
        if alpha == 0.0 or a.root.is_nil or a.root.n_blocks == 0:
            return Matrix(NIL, a.params, a.leaf_kind, a.block_size, a.symmetric)
        self._local_only("scale")
        return self._wrap(algebra.scale(a.geometry, a.root.require(), float(alpha)), a)

    def add_scaled_identity(self, a: Matrix, c: float) -> Matrix:
        """session.py:156-158 / ops.py:253-345: A + c*I on the logical diagonal."""
        from . import algebra  # noqa: PLC0415

        if c == 0.0:
            return a
        self._local_only("add_scaled_identity")
        if self.device.type != "cuda":
            raise DeviceUnavailableError("add_scaled_identity runs on the CUDA path")
        base = None if (a.root.is_nil or a.root.n_blocks == 0) else a.root.require()
        return self._wrap(algebra.add_scaled_identity(a.geometry, base, float(c), self.device), a)

    def truncate(self, a: Matrix, spec) -> tuple[Matrix, float]:
        """session.py:173-185: global Frobenius truncation; returns (matrix, removed norm)."""
        from . import algebra  # noqa: PLC0415

        if not isinstance(spec, TruncationSpec):
            spec = TruncationSpec(float(spec))
        if a.root.is_nil or a.root.n_blocks == 0 or spec.tau == 0.0:
            return a, 0.0
        self._local_only("truncate")
        out, removed = algebra.truncate(a.geometry, a.root.require(), spec.tau, a.symmetric)
        if out is a.root.blockset:
            return a, 0.0
        return self._wrap(out, a), removed

    # -- inspection -----------------------------------------------------------------------------

    def _host(self, a: Matrix):
        if a.root.is_nil or a.root.blockset is None:
            bs = a.block_size
            return np.zeros(0, np.int64), np.zeros((0, bs, bs)), np.zeros(0)
        return self._gathered(a.root.blockset).to_host()

    @staticmethod
    def _map_symmetric(a: Matrix, rows, cols):
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        if a.symmetric:
            swap = rows > cols
            rows, cols = np.where(swap, cols, rows), np.where(swap, rows, cols)
        return rows, cols

    def get_elements(self, a: Matrix, rows, cols) -> np.ndarray:
        rows, cols = self._map_symmetric(a, rows, cols)
        k, b, _ = self._host(a)
        return bridge.get_elements(a.geometry, k, b, rows, cols)

    extract_elements = get_elements

    def to_dense(self, a: Matrix) -> np.ndarray:
        k, b, _ = self._host(a)
        return bridge.to_dense(a.geometry, k, b, a.symmetric)

    def tree_stats(self, a: Matrix) -> TreeStats:
        k, b, _ = self._host(a)
        if a.root.is_nil:
            return TreeStats()
        return bridge.tree_stats(a.geometry, k, b, a.root.explicit_zero)

    def canonical(self, a: Matrix) -> bytes:
        if a.root.is_nil:
            return b"N"
        k, b, _ = self._host(a)
        return bridge.canonical_bytes(a.geometry, k, b, a.root.explicit_zero)

    def norm(self, a: Matrix) -> float:
        k, _, s = self._host(a)
        return bridge.tree_norm(a.geometry, k, s)

    def write_coordinate(self, a: Matrix, path):
        """quadtree.write_coordinate_text (quadtree.py:348-376)."""
        d = self.to_dense(a)
        rr, cc = np.nonzero(d)
        n = a.params.n_logical
        with open(path, "w") as fh:
            fh.write("% coordinate real general\n")
            fh.write(f"{n} {n} {rr.size}\n")
            for i, j in zip(rr, cc):
                fh.write(f"{i + 1} {j + 1} {float(d[i, j])!r}\n")

    def total_bytes_received(self) -> int:
        if not self.last_stats:
            return 0
        return sum(s.bytes_received for s in self.last_stats)


class _EngineInfo:
    """What the reference's ``session.last_engine`` exposes for the approximate variant:
    ``prune_log`` = bounds of the pruned subproducts (engine.py:156, 273-275). The product itself
    only needs the per-triple survival test (approximate.Pruner.filter); the log -- ~10^5 bounds --
    is computed from the same node tables on first read and kept."""

    def __init__(self, source, pairs_per_level: list | None = None):
        self._source = source  # an approximate.Pruner, or a ready log (list / device tensor)
        self._list = None
        self._pairs = pairs_per_level

    @property
    def prune_log(self) -> list:
        if self._list is None:
            src = self._source
            log = src.result().prune_log if hasattr(src, "result") else src
            self._list = log.tolist() if isinstance(log, torch.Tensor) else list(log)
        return self._list

    @property
    def pairs_per_level(self) -> list:
        if self._pairs is None:
            src = self._source
            self._pairs = src.result().pairs_per_level if hasattr(src, "result") else []
        return self._pairs


def _read_coordinate_text(path):
    """quadtree.read_coordinate_text (quadtree.py:379-402)."""
    rows, cols, vals = [], [], []
    header = None
    with open(path) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("%"):
                continue
            fields = line.split()
            if header is None:
                header = (int(fields[0]), int(fields[1]), int(fields[2]))
                continue
            rows.append(int(fields[0]) - 1)
            cols.append(int(fields[1]) - 1)
            vals.append(float(fields[2]))
    if header is None:
        raise ConfigurationError(f"{path}: no header line found")
    n, m, nnz = header
    if n != m:
        raise ConfigurationError(f"{path}: only square matrices are supported, header says {n} x {m}")
    if len(rows) != nnz:
        raise ConfigurationError(f"{path}: header says {nnz} entries, found {len(rows)}")
    return n, np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64), np.array(vals)
