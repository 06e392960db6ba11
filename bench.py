"""Benchmark of the hot path: C = A*B block-sparse quadtree multiply (FP64) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5-64] [--impl ours|reference]

One step = one full product of the configured BASELINE workload (symbolic phase + DMMA numeric
phase + exact-zero compaction) through the drop-in API's multiply path, inputs resident in HBM
(inputs are larger than L2, so no flush is needed between steps). Prints ONE JSON line (rank 0).
Default workload: C5-64 (BASELINE configs[4]: banded N = 2^20, half-bandwidth 1024, bs 64 --
the largest configuration that fits one B200, 70 GB of operands and result); N > 1 runs it
strong-scaled (the same product partitioned over the GPUs).

  metric  leaf-GEMM GFLOP/s (FP64) = executed flops / time: 2*bs^3 per block triple (SURVEY.md
          8(d)), i.e. 2*bs^2*32 per 32-deep k panel; block pairs (and k panels of a pair) whose
          nonzero-column / nonzero-row masks do not meet multiply to exact zeros and are skipped,
          so only the executed ones count (config.triples_structural is the block-level count)
  e2e     the same metric through MatrixSession.multiply with host (pinned) operands: H2D of A
          and B and D2H of C inside the timed region
  roofline  the numeric kernel (dominant) against the measured FP64 tensor peak (a DMMA
          microbenchmark run in-process; MEASURED_PEAKS.json has no FP64 figure)
  cpu_baseline  the numpy oracle port (reference algorithm) on a bounded sample, all host cores

``--impl reference`` times the reference's algorithm on the host CPU (the oracle port: the
reference is pure Python and does not travel to the GPU box) on a bounded sample per step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

DEFAULT_CONFIG = "C5-64"  # the largest single-GPU BASELINE config (configs[4], bs 64)
FP64_NOMINAL_TFLOPS = 37.0  # B200 FP64 tensor datasheet class figure; floor of the roofline peak


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default=DEFAULT_CONFIG)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-target-s", type=float, default=12.0)
    p.add_argument("--scaling", choices=["weak", "strong"], default=None,
                   help="N>1: weak = banded n grows with N (default for C2), strong = fixed n (C5)")
    return p.parse_args()


# ---------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        # nvidia-smi's own start-up (NVML init) must not overlap the timed region
        t0 = time.time()
        while not self.rows and time.time() - t0 < 3.0:
            time.sleep(0.01)

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for nm, v in zip(names, r[3:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def bind_to_gpu_numa(index: int):
    """Restricts this process to the CPUs local to GPU `index` (NVML CPU affinity), so pinned host
    buffers are first-touched on the GPU's NUMA node. Returns the previous affinity (or None)."""
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = {w * 64 + b for w, word in enumerate(words) for b in range(64) if (word >> b) & 1}
        prev = os.sched_getaffinity(0)
        cpus &= prev
        if cpus and cpus != prev:
            os.sched_setaffinity(0, cpus)
            return prev
    except Exception:  # noqa: BLE001 -- best effort (no NVML, containers without affinity rights)
        return None
    return None


# ---------------------------------------------------------------------------------------------
# CPU side: oracle port on a bounded sample
# ---------------------------------------------------------------------------------------------

def cpu_sample(cfg_name: str, target_s: float, threads: int):
    """Builds a bounded sample of the workload for the oracle port: the first R C block rows of
    the product (their A rows and the B rows they touch), R sized by a short probe so one pass
    takes about target_s seconds on `threads` host threads."""
    from oracle import spgemm_oracle as O
    from paper_2011_11762_b200 import generators as G

    cfg = G.CONFIGS[cfg_name]
    geom = cfg.geometry
    pat = G.config_pattern(cfg)
    if cfg.kind == "decay":
        _, (ka, ba), (kb, bb) = G.config_operands_host(cfg)
    else:
        ka, kb = G.config_keys(cfg, 0), G.config_keys(cfg, 1)
        ba = bb = None
    ai, ak = geom.decode(ka)
    bk, _ = geom.decode(kb)
    og = O.Geom(cfg.n, cfg.bs, cfg.bs)

    def sample(rows_hi):
        sel = ai < rows_hi
        ka_s = ka[sel]
        kb_s = kb[np.isin(bk, np.unique(ak[sel]))]
        if ba is None:
            a_s = G.host_blocks(geom, ka_s, cfg.seed, 0, pat, cfg.half_bw)
            b_s = G.host_blocks(geom, kb_s, cfg.seed, 1, pat, cfg.half_bw)
        else:
            a_s = ba[np.searchsorted(ka, ka_s)]
            b_s = bb[np.searchsorted(kb, kb_s)]
        return ka_s, a_s, kb_s, b_s

    def run(s):
        t0 = time.perf_counter()
        _, _, T = O.multiply(og, *[s[0], s[1], s[2], s[3]], threads=threads)
        return time.perf_counter() - t0, T

    probe_rows = max(1, min(geom.nbg // 64, 32))
    s = sample(probe_rows)
    dt, T = run(s)
    rows = int(min(geom.nbg, max(1, probe_rows * target_s / max(dt, 1e-3))))
    s = sample(rows)
    return cfg, s, run, rows


def cpu_baseline(cfg_name: str, target_s: float) -> dict:
    from oracle import spgemm_oracle as O

    threads = O.default_threads()
    cfg, s, run, rows = cpu_sample(cfg_name, target_s, threads)
    dt, T = run(s)
    return {"value": 2.0 * cfg.bs ** 3 * T / dt / 1e9, "unit": "GFLOP/s", "cores": threads,
            "kind": "port",
            "sample": f"{cfg_name}: first {rows} of {cfg.geometry.nbg} C block rows ({T} triples) "
                      f"through oracle/spgemm_oracle.py (reference summation order, numpy/OpenBLAS "
                      f"dgemm per block, {threads} threads), {dt:.2f} s"}


# ---------------------------------------------------------------------------------------------
# FP64 tensor peak (roofline denominator)
# ---------------------------------------------------------------------------------------------

def fp64_peak(lib, torch, dev) -> dict:
    import ctypes

    sink = torch.zeros(1, dtype=torch.float64, device=dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    out = {}
    for kind, name, threads, iters in ((0, "dmma", 256, 40000), (1, "dfma", 256, 200000)):
        flops = ctypes.c_double(0)
        best = 0.0
        for rep in range(4):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            st = torch.cuda.current_stream(dev)
            s.record(st)
            rc = lib.qm_fp64_peak_kernel(kind, sms * 4, threads, iters, sink.data_ptr(),
                                         ctypes.byref(flops), st.cuda_stream)
            e.record(st)
            e.synchronize()
            if rc:
                raise RuntimeError("fp64 peak kernel failed")
            if rep:
                best = max(best, flops.value / (s.elapsed_time(e) * 1e-3) / 1e12)
        out[name] = best
    return out


# ---------------------------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2011_11762_b200 import MatrixSession, _ffi, spgemm
    from paper_2011_11762_b200 import generators as G

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % torch.cuda.device_count()
    prev_affinity = bind_to_gpu_numa(local)  # before any pinned allocation (e2e host buffers)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    backend = os.environ.get("QM_DIST_BACKEND", "nccl")  # gloo: host-staged (tests, 1 GPU)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cdev = dev if backend == "nccl" else torch.device("cpu")  # where timing collectives run
    lib = _ffi.load()
    base = G.CONFIGS[args.config]
    scaling = args.scaling or ("strong" if base.name.startswith("C5") or base.kind != "banded" else "weak")
    cfg = base
    if world > 1 and scaling == "weak":
        if base.kind != "banded":
            raise SystemExit("weak scaling is defined for the banded configs (n grows with the GPU count)")
        cfg = G.BaselineConfig(f"{base.name}-x{world}", "banded", base.n * world, base.bs,
                               half_bw=base.half_bw, seed=base.seed)
    ses = MatrixSession(device=dev)
    stream = torch.cuda.Stream(dev)
    dist_stats = {}

    def barrier():
        if world > 1:
            dist.barrier()

    if world == 1:
        geom, a, b = G.config_operands_device(cfg, dev)
        if cfg.same_operand:
            b = a
        layout = _ffi.make_layout(geom.params, geom.bs)

        def step(stats=None, events=None):
            return spgemm.multiply_blocks(layout, a, b, stream=stream, stats=stats, events=events)
    else:
        from paper_2011_11762_b200 import distributed as D

        geom = cfg.geometry
        layout = _ffi.make_layout(geom.params, geom.bs)
        parts = []
        b_is_a = cfg.same_operand
        if cfg.kind == "decay":  # host-built operand (C = A*A); each rank keeps its key range of A
            from paper_2011_11762_b200.blocks import BlockSet

            _, (ka, ba), _ = G.config_operands_host(cfg)
            lo, hi = (ka.size * rank) // world, (ka.size * (rank + 1)) // world
            parts = [BlockSet.from_numpy(ka[lo:hi], ba[lo:hi], None, dev).compute_meta()] * 2
        else:
            for m in (0, 1):
                keys = G.config_keys(cfg, m)
                lo, hi = (keys.size * rank) // world, (keys.size * (rank + 1)) // world
                parts.append(G.device_blocks(geom, keys[lo:hi], cfg.seed, m, G.config_pattern(cfg),
                                             cfg.half_bw, dev))
        a, b = parts
        comm = D.Comm()
        backend = D.CudaBackend(stream)

        def step(stats=None, events=None):
            if events is not None:
                events["symbolic"].record(stream)
            c, ds = D.multiply(comm, layout, a, b, backend=backend, b_is_a=b_is_a)
            if events is not None:
                events["numeric"].record(stream)
                events["end"].record(stream)
            if stats is not None:
                stats.n_triples = ds.n_triples_global
                stats.n_c = ds.n_c_global
                # executed flops: 2*bs^2 per executed k row summed over the ranks (as on one GPU,
                # where k panels skipped by the support masks are not counted)
                kr = torch.tensor([float(ds.k_rows)], dtype=torch.float64, device=cdev)
                dist.all_reduce(kr, op=dist.ReduceOp.MIN)
                if kr.item() >= 0:
                    kr = torch.tensor([float(ds.k_rows)], dtype=torch.float64, device=cdev)
                    dist.all_reduce(kr)
                    stats.flops = 2 * geom.bs ** 2 * int(kr.item())
                else:
                    stats.flops = 2 * geom.bs ** 3 * ds.n_triples_global
                dist_stats["last"] = ds
            return c

    if world == 1:
        a._bench_layout = layout  # (for the row-index timing of operand_meta_timing)
    meta = operand_meta_timing(lib, torch, a, stream) if world == 1 else None
    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 0)):
            step()
        torch.cuda.synchronize()
        stats = spgemm.MultiplyStats()
        step(stats=stats)
        torch.cuda.synchronize()
        evs = [{k: torch.cuda.Event(enable_timing=True) for k in ("symbolic", "numeric", "end", "done")}
               for _ in range(args.steps)]
        t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # Working sets that fit in L2 (C1) would be timed warm: flush L2 between the timed steps
        # (a write of twice the L2 size, outside each step's own events) and sum the step times.
        l2_bytes = int(getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 126 << 20))
        work_bytes = 8 * geom.bs ** 2 * (a.n + b.n + stats.n_c)
        flush = world == 1 and work_bytes < 2 * l2_bytes
        scratch = torch.empty(2 * l2_bytes // 4, dtype=torch.int32, device=dev) if flush else None
        clocks = ClockSampler(local)
        barrier()
        torch.cuda.synchronize()
        clocks.start()
        l0 = lib.qm_launch_count()
        t_start.record(stream)
        for k in range(args.steps):
            if flush:
                scratch.fill_(k)
            c = step(events=evs[k])
            evs[k]["done"].record(stream)
            del c
        t_end.record(stream)
        torch.cuda.synchronize()
        launches = lib.qm_launch_count() - l0
        clock = clocks.stop()
        barrier()
    if flush:
        total_ms = sum(e["symbolic"].elapsed_time(e["done"]) for e in evs)
    else:
        total_ms = t_start.elapsed_time(t_end)
    numeric_ms = [e["numeric"].elapsed_time(e["end"]) for e in evs]
    symbolic_ms = [e["symbolic"].elapsed_time(e["numeric"]) for e in evs]
    if world > 1:
        t = torch.tensor([total_ms], device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    flops = stats.flops
    value = flops * args.steps / (total_ms * 1e-3) / 1e9  # global flops of the product / max time
    ms_per_step = total_ms / args.steps
    nk_ms = statistics.mean(numeric_ms)
    bs = geom.bs
    alg_bytes = 8 * bs * bs * (a.n + b.n + stats.n_c) + 8 * (a.n + b.n + stats.n_c) + 8 * stats.n_triples
    # the kernel the library selects for this product (bs 16 groups / bs 32 quads of C blocks for long
    # k lists, the per-block kernels otherwise; multi-GPU products use the pooled per-block kernel)
    masked = int(spgemm._use_masks(a, b)) if world == 1 else 0
    numeric_kernel = "k_numeric_tma"
    if world == 1:
        import ctypes

        lay = _ffi.make_layout(geom.params, geom.bs)
        numeric_kernel = lib.qm_numeric_kernel(ctypes.byref(lay), stats.n_c_symbolic, stats.n_triples, masked,
                                               0).decode()
    traffic, traffic_note = committed_traffic(cfg.name, numeric_kernel)
    peaks = fp64_peak(lib, torch, dev)
    peak = max(peaks["dmma"], peaks["dfma"], FP64_NOMINAL_TFLOPS)
    if world > 1:  # the events bracket the whole distributed step; per-GPU share of the flops
        nk_ms = statistics.mean(symbolic_ms)
        achieved = flops / world / (nk_ms * 1e-3) / 1e12
    else:
        achieved = flops / (nk_ms * 1e-3) / 1e12
    counts = structural_counts(geom, a, b, world, cfg)
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "GFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: block-keyed uniform[-1,1] values (numpy PCG64 streams, generated on device)",
        "config": workload_config(cfg, counts, world),
        "result": {"nnzb_c": stats.n_c, "triples_executed": stats.n_triples, "zero_blocks": stats.zero_blocks,
                   "note": "triples_executed = block pairs whose nonzero-column / nonzero-row masks meet "
                           "(the others multiply to exact zeros and are skipped); the metric counts "
                           "executed flops (2*bs^2 per executed k row)"},
        "l2": (f"working set {work_bytes / 1e6:.0f} MB < 2x L2: L2 flushed between timed steps (a "
               f"{2 * l2_bytes >> 20} MiB write outside each step's events)" if flush
               else "inputs larger than L2 (no flush)"),
        "phases_ms": {"symbolic": round(statistics.mean(symbolic_ms), 4), "numeric": round(nk_ms, 4)},
        "roofline": {"bound": "tensor", "kernel": numeric_kernel, "achieved": round(achieved, 3),
                     "peak": round(peak, 3), "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
                     "peak_source": f"max(measured DMMA {peaks['dmma']:.2f}, measured DFMA "
                                    f"{peaks['dfma']:.2f}, nominal {FP64_NOMINAL_TFLOPS}) TFLOP/s; "
                                    "MEASURED_PEAKS.json has no FP64 figure",
                     "algorithmic_bytes": alg_bytes,
                     "hbm_gbs_at_alg_bytes": round(alg_bytes / (nk_ms * 1e-3) / 1e9, 1),
                     "traffic": traffic,
                     "traffic_note": traffic_note},
        "clocks": clock,
        "gpu_launches": int(launches),
        "launches_per_step": round(launches / args.steps, 2),
    }
    if meta is not None:
        line["operand_metadata"] = meta
    if world > 1:
        ds = dist_stats["last"]
        v = torch.tensor([ds.bytes_received, ds.t_range[1] - ds.t_range[0], ds.n_c_local],
                         dtype=torch.float64, device=cdev)
        allv = [torch.zeros_like(v) for _ in range(world)]
        dist.all_gather(allv, v)
        m = torch.stack(allv).cpu().numpy()
        line["distributed"] = {
            "bytes_received_per_gpu": {"min": int(m[:, 0].min()), "mean": float(m[:, 0].mean()),
                                       "max": int(m[:, 0].max())},
            "triples_per_gpu": {"min": int(m[:, 1].min()), "max": int(m[:, 1].max())},
            "phases_s_rank0": {k: round(x, 5) for k, x in ds.phase_s.items()},
            "mode": ds.mode,  # fused (TMA reads of peer pools) / staged (halo gather) / exchange (NCCL)
            "rank0": {k: v for k, v in ds.extra.items() if isinstance(v, (int, float))},
        }
        line["roofline"]["note"] = ("multi-GPU: 'numeric' phase = the whole distributed step "
                                    "(structure gather + symbolic + exchange + numeric)")
    if not args.no_e2e and world == 1:
        host = HostOperands(torch, a, None if cfg.same_operand else b)
        step = None  # noqa: F841 -- the timed loop's closure held the device operands
        a = b = None  # the e2e loop double-buffers its own device copies (C5: 2 x 35 GB + 2 x 35 GB of C)
        torch.cuda.empty_cache()
        try:
            line["e2e"] = run_e2e(args, torch, ses, geom, host, dev)
        except (RuntimeError, MemoryError) as e:  # e.g. a host that cannot pin the operands: keep the line
            line["e2e"] = {"value": None, "unit": "GFLOP/s", "error": f"{type(e).__name__}: {str(e)[:300]}"}
        else:
            try:
                line["e2e"]["pcie"] = pcie_floor(torch, dev, line["e2e"])
            except (RuntimeError, MemoryError) as e:
                line["e2e"]["pcie"] = {"error": f"{type(e).__name__}: {str(e)[:300]}"}
        del host
    elif not args.no_e2e:
        line["e2e"] = run_e2e_distributed(args, torch, geom, a, b, dev, world, dist, cdev)
    if prev_affinity is not None:
        line.setdefault("e2e", {})["numa_bound"] = True
        os.sched_setaffinity(0, prev_affinity)  # the CPU baseline uses every host core
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args.config, args.cpu_target_s)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        from paper_2011_11762_b200 import distributed as D

        D.release_peer_mappings()
        dist.barrier()
        dist.destroy_process_group()


METRIC = "block-sparse multiply leaf-GEMM GFLOP/s (FP64)"


def workload_config(cfg, counts: dict, world: int) -> dict:
    """The workload definition both arms print (identical dicts): the BASELINE configuration and
    its block-level structure (structural counts: every block pair with a matching k)."""
    return {"workload": cfg.name, "kind": cfg.kind, "n": cfg.n, "block_size": cfg.bs,
            "half_bandwidth": cfg.half_bw, "leaf_dim": cfg.bs, **counts,
            "parallelism": f"keyrange-partition dp{world}" if world > 1 else "single"}


def structural_counts(geom, a, b, world, cfg) -> dict:
    """Block-level structure of the product measured on the device (the symbolic phase without the
    exact-zero filter); the reference arm computes the same numbers on the host
    (generators.structure_counts) -- equal by construction, tested."""
    if world > 1:
        from paper_2011_11762_b200 import generators as G

        return G.structure_counts(cfg)
    from paper_2011_11762_b200 import _ffi, spgemm

    st = spgemm.SymbolicState(_ffi.make_layout(geom.params, geom.bs), a.keys, a.n, b.keys, b.n)
    return {"nnzb_a": a.n, "nnzb_b": b.n, "nnzb_c_structural": st.n_c, "triples_structural": st.n_t}


KERNEL_SOURCES = {
    "k_numeric_tma": ("csrc/qm_numeric_tma.cu", "csrc/qm_tma.cuh", "csrc/qm_common.cuh"),
    "k_numeric_quad32": ("csrc/qm_numeric_quad.cu", "csrc/qm_tma.cuh", "csrc/qm_common.cuh"),
    "k_numeric_group16": ("csrc/qm_numeric_group.cu", "csrc/qm_tma.cuh", "csrc/qm_common.cuh"),
}


def kernel_source_sha(kernel: str = "k_numeric_tma") -> str:
    """sha256 (16 hex) of a numeric kernel's sources: a committed ncu traffic figure is used only
    for the kernel it was captured on."""
    import hashlib

    h = hashlib.sha256()
    for rel in KERNEL_SOURCES[kernel]:
        h.update((ROOT / "paper_2011_11762_b200" / rel).read_bytes())
    return h.hexdigest()[:16]


def committed_traffic(workload: str, kernel: str = "k_numeric_tma"):
    """DRAM read+write bytes of one launch of the workload's numeric kernel from the committed ncu
    capture (profiles/ncu_traffic.json), or None when there is none for this kernel and source."""
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    entry = json.loads(tfile.read_text()).get(workload, {}) if tfile.exists() else {}
    if not entry:
        return None, f"no committed ncu capture for {workload}"
    if entry.get("kernel", "k_numeric_tma") != kernel or kernel not in KERNEL_SOURCES:
        return None, (f"the committed ncu capture for {workload} is of {entry.get('kernel', 'k_numeric_tma')}, "
                      f"not {kernel}: not used")
    sha = kernel_source_sha(kernel)
    if entry.get("kernel_src_sha") != sha:
        return None, (f"committed ncu capture for {workload} is of kernel source "
                      f"{entry.get('kernel_src_sha')}, not the current {sha}: not used")
    return entry["traffic_bytes"], (f"dram__bytes_read.sum + dram__bytes_write.sum of one {kernel} "
                                    f"launch, ncu capture {entry.get('capture')} (kernel source {sha}; "
                                    "profiles/ncu_traffic.json)")


def operand_meta_timing(lib, torch, a, stream) -> dict:
    """Operand metadata (norms, support masks, NaN/Inf flags) is computed by the producer of a
    block set, in the same pass that writes or first reads it (qm_generate_blocks + qm_block_meta,
    qm_build_fill_meta): the reference likewise stores each leaf's block norms with the leaf. It is
    not part of a product step; this times that one pass over A once, for the record."""
    from paper_2011_11762_b200 import _ffi

    n = a.n
    m = torch.empty((3, n), dtype=torch.int64, device=a.device)
    sq = torch.empty(n, dtype=torch.float64, device=a.device)
    nf = torch.zeros(2, dtype=torch.int64, device=a.device)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    best = float("inf")
    for _ in range(3):
        torch.cuda.synchronize()
        ev[0].record(stream)
        _ffi.check(lib.qm_block_meta(a.bs, n, _ffi.ptr(a.blocks), _ffi.ptr(sq), 0, 0, _ffi.ptr(m), _ffi.ptr(nf),
                                     _ffi.stream_handle(stream)), "qm_block_meta")
        ev[1].record(stream)
        torch.cuda.synchronize()
        best = min(best, ev[0].elapsed_time(ev[1]))
    nbytes = a.blocks.numel() * 8 + n * (8 + 24)
    # the row index (the operand's row-sorted view the symbolic phase reads) is metadata too: built
    # on the block set's first use as a factor and kept with it; timed here once, for the record
    from paper_2011_11762_b200 import spgemm  # noqa: PLC0415
    from paper_2011_11762_b200.blocks import BlockSet  # noqa: PLC0415

    ix_ms = None
    if spgemm.row_index_enabled():
        geom_lay = getattr(a, "_bench_layout", None)
        if geom_lay is not None:
            tmp = BlockSet(a.keys, a.blocks, a.sumsq, a.masks, a.masks_full)
            tb = float("inf")
            for _ in range(3):
                tmp.__dict__.pop("_row_index", None)
                torch.cuda.synchronize()
                ev[0].record(stream)
                tmp.row_index(geom_lay, stream)
                ev[1].record(stream)
                torch.cuda.synchronize()
                tb = min(tb, ev[0].elapsed_time(ev[1]))
            ix_ms = round(tb, 4)
    return {"where": "computed once by the operands' producer (device generator -> qm_block_meta; "
                     "qm_build_fill_meta for matrix_from_triplets), not inside the product step; "
                     "the e2e step copies it with the blocks",
            "kernel": "k_block_meta", "ms_per_operand": round(best, 4),
            "gbs": round(nbytes / (best * 1e-3) / 1e9, 1),
            "row_index": {"where": "built on the operand's first use as a factor (qm_row_index_build: the "
                                   "row-sorted view the symbolic phase reads), kept with the block set; the "
                                   "e2e step's fresh operands build it inside the step",
                          "ms_per_operand": ix_ms}}


class HostOperands:
    """Pinned host copies of the operands (keys, blocks, norms, support masks) for the e2e loop."""

    def __init__(self, torch, a, b):
        def pinned(t):
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t)
            return h

        self.same = b is None
        self.sets = [a] if b is None else [a, b]
        self.tensors = []
        self.full = []
        for x in self.sets:
            x.support_masks()
            self.tensors.append([pinned(t) for t in (x.keys, x.blocks, x.sumsq, x.masks)])
            self.full.append(x.masks_full)
        self.sets = None
        self.nbytes = sum(t.numel() * t.element_size() for ts in self.tensors for t in ts)


def run_e2e(args, torch, ses, geom, host: HostOperands, dev, timeline: dict | None = None):
    """MatrixSession.multiply with host (pinned) operands, as a pipelined serving loop: every step
    copies its operands host->device (keys, blocks, norms and support masks -- the stored matrix)
    and its result C device->host, on dedicated copy streams with double-buffered device inputs, so
    step k's D2H, step k+1's H2D and step k's product overlap (PCIe is full duplex). Timed with
    CUDA events from the first H2D to the last D2H. Device memory: two input slots plus at most two
    results alive (the product of step k and the result of step k-1 still being copied out); the
    host frees the result of step k-2 only once its D2H has completed (it has long finished by then
    in a PCIe-bound pipeline), so C5-64's 4 x 35 GB fit in HBM with no allocator stall. One pinned
    host result buffer (the host never reads it: D2H copies are stream-ordered)."""
    from paper_2011_11762_b200.blocks import BlockSet

    nset = len(host.tensors)
    h2d = host.nbytes
    dev_in = [[[torch.empty_like(t, device=dev) for t in ts] for ts in host.tensors] for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    compute = torch.cuda.current_stream(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    h2d_done = [ev(), ev()]
    used = [None, None]
    out_host = {}
    live = []  # (result, its D2H-done event)

    def mark(name, stream):  # optional per-step timeline (scripts/e2e_c5_probe.py)
        if timeline is not None:
            e = ev()
            e.record(stream)
            timeline.setdefault(name, []).append((e, time.perf_counter()))

    def issue_h2d(k):
        slot = k % 2
        with torch.cuda.stream(s_in):
            if used[slot] is not None:
                s_in.wait_event(used[slot])  # the product of step k-2 has finished reading this slot
            mark("h2d_start", s_in)
            for dts, hts in zip(dev_in[slot], host.tensors):
                for d, h in zip(dts, hts):
                    d.copy_(h, non_blocking=True)
            h2d_done[slot].record(s_in)
            mark("h2d_end", s_in)

    def operand(slot, i):
        k, blk, sq, m = dev_in[slot][i]
        return BlockSet(k, blk, sq, masks=m, masks_full=host.full[i])

    def step(k):
        slot = k % 2
        # The result of step k-2 is released only once its D2H has completed (host-side event wait;
        # it finished long ago in a PCIe-bound pipeline), so its memory is reusable by this step's
        # product at once. (record_stream on the copy stream would instead defer the reuse until
        # everything queued there -- the D2H of step k-1 too -- had drained: the allocator would
        # then fall back to a fresh 35 GB cudaMalloc and a device-wide synchronisation.)
        while len(live) > 1:
            old, done_ev = live.pop(0)
            done_ev.synchronize()
            del old
        compute.wait_event(h2d_done[slot])
        mark("product_start", compute)
        da = operand(slot, 0)
        db = da if nset == 1 else operand(slot, 1)
        c = ses.multiply(ses.matrix_from_blockset(geom, da), ses.matrix_from_blockset(geom, db))
        done = ev()
        done.record(compute)
        mark("product_end", compute)
        used[slot] = done
        cs = c.root.blockset
        parts = (("k", cs.keys), ("b", cs.blocks), ("s", cs.sumsq))
        for name, src in parts:
            if name not in out_host or out_host[name].numel() < src.numel():
                out_host[name] = torch.empty(src.numel(), dtype=src.dtype, pin_memory=True)
        d2h_ev = ev()
        with torch.cuda.stream(s_out):
            s_out.wait_event(done)
            mark("d2h_start", s_out)
            for name, src in parts:
                out_host[name][:src.numel()].copy_(src.reshape(-1), non_blocking=True)
            d2h_ev.record(s_out)
            mark("d2h_end", s_out)
        live.append((c, d2h_ev))
        return sum(t.numel() * t.element_size() for _, t in parts)

    # the same K as the device-timed loop (a serving loop of K products: the pipeline's fill and
    # drain -- one product and one D2H not overlapped with copies -- are amortised over K steps)
    steps = max(3, min(args.steps, 50))
    issue_h2d(0)
    step(0)  # warm-up (allocations, pinned output buffers)
    torch.cuda.synchronize()
    used[0] = used[1] = None
    live.clear()
    torch.cuda.synchronize()
    if timeline is not None:
        timeline.clear()
    start, end = ev(), ev()
    start.record(s_in)
    if timeline is not None:
        timeline["t0"] = (start, time.perf_counter())
    issue_h2d(0)
    d2h = 0
    for k in range(steps):
        if k + 1 < steps:
            issue_h2d(k + 1)
        d2h = step(k)
    end.record(s_out)
    torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    flops = ses.last_multiply.flops
    live.clear()
    # the box's pinned-copy bandwidth at the e2e's own transfer size (one operand's blocks tensor
    # each way and both at once; large copies run slower than 1 GiB ones here)
    big = host.tensors[0][1]
    d_a, d_b = dev_in[0][0][1], dev_in[1][0][1]
    h_o = out_host["b"][:big.numel()].view(big.shape)
    bw = {}
    for mode in ("h2d", "d2h", "both"):
        torch.cuda.synchronize()
        e0, e1, e2 = ev(), ev(), ev()
        e0.record(s_in)
        s_out.wait_event(e0)
        if mode != "d2h":
            with torch.cuda.stream(s_in):
                d_a.copy_(big, non_blocking=True)
        if mode != "h2d":
            with torch.cuda.stream(s_out):
                h_o.copy_(d_b, non_blocking=True)
        e2.record(s_out)
        s_in.wait_event(e2)
        e1.record(s_in)
        torch.cuda.synchronize()
        nbytes = big.numel() * 8 * (2 if mode == "both" else 1)
        bw[f"{mode}_gbs"] = round(nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
    del dev_in
    return {"value": round(flops * steps / (ms * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": steps,
            "ms_per_step": round(ms / steps, 3), "api": "MatrixSession.multiply",
            "pipelining": "H2D(k+1) | product(k) | D2H(k) on separate streams, double-buffered inputs",
            "h2d_contents": "keys, blocks, norms and support masks of A and B (the stored matrices)",
            "pcie_at_transfer_size": {**bw, "bytes_per_copy": int(big.numel() * 8),
                                      "floor_ms_per_step": round((h2d + d2h) / (bw["both_gbs"] * 1e9) * 1e3, 3),
                                      "frac_of_floor": round((h2d + d2h) / (bw["both_gbs"] * 1e9) * 1e3 / (ms / steps), 3)}}


def pcie_floor(torch, dev, e2e, mib=1024):
    """Pinned copy bandwidth of this box measured right after the e2e run (outside its timed
    region): H2D alone, D2H alone, both directions at once. The e2e step moves its H2D and D2H
    bytes concurrently, so its floor is (h2d + d2h bytes) / bidirectional bandwidth."""
    n = mib * 2**20 // 8
    h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d_in = torch.empty(n, dtype=torch.float64, device=dev)
    d_out = torch.empty(n, dtype=torch.float64, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def timed(h2d, d2h):
        best = float("inf")
        for _ in range(3):
            torch.cuda.synchronize(dev)
            e = [ev(), ev(), ev(), ev()]
            e[0].record(s1)
            s2.wait_event(e[0])
            if h2d:
                with torch.cuda.stream(s1):
                    d_in.copy_(h_in, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    h_out.copy_(d_out, non_blocking=True)
            e[1].record(s1)
            e[2].record(s2)
            s1.wait_event(e[2])
            e[3].record(s1)
            torch.cuda.synchronize(dev)
            best = min(best, e[0].elapsed_time(e[3]))
        return (h2d + d2h) * n * 8 / (best * 1e-3) / 1e9

    bw = {"h2d_gbs": round(timed(1, 0), 1), "d2h_gbs": round(timed(0, 1), 1),
          "bidir_gbs": round(timed(1, 1), 1)}
    floor = (e2e["h2d_bytes_per_step"] + e2e["d2h_bytes_per_step"]) / (bw["bidir_gbs"] * 1e9) * 1e3
    bw["floor_ms_per_step"] = round(floor, 3)
    bw["frac_of_floor"] = round(floor / e2e["ms_per_step"], 3)
    bw["note"] = f"{mib} MiB pinned buffers, best of 3, measured after the e2e loop"
    del h_in, h_out, d_in, d_out
    return bw


def run_e2e_distributed(args, torch, geom, a, b, dev, world, dist, cdev):
    """N > 1: MatrixSession(n_workers=N).multiply on each rank's host-resident key range of A and
    B (pinned H2D inside the timed region), the distributed product, D2H of the rank's C range."""
    from paper_2011_11762_b200 import MatrixSession
    from paper_2011_11762_b200.blocks import BlockSet

    ses = MatrixSession(n_workers=world, device=dev)
    pin = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t)  # noqa: E731
    ha = [pin(t) for t in (a.keys, a.blocks, a.sumsq)]
    hb = [pin(t) for t in (b.keys, b.blocks, b.sumsq)]
    h2d = sum(t.numel() * t.element_size() for t in ha + hb)

    def step():
        da = BlockSet(*[t.to(dev, non_blocking=True) for t in ha])
        db = BlockSet(*[t.to(dev, non_blocking=True) for t in hb])
        c = ses.multiply(ses.matrix_from_blockset(geom, da), ses.matrix_from_blockset(geom, db))
        cs = c.root.blockset if not c.root.is_nil else BlockSet.empty(geom.bs, dev)
        outs = [t.to("cpu", non_blocking=True) for t in (cs.keys, cs.blocks, cs.sumsq)]
        return sum(t.numel() * t.element_size() for t in outs)

    steps = max(1, min(args.steps, 3))
    step()
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    d2h = 0
    for _ in range(steps):
        d2h = step()
    e.record()
    torch.cuda.synchronize()
    t = torch.tensor([s.elapsed_time(e)], device=cdev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    flops = ses.last_multiply.flops
    return {"value": round(flops * steps / (ms * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": steps,
            "ms_per_step": round(ms / steps, 3), "api": "MatrixSession(n_workers=N).multiply",
            "note": "per-rank bytes (rank 0); each rank copies its own key range in and its C range out"}


# ---------------------------------------------------------------------------------------------
# reference arm (host CPU, oracle port)
# ---------------------------------------------------------------------------------------------

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle import spgemm_oracle as O

    threads = O.default_threads()
    target = max(1.0, min(args.cpu_target_s, 100.0 / max(1, args.steps + args.warmup)))  # whole run ~3 min
    cfg, s, run, rows = cpu_sample(args.config, target, threads)
    for _ in range(max(args.warmup, 0)):
        run(s)
    times = []
    T = 0
    for _ in range(args.steps):
        dt, T = run(s)
        times.append(dt)
    tot = sum(times)
    value = 2.0 * cfg.bs ** 3 * T * args.steps / tot / 1e9
    sample = (f"{cfg.name}: first {rows} of {cfg.geometry.nbg} C block rows ({T} triples) per step; "
              f"oracle/spgemm_oracle.py = the reference's algorithm and summation order on numpy/"
              f"OpenBLAS dgemm, {threads} host threads")
    from paper_2011_11762_b200 import generators as G

    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(tot / args.steps * 1e3, 2),
        "higher_is_better": True,
        "scaling": "strong" if cfg.name.startswith("C5") or cfg.kind != "banded" else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: block-keyed uniform[-1,1] values (numpy PCG64 streams)",
        "config": workload_config(cfg, G.structure_counts(cfg), world),
        "sampling": {"c_block_rows": rows, "of": cfg.geometry.nbg, "triples_per_step": T,
                     "note": "each step multiplies a bounded sample of the workload (its first C block "
                             "rows, complete); the value is the sample's leaf-GEMM rate"},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
