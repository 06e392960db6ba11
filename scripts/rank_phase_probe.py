"""Where one rank's time goes in a multi-GPU product (C4 decay by default): every kernel of the
rank's partitioned symbolic phase and numeric phase with its device duration (torch.profiler /
CUPTI), the span from the first kernel's start to the last one's end, and the host wall time of the
same calls -- the gaps between kernels are host enqueue / synchronisation time.

    python scripts/rank_phase_probe.py [CONFIG] [WORLD] [RANK ...]
"""
import sys
import time
from collections import defaultdict

sys.path.insert(0, ".")
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2011_11762_b200 import _ffi, spgemm
from paper_2011_11762_b200 import generators as G

dev = torch.device("cuda:0")
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ranks = [int(x) for x in sys.argv[3:]] or [0, 1]
cfg = G.CONFIGS[name]
geom, a, b = G.config_operands_device(cfg, dev)
if cfg.same_operand:
    b = a
lay = _ffi.make_layout(geom.params, geom.bs)
use = spgemm._use_masks(a, b)
am = a.masks[1] if use else None
bm = b.masks[0] if use else None
print(f"{name}: nA={a.n} nB={b.n} nbg={geom.nbg} masks={use}", flush=True)


def run(part):
    s2 = spgemm.SymbolicState(lay, a.keys, a.n, b.keys, b.n, None, am, bm, part=part)
    k2, t2 = s2.keys()
    plan = spgemm.SymbolicPlan(s2.n_c, s2.n_t, k2, t2, s2.triples(t2))
    torch.cuda.synchronize()
    h1 = time.perf_counter()
    spgemm.numeric(lay, a, b, plan)
    return s2, h1


for part in [None] + [(world, r) for r in ranks]:
    for _ in range(3):
        run(part)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        s2, h1 = run(part)
        torch.cuda.synchronize()
        h2 = time.perf_counter()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    agg = defaultdict(lambda: [0, 0.0])
    print(f"--- part={part} nC={s2.n_c} nT={s2.n_t} host symbolic {1e3 * (h1 - h0):.3f} ms, numeric "
          f"{1e3 * (h2 - h1):.3f} ms", flush=True)
    t0 = evs[0].time_range.start if evs else 0
    for e in evs:
        print(f"   {(e.time_range.start - t0) / 1e3:8.3f} ms  {e.time_range.elapsed_us() / 1e3:7.3f} ms  {e.name[:90]}")
        agg[e.name[:60]][0] += 1
        agg[e.name[:60]][1] += e.time_range.elapsed_us()
    if evs:
        span = (evs[-1].time_range.end - t0) / 1e3
        busy = sum(e.time_range.elapsed_us() for e in evs) / 1e3
        print(f"   span {span:.3f} ms, kernels busy {busy:.3f} ms, launches {len(evs)}", flush=True)
