"""Timeline of one rank's staged step (scaling_projection.py's step): every GPU kernel / copy with
its start and duration (torch.profiler / CUPTI) and the host's top ops, to see where a rank's
time goes between the symbolic phase, the staged numeric phase and compaction.

    python scripts/staged_probe.py [CONFIG] [WORLD] [RANK] [LINK_GBS]
"""
import sys
import time

sys.path.insert(0, ".")
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2011_11762_b200 import _ffi, spgemm
from paper_2011_11762_b200 import distributed as D
from paper_2011_11762_b200 import generators as G

dev = torch.device("cuda:0")
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
r = int(sys.argv[3]) if len(sys.argv) > 3 else 4
link = float(sys.argv[4]) if len(sys.argv) > 4 else 770.0
cfg = G.CONFIGS[name]
geom, a, b = G.config_operands_device(cfg, dev)
b_is_a = cfg.same_operand
if b_is_a:
    b = a
lay = _ffi.make_layout(geom.params, geom.bs)
use = spgemm._use_masks(a, b)
am, bm = (a.masks[1], b.masks[0]) if use else (None, None)
masks = (a.masks[1], b.masks[0], a.masks[2], b.masks[2]) if use else None
a_off = [(a.n * q) // world for q in range(world + 1)]
b_off = a_off if b_is_a else [(b.n * q) // world for q in range(world + 1)]
blk = geom.bs * geom.bs * 8
pa = [a.blocks.data_ptr() + a_off[q] * blk for q in range(world)]
pb = [b.blocks.data_ptr() + b_off[q] * blk for q in range(world)]
marks = {}


def step():
    t = time.perf_counter
    marks["t0"] = t()
    st = spgemm.SymbolicState(lay, a.keys, a.n, b.keys, b.n, None, am, bm, part=(world, r))
    ck, ct = st.keys()
    tri = st.triples(ct)
    marks["sym"] = t()
    info = {}
    c, nz, zc = D.staged_numeric(lay, tri, ct, ck, r, a_off, b_off, pa, pb, a.blocks[a_off[r]:a_off[r + 1]],
                                 b.blocks[b_off[r]:b_off[r + 1]], b_is_a, masks, info=info,
                                 emulate_link_gbs=link if link > 0 else None)
    marks["num"] = t()
    c = spgemm.compact(geom.bs, c, nz, _ffi.read_i64(zc))
    marks["end"] = t()
    return info


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    info = step()
    torch.cuda.synchronize()
print({k: v for k, v in info.items() if not k.startswith("_")})
print("host ms: symbolic %.3f  staged_numeric %.3f  compact %.3f" % (
    1e3 * (marks["sym"] - marks["t0"]), 1e3 * (marks["num"] - marks["sym"]), 1e3 * (marks["end"] - marks["num"])))
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
for e in evs:
    print(f"   {(e.time_range.start - t0) / 1e3:8.3f} ms  {e.time_range.elapsed_us() / 1e3:7.3f} ms  {e.name[:80]}")
print(f"   span {(evs[-1].time_range.end - t0) / 1e3:.3f} ms")
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
# plain timing
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    e0, e1 = E(), E()
    e0.record()
    step()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("step ms", [round(x, 3) for x in ts])

# host-side cost of each call of the step (no profiler): perf_counter around every call, GPU
# synchronised only where the code itself synchronises
def step_timed():
    t = time.perf_counter
    T = [t()]
    st = spgemm.SymbolicState(lay, a.keys, a.n, b.keys, b.n, None, am, bm, part=(world, r))
    T.append(t())
    ck, ct = st.keys()
    T.append(t())
    tri = st.triples(ct)
    T.append(t())
    info = {}
    c, nz, zc = D.staged_numeric(lay, tri, ct, ck, r, a_off, b_off, pa, pb, a.blocks[a_off[r]:a_off[r + 1]],
                                 b.blocks[b_off[r]:b_off[r + 1]], b_is_a, masks, info=info,
                                 emulate_link_gbs=link if link > 0 else None)
    T.append(t())
    n0 = _ffi.read_i64(zc)
    T.append(t())
    c = spgemm.compact(geom.bs, c, nz, n0)
    T.append(t())
    return [1e3 * (y - x) for x, y in zip(T, T[1:])]


rows = []
for _ in range(8):
    torch.cuda.synchronize()
    rows.append(step_timed())
med = [sorted(col)[len(col) // 2] for col in zip(*rows)]
print("host ms per call (median): count_part %.3f keys %.3f triples %.3f staged_numeric %.3f read %.3f compact %.3f"
      % tuple(med))
