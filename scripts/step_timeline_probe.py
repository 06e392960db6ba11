"""CUPTI timeline of consecutive single-GPU products (spgemm.multiply_blocks) of one config: every
kernel's start / duration, so the GPU idle time between phases (host enqueue, count read-back) is
visible. python scripts/step_timeline_probe.py [CONFIG]"""
import sys

sys.path.insert(0, ".")
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2011_11762_b200 import _ffi, spgemm
from paper_2011_11762_b200 import generators as G

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
dev = torch.device("cuda:0")
cfg = G.CONFIGS[name]
geom, a, b = G.config_operands_device(cfg, dev)
if cfg.same_operand:
    b = a
lay = _ffi.make_layout(geom.params, geom.bs)
st = torch.cuda.Stream(dev)
for _ in range(3):
    spgemm.multiply_blocks(lay, a, b, stream=st)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        spgemm.multiply_blocks(lay, a, b, stream=st)
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
             key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev_end = t0
busy = 0.0
for e in evs:
    gap = (e.time_range.start - prev_end) / 1e3
    print(f"{(e.time_range.start - t0) / 1e3:8.3f} ms  gap {gap:6.3f}  dur {e.time_range.elapsed_us() / 1e3:7.3f}  {e.name[:70]}")
    prev_end = max(prev_end, e.time_range.end)
    busy += e.time_range.elapsed_us() / 1e3
print(f"span {(prev_end - t0) / 1e3:.3f} ms for 2 products, kernels busy {busy:.3f} ms")
