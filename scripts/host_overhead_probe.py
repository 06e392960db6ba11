"""Host-side cost of one small product (C1): cProfile of back-to-back multiply_blocks calls, and
the host wall per call vs its device time. Small products are host-enqueue-bound, so the host
cost of each library call is device idle time.

    python scripts/host_overhead_probe.py [CONFIG]
"""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_2011_11762_b200 import generators as G
from paper_2011_11762_b200 import _ffi, spgemm

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
dev = torch.device("cuda:0")
cfg = G.CONFIGS[name]
geom, a, b = G.config_operands_device(cfg, dev)
lay = _ffi.make_layout(geom.params, geom.bs)
if cfg.same_operand:
    b = a
st = torch.cuda.current_stream()
for _ in range(20):
    spgemm.multiply_blocks(lay, a, b, stream=st)
torch.cuda.synchronize()
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
n = 200
e0, e1 = E(), E()
t0 = time.perf_counter()
e0.record(st)
for _ in range(n):
    spgemm.multiply_blocks(lay, a, b, stream=st)
e1.record(st)
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"{name}: back-to-back {e0.elapsed_time(e1) / n:.4f} ms/call device, {(t1 - t0) / n * 1e3:.4f} ms/call host")
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    spgemm.multiply_blocks(lay, a, b, stream=st)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
