"""Host time of one single-GPU product (spgemm.multiply_blocks) by Python function: cProfile over
200 consecutive C1 products (GPU work is tiny there, so the host path dominates)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_2011_11762_b200 import _ffi, spgemm
from paper_2011_11762_b200 import generators as G

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
dev = torch.device("cuda:0")
cfg = G.CONFIGS[name]
geom, a, b = G.config_operands_device(cfg, dev)
lay = _ffi.make_layout(geom.params, geom.bs)
st = torch.cuda.Stream(dev)
for _ in range(20):
    spgemm.multiply_blocks(lay, a, b, stream=st)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(200):
    spgemm.multiply_blocks(lay, a, b, stream=st)
torch.cuda.synchronize()
print(f"wall per product {1e3 * (time.perf_counter() - t) / 200:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    spgemm.multiply_blocks(lay, a, b, stream=st)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
