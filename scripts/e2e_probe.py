"""Per-step timeline of the pipelined e2e loop (H2D / compute / D2H), to find where time goes."""
import sys, os, time, json
sys.path.insert(0, '.')
import torch, numpy as np
from paper_2011_11762_b200 import MatrixSession
from paper_2011_11762_b200 import generators as G
from paper_2011_11762_b200.blocks import BlockSet
dev = torch.device("cuda:0")
cfg = G.CONFIGS["C2-131072"]
geom, a, b = G.config_operands_device(cfg, dev)
ses = MatrixSession(device=dev)
pin = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t)
hin = [pin(t) for t in (a.keys, a.blocks, a.sumsq, b.keys, b.blocks, b.sumsq)]
din = [[torch.empty_like(t, device=dev) for t in hin] for _ in range(2)]
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
comp = torch.cuda.current_stream()
E = lambda: torch.cuda.Event(enable_timing=True)
c0 = ses.multiply(ses.matrix_from_blockset(geom, a), ses.matrix_from_blockset(geom, b)).root.blockset
hout = [[torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in (c0.keys, c0.blocks, c0.sumsq)] for _ in range(2)]
torch.cuda.synchronize()
steps = 8
ev = {k: [E() for _ in range(steps)] for k in ("h0", "h1", "c0", "c1", "d0", "d1")}
t0 = E(); t0.record(s_in)
used = [None, None]
def h2d(k):
    with torch.cuda.stream(s_in):
        if used[k % 2] is not None: s_in.wait_event(used[k % 2])
        ev["h0"][k].record(s_in)
        for d, h in zip(din[k % 2], hin): d.copy_(h, non_blocking=True)
        ev["h1"][k].record(s_in)
wall = []
h2d(0)
for k in range(steps):
    if k + 1 < steps: h2d(k + 1)
    comp.wait_event(ev["h1"][k])
    ev["c0"][k].record(comp)
    tw = time.perf_counter()
    t = din[k % 2]
    c = ses.multiply(ses.matrix_from_blockset(geom, BlockSet(t[0], t[1], t[2])), ses.matrix_from_blockset(geom, BlockSet(t[3], t[4], t[5]))).root.blockset
    wall.append(time.perf_counter() - tw)
    ev["c1"][k].record(comp)
    used[k % 2] = ev["c1"][k]
    with torch.cuda.stream(s_out):
        s_out.wait_event(ev["c1"][k])
        ev["d0"][k].record(s_out)
        for o, src in zip(hout[k % 2], (c.keys, c.blocks, c.sumsq)): o.copy_(src, non_blocking=True); src.record_stream(s_out)
        ev["d1"][k].record(s_out)
torch.cuda.synchronize()
for k in range(steps):
    f = lambda e: t0.elapsed_time(ev[e][k])
    print(f"step {k}: H2D {f('h0'):7.1f}-{f('h1'):7.1f}  compute {f('c0'):7.1f}-{f('c1'):7.1f} (host wall {wall[k]*1e3:.1f} ms)  D2H {f('d0'):7.1f}-{f('d1'):7.1f}")
