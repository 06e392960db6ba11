"""Where the symbolic phase's time goes: host time of each library call vs device time.

    python scripts/symbolic_probe.py [CONFIG ...]
"""
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_2011_11762_b200 import generators as G
from paper_2011_11762_b200 import _ffi, spgemm

dev = torch.device("cuda:0")
E = lambda: torch.cuda.Event(enable_timing=True)
for name in sys.argv[1:] or ["C1", "C3", "C2-131072"]:
    cfg = G.CONFIGS[name]
    geom, a, b = G.config_operands_device(cfg, dev)
    lay = _ffi.make_layout(geom.params, geom.bs)
    if cfg.same_operand:
        b = a
    st = torch.cuda.current_stream()
    rows = []
    for it in range(25):
        torch.cuda.synchronize()
        e = [E() for _ in range(4)]
        h = [time.perf_counter()]
        e[0].record(st)
        s = spgemm.SymbolicState(lay, a.keys, a.n, b.keys, b.n, st)
        h.append(time.perf_counter())
        e[1].record(st)
        ck, ct = s.keys()
        h.append(time.perf_counter())
        e[2].record(st)
        s.triples(ct)
        h.append(time.perf_counter())
        e[3].record(st)
        torch.cuda.synchronize()
        h.append(time.perf_counter())
        if it >= 5:
            rows.append([e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3]),
                         (h[1] - h[0]) * 1e3, (h[2] - h[1]) * 1e3, (h[3] - h[2]) * 1e3,
                         (h[4] - h[0]) * 1e3])
    med = [sorted(c)[len(c) // 2] for c in zip(*rows)]
    print(f"{name}: nA={a.n} nB={b.n} nC={s.n_c} nT={s.n_t}")
    print("  device ms  count %.3f  keys %.3f  triples %.3f" % tuple(med[:3]))
    print("  host   ms  count %.3f  keys %.3f  triples %.3f  total(wall, synced) %.3f" % tuple(med[3:]))

    # whole multiply: host wall per call vs device time of its phases
    ev = {k: E() for k in ("symbolic", "numeric", "end")}
    walls, dev_ms = [], []
    for it in range(25):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0 = E(); e0.record(st)
        spgemm.multiply_blocks(lay, a, b, stream=st, events=ev)
        e1 = E(); e1.record(st)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        if it >= 5:
            walls.append((t1 - t0) * 1e3)
            dev_ms.append([e0.elapsed_time(ev["symbolic"]), ev["symbolic"].elapsed_time(ev["numeric"]),
                           ev["numeric"].elapsed_time(ev["end"]), ev["end"].elapsed_time(e1),
                           e0.elapsed_time(e1)])
    med = [sorted(c)[len(c) // 2] for c in zip(*dev_ms)]
    print("  multiply_blocks: host wall %.3f ms; device: pre %.3f symbolic %.3f numeric %.3f "
          "post %.3f total %.3f" % (sorted(walls)[len(walls) // 2], *med))
    # back-to-back calls (as bench.py times them)
    torch.cuda.synchronize()
    e0 = E(); e0.record(st)
    for it in range(20):
        spgemm.multiply_blocks(lay, a, b, stream=st)
    e1 = E(); e1.record(st)
    torch.cuda.synchronize()
    print("  back-to-back: %.3f ms/call" % (e0.elapsed_time(e1) / 20))
