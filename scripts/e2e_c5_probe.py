"""Per-step timeline of bench.py's pipelined e2e loop on C5-64 (H2D / product / D2H events plus
host enqueue times), and the pinned-copy bandwidth for transfers of the e2e's own sizes."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2011_11762_b200 import MatrixSession  # noqa: E402
from paper_2011_11762_b200 import generators as G  # noqa: E402

cfg = G.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5-64"]
dev = torch.device("cuda:0")
bench.bind_to_gpu_numa(0)
geom, a, b = G.config_operands_device(cfg, dev)
host = bench.HostOperands(torch, a, b)
a = b = None
torch.cuda.empty_cache()
ses = MatrixSession(device=dev)


class A:
    steps = 6


tl = {}
out = bench.run_e2e(A, torch, ses, geom, host, dev, timeline=tl)
t0e, t0h = tl.pop("t0")
rows = []
for k in range(A.steps):
    r = {}
    for name, lst in tl.items():
        if k < len(lst):
            e, h = lst[k]
            r[name] = round(t0e.elapsed_time(e), 1)
            r[name + "_host"] = round((h - t0h) * 1e3, 1)
    rows.append(r)
    print(json.dumps(r))
print(json.dumps(out))
# copy bandwidth at the e2e's transfer sizes (one 17.7 GB blocks tensor each way, and both at once)
hb = host.tensors[0][1]
db = torch.empty_like(hb, device=dev)
ho = torch.empty_like(hb, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
res = {}
for mode in ("h2d", "d2h", "both"):
    torch.cuda.synchronize()
    e0, e1, e2 = E(), E(), E()
    e0.record(s1)
    s2.wait_event(e0)
    if mode in ("h2d", "both"):
        with torch.cuda.stream(s1):
            db.copy_(hb, non_blocking=True)
    if mode in ("d2h", "both"):
        with torch.cuda.stream(s2):
            ho.copy_(db, non_blocking=True)
    e2.record(s2)
    s1.wait_event(e2)
    e1.record(s1)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    nbytes = hb.numel() * 8 * (2 if mode == "both" else 1)
    res[mode] = {"ms": round(ms, 1), "gbs": round(nbytes / ms / 1e6, 1)}
print(json.dumps({"big_copies": res, "bytes_each": hb.numel() * 8}))
