"""Phase timing of the partitioned symbolic phase for one simulated rank (CUDA events around each
library call, after a warm-up), next to the global symbolic phase of the same product.

    python scripts/partition_probe.py [config] [world] [rank]
"""
import json
import sys

sys.path.insert(0, ".")
import torch

from paper_2011_11762_b200 import _ffi, spgemm
from paper_2011_11762_b200 import generators as G

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rank = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dev = torch.device("cuda:0")
base = G.CONFIGS[name]
cfg = base if world == 1 or base.kind != "banded" or name.startswith("C5") else \
    G.BaselineConfig(f"{name}-x{world}", "banded", base.n * world, base.bs, half_bw=base.half_bw)
geom, a, b = G.config_operands_device(cfg, dev)
if cfg.same_operand:
    b = a
lay = _ffi.make_layout(geom.params, geom.bs)
use = spgemm._use_masks(a, b)
am, bm = (a.masks[1], b.masks[0]) if use else (None, None)
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def run(part):
    ev = [E() for _ in range(4)]
    torch.cuda.synchronize()
    ev[0].record()
    st = spgemm.SymbolicState(lay, a.keys, a.n, b.keys, b.n, None, am, bm, part=part)
    ev[1].record()
    ck, ct = st.keys()
    ev[2].record()
    st.triples(ct)
    ev[3].record()
    torch.cuda.synchronize()
    return {"count_ms": ev[0].elapsed_time(ev[1]), "keys_ms": ev[1].elapsed_time(ev[2]),
            "triples_ms": ev[2].elapsed_time(ev[3]), "n_c": st.n_c, "n_t": st.n_t}


for part in (None, (world, rank)):
    run(part)
    r = min((run(part) for _ in range(5)), key=lambda x: x["count_ms"] + x["keys_ms"] + x["triples_ms"])
    print(json.dumps({"config": cfg.name, "part": part, **{k: round(v, 4) if isinstance(v, float) else v
                                                        for k, v in r.items()}}), flush=True)
