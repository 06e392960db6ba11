"""Device time of the symbolic phase on the GLOBAL structure of the weak-scaling bench at N GPUs
(every rank runs count + C keys globally, then emits only its own triple range)."""
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_2011_11762_b200 import _ffi, spgemm
from paper_2011_11762_b200 import generators as G

dev = torch.device("cuda:0")
E = lambda: torch.cuda.Event(enable_timing=True)
for world in (1, 2, 4, 8):
    cfg = G.BaselineConfig(f"C2-131072-x{world}", "banded", 131072 * world, 64, half_bw=512, seed=0)
    geom = cfg.geometry
    ka = torch.from_numpy(G.config_keys(cfg, 0)).to(dev)
    kb = torch.from_numpy(G.config_keys(cfg, 1)).to(dev)
    lay = _ffi.make_layout(geom.params, geom.bs)
    st = torch.cuda.current_stream()
    res = []
    for it in range(8):
        torch.cuda.synchronize()
        e0, e1, e2, e3 = E(), E(), E(), E()
        e0.record(st)
        s = spgemm.SymbolicState(lay, ka, ka.numel(), kb, kb.numel(), st)
        e1.record(st)
        ck, ct = s.keys()
        e2.record(st)
        t = s.n_t
        s.triples(ct, 0, t // world)  # one rank's share
        e3.record(st)
        torch.cuda.synchronize()
        if it >= 3:
            res.append((e0.elapsed_time(e1), e1.elapsed_time(e2), e2.elapsed_time(e3)))
    med = [sorted(c)[len(c) // 2] for c in zip(*res)]
    print(f"N={world}: global nA={ka.numel()} nC={s.n_c} nT={s.n_t}: count {med[0]:.3f} keys {med[1]:.3f} "
          f"own triples {med[2]:.3f} ms (rank's numeric at 35 TF: {2 * 64**3 * (t // world) / 35e12 * 1e3:.2f} ms)")

# strong-scaling configs: the global count + keys phases every rank repeats, vs one rank's numeric
for name in ("C4", "C5-64", "C5-32"):
    cfg = G.CONFIGS[name]
    geom, a, b = G.config_operands_device(cfg, dev) if name == "C4" else (cfg.geometry, None, None)
    if a is not None:
        ka = a.keys
        kb = ka if cfg.same_operand else b.keys
    else:
        ka = torch.from_numpy(G.config_keys(cfg, 0)).to(dev)
        kb = torch.from_numpy(G.config_keys(cfg, 1)).to(dev)
    lay = _ffi.make_layout(geom.params, geom.bs)
    st = torch.cuda.current_stream()
    res = []
    for it in range(6):
        torch.cuda.synchronize()
        e0, e1, e2 = E(), E(), E()
        e0.record(st)
        s = spgemm.SymbolicState(lay, ka, ka.numel(), kb, kb.numel(), st)
        e1.record(st)
        ck, ct = s.keys()
        e2.record(st)
        torch.cuda.synchronize()
        if it >= 2:
            res.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
    med = [sorted(c)[len(c) // 2] for c in zip(*res)]
    t8 = 2 * geom.bs ** 3 * s.n_t / 8 / 36e12 * 1e3
    print(f"{name}: nA={ka.numel()} nC={s.n_c} nT={s.n_t}: global count {med[0]:.3f} keys {med[1]:.3f} ms; "
          f"one rank's numeric at N=8 ~{t8:.2f} ms")
    del a, b
