"""Projected multi-GPU efficiency from per-rank components MEASURED on one B200 (only one GPU is
available; this is a projection, not a scaling measurement).

For P ranks the product is partitioned exactly as distributed.multiply does it (contiguous C key
ranges of equal triple count; A and B owned in equal contiguous key ranges). Each rank's
components are timed on the GPU with CUDA events:
  symbolic   the global count + C-key phase every rank repeats, then the rank's own triples;
  numeric    the numeric kernel on the rank's triple range (operands resident);
and its exchange is modelled from the partition's actual halo: unique A/B blocks its triples
reference outside its own key ranges, at 770 GB/s per direction over NVLink (B200_PROFILING.md).
T(P) = max over ranks (symbolic + exchange + numeric); E(P) = T(1) / T(P) for weak scaling (C2
with n = 131072*P) and T(1) / (P * T(P)) for strong scaling (C4, C5-64).

    python scripts/scaling_projection.py [--out profiles/scaling_projection_rXX.json]
"""
import argparse
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2011_11762_b200 import _ffi, spgemm
from paper_2011_11762_b200 import distributed as D
from paper_2011_11762_b200 import generators as G

NVLINK = 770e9
dev = torch.device("cuda:0")
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def timed(fn, reps=3):
    best, out = float("inf"), None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = E(), E()
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, out


def project(cfg, world):
    geom, a, b = G.config_operands_device(cfg, dev)
    if cfg.same_operand:
        b = a
    lay = _ffi.make_layout(geom.params, geom.bs)
    use = spgemm._use_masks(a, b)
    am = a.masks[1] if use else None
    bm = b.masks[0] if use else None

    def sym_global():
        st = spgemm.SymbolicState(lay, a.keys, a.n, b.keys, b.n, None, am, bm)
        ck, ct = st.keys()
        return st, ck, ct

    t_glob, (st, ck, ct) = timed(sym_global)
    cb, tb = D.partition(ct, world)
    a_cut = [(a.n * r) // world for r in range(world + 1)]
    b_cut = [(b.n * r) // world for r in range(world + 1)]
    ranks = []
    for r in range(world):
        lo, hi = tb[r], tb[r + 1]
        m0, m1 = cb[r], cb[r + 1]
        t_tri, tri = timed(lambda: st.triples(ct, lo, hi))
        plan = spgemm.SymbolicPlan(m1 - m0, hi - lo, ck[m0:m1].contiguous(), (ct[m0:m1 + 1] - lo).contiguous(), tri)
        t_num, _ = timed(lambda: spgemm.numeric(lay, a, b, plan))
        t2 = tri.view(-1, 2).long()
        ua, ub = torch.unique(t2[:, 0]), torch.unique(t2[:, 1])
        rem_a = int(((ua < a_cut[r]) | (ua >= a_cut[r + 1])).sum())
        rem_b = int(((ub < b_cut[r]) | (ub >= b_cut[r + 1])).sum())
        halo = (rem_a + rem_b) * geom.bs * geom.bs * 8
        t_x = halo / NVLINK * 1e3
        ranks.append({"rank": r, "triples": hi - lo, "symbolic_ms": t_glob + t_tri, "numeric_ms": t_num,
                      "halo_bytes": halo, "exchange_ms_model": t_x, "total_ms": t_glob + t_tri + t_num + t_x})
    del a, b
    torch.cuda.empty_cache()
    return {"T_ms": max(x["total_ms"] for x in ranks), "ranks": ranks}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    res = {}
    for name, strong in (("C2", False), ("C4", True), ("C5-64", True)):
        rows = {}
        for world in (1, 2, 4, 8):
            cfg = (G.BaselineConfig(f"C2-{131072 * world}", "banded", 131072 * world, 64, half_bw=512)
                   if not strong else G.CONFIGS[name])
            rows[world] = project(cfg, world)
        t1 = rows[1]["T_ms"]
        for world, r in rows.items():
            r["efficiency"] = t1 / (world * r["T_ms"]) if strong else t1 / r["T_ms"]
            print(f"{name} P={world}: T={r['T_ms']:.3f} ms  E={r['efficiency']:.3f}  "
                  f"max rank: sym {max(x['symbolic_ms'] for x in r['ranks']):.3f} "
                  f"num {max(x['numeric_ms'] for x in r['ranks']):.3f} "
                  f"xchg {max(x['exchange_ms_model'] for x in r['ranks']):.3f} ms", flush=True)
        res[name] = {"scaling": "strong" if strong else "weak", "per_world": rows}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
