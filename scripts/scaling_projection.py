"""Projected multi-GPU efficiency from per-rank components MEASURED on one B200 (only one GPU is
available; this is a projection, not a scaling measurement).

For P ranks the product is partitioned exactly as distributed.multiply does it (contiguous C key
ranges of equal triple count; A and B owned in equal contiguous key ranges). Each rank's
components are timed on the GPU with CUDA events:
  symbolic   the rank's partitioned symbolic phase (qm_spgemm_count_part: the O(nA) tile-work pass
             and cut, then count / keys / triples of its own C key range only);
  numeric    the numeric kernel on the rank's triples (operands resident);
and its exchange is modelled from the partition's actual halo: unique A/B blocks its triples
reference outside its own key ranges, at 770 GB/s per direction over NVLink (B200_PROFILING.md),
serialised before the numeric phase ("exchange" mode), or -- distributed.py's "auto" rule -- the
fused mode when every remote block reference read over NVLink costs at most a quarter of the
numeric time: max(numeric, remote references / 770 GB/s), the TMA reads overlapping the DMMAs.
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
    a_cut = [(a.n * r) // world for r in range(world + 1)]
    b_cut = [(b.n * r) // world for r in range(world + 1)]
    ranks = []
    for r in range(world):
        def sym_rank():  # the rank's own share: partition pass + count + keys + triples
            s2 = spgemm.SymbolicState(lay, a.keys, a.n, b.keys, b.n, None, am, bm, part=(world, r))
            if s2.n_c == 0:
                return s2, None
            k2, t2_ = s2.keys()
            return s2, spgemm.SymbolicPlan(s2.n_c, s2.n_t, k2, t2_, s2.triples(t2_))
        t_sym, (s2, plan) = timed(sym_rank)
        if plan is None:
            ranks.append({"rank": r, "triples": 0, "symbolic_ms": t_sym, "numeric_ms": 0.0, "halo_bytes": 0,
                          "exchange_ms_model": 0.0, "fused_ms_model": 0.0, "total_ms": t_sym})
            continue
        t_num, _ = timed(lambda: spgemm.numeric(lay, a, b, plan))
        t2 = plan.tri.view(-1, 2).long()
        ua, ub = torch.unique(t2[:, 0]), torch.unique(t2[:, 1])
        rem_a = int(((ua < a_cut[r]) | (ua >= a_cut[r + 1])).sum())
        rem_b = int(((ub < b_cut[r]) | (ub >= b_cut[r + 1])).sum())
        blk = geom.bs * geom.bs * 8
        halo = (rem_a + rem_b) * blk
        refs = int(((t2[:, 0] < a_cut[r]) | (t2[:, 0] >= a_cut[r + 1])).sum() +
                   ((t2[:, 1] < b_cut[r]) | (t2[:, 1] >= b_cut[r + 1])).sum()) * blk
        t_x = halo / NVLINK * 1e3
        # fused mode (distributed.py "auto" rule): the kernel's TMA reads every remote block
        # reference over NVLink, overlapped with the DMMAs of earlier stages
        t_f = refs / NVLINK * 1e3
        fused = world > 1 and t_f <= 0.25 * t_num
        tot = t_sym + (max(t_num, t_f) if fused else t_num + t_x)
        ranks.append({"rank": r, "triples": s2.n_t, "key_range": list(s2.key_range), "symbolic_ms": t_sym,
                      "numeric_ms": t_num, "halo_bytes": halo, "remote_ref_bytes": refs,
                      "exchange_ms_model": t_x, "fused_ms_model": t_f, "mode": "fused" if fused else "exchange",
                      "total_ms": tot})
    del a, b
    torch.cuda.empty_cache()
    return {"T_ms": max(x["total_ms"] for x in ranks), "global_symbolic_ms": t_glob, "ranks": ranks}


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
                  f"xchg {max(x['exchange_ms_model'] for x in r['ranks']):.3f} "
                  f"modes {sorted(set(x.get('mode', '-') for x in r['ranks']))}", flush=True)
        res[name] = {"scaling": "strong" if strong else "weak", "per_world": rows}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
