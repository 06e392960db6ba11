"""C4 approximate (norm-pruned) multiply vs the regular product on one B200: time per product
(median of 5, synchronised wall clock), executed triples, pruned tasks, and the prune phase alone.

    python scripts/approx_probe.py [--out profiles/R2_approx.json]
"""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_2011_11762_b200 import MatrixSession, approximate
from paper_2011_11762_b200 import generators as G


def timed(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return sorted(ts)[len(ts) // 2], out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    ses = MatrixSession(device=dev)
    geom, a, _ = G.config_operands_device(G.CONFIGS["C4"], dev)
    ma = ses.matrix_from_blockset(geom, a)
    na = ses.norm(ma)
    res = {}
    dt, _ = timed(lambda: ses.multiply(ma, ma))
    res["regular"] = {"ms": round(dt * 1e3, 3), "triples": ses.last_multiply.n_triples, "c_blocks": ses.last_multiply.n_c}
    print(json.dumps(res["regular"]), flush=True)
    for rel in (1e-10, 1e-6, 1e-3):
        tau = rel * na * na
        dt, _ = timed(lambda: ses.multiply(ma, ma, "approximate", tau))
        pt, pr = timed(lambda: approximate.prune(geom, a, a, tau))
        row = {"tau_rel": rel, "ms": round(dt * 1e3, 3), "prune_ms": round(pt * 1e3, 3),
               "triples": ses.last_multiply.n_triples, "c_blocks": ses.last_multiply.n_c,
               "pruned_tasks": len(ses.last_engine.prune_log), "levels": len(pr.pairs_per_level)}
        res[f"approximate_{rel:g}"] = row
        print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
