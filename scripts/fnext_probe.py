"""Measurements of the SURVEY 8(f) rows (the callers either side of the multiply) on one B200:

  construct  matrix_from_triplets on the device (qm_build_*, triplets H2D included) vs the host
             build (bit-identical numpy restatement) -- entries/s;
  add/scale  block algebra (qm_axpby_blocks) on two C2-131072 products -- HBM GB/s;
  truncate   global Frobenius truncation of a C2-131072 product;
  approx     approximate (norm-pruned) multiply on C4 vs the regular product.

    python scripts/fnext_probe.py [--out profiles/fnext_rXX.json]
"""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2011_11762_b200 import MatrixSession, construct
from paper_2011_11762_b200 import generators as G
from paper_2011_11762_b200.layout import Geometry, MatrixParams


def timed(fn, reps=5):
    ts = []
    out = fn()  # warm-up (lazy module loading, allocator growth)
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return sorted(ts)[len(ts) // 2], out


def banded_triplets(n, hb, seed=0):
    d = np.arange(-hb, hb + 1)
    rows = np.repeat(np.arange(n, dtype=np.int64), d.size)
    cols = rows + np.tile(d, n)
    keep = (cols >= 0) & (cols < n)
    rows, cols = rows[keep], cols[keep]
    vals = np.random.default_rng(seed).uniform(-1, 1, rows.size)
    return rows, cols, vals


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    ses = MatrixSession(device=dev)
    res = {}

    # -- construction -------------------------------------------------------------------------
    for n, hb in ((16384, 512), (131072, 512)):
        r, c, v = banded_triplets(n, hb)
        dt, m = timed(lambda: ses.matrix_from_triplets(n, r, c, v, leaf_dim=64, block_size=64), reps=3)
        row = {"entries": int(r.size), "device_s": dt, "device_entries_per_s": r.size / dt,
               "blocks": int(m.root.n_blocks), "triplet_bytes_h2d": int(r.size * 24)}
        if n <= 16384:
            geom = Geometry(MatrixParams.create(n, 64), 64)
            th, _ = timed(lambda: construct.blocks_from_triplets(geom, r, c, v), reps=1)
            row.update(host_s=th, host_entries_per_s=r.size / th)
        res[f"construct_banded_n{n}_hb{hb}"] = row
        print("construct", n, row, flush=True)

    # -- block algebra on products --------------------------------------------------------------
    cfg = G.CONFIGS["C2-131072"]
    geom, a, b = G.config_operands_device(cfg, dev)
    ma, mb = ses.matrix_from_blockset(geom, a), ses.matrix_from_blockset(geom, b)
    c1 = ses.multiply(ma, mb)
    c2 = ses.multiply(mb, ma)
    nb = c1.root.n_blocks
    blk = 8 * geom.bs * geom.bs
    dt, s = timed(lambda: ses.add(c1, c2, 1.0, -0.5))
    union = s.root.n_blocks
    res["add_C2-131072"] = {"s": dt, "blocks_in": [nb, c2.root.n_blocks], "blocks_out": union,
                            "hbm_bytes": (nb + c2.root.n_blocks + union) * blk,
                            "GBps": (nb + c2.root.n_blocks + union) * blk / dt / 1e9}
    dt, _ = timed(lambda: ses.scale(c1, 0.75))
    res["scale_C2-131072"] = {"s": dt, "hbm_bytes": 2 * nb * blk, "GBps": 2 * nb * blk / dt / 1e9}
    fro = ses.norm(c1)
    dt, (t_m, removed) = timed(lambda: ses.truncate(c1, 1e-3 * fro))
    res["truncate_C2-131072"] = {"s": dt, "tau": 1e-3 * fro, "blocks_in": nb,
                                 "blocks_out": t_m.root.n_blocks, "removed_norm": removed}
    print({k: v for k, v in res.items() if not k.startswith("construct")}, flush=True)
    del c1, c2, s, t_m, ma, mb, a, b
    torch.cuda.empty_cache()

    # -- approximate multiply ------------------------------------------------------------------
    cfg = G.CONFIGS["C4"]
    geom, a, _ = G.config_operands_device(cfg, dev)
    ma = ses.matrix_from_blockset(geom, a)
    dt_reg, c = timed(lambda: ses.multiply(ma, ma), reps=3)
    na = ses.norm(ma)
    for rel in (1e-10, 1e-6):
        tau = rel * na * na
        dt, ca = timed(lambda: ses.multiply(ma, ma, "approximate", tau), reps=3)
        log = ses.last_engine.prune_log if ses.last_engine is not None else []
        res[f"approximate_C4_tau{rel:g}"] = {
            "s": dt, "regular_s": dt_reg, "tau": tau, "blocks": ca.root.n_blocks,
            "regular_blocks": c.root.n_blocks, "pruned_tasks": len(log),
            "pruned_bound_sum": float(sum(log))}
        print("approx", rel, res[f"approximate_C4_tau{rel:g}"], flush=True)

    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
