"""Projected multi-GPU efficiency from each rank's pipeline RUN on one B200 (only one GPU is
available; this is a projection, not a scaling measurement).

For P ranks the product is partitioned exactly as distributed.multiply does it (qm_spgemm_count_part:
contiguous C key ranges of equal executed work; A and B owned in equal contiguous key ranges). Each
rank's whole step is executed on the GPU and timed with one pair of CUDA events (host enqueue and
synchronisation gaps included, as in the real product):
  symbolic  the rank's partitioned symbolic phase over the global structure's row indexes (kept
            with the distributed operands after their first product): tile work + cut, then count
            / keys / triples of its own C key range only;
  numeric   distributed.staged_numeric: the rank's C blocks whose triples are all local run first
            while k_halo_gather copies the halo (every block owned by another rank, once); the
            numeric kernel's claims of the other C blocks wait for the gather grid. The "peer" pools
            are slices of the operand pools on this GPU, and the gather is held until halo bytes /
            770 GB/s have elapsed (halo_min_ns: the measured NVLink peer-copy bandwidth,
            B200_PROFILING.md), so the halo arrives no earlier than it would over NVLink;
  compaction the exact-zero count read-back and drop.
T(P) = max over ranks; E(P) = T(1) / T(P) for weak scaling (C2 with n = 131072*P) and
T(1) / (P * T(P)) for strong scaling (C4, C5-64), T(1) = the single-GPU product (spgemm.multiply_blocks)
timed the same way.

    python scripts/scaling_projection.py [--out profiles/R2_scaling_projection.json] [--configs C4 ...]
"""
import argparse
import json
import sys

sys.path.insert(0, ".")
import torch

from paper_2011_11762_b200 import _ffi, spgemm
from paper_2011_11762_b200 import distributed as D
from paper_2011_11762_b200 import generators as G

NVLINK_GBS = 770.0
dev = torch.device("cuda:0")
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def timed(fn, reps=5):
    """Median of `reps` runs (after one warm-up) of fn between two events on the current stream."""
    fn()
    ts, out = [], None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = E(), E()
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2], out


def peers(t, off):
    blk = t.shape[1] * t.shape[2] * t.element_size()
    return [t.data_ptr() + off[r] * blk for r in range(len(off) - 1)]


def project(cfg, world):
    geom, a, b = G.config_operands_device(cfg, dev)
    b_is_a = cfg.same_operand
    if b_is_a:
        b = a
    lay = _ffi.make_layout(geom.params, geom.bs)
    use = spgemm._use_masks(a, b)
    am = a.masks[1] if use else None
    bm = b.masks[0] if use else None
    masks = (a.masks[1], b.masks[0], a.masks[2], b.masks[2]) if use else None
    if world == 1:
        t1, _ = timed(lambda: spgemm.multiply_blocks(lay, a, b))
        return {"T_ms": t1, "ranks": [{"rank": 0, "total_ms": t1}]}
    a_off = [(a.n * r) // world for r in range(world + 1)]
    b_off = a_off if b_is_a else [(b.n * r) // world for r in range(world + 1)]
    pa, pb = peers(a.blocks, a_off), peers(b.blocks, b_off)
    # the global structure's row indexes: metadata of the distributed operands, gathered and built
    # on the first product and reused while the ranks multiply the same block sets (distributed.py)
    ixs = D.CudaBackend().row_indexes(lay, a.keys, b.keys, a.masks[1] if use else None, b.masks[0] if use else None,
                                      a.masks[2] if use else None, b.masks[2] if use else None, b_is_a)
    ranks = []
    for r in range(world):
        info = {}

        def step():  # the rank's product: partitioned symbolic, staged numeric, compaction
            st = spgemm.SymbolicState(lay, a.keys, a.n, b.keys, b.n, None, am, bm, part=(world, r), ix=ixs[0])
            if st.n_c == 0:
                return st
            ck, ct = st.keys()
            tri = st.triples(ct)
            info.clear()
            c, nz, zc = D.staged_numeric(lay, tri, ct, ck, r, a_off, b_off, pa, pb,
                                         a.blocks[a_off[r]:a_off[r + 1]], b.blocks[b_off[r]:b_off[r + 1]],
                                         b_is_a, masks, info=info, emulate_link_gbs=NVLINK_GBS)
            c = spgemm.compact(geom.bs, c, nz, _ffi.read_i64(zc))
            return st

        t_rank, st = timed(step)

        def sym_only():
            s2 = spgemm.SymbolicState(lay, a.keys, a.n, b.keys, b.n, None, am, bm, part=(world, r), ix=ixs[0])
            if s2.n_c:
                k2, t2 = s2.keys()
                s2.triples(t2)
            return s2

        t_sym, _ = timed(sym_only)
        ranks.append({"rank": r, "triples": st.n_t, "c_blocks": st.n_c, "key_range": [int(x) for x in st.key_range],
                      "total_ms": t_rank, "symbolic_ms": t_sym, "halo_bytes": info.get("halo_bytes", 0),
                      "halo_link_ms": info.get("halo_bytes", 0) / (NVLINK_GBS * 1e9) * 1e3,
                      "local_c_blocks": info.get("local_c_blocks", 0)})
    del a, b
    torch.cuda.empty_cache()
    return {"T_ms": max(x["total_ms"] for x in ranks), "ranks": ranks}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--configs", nargs="*", default=["C2", "C4", "C5-64"])
    args = ap.parse_args()
    res = {"method": "each rank's step run on one B200 (symbolic + staged numeric with the halo gather "
                     f"held to {NVLINK_GBS} GB/s + compaction), CUDA events; max over ranks"}
    for name in args.configs:
        strong = name != "C2"
        rows = {}
        for world in (1, 2, 4, 8):
            cfg = (G.BaselineConfig(f"C2-{131072 * world}", "banded", 131072 * world, 64, half_bw=512)
                   if not strong else G.CONFIGS[name])
            rows[world] = project(cfg, world)
        t1 = rows[1]["T_ms"]
        for world, r in rows.items():
            r["efficiency"] = t1 / (world * r["T_ms"]) if strong else t1 / r["T_ms"]
            rk = r["ranks"]
            print(f"{name} P={world}: T={r['T_ms']:.3f} ms  E={r['efficiency']:.3f}  "
                  f"max rank sym {max(x.get('symbolic_ms', 0) for x in rk):.3f} "
                  f"halo {max(x.get('halo_bytes', 0) for x in rk) / 1e6:.1f} MB "
                  f"({max(x.get('halo_link_ms', 0) for x in rk):.3f} ms at NVLink) "
                  f"local C {min(x.get('local_c_blocks', 0) / max(x.get('c_blocks', 1), 1) for x in rk):.2f}",
                  flush=True)
        res[name] = {"scaling": "strong" if strong else "weak", "per_world": rows}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
