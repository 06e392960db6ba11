"""Times the REAL reference multiply (quadmat.MatrixSession.multiply, pkg/src/quadmat/session.py:
160-171) on this host, the way its own harness does (bench.py:104-120): a fresh
MatrixSession(n_workers=W, mode="threaded") per repeat, threadpool_limits(1), perf_counter around
the multiply only, median of the repeats. Inputs are the identical block-keyed arrays the GPU path
consumes (generators.config_operands_host), handed to quadmat through matrix_from_triplets.

    PYTHONPATH=baseline/_ref python scripts/reference_cpu_timing.py [out.json]

Layouts: L64 (leaf_dim = block_size = 64, the literal BASELINE layout) and L256 (leaf 256, bs 64:
the reference bench's default, bench.py:36-37); W = 1 and W = all host cores. SURVEY.md 8(d)."""

from __future__ import annotations

import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))


def triplets(keys, blocks, geom):
    bi, bj = geom.decode(keys)
    bs = geom.bs
    nz = blocks != 0
    m, r, c = np.nonzero(nz)
    return bi[m] * bs + r, bj[m] * bs + c, blocks[nz]


def main(out=None):
    import quadmat
    from threadpoolctl import threadpool_limits

    from paper_2011_11762_b200 import generators as G

    cores = len(os.sched_getaffinity(0))
    rows = []
    for name, reps in (("C1", 3), ("C2-16384", 3)):
        cfg = G.CONFIGS[name]
        geom, (ka, ba), (kb, bb) = G.config_operands_host(cfg)
        ta, tb = triplets(ka, ba, geom), triplets(kb, bb, geom)
        T = G.structure_counts(cfg)["triples_structural"]
        for leaf in (64, 256):
            for w in sorted({1, cores}):
                times = []
                for _ in range(reps):
                    s = quadmat.MatrixSession(n_workers=w, mode="threaded")
                    a = s.matrix_from_triplets(cfg.n, *ta, leaf_dim=leaf, block_size=cfg.bs)
                    b = s.matrix_from_triplets(cfg.n, *tb, leaf_dim=leaf, block_size=cfg.bs)
                    with threadpool_limits(limits=1):
                        t0 = time.perf_counter()
                        s.multiply(a, b)
                        times.append(time.perf_counter() - t0)
                    del s, a, b
                wall = statistics.median(times)
                row = {"workload": name, "leaf_dim": leaf, "block_size": cfg.bs, "workers": w,
                       "host_cores": cores, "wall_s": round(wall, 4), "repeats": times,
                       "leaf_gemm_gflops": round(2.0 * cfg.bs ** 3 * T / wall / 1e9, 4)}
                print(json.dumps(row), flush=True)
                rows.append(row)
    if out:
        Path(out).write_text(json.dumps({"what": "reference quadmat.MatrixSession.multiply on the host "
                                                 "(mode threaded, threadpool_limits(1), median)",
                                         "rows": rows}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
