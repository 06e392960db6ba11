"""Where grouping C blocks pays: banded products of growing bandwidth (average k-list length L = nT/nC)
at bs 16 (groups vs the per-block cp.async kernel) and bs 32 (quads vs the per-block TMA kernel).
The library's gates (L >= 4 / L >= 8) sit at the measured crossovers."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2011_11762_b200 import MatrixSession, spgemm, _ffi

ses = MatrixSession(device="cuda:0")
E = lambda: torch.cuda.Event(enable_timing=True)
n = 65536
for bs, leaf, hbs in ((16, 128, (8, 16, 24, 32, 48, 64, 128)), (32, 32, (16, 32, 48, 64, 96, 128, 256))):
    for hb in hbs:
        d = np.arange(-hb, hb + 1)
        rows = np.repeat(np.arange(n), d.size)
        cols = rows + np.tile(d, n)
        keep = (cols >= 0) & (cols < n)
        rows, cols = rows[keep], cols[keep]
        vals = np.random.default_rng(0).uniform(-1, 1, rows.size)
        a = ses.matrix_from_triplets(n, rows, cols, vals, leaf_dim=leaf, block_size=bs)
        del rows, cols, vals
        lay = _ffi.make_layout(a.params, bs)
        x = a.root.require()
        out = []
        for grouped in ("1", "0"):
            os.environ["QM_G16_GROUPS"] = grouped
            os.environ["QM_QUAD32"] = grouped
            res = []
            for it in range(8):
                ev = {k: E() for k in ("symbolic", "numeric", "end")}
                st = spgemm.MultiplyStats()
                spgemm.multiply_blocks(lay, x, x, events=ev, stats=st)
                torch.cuda.synchronize()
                if it >= 3:
                    res.append(ev["numeric"].elapsed_time(ev["end"]))
            out.append(float(np.median(res)))
        L = st.n_triples / st.n_c_symbolic
        print(f"bs {bs} hb {hb:4d}: L = {L:5.2f}  grouped {out[0]:.3f} ms  per-block {out[1]:.3f} ms  "
              f"ratio {out[1] / out[0]:.2f}", flush=True)
        del a, x
        torch.cuda.empty_cache()
