"""Per-phase device time of the product for the reference's default-style layouts (leaf 128 with
bs 16/32/64), TMA vs cp.async numeric kernel (QM_NUMERIC); bs 16 also with single-row groups
(QM_GROUP_ROWS=1)."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2011_11762_b200 import MatrixSession, spgemm, _ffi

n, hb = 32768, 256
rng = np.random.default_rng(0)
d = np.arange(-hb, hb + 1)
rows = np.repeat(np.arange(n), d.size)
cols = rows + np.tile(d, n)
keep = (cols >= 0) & (cols < n)
rows, cols = rows[keep], cols[keep]
vals = rng.uniform(-1, 1, rows.size)
ses = MatrixSession(device="cuda:0")
E = lambda: torch.cuda.Event(enable_timing=True)
for leaf, bs in ((128, 16), (128, 32), (32, 32), (128, 64)):
    a = ses.matrix_from_triplets(n, rows, cols, vals, leaf_dim=leaf, block_size=bs)
    layout = _ffi.make_layout(a.params, bs)
    bsx = a.root.require()
    for impl in (("tma", "tma-rows1", "cpasync") if bs == 16 else ("tma", "cpasync")):
        os.environ["QM_NUMERIC"] = impl.split("-")[0]
        os.environ["QM_GROUP_ROWS"] = "1" if impl.endswith("rows1") else "2"
        res = []
        for it in range(6):
            ev = {k: E() for k in ("symbolic", "numeric", "end")}
            st = spgemm.MultiplyStats()
            spgemm.multiply_blocks(layout, bsx, bsx, events=ev, stats=st)
            torch.cuda.synchronize()
            if it >= 2:
                res.append((ev["symbolic"].elapsed_time(ev["numeric"]), ev["numeric"].elapsed_time(ev["end"])))
        sym, num = np.median(np.array(res), axis=0)
        print(f"leaf {leaf} bs {bs} {impl:10s}: T={st.n_triples} nC={st.n_c_symbolic} symbolic {sym:.3f} ms "
              f"numeric {num:.3f} ms = {st.flops / num / 1e9:.2f} TFLOP/s")
