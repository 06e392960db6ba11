"""bs 16 grouped kernel vs problem size: numeric phase of a banded product (leaf 128, bs 16) for several
n, to separate the kernel's steady-state rate from its ramp-up / tail on a sub-millisecond launch.
    python scripts/bs16_size_probe.py [n ...]"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2011_11762_b200 import MatrixSession, spgemm, _ffi

hb = 256
ses = MatrixSession(device="cuda:0")
E = lambda: torch.cuda.Event(enable_timing=True)
for n in [int(x) for x in sys.argv[1:]] or [32768, 131072]:
    rng = np.random.default_rng(0)
    d = np.arange(-hb, hb + 1)
    rows = np.repeat(np.arange(n), d.size)
    cols = rows + np.tile(d, n)
    keep = (cols >= 0) & (cols < n)
    rows, cols = rows[keep], cols[keep]
    vals = rng.uniform(-1, 1, rows.size)
    a = ses.matrix_from_triplets(n, rows, cols, vals, leaf_dim=128, block_size=16)
    del rows, cols, vals
    layout = _ffi.make_layout(a.params, 16)
    bsx = a.root.require()
    res = []
    for it in range(7):
        ev = {k: E() for k in ("symbolic", "numeric", "end")}
        st = spgemm.MultiplyStats()
        spgemm.multiply_blocks(layout, bsx, bsx, events=ev, stats=st)
        torch.cuda.synchronize()
        if it >= 2:
            res.append((ev["symbolic"].elapsed_time(ev["numeric"]), ev["numeric"].elapsed_time(ev["end"])))
    sym, num = np.median(np.array(res), axis=0)
    print(f"n {n} bs 16: T={st.n_triples} nC={st.n_c_symbolic} symbolic {sym:.3f} ms numeric {num:.3f} ms = "
          f"{st.flops / num / 1e9:.2f} TFLOP/s", flush=True)
    del a, bsx
    torch.cuda.empty_cache()
