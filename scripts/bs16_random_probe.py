"""bs 16 on a random block pattern (8 blocks per block row, leaf 128): grouped kernel vs the per-block
cp.async kernel -- groups pay only when a stage's k is shared by several members."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2011_11762_b200 import MatrixSession, spgemm, _ffi

bs, leaf = 16, 128
ses = MatrixSession(device="cuda:0")
E = lambda: torch.cuda.Event(enable_timing=True)
for n, per_row in ((32768, 8), (32768, 32)):
    nb = n // bs
    rng = np.random.default_rng(1)
    bi = np.repeat(np.arange(nb), per_row)
    bj = rng.integers(0, nb, bi.size)
    r = (bi[:, None, None] * bs + np.arange(bs)[None, :, None] + np.zeros((1, 1, bs), int)).ravel()
    c = (bj[:, None, None] * bs + np.zeros((1, bs, 1), int) + np.arange(bs)[None, None, :]).ravel()
    v = rng.uniform(-1, 1, r.size)
    a = ses.matrix_from_triplets(n, r, c, v, leaf_dim=leaf, block_size=bs)
    lay = _ffi.make_layout(a.params, bs)
    x = a.root.require()
    for impl in ("tma", "cpasync", "tma", "cpasync"):
        os.environ["QM_NUMERIC"] = impl
        res = []
        for it in range(7):
            ev = {k: E() for k in ("symbolic", "numeric", "end")}
            st = spgemm.MultiplyStats()
            spgemm.multiply_blocks(lay, x, x, events=ev, stats=st)
            torch.cuda.synchronize()
            if it >= 2:
                res.append(ev["numeric"].elapsed_time(ev["end"]))
        num = float(np.median(res))
        print(f"random n={n} per_row={per_row} bs 16 {impl:8s}: T={st.n_triples} nC={st.n_c_symbolic} numeric {num:.3f} ms = "
              f"{st.flops / num / 1e9:.2f} TFLOP/s", flush=True)
