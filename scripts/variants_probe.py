"""symmetric_square / rank_k / symmetric products on the decay config (C4's symmetric A stored as
its upper leaves) against the regular product -- the purification-style use of the library."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2011_11762_b200 import MatrixSession
from paper_2011_11762_b200 import generators as G

dev = torch.device("cuda:0")
ses = MatrixSession(device=dev)
cfg = G.CONFIGS["C4"]
geom, (ka, ba), _ = G.config_operands_host(cfg)
bi, bj = geom.decode(ka)
up = (bi // geom.nbl) <= (bj // geom.nbl)
full = ses.matrix_from_blocks(geom, ka, ba)
sym = ses.matrix_from_blocks(geom, ka[up], ba[up], symmetric=True)


def timed(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return sorted(ts)[len(ts) // 2] * 1e3, out


t_reg, c = timed(lambda: ses.multiply(full, full))
print(f"regular A*A: {t_reg:.3f} ms, blocks {c.root.n_blocks}")
t_rk, c2 = timed(lambda: ses.multiply(full, None, "rank_k"))
print(f"rank_k A*A^T (upper): {t_rk:.3f} ms, blocks {c2.root.n_blocks}")
t_ss, c3 = timed(lambda: ses.multiply(sym, None, "symmetric_square"))
print(f"symmetric_square (A stored upper): {t_ss:.3f} ms, blocks {c3.root.n_blocks}")
