"""Throughput of the drop-in with the reference's default layout (leaf_dim=128, block_size=16) and
bs=32/64 for comparison, through MatrixSession (triplets -> device build -> multiply)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2011_11762_b200 import MatrixSession
n, hb = 32768, 256
rng = np.random.default_rng(0)
d = np.arange(-hb, hb + 1)
rows = np.repeat(np.arange(n), d.size); cols = rows + np.tile(d, n)
keep = (cols >= 0) & (cols < n); rows, cols = rows[keep], cols[keep]
vals = rng.uniform(-1, 1, rows.size)
ses = MatrixSession(device="cuda:0")
for leaf, bs in ((128, 16), (128, 32), (128, 64), (64, 64)):
    a = ses.matrix_from_triplets(n, rows, cols, vals, leaf_dim=leaf, block_size=bs)
    for _ in range(2): ses.multiply(a, a)
    ts = []
    for _ in range(8):
        torch.cuda.synchronize(); t = time.perf_counter()
        c = ses.multiply(a, a)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    dt = sorted(ts)[len(ts) // 2]
    print("  per call ms:", " ".join(f"{x*1e3:.2f}" for x in ts))
    f = ses.last_multiply.flops
    print(f"leaf {leaf} bs {bs}: triples {ses.last_multiply.n_triples} {dt*1e3:.2f} ms  {f/dt/1e12:.2f} TFLOP/s")
