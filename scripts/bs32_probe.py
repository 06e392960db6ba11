"""One bs-32 product (banded n=32768, hb=256, leaf 128) for launch lists / ncu."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2011_11762_b200 import MatrixSession

n, hb = 32768, 256
d = np.arange(-hb, hb + 1)
rows = np.repeat(np.arange(n), d.size)
cols = rows + np.tile(d, n)
keep = (cols >= 0) & (cols < n)
rows, cols = rows[keep], cols[keep]
vals = np.random.default_rng(0).uniform(-1, 1, rows.size)
ses = MatrixSession(device="cuda:0")
a = ses.matrix_from_triplets(n, rows, cols, vals, leaf_dim=int(sys.argv[1]) if len(sys.argv) > 1 else 32,
                             block_size=32)
for _ in range(3):
    c = ses.multiply(a, a)
torch.cuda.synchronize()
print("ok", c.root.n_blocks)
