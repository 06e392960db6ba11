import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2011_11762_b200 import MatrixSession
from oracle import spgemm_oracle as O
ses = MatrixSession(device="cuda:0")
for bs in (16, 32, 64):
    n = 4 * bs
    rng = np.random.default_rng(0)
    da = np.zeros((n, n)); db = np.zeros((n, n))
    da[:bs, :bs] = rng.uniform(-1, 1, (bs, bs)) * 1e-310     # subnormal operands
    db[:bs, :bs] = rng.uniform(-1, 1, (bs, bs))
    da[bs:2*bs, bs:2*bs] = 1e-160; db[bs:2*bs, bs:2*bs] = 1e-160   # products underflow to subnormal
    da[2*bs, 2*bs] = np.nan; db[2*bs, 2*bs] = 1.0
    da[3*bs, 3*bs] = np.inf; db[3*bs, 3*bs] = 2.0
    r, c = np.nonzero(da != 0); a = ses.matrix_from_triplets(n, r, c, da[r, c], leaf_dim=bs, block_size=bs)
    r, c = np.nonzero(db != 0); b = ses.matrix_from_triplets(n, r, c, db[r, c], leaf_dim=bs, block_size=bs)
    got = ses.to_dense(ses.multiply(a, b))
    want = da @ db
    # block-sparse semantics: NaN/Inf spread only inside the stored blocks they sit in
    for q in (2, 3):
        sl = slice(q * bs, (q + 1) * bs)
        want[sl, :] = 0.0
        want[sl, sl] = da[sl, sl] @ db[sl, sl]
    same = np.array_equal(got, want, equal_nan=True)
    print(bs, "equal:", same, "min nonzero |got|:", np.min(np.abs(got[got != 0])) if np.any(got != 0) else None,
          "want block0 nonzero:", np.count_nonzero(want[:bs,:bs]), "got:", np.count_nonzero(got[:bs,:bs]),
          "block1 want/got nz:", np.count_nonzero(want[bs:2*bs,bs:2*bs]), np.count_nonzero(got[bs:2*bs,bs:2*bs]))
