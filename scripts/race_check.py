import torch, sys, os
sys.path.insert(0, '.')
from paper_2011_11762_b200 import spgemm, _ffi
from paper_2011_11762_b200 import generators as G
dev = torch.device('cuda:0')
cfg = G.CONFIGS["C2-16384"]
geom, a, b = G.config_operands_device(cfg, dev)
layout = _ffi.make_layout(geom.params, geom.bs)
plan = spgemm.symbolic(layout, a, b)
ref, _, _ = spgemm.numeric(layout, a, b, plan)
torch.cuda.synchronize()
tptr = plan.c_tptr.cpu(); tri = plan.tri.view(-1, 2).long().cpu()
found = 0
for it in range(int(os.environ.get("ITERS", "200"))):
    c, _, _ = spgemm.numeric(layout, a, b, plan)
    torch.cuda.synchronize()
    bad = ((c.blocks - ref.blocks).abs().amax(dim=(1, 2)) > 0).nonzero().flatten().tolist()
    if not bad:
        continue
    found += 1
    print("iter", it, "bad", bad, flush=True)
    for m in bad[:2]:
        D = c.blocks[m] - ref.blocks[m]
        rows = (D.abs().amax(dim=1) > 1e-9).nonzero().flatten().tolist()
        cols = (D.abs().amax(dim=0) > 1e-9).nonzero().flatten().tolist()
        print(" m", m, "ntrip", int(tptr[m+1]-tptr[m]), "bad rows", rows[:8], len(rows), "bad cols", cols[:8], len(cols), "maxdiff", D.abs().max().item())
        # compare with single panel products of this block's triples
        best = None
        for t in range(int(tptr[m]), int(tptr[m+1])):
            A = a.blocks[tri[t,0]]; B = b.blocks[tri[t,1]]
            for p in range(2):
                P = A[:, 32*p:32*p+32] @ B[32*p:32*p+32, :]
                for sgn in (1.0, -1.0):
                    r = (D - sgn*P).abs().max().item()
                    if best is None or r < best[0]: best = (r, t - int(tptr[m]), p, sgn)
        print("  closest single panel product: resid %.3e triple %d panel %d sign %+.0f" % best, flush=True)
    if found >= 3:
        break
print("done, failures", found)
