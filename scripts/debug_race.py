import torch, sys, os
sys.path.insert(0, '.')
from paper_2011_11762_b200 import distributed as D, spgemm, _ffi
from paper_2011_11762_b200.blocks import BlockSet
from paper_2011_11762_b200 import generators as G
dev = torch.device('cuda:0')
cfg = G.CONFIGS[os.environ.get("CFG", "C2-16384")]
geom, a, b = G.config_operands_device(cfg, dev)
layout = _ffi.make_layout(geom.params, geom.bs)
ref = spgemm.multiply_blocks(layout, a, b)
plan = spgemm.symbolic(layout, a, b)
def cmp(tag, c):
    bad = ((c.blocks - ref.blocks).abs().amax(dim=(1,2)) > 0).nonzero().flatten()
    print(tag, bad.numel(), bad[:4].tolist(), flush=True)
mode = sys.argv[1]
for i in range(12):
    if mode == "fresh":   # fresh copies of the operands every time
        a2 = BlockSet(a.keys, a.blocks.clone(), a.sumsq); b2 = BlockSet(b.keys, b.blocks.clone(), b.sumsq)
        c, nz, zc = spgemm.numeric(layout, a2, b2, plan)
    elif mode == "freshsync":
        a2 = BlockSet(a.keys, a.blocks.clone(), a.sumsq); b2 = BlockSet(b.keys, b.blocks.clone(), b.sumsq)
        torch.cuda.synchronize()
        c, nz, zc = spgemm.numeric(layout, a2, b2, plan)
    elif mode == "same":
        c, nz, zc = spgemm.numeric(layout, a, b, plan)
    elif mode == "local":
        c, _ = D.multiply(D.LocalComm(), layout, a, b)
    torch.cuda.synchronize()
    cmp(f"{mode} {i}", c)
