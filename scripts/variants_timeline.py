"""Device time of each stage of symmetric_square on the decay config (CUDA events around the
variant's steps), to see what beyond the half product it costs."""
import sys

sys.path.insert(0, ".")
import torch

from paper_2011_11762_b200 import MatrixSession, _ffi, spgemm, variants
from paper_2011_11762_b200 import generators as G

dev = torch.device("cuda:0")
ses = MatrixSession(device=dev)
cfg = G.CONFIGS["C4"]
geom, (ka, ba), _ = G.config_operands_host(cfg)
bi, bj = geom.decode(ka)
up = (bi // geom.nbl) <= (bj // geom.nbl)
sym = ses.matrix_from_blocks(geom, ka[up], ba[up], symmetric=True)
s = sym.root.blockset
s.support_masks()
lay = _ffi.make_layout(geom.params, geom.bs)
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
for it in range(4):
    torch.cuda.synchronize()
    ev = [E() for _ in range(6)]
    ev[0].record()
    x = variants.expand_symmetric(geom, s)
    ev[1].record()
    plan = spgemm.symbolic(lay, x, x)
    ev[2].record()
    plan2 = spgemm.symbolic(lay, x, x, upper=True)
    ev[3].record()
    c, nz, zc = spgemm.numeric(lay, x, x, plan2)
    ev[4].record()
    torch.cuda.synchronize()
    ev[5].record()
    torch.cuda.synchronize()
    if it:
        print("expand %.3f symbolic %.3f symbolic-upper %.3f numeric %.3f ms (triples %d -> %d)" % (
            ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]),
            ev[3].elapsed_time(ev[4]), plan.n_triples, plan2.n_triples))
