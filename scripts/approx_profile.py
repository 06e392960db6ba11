import sys, cProfile, pstats, time
sys.path.insert(0, ".")
import torch
from paper_2011_11762_b200 import MatrixSession
from paper_2011_11762_b200 import generators as G
dev = torch.device("cuda:0")
ses = MatrixSession(device=dev)
geom, a, _ = G.config_operands_device(G.CONFIGS["C4"], dev)
ma = ses.matrix_from_blockset(geom, a)
na = ses.norm(ma)
tau = 1e-10 * na * na
for _ in range(2): ses.multiply(ma, ma, "approximate", tau)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
ses.multiply(ma, ma, "approximate", tau); torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
