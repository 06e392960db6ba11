import socket, torch, torch.distributed as dist, sys, os
sys.path.insert(0, '.')
from paper_2011_11762_b200 import distributed as D, spgemm, _ffi
from paper_2011_11762_b200 import generators as G
dev = torch.device('cuda:0')
cfg = G.CONFIGS[os.environ.get("CFG", "C2-16384")]
geom, a, b = G.config_operands_device(cfg, dev)
layout = _ffi.make_layout(geom.params, geom.bs)
ref = spgemm.multiply_blocks(layout, a, b)
for i in range(6):
    r = spgemm.multiply_blocks(layout, a, b)
    print("ref again", i, torch.equal(r.blocks, ref.blocks), flush=True)
for i in range(4):
    c, _ = D.multiply(D.LocalComm(), layout, a, b)
    print("local", i, torch.equal(c.blocks, ref.blocks), flush=True)
with socket.socket() as s_:
    s_.bind(("127.0.0.1", 0)); port = s_.getsockname()[1]
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=dev)
comm = D.Comm()
for i in range(6):
    c, _ = D.multiply(comm, layout, a, b)
    torch.cuda.synchronize()
    bad = ((c.blocks - ref.blocks).abs().amax(dim=(1,2)) > 0).nonzero().flatten()
    print("nccl", i, torch.equal(c.blocks, ref.blocks), bad.numel(), bad[:5].tolist(), flush=True)
dist.destroy_process_group()
