import socket, torch, torch.distributed as dist, sys
sys.path.insert(0, '.')
from paper_2011_11762_b200 import distributed as D, spgemm, _ffi
from paper_2011_11762_b200 import generators as G
dev = torch.device('cuda:0')
cfg = G.CONFIGS['C2-16384']
geom, a, b = G.config_operands_device(cfg, dev)
layout = _ffi.make_layout(geom.params, geom.bs)
ref = spgemm.multiply_blocks(layout, a, b)
with socket.socket() as s_:
    s_.bind(("127.0.0.1", 0)); port = s_.getsockname()[1]
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=dev)
comm = D.Comm()
need = torch.arange(a.n, device=dev)
pool, r, s, n = D._fetch(comm, D.CudaBackend(), a.blocks, [0, a.n], need)
torch.cuda.synchronize()
print("pool equal", torch.equal(pool, a.blocks), pool.shape, a.blocks.shape)
k2, _ = comm.allgather_varlen(a.keys)
print("keys equal", torch.equal(k2, a.keys))
c2, st = D.multiply(comm, layout, a, b)
torch.cuda.synchronize()
print("c equal", torch.equal(c2.keys, ref.keys), torch.equal(c2.blocks, ref.blocks))
d = (c2.blocks - ref.blocks).abs().max().item(); print("maxdiff", d, ref.blocks.abs().max().item())
bad = ((c2.blocks - ref.blocks).abs().amax(dim=(1,2)) > 0).nonzero().flatten()
print("bad blocks", bad.numel(), bad[:10].tolist())
c3, st3 = D.multiply(D.LocalComm(), layout, a, b)
print("local equal", torch.equal(c3.blocks, ref.blocks))
c4, _ = D.multiply(comm, layout, a, b)
torch.cuda.synchronize()
print("again equal", torch.equal(c4.blocks, ref.blocks), torch.equal(c4.blocks, c2.blocks))
dist.destroy_process_group()
