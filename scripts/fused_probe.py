"""3-rank fused-mode probe on one GPU with faulthandler (debugging aid)."""
import faulthandler, os, socket, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, torch.multiprocessing as mp

def worker(rank, world, port):
    faulthandler.enable()
    import torch.distributed as dist
    from paper_2011_11762_b200 import _ffi, spgemm
    from paper_2011_11762_b200 import distributed as D
    from paper_2011_11762_b200 import generators as G
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
    cfg = G.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2-16384"]
    geom = cfg.geometry
    parts = []
    for m in (0, 1):
        keys = G.config_keys(cfg, m)
        cut = np.r_[0, np.sort(np.random.default_rng(m).choice(keys.size, world - 1, replace=False)), keys.size]
        parts.append(G.device_blocks(geom, keys[cut[rank]:cut[rank + 1]], cfg.seed, m, G.config_pattern(cfg), cfg.half_bw, dev))
    layout = _ffi.make_layout(geom.params, geom.bs)
    comm = D.Comm()
    print(rank, "start", flush=True)
    c, st = D.multiply(comm, layout, parts[0], parts[1], mode="fused")
    print(rank, "done", c.n, st.mode, flush=True)
    torch.cuda.synchronize(); dist.barrier(); print(rank, "exit", flush=True)
    dist.destroy_process_group()

if __name__ == "__main__":
    world = int(os.environ.get("WORLD", "3"))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
    mp.spawn(worker, args=(world, port), nprocs=world, join=True)
