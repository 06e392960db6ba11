"""The multi-GPU product with its real CUDA backend at world size 2 and 3 -- several ranks on the
one available B200, collectives over gloo (host-staged), so no GPU kernel ever waits on another
rank. Checks the gathered distributed product equals the single-GPU product bit for bit (every C
block's k sum is computed by one rank in the same order), balanced triples, halo traffic."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg_name, outdir, mode="exchange"):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from paper_2011_11762_b200 import _ffi, spgemm
    from paper_2011_11762_b200 import distributed as D
    from paper_2011_11762_b200 import generators as G

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    full = None
    if cfg_name == "masked":  # partial block supports: the support-mask filter runs distributed
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        import helpers

        from paper_2011_11762_b200 import MatrixSession
        from paper_2011_11762_b200.blocks import BlockSet

        ses = MatrixSession(device=dev)
        mats = [helpers.build(ses, helpers.banded_support_decay(2048, 20, 7 + m), 64, 64) for m in (0, 1)]
        geom = mats[0].geometry
        full = [m.root.blockset for m in mats]
        parts = []
        for m in (0, 1):
            n = full[m].n
            cut = np.r_[0, np.sort(np.random.default_rng(m).choice(n, world - 1, replace=False)), n]
            sl = slice(int(cut[rank]), int(cut[rank + 1]))
            parts.append(BlockSet(full[m].keys[sl].clone(), full[m].blocks[sl].clone(), full[m].sumsq[sl].clone()))
    else:
        cfg = (G.CONFIGS[cfg_name] if cfg_name in G.CONFIGS else
               G.BaselineConfig("t", "banded", 96, 32, half_bw=20) if cfg_name == "tiny" else
               G.BaselineConfig("r", "random", 8192, 64, per_row=8))
        geom = cfg.geometry
        parts = []
        for m in (0, 1):
            keys = G.config_keys(cfg, m)
            cut = np.r_[0, np.sort(np.random.default_rng(m).choice(keys.size, world - 1, replace=False)), keys.size]
            if cfg_name == "tiny":  # rank 0 owns no block (its pool is empty; peers still map it)
                cut = np.r_[0, 0, np.sort(np.random.default_rng(m).choice(np.arange(1, keys.size), world - 2,
                                                                          replace=False)), keys.size]
            parts.append(G.device_blocks(geom, keys[cut[rank]:cut[rank + 1]], cfg.seed, m, G.config_pattern(cfg),
                                         cfg.half_bw, dev))
    layout = _ffi.make_layout(geom.params, geom.bs)
    comm = D.Comm()
    c, st = D.multiply(comm, layout, parts[0], parts[1], mode=mode)
    assert st.mode == mode
    if mode in ("fused", "staged"):  # a repeated product reuses the cached peer mappings, bitwise equal
        mapped = dict(D._IPC_MAPPED)
        c2, st2 = D.multiply(comm, layout, parts[0], parts[1], mode=mode)
        assert st2.mode == mode and D._IPC_MAPPED == mapped
        assert torch.equal(c2.keys, c.keys) and torch.equal(c2.blocks, c.blocks)
    keys, _ = comm.allgather_varlen(c.keys)
    blocks, _ = comm.allgather_varlen(c.blocks.reshape(-1))
    info = torch.tensor([st.bytes_received, st.t_range[1] - st.t_range[0]], dtype=torch.int64)
    allinfo = [torch.zeros_like(info) for _ in range(world)]
    dist.all_gather(allinfo, info)
    if rank == 0:
        if full is None:
            full = [G.device_blocks(geom, G.config_keys(cfg, m), cfg.seed, m, G.config_pattern(cfg), cfg.half_bw,
                                    dev) for m in (0, 1)]
        ref = spgemm.multiply_blocks(layout, full[0], full[1])
        np.savez(os.path.join(outdir, "out.npz"),
                 same_keys=torch.equal(keys, ref.keys), same_blocks=torch.equal(blocks.view(ref.blocks.shape), ref.blocks)
                 if blocks.numel() == ref.blocks.numel() else False,
                 info=torch.stack(allinfo).numpy())
    torch.cuda.synchronize()
    D.release_peer_mappings()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["exchange", "fused", "staged"])
@pytest.mark.parametrize("world,cfg", [(2, "C1"), (3, "C2-16384"), (2, "random"), (3, "masked"), (4, "tiny")])
def test_multirank_cuda_backend_equals_single_gpu(tmp_path, world, cfg, mode):
    """mode "fused": the numeric kernel reads remote blocks through CUDA-IPC-mapped peer pools
    (qm_numeric_pools_ex) instead of an exchange; mode "staged": k_halo_gather pulls the halo
    from the mapped pools while local-only C blocks compute (the numeric kernel is its programmatic
    dependent) -- here the peers share the one GPU."""
    mp.spawn(_worker, args=(world, _free_port(), cfg, str(tmp_path), mode), nprocs=world, join=True)
    out = np.load(tmp_path / "out.npz")
    assert bool(out["same_keys"]) and bool(out["same_blocks"])
    info = out["info"]
    assert info[:, 0].sum() > 0  # blocks crossed ranks
    tr = info[:, 1]
    if cfg != "masked":  # (masked products are balanced on executed k panels, not triples)
        assert tr.max() - tr.min() <= 17 + 1  # balanced by triples within one C block's k list
