import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2011_11762_b200 import _ffi, spgemm, generators as G
dev = torch.device("cuda:0")
E = lambda: torch.cuda.Event(enable_timing=True)
for cfg in [G.BaselineConfig("b", "banded", 4096, 64, half_bw=256), G.BaselineConfig("b", "banded", 8192, 64, half_bw=512),
            G.BaselineConfig("b", "banded", 12288, 64, half_bw=512), G.BaselineConfig("r", "random", 16384, 64, per_row=4)]:
    geom, a, b = G.config_operands_device(cfg, dev)
    lay = _ffi.make_layout(geom.params, geom.bs)
    for mode in ("rank", "smallsort", "rank", "smallsort"):
        os.environ["QM_RANK_ORDER"] = "1" if mode == "rank" else "0"
        os.environ["QM_SMALL_SORT"] = "0" if mode == "rank" else "1"
        res = []
        for it in range(40):
            ev = {k: E() for k in ("symbolic", "numeric", "end")}
            st = spgemm.MultiplyStats()
            t0 = E(); t0.record()
            spgemm.multiply_blocks(lay, a, b, events=ev, stats=st)
            t1 = E(); t1.record()
            torch.cuda.synchronize()
            if it >= 10: res.append((ev["symbolic"].elapsed_time(ev["numeric"]), t0.elapsed_time(t1)))
        sym, tot = np.median(np.array(res), axis=0)
        print(f"{cfg.kind} n={cfg.n}: nC={st.n_c_symbolic} {mode:9s} symbolic {sym*1e3:.1f} us  product {tot*1e3:.1f} us", flush=True)
