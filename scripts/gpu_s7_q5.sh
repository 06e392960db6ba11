# bs 32 quad kernel as the default: full GPU suite + A/B on several bs 32 products.
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
cat > /tmp/bs32_ab.py <<'PY'
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2011_11762_b200 import _ffi, spgemm, generators as G
dev = torch.device("cuda:0")
E = lambda: torch.cuda.Event(enable_timing=True)
for cfg in [G.BaselineConfig("b", "banded", 131072, 32, half_bw=512), G.BaselineConfig("r", "random", 32768, 32, per_row=8),
            G.BaselineConfig("b2", "banded", 16384, 32, half_bw=128), G.BaselineConfig("r2", "random", 131072, 32, per_row=16)]:
    geom, a, b = G.config_operands_device(cfg, dev)
    lay = _ffi.make_layout(geom.params, geom.bs)
    for q in ("1", "0", "1", "0"):
        os.environ["QM_QUAD32"] = q
        res = []
        for it in range(8):
            ev = {k: E() for k in ("symbolic", "numeric", "end")}
            st = spgemm.MultiplyStats()
            spgemm.multiply_blocks(lay, a, b, events=ev, stats=st)
            torch.cuda.synchronize()
            if it >= 3: res.append(ev["numeric"].elapsed_time(ev["end"]))
        num = float(np.median(res))
        print(f"{cfg.kind} n={cfg.n} quad={q}: T={st.n_triples} nC={st.n_c_symbolic} numeric {num:.3f} ms = {st.flops / num / 1e9:.2f} TFLOP/s", flush=True)
PY
timeout 900 python /tmp/bs32_ab.py 2>&1 | grep -v Warn
