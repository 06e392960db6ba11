"""Host cost of individual library calls of one small product (C1), GPU idle vs queued:
workspace queries (CUB size queries), qm_spgemm_count (launches + sync), torch allocations."""
import ctypes
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_2011_11762_b200 import generators as G
from paper_2011_11762_b200 import _ffi, spgemm

cfg = G.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
dev = torch.device("cuda:0")
geom, a, b = G.config_operands_device(cfg, dev)
lay = _ffi.make_layout(geom.params, geom.bs)
lib = _ffi.load()
lp = ctypes.byref(lay)
st = torch.cuda.current_stream()
N = 2000


def t(fn, n=N):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


print("qm_spgemm_workspace_bytes   %.2f us" % t(lambda: lib.qm_spgemm_workspace_bytes(lp, a.n, b.n)))
print("qm_spgemm_fill_ws_bytes     %.2f us" % t(lambda: lib.qm_spgemm_fill_workspace_bytes(lp, 1016)))
print("qm_numeric_workspace_bytes  %.2f us" % t(lambda: lib.qm_numeric_workspace_bytes(64, 1016, 4884)))
print("torch.empty (device)        %.2f us" % t(lambda: torch.empty(1000, dtype=torch.int64, device=dev)))
print("torch.zeros (device)        %.2f us" % t(lambda: torch.zeros(1, dtype=torch.int64, device=dev)))
print("SymbolicState (count+sync)  %.2f us" % t(lambda: spgemm.SymbolicState(lay, a.keys, a.n, b.keys, b.n, st), 500))
s = spgemm.SymbolicState(lay, a.keys, a.n, b.keys, b.n, st)
plan = spgemm.symbolic(lay, a, b, st)
print("symbolic (count+fill)       %.2f us" % t(lambda: spgemm.symbolic(lay, a, b, st), 500))
print("numeric (launch only)       %.2f us" % t(lambda: spgemm.numeric(lay, a, b, plan, st), 200))
print("multiply_blocks             %.2f us" % t(lambda: spgemm.multiply_blocks(lay, a, b, st), 500))
# GPU kept busy: host-side cost of queueing a numeric call
big = torch.empty(1 << 28, dtype=torch.uint8, device=dev)
def busy_numeric():
    torch.cuda._sleep(20_000_000)
    t0 = time.perf_counter()
    spgemm.numeric(lay, a, b, plan, st)
    return time.perf_counter() - t0
ts = [busy_numeric() for _ in range(20)]
torch.cuda.synchronize()
print("numeric host enqueue (GPU busy) %.2f us" % (sorted(ts)[10] * 1e6))
# raw qm_numeric call (GPU busy)
out_b = torch.empty((plan.n_c, geom.bs, geom.bs), dtype=torch.float64, device=dev)
out_s = torch.empty(plan.n_c, dtype=torch.float64, device=dev)
nz = torch.empty(plan.n_c, dtype=torch.uint8, device=dev)
zc = torch.empty(1, dtype=torch.int64, device=dev)
wb = lib.qm_numeric_workspace_bytes(geom.bs, plan.n_c, plan.n_triples)
ws = torch.empty(wb, dtype=torch.uint8, device=dev)
P = _ffi.ptr
def busy_raw():
    torch.cuda._sleep(20_000_000)
    t0 = time.perf_counter()
    lib.qm_numeric(lp, P(a.keys), P(a.blocks), a.n, P(b.blocks), b.n, P(plan.tri), P(plan.c_tptr),
                   P(plan.c_keys), plan.n_c, plan.n_triples, P(out_b), P(out_s), P(nz), P(zc), P(ws), wb,
                   _ffi.stream_handle(st))
    return time.perf_counter() - t0
ts = [busy_raw() for _ in range(20)]
torch.cuda.synchronize()
print("qm_numeric ctypes call (GPU busy) %.2f us" % (sorted(ts)[10] * 1e6))
