"""Latency of reading a device int64 to the host while a large D2H copy saturates PCIe:
mapped-memory write by a kernel (qm_read_i64) vs an 8-byte cudaMemcpyAsync on another stream vs
a host poll of a mapped flag set by the kernel stream."""
import sys
import time

sys.path.insert(0, ".")
import ctypes

import torch

from paper_2011_11762_b200 import _ffi

dev = torch.device("cuda:0")
lib = _ffi.load()
n = 2 * 1024**3 // 8
d_big = torch.empty(n, dtype=torch.float64, device=dev)
h_big = torch.empty(n, dtype=torch.float64, pin_memory=True)
v = torch.full((2,), 7, dtype=torch.int64, device=dev)
h8 = torch.empty(2, dtype=torch.int64, pin_memory=True)
s_copy, s_work, s_small = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def with_d2h(fn, label):
    torch.cuda.synchronize()
    with torch.cuda.stream(s_copy):
        h_big.copy_(d_big, non_blocking=True)  # ~40 ms of D2H traffic
    time.sleep(0.005)
    t = time.perf_counter()
    fn()
    dt = time.perf_counter() - t
    torch.cuda.synchronize()
    print(f"{label}: {dt * 1e3:.3f} ms (during a 2 GiB D2H)")


def alone(fn, label):
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn()
    print(f"{label}: {(time.perf_counter() - t) * 1e3:.3f} ms (idle link)")


def mapped():
    out = (ctypes.c_int64 * 2)()
    _ffi.check(lib.qm_read_i64(_ffi.ptr(v), 2, out, _ffi.stream_handle(s_work)), "read")


def memcpy_small():
    with torch.cuda.stream(s_small):
        h8.copy_(v, non_blocking=True)
    s_small.synchronize()


for f, name in ((mapped, "mapped write (qm_read_i64)"), (memcpy_small, "8-byte cudaMemcpyAsync")):
    for _ in range(2):
        alone(f, name)
        with_d2h(f, name)
