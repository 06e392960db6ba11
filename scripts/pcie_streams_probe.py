"""Pinned copy bandwidth with the copy split over 1/2/4 streams per direction (copy engines)."""
import torch

n = 2 * 1024**3 // 8
dev = torch.device("cuda:0")
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_in = torch.empty(n, dtype=torch.float64, device=dev)
d_out = torch.empty(n, dtype=torch.float64, device=dev)
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def run(k, h2d, d2h):
    streams = [torch.cuda.Stream() for _ in range(2 * k)]
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = E(), E()
        e0.record()
        for s in streams:
            s.wait_event(e0)
        c = n // k
        for i in range(k):
            if h2d:
                with torch.cuda.stream(streams[i]):
                    d_in[i * c:(i + 1) * c].copy_(h_in[i * c:(i + 1) * c], non_blocking=True)
            if d2h:
                with torch.cuda.stream(streams[k + i]):
                    h_out[i * c:(i + 1) * c].copy_(d_out[i * c:(i + 1) * c], non_blocking=True)
        for s in streams:
            e = E()
            e.record(s)
            torch.cuda.current_stream().wait_event(e)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return (h2d + d2h) * n * 8 / (best * 1e-3) / 1e9


for k in (1, 2, 4):
    print(f"streams/direction {k}: H2D {run(k, 1, 0):.1f}  D2H {run(k, 0, 1):.1f}  both {run(k, 1, 1):.1f} GB/s")
