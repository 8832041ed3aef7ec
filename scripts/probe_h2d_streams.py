"""Pinned H2D throughput of 2.1 MB copies (one Llama-70B decode step's K + V) issued on 1, 2 or 4
streams in flight, and of the full da_forward_host step pipelined over 1 or 2 streams."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

dev = torch.device("cuda", 0)
nb = 2113536
n = 200
for k in (1, 2, 4):
    hs = [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(k)]
    ds = [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(k)]
    sts = [torch.cuda.Stream() for _ in range(k)]
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sts[0])
        for s in sts[1:]:
            s.wait_event(e0)
        for i in range(n):
            j = i % k
            with torch.cuda.stream(sts[j]):
                ds[j].copy_(hs[j], non_blocking=True)
        for s in sts[1:]:
            ev = torch.cuda.Event()
            ev.record(s)
            sts[0].wait_event(ev)
        e1.record(sts[0])
        e1.synchronize()
        ms = e0.elapsed_time(e1)
    print(f"{k} stream(s): {nb * n / (ms * 1e-3) / 1e9:.1f} GB/s ({ms * 1e3 / n:.1f} us per 2.1 MB copy)", flush=True)
