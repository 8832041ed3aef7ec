"""Where the e2e (host-buffer) step time goes: raw pinned H2D bandwidth, the host-side enqueue cost of
da_forward_host, and the device time per step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_00028_b200 as dec  # noqa: E402
from paper_2604_00028_b200 import _lib as L  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
for mb in (1, 2, 4, 16, 64):
    h = torch.empty(mb << 20, dtype=torch.uint8).pin_memory()
    d = torch.empty(mb << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 50
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(n):
            d.copy_(h, non_blocking=True)
        e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"H2D {mb:3d} MB pinned: {ms * 1e3:8.1f} us  {mb * 1.048576 / ms:6.1f} GB/s")

cfg = synth.CONFIGS["llama70b"]
b, hq, hkv, lk = cfg["batch"], cfg["h_q"], cfg["h_kv"], cfg["l_k"]
inp = synth.make_inputs(b, hq, hkv, lk, seed=2000)
q, k, v = (inp[n].contiguous().pin_memory() for n in ("q", "k", "v"))
out = torch.empty((b, hq, 128), dtype=torch.bfloat16).pin_memory()
lse = torch.empty((b, hq), dtype=torch.float32).pin_memory()
staging = dec.HostStaging(dev)
plan = dec.make_plan(b, hq, hkv, lk, policy="seq_aware_sm")
for _ in range(5):
    dec.forward_host(plan, q, k, v, None, out=out, lse=lse, staging=staging, stream=s)
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for _ in range(n):
    L.da_plan_make(b, hq, hkv, lk, 128, 1, 0, 148, L.POLICIES["seq_aware_sm"], 0)
t1 = time.perf_counter()
print(f"da_plan_make via ctypes: {(t1 - t0) / n * 1e6:.1f} us")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
t0 = time.perf_counter()
for _ in range(n):
    dec.forward_host(plan, q, k, v, None, out=out, lse=lse, staging=staging, stream=s)
t1 = time.perf_counter()
e1.record(s)
e1.synchronize()
print(f"forward_host: host enqueue {(t1 - t0) / n * 1e6:.1f} us/step, device {e0.elapsed_time(e1) / n * 1e3:.1f} us/step")
buf = staging.get(0)
nbytes = L.da_forward_host_bytes(plan, lk, 0, L.DA_BF16)
t0 = time.perf_counter()
e0.record(s)
for _ in range(n):
    L.da_forward_host(plan, q, k, v, lk, None, 0.0, L.DA_BF16, out, lse, buf, nbytes, s)
t1 = time.perf_counter()
e1.record(s)
e1.synchronize()
print(f"raw ctypes da_forward_host: host enqueue {(t1 - t0) / n * 1e6:.1f} us/step, device {e0.elapsed_time(e1) / n * 1e3:.1f} us/step")

# joint [2, ...] KV + out|lse allocations (one DMA each way) vs separate pinned tensors, interleaved
kvj = torch.empty((2,) + tuple(k.shape), dtype=torch.bfloat16).pin_memory()
kvj[0].copy_(k)
kvj[1].copy_(v)
ob = b * hq * 128 * 2
ol = torch.empty(ob + 4 * b * hq, dtype=torch.uint8).pin_memory()
outj, lsej = ol[:ob].view(torch.bfloat16).view(b, hq, 128), ol[ob:].view(torch.float32).view(b, hq)
for rep in range(3):
    for name, (kk, vv, oo, ll) in (("separate", (k, v, out, lse)), ("joint", (kvj[0], kvj[1], outj, lsej))):
        for _ in range(5):
            dec.forward_host(plan, q, kk, vv, None, out=oo, lse=ll, staging=staging, stream=s)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(n):
            dec.forward_host(plan, q, kk, vv, None, out=oo, lse=ll, staging=staging, stream=s)
        e1.record(s)
        e1.synchronize()
        print(f"{name:9s}: {e0.elapsed_time(e1) / n * 1e3:.1f} us/step")
