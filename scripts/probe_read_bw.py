"""Read-only HBM bandwidth reference (development tool): torch reductions over a 4 GiB buffer,
CUDA events, best of 10 - the read-side ceiling the split-KV kernel's GB/s is compared with
(MEASURED_PEAKS.json's copy figure counts a read and a write per byte).

    python scripts/probe_read_bw.py      (on the GPU box)"""
import torch

if __name__ == "__main__":
    n = 2 << 30                                   # 2 Gi bf16 = 4 GiB
    x = torch.randn(n // 1024, 1024, device="cuda").to(torch.bfloat16)
    for name, fn in (("sum(dtype=f32)", lambda: x.sum(dtype=torch.float32)),
                     ("amax", lambda: x.amax()),
                     ("sum over rows", lambda: x.sum(dim=0, dtype=torch.float32))):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b) * 1e-3)
        print(f"{name:16s} {x.numel() * 2 / best / 1e9:8.1f} GB/s read ({best * 1e6:.0f} us for {x.numel() * 2 >> 20} MiB)",
              flush=True)
