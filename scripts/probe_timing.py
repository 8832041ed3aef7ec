"""Quick CUDA-graph timing probe of the forward path (development tool).

python scripts/probe_timing.py  -> prints us/step and GB/s for a few shapes/policies.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2604_00028_b200 as dec
import synth

L2 = torch.cuda.get_device_properties(0).L2_cache_size


def bytes_step(b, hq, hkv, lk):
    return 4 * b * lk * hkv * 128 + 4 * b * hq * 128 + 4 * b * hq


def bench(b, hq, hkv, lk, policy="seq_aware", forced=0, combine=None, steps=200, reps=5, pack=True,
          rotate=True, path=None):
    kvb = 4 * b * lk * hkv * 128
    nbuf = max(1, min(256, -(-2 * L2 // kvb))) if rotate else 1
    ins = [synth.make_inputs(b, hq, hkv, lk, device="cuda", seed=i) for i in range(min(nbuf, 2))]
    ks = [ins[i % len(ins)]["k"].clone() for i in range(nbuf)]
    vs = [ins[i % len(ins)]["v"].clone() for i in range(nbuf)]
    q, seq = ins[0]["q"], ins[0]["seqlens"]
    plan = dec.make_plan(b, hq, hkv, lk, pack_gqa=pack, policy=policy, forced_splits=forced,
                         combine_mode=combine, path=path)
    ws = dec.workspace_for(plan, q.device)
    out = torch.empty_like(q)
    lse = torch.empty(b, hq, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(3):
            dec.forward(plan, q, ks[i % nbuf], vs[i % nbuf], seq, out=out, lse=lse, workspace=ws)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(steps):
                dec.forward(plan, q, ks[i % nbuf], vs[i % nbuf], seq, out=out, lse=lse, workspace=ws)
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / steps)
    ts.sort()
    us = ts[len(ts) // 2]
    gbs = bytes_step(b, hq, hkv, lk) / (us * 1e-6) / 1e9
    print(f"B={b:4d} HQ={hq:3d} HKV={hkv:2d} L={lk:7d} pack={int(pack)} {policy:9s} s={plan.num_splits:3d} "
          f"comb={plan.combine_mode} path={plan.path} nbuf={nbuf:3d}: {us:9.2f} us/step  {gbs:8.1f} GB/s", flush=True)
    return us


if __name__ == "__main__":
    for lk in (128, 256, 384, 512):
        for hkv in (1, 2, 8):
            bench(1, 8 * hkv, hkv, lk, "guarded")
            bench(1, 8 * hkv, hkv, lk, "seq_aware")
    bench(1, 8, 1, 192, "fixed", 1)
    bench(1, 8, 1, 64, "fixed", 1)
    for s in (1, 2, 3, 4, 6, 8):
        bench(1, 8, 1, 512, "fixed", s)
    for s in (2, 3, 4, 8, 16):
        bench(1, 8, 1, 512, "fixed", s, combine=2)
    bench(1, 8, 1, 512, "guarded", rotate=False)
    bench(1, 8, 1, 512, "seq_aware", rotate=False)
    bench(1, 64, 8, 512, "seq_aware", pack=False)
    bench(1, 64, 8, 131072, "seq_aware", steps=20)
    bench(1, 64, 8, 131072, "fixed", 32, steps=20)
    bench(1, 64, 8, 131072, "fixed", 64, steps=20)
    bench(128, 64, 8, 8192, "seq_aware", steps=5, reps=3)
    bench(128, 64, 8, 8192, "seq_aware", steps=5, reps=3, pack=False)
