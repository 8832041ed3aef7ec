"""Paged decode latency on the headline shapes with the page pools rotated through > 2x L2 (cold L2,
like bench.py): the pre-wait page prefetch steered by the block table."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_00028_b200 as dec  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
l2 = torch.cuda.get_device_properties(0).L2_cache_size
timer = bench.Timer(dev)
stream = torch.cuda.Stream()
for (b, hq, hkv, lk) in ((1, 64, 8, 512), (1, 8, 1, 512), (4, 32, 4, 1024)):
    for ps in (64, 256):
        inp = synth.make_inputs(b, hq, hkv, lk, device=dev, seed=7)
        P = -(-lk // ps)
        pool_bytes = 4 * b * P * ps * hkv * 128
        nbuf = max(2, min(512, -(-3 * l2 // pool_bytes)))
        g0 = torch.Generator(device="cpu").manual_seed(1)
        perm = torch.randperm(b * P, generator=g0).to(dev)
        kp0 = torch.empty((b * P, ps, hkv, 128), dtype=torch.bfloat16, device=dev)
        vp0 = torch.empty_like(kp0)
        kp0[perm] = inp["k"].reshape(b * P, ps, hkv, 128)
        vp0[perm] = inp["v"].reshape(b * P, ps, hkv, 128)
        kps = kp0.unsqueeze(0).repeat(nbuf, 1, 1, 1, 1)
        vps = vp0.unsqueeze(0).repeat(nbuf, 1, 1, 1, 1)
        table = perm.view(b, P).to(torch.int32).contiguous()
        plan = dec.make_plan(b, hq, hkv, lk, policy="seq_aware_sm")
        steps = 200
        with torch.cuda.stream(stream):
            for i in range(3):
                dec.forward_paged(plan, inp["q"], kps[i % nbuf], vps[i % nbuf], table, None)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for i in range(steps):
                dec.forward_paged(plan, inp["q"], kps[i % nbuf], vps[i % nbuf], table, None)
        ts = [timer.time_replay(g, stream) * 1e3 / steps for _ in range(7)]
        print(f"paged B={b} H_Q={hq} H_KV={hkv} L={lk} page={ps} s={plan.num_splits} nbuf={nbuf}: "
              f"{statistics.median(ts):.3f} us/step", flush=True)
        del g, kps, vps
        torch.cuda.empty_cache()
