"""The peer-exchange step at one rank (world size 1 NCCL group + torch symmetric memory) on the
per-rank shard of the long-context config at P = 2, 4, 8 (B = 1, H_Q = 64, H_KV = 8,
L_K = 131072 / P), CUDA-graph replay, KV rotated past L2:
  fwd    the forward alone (fp32 partial into a local buffer)
  one    da_forward_peer_combine (1 launch: publish + wait + cross-rank combine in the forward)
  fused  da_forward_peer -> da_combine_peers (2 launches)
  split  forward -> da_peer_signal -> da_combine_peers (3 launches)"""
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2604_00028_b200 as dec  # noqa: E402
import synth  # noqa: E402
from paper_2604_00028_b200.dist import PeerSeqShardedDecode  # noqa: E402


def graph_us(fn, nbuf, steps=int(os.environ.get("PROBE_STEPS", "50")), reps=int(os.environ.get("PROBE_REPS", "7"))):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(3):
            fn(i % nbuf)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(steps):
            fn(i % nbuf)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st)
            g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / steps)
    return sorted(ts)[len(ts) // 2]


def main():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    for P in [int(x) for x in (sys.argv[1:] or ["1", "2", "4", "8"])]:
        lk = 131072 // P
        inp = synth.make_inputs(1, 64, 8, lk, seed=1700, device="cuda")
        nbuf = max(2, (400 << 20) // (inp["k"].numel() * 4) + 1)
        ks = [inp["k"].clone() for _ in range(nbuf)]
        vs = [inp["v"].clone() for _ in range(nbuf)]
        out = torch.empty((1, 64, 128), dtype=torch.bfloat16, device="cuda")
        lse = torch.empty((1, 64), dtype=torch.float32, device="cuda")
        o32 = torch.empty((1, 64, 128), dtype=torch.float32, device="cuda")
        res = {"fwd": [], "one": [], "fused": [], "split": []}
        plan = None
        for _ in range(2):
            sd = {f: PeerSeqShardedDecode(1, 64, 8, lk, device="cuda", fused=f != "split", one_kernel=f == "one",
                                          policy=os.environ.get("PROBE_POLICY", "seq_aware_sm"))
                  for f in ("one", "fused", "split")}
            plan = sd["fused"].plan
            ws = dec.workspace_for(plan, torch.device("cuda"))
            res["fwd"].append(graph_us(lambda i: dec.forward(plan, inp["q"], ks[i], vs[i], None, out=o32, lse=lse,
                                                             workspace=ws, out_dtype=torch.float32), nbuf))
            for f in ("one", "fused", "split"):
                res[f].append(graph_us(lambda i, f=f: sd[f].step(inp["q"], ks[i], vs[i], None, out, lse), nbuf))
            del sd
        r = {k: min(v) for k, v in res.items()}
        print(f"P={P} shard L_K={lk} s={plan.num_splits} mode={plan.combine_mode}: fwd {r['fwd']:.2f} us, "
              f"one-kernel step {r['one']:.2f} us, fused (2 launches) {r['fused']:.2f} us, split (3 launches) "
              f"{r['split']:.2f} us", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
