"""Per-CTA timeline of the one-kernel sequence-sharded step (da_forward_peer_combine) from a
-DDECATTN_TRACE build at world size 1 (development tool):
DECATTN_LIB=paper_2604_00028_b200/lib/variants/libdecattn_trace.so python scripts/trace_peer.py [P]
Slots (globaltimer ns, relative to the previous step's end stamp): 1 after griddepcontrol.wait,
26 epilogue start, 29 cluster pushes received, 47 rows stored, 48 after the publish (count /
last-CTA release), 49 after every rank's flag, 30 CTA end (rows merged and stored)."""
import ctypes
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2604_00028_b200 import _lib as L  # noqa: E402
from paper_2604_00028_b200.dist import PeerSeqShardedDecode  # noqa: E402
import synth  # noqa: E402

L.LIB.da_trace_fetch.argtypes = [ctypes.c_void_p, ctypes.c_int]

if __name__ == "__main__":
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        os.environ["MASTER_PORT"] = str(s.getsockname()[1])
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    lk = 131072 // P
    inp = synth.make_inputs(1, 64, 8, lk, seed=3, device="cuda")
    nbuf = 8
    ks = [inp["k"].clone() for _ in range(nbuf)]
    vs = [inp["v"].clone() for _ in range(nbuf)]
    for one in (True, False):
        sd = PeerSeqShardedDecode(1, 64, 8, lk, device="cuda", policy="seq_aware_sm", one_kernel=one)
        out = torch.empty((1, 64, 128), dtype=torch.bfloat16, device="cuda")
        lse = torch.empty((1, 64), dtype=torch.float32, device="cuda")
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for i in range(3):
                sd.step(inp["q"], ks[i % nbuf], vs[i % nbuf], None, out, lse)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(20):
                sd.step(inp["q"], ks[i % nbuf], vs[i % nbuf], None, out, lse)
        for _ in range(3):
            with torch.cuda.stream(st):
                g.replay()
            torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * (64 * 64))()
        L.LIB.da_trace_fetch(ctypes.addressof(buf), 64 * 64)
        rows = [[buf[c * 64 + j] for j in range(64)] for c in range(64)]
        t0 = min(r[63] for r in rows if r[63])
        print(f"== P={P} shard L_K={lk} one_kernel={sd.one_kernel} s={sd.plan.num_splits} "
              f"combine={sd.plan.combine_mode}; ns after the previous step's end stamp")
        for c in (0, 1, 9, 10, 40, 63):
            r = rows[c]
            print(f"  cta{c:2d}: " + " ".join(f"{n}={int(r[j]) - t0}" for n, j in
                                            (("wait", 1), ("epi", 26), ("push_in", 29), ("stored", 47),
                                             ("pub", 48), ("flags", 49), ("end", 30)) if r[j]))
        for n, j in (("epi", 26), ("push_in", 29), ("stored", 47), ("pub", 48), ("flags", 49), ("end", 30)):
            v = [int(r[j]) - t0 for r in rows if r[j]]
            if v:
                print(f"  {n:8s} min {min(v):6d} max {max(v):6d} (of {len(v)} traced CTAs)")
    dist.destroy_process_group()
