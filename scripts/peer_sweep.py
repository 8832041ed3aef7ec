"""Randomised parity sweep of the sequence-sharded step at world size 1 (development tool): random
shapes / policies / lengths through PeerSeqShardedDecode with the one-kernel LL exchange and the
two-launch exchange, several consecutive steps each (both slot parities), against the fp64 oracle.

    python scripts/peer_sweep.py [n_cases] [seed]
"""
import os
import random
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from oracle import attention as OA  # noqa: E402
from paper_2604_00028_b200.dist import PeerSeqShardedDecode  # noqa: E402
from tests.helpers import assert_lse_close, assert_out_close  # noqa: E402

if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        os.environ["MASTER_PORT"] = str(s.getsockname()[1])
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    fails = 0
    for i in range(n):
        hkv = rng.choice([1, 2, 4, 8])
        G = rng.choice([1, 2, 8, 8, 16])
        b = rng.choice([1, 1, 2, 3, 6])
        lk = rng.choice([64, 300, 512, 1000, 2048, 4097, 9000])
        policy = rng.choice(["guarded", "seq_aware", "seq_aware_sm", "dynamic"])
        one = rng.random() < 0.7
        variant = rng.choice(["normal", "peaked", "ragged"])
        try:
            inp = synth.make_inputs(b, G * hkv, hkv, lk, seed=9000 + i, variant=variant, device="cuda")
            sd = PeerSeqShardedDecode(b, G * hkv, hkv, lk, device="cuda", policy=policy, one_kernel=one)
            ref_o, ref_l = OA.decode_attention(*(synth.to_f64(inp[k]) for k in ("q", "k", "v", "seqlens")))
            out = torch.empty((b, G * hkv, 128), dtype=torch.bfloat16, device="cuda")
            lse = torch.empty((b, G * hkv), dtype=torch.float32, device="cuda")
            for _ in range(3):
                out.fill_(float("nan"))
                sd.step(inp["q"], inp["k"], inp["v"], inp["seqlens"], out, lse)
                torch.cuda.synchronize()
                assert_out_close(synth.to_f64(out), ref_o)
                assert_lse_close(synth.to_f64(lse), ref_l)
            assert int(sd.epoch.item()) == 3 and int(sd.counter.item()) == 0
        except Exception as e:   # noqa: BLE001 - report and continue
            fails += 1
            print(f"FAIL case {i}: B={b} H_KV={hkv} G={G} L={lk} {policy} one_kernel={one} {variant}: {e}", flush=True)
    print(f"{n} cases, {fails} failures", flush=True)
    dist.destroy_process_group()
