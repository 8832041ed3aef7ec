"""Randomised GPU parity sweep against the fp64 oracle (development tool; the pinned cases live in
tests/test_gpu_parity.py): random (B, H_KV, G, L_K, policy, combine, variant, pack_gqa, paged,
sequence-shard offset) draws, every output element and lse checked with the test tolerances
(DESIGN.md C-amb-14).  Round 2 adds long lengths (tail-balanced cluster splits), explicit combine
modes and da_plan_set_seq_offset shards (whole-sequence lengths in, the shard's part attended),
and plans forced onto the tcgen05 kernel.

    python scripts/parity_sweep.py [n_cases] [seed]
"""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_00028_b200 as dec  # noqa: E402
import synth  # noqa: E402
from oracle import attention as OA  # noqa: E402
from tests.helpers import assert_lse_close, assert_out_close  # noqa: E402

if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
    fails = 0
    for i in range(n):
        hkv = rng.choice([1, 1, 2, 3, 4, 8])
        G = rng.choice([1, 2, 4, 5, 8, 8, 12, 16, 24, 64])
        b = rng.choice([1, 1, 2, 3, 5, 8])
        lk = rng.choice([1, 7, 63, 64, 65, 100, 300, 511, 512, 513, 1000, 2048, 3000, 4097, 6000, 16448, 40000])
        if lk > 10000:            # keep the fp64 oracle fast: few query heads and sequences
            b, G = min(b, 2), min(G, 8)
        policy = rng.choice(["guarded", "seq_aware", "seq_aware_sm", "evolved", "dynamic", "fixed"])
        forced = rng.randint(1, 40) if policy == "fixed" else 0
        variant = rng.choice(["normal", "peaked", "ragged"])
        pack = rng.random() < 0.85
        l_cap = lk + rng.choice([0, 0, 64, 129])
        comb, offset = None, 0
        try:
            inp = synth.make_inputs(b, G * hkv, hkv, lk, l_cap=l_cap, seed=5000 + i, variant=variant, device="cuda")
            if policy == "fixed" and forced > 1 and rng.random() < 0.5:
                comb = 1 if forced <= 16 and rng.random() < 0.6 else 2
            offset = rng.choice([0, 0, 0, 64, 1000, 77777])
            # the tcgen05 kernel forced on a fifth of the packed static plans (any G >= 2; the
            # planner alone picks it only for wide groups on long enough splits)
            path = 2 if (pack and G >= 2 and policy != "dynamic" and comb != 1 and rng.random() < 0.2) else None
            if comb == 1 and dec.make_plan(b, G * hkv, hkv, lk, pack_gqa=pack, policy=policy, forced_splits=forced,
                                           path=path).path == dec.DA_PATH_TC:
                comb = 2          # the tcgen05 kernel has no cluster combine (da_plan_set_combine rejects it)
            plan = dec.make_plan(b, G * hkv, hkv, lk, pack_gqa=pack, policy=policy, forced_splits=forced,
                                 combine_mode=comb, seq_offset=offset, path=path)
            seq_arg = inp["seqlens"]
            if offset:                # a shard: whole-sequence lengths in; some end before the shard
                seq_arg = inp["seqlens"] + offset
                if b >= 2:
                    seq_arg[0] = rng.randint(0, offset)
                inp["seqlens"] = (seq_arg.to(torch.int64) - offset).clamp(0, l_cap).to(torch.int32)
            odt = rng.choice([torch.bfloat16, torch.float32])
            if rng.random() < 0.25 and policy != "dynamic":   # paged: the same cache in a shuffled page pool
                ps = rng.choice([64, 128, 256])
                npg = -(-l_cap // ps)
                k = torch.zeros((b, npg * ps, hkv, 128), dtype=torch.bfloat16, device="cuda")
                v = torch.zeros_like(k)
                k[:, :l_cap], v[:, :l_cap] = inp["k"], inp["v"]
                perm = torch.randperm(b * npg, device="cuda")
                kp = torch.empty((b * npg, ps, hkv, 128), dtype=torch.bfloat16, device="cuda")
                vp = torch.empty_like(kp)
                kp[perm] = k.reshape(b * npg, ps, hkv, 128)
                vp[perm] = v.reshape(b * npg, ps, hkv, 128)
                table = perm.view(b, npg).to(torch.int32).contiguous()
                out, lse = dec.forward_paged(plan, inp["q"], kp, vp, table, seq_arg, out_dtype=odt)
            else:
                out, lse = dec.forward(plan, inp["q"], inp["k"], inp["v"], seq_arg, out_dtype=odt)
            torch.cuda.synchronize()
            ref_o, ref_l = OA.decode_attention(*(synth.to_f64(inp[k]) for k in ("q", "k", "v", "seqlens")))
            assert_out_close(synth.to_f64(out), ref_o)
            assert_lse_close(synth.to_f64(lse), ref_l)
        except Exception as e:   # noqa: BLE001 - report and continue the sweep
            fails += 1
            print(f"FAIL case {i}: B={b} H_KV={hkv} G={G} L={lk} cap={l_cap} {policy} s={forced} {variant} "
                  f"pack={pack} comb={comb} offset={offset} path={plan.path if 'plan' in dir() else '?'}: {e}", flush=True)
    print(f"{n} cases, {fails} failures", flush=True)
