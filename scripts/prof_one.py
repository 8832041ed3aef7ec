"""One shape's forward, eager, a few times (development tool: the target of an ncu capture).

    python scripts/prof_one.py B H_Q H_KV L_K policy [forced] [combine]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2604_00028_b200 as dec
import synth

if __name__ == "__main__":
    b, hq, hkv, lk = (int(x) for x in sys.argv[1:5])
    pol = sys.argv[5]
    forced = int(sys.argv[6]) if len(sys.argv) > 6 else 0
    comb = int(sys.argv[7]) if len(sys.argv) > 7 else None
    inp = synth.make_inputs(b, hq, hkv, lk, device="cuda", seed=3)
    plan = dec.make_plan(b, hq, hkv, lk, policy=pol, forced_splits=forced, combine_mode=comb)
    ws = dec.workspace_for(plan, inp["q"].device)
    for _ in range(8):
        dec.forward(plan, inp["q"], inp["k"], inp["v"], None, workspace=ws)
    torch.cuda.synchronize()
    print(f"ok s={plan.num_splits} comb={plan.combine_mode}")
