"""Launch the TP-8 slice decode step (guarded s=1, then seq-aware s=3) 50 times each (profiling target)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_00028_b200 as dec
import synth

w = synth.make_inputs(1, 8, 1, 512, device="cuda", seed=3)
for pol in ("seq_aware", "guarded"):
    plan = dec.make_plan(1, 8, 1, 512, policy=pol)
    for _ in range(50):
        dec.forward(plan, w["q"], w["k"], w["v"], None)
torch.cuda.synchronize()
print("ok")
