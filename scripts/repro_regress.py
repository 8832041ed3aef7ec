import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "scripts"))
import torch
import sweeps
from sweeps import dec
for (b, hkv, lk) in [(1, 8, 128), (1, 32, 128), (1, 32, 256)]:
    cfg = dict(batch=b, h_q=8 * hkv, h_kv=hkv, l_k=lk)
    plans = [dec.make_plan(b, 8 * hkv, hkv, lk, policy=p) for p in sweeps.REG_POLICIES]
    print(cfg, [(p.num_splits, p.combine_mode) for p in plans], flush=True)
    t, raw = sweeps.timed_graphs(cfg, plans, sweeps.steps_for(cfg), 3, 7, control=True, raw=True)
    print("  ", [round(x[0], 3) for x in t], flush=True)
