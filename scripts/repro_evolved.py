import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2604_00028_b200 as dec
from oracle import attention as OA
from tests.helpers import assert_out_close, assert_lse_close
cfgs = [(1, 256, 32, 128), (1, 64, 8, 128), (2, 256, 32, 128), (1, 256, 32, 256), (1, 256, 32, 512), (1, 256, 32, 1024)]
for (b, hq, hkv, lk) in cfgs:
    for pol in sys.argv[1].split(","):
        inp = synth.make_inputs(b, hq, hkv, lk, device="cuda", seed=1)
        plan = dec.make_plan(b, hq, hkv, lk, policy=pol)
        print(b, hq, hkv, lk, pol, "s", plan.num_splits, "comb", plan.combine_mode, "grid", plan.grid_x, plan.grid_y, plan.grid_z, "rows", plan.rows_per_cta, flush=True)
        out, lse = dec.forward(plan, inp["q"], inp["k"], inp["v"], None)
        torch.cuda.synchronize()
        ro, rl = OA.decode_attention(*(synth.to_f64(inp[n]) for n in ("q", "k", "v", "seqlens")))
        assert_out_close(synth.to_f64(out), ro); assert_lse_close(synth.to_f64(lse), rl)
        print("  ok", flush=True)
