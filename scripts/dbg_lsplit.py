import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2604_00028_b200 as dec, synth
from oracle import attention as OA
def run(b,hq,hkv,lk,s,comb=None,pol="fixed"):
    inp = synth.make_inputs(b,hq,hkv,lk,seed=5,device="cuda")
    plan = dec.make_plan(b,hq,hkv,lk,policy=pol,forced_splits=s,combine_mode=comb)
    out,lse = dec.forward(plan, inp["q"],inp["k"],inp["v"],inp["seqlens"])
    torch.cuda.synchronize()
    ro, rl = OA.decode_attention(*(synth.to_f64(inp[n]) for n in ("q","k","v","seqlens")))
    o = synth.to_f64(out); l = synth.to_f64(lse)
    bad = ~np.isfinite(o)
    err = np.nanmax(np.abs(o-ro)) if np.isfinite(o).any() else -1
    print(f"B{b} HQ{hq} HKV{hkv} L{lk} s={plan.num_splits} comb={plan.combine_mode} grid=({plan.grid_x},{plan.grid_y},{plan.grid_z}) thr={plan.block_threads}: nonfinite={bad.sum()} rows={sorted(set(zip(*np.nonzero(bad.any(-1)))))[:8]} maxerr={err:.3g} lseerr={np.nanmax(np.abs(l-rl)):.3g}", flush=True)
for args in [(1,8,1,64,1),(1,8,1,128,1),(1,8,1,128,2,2),(1,8,1,128,2,1),(1,8,1,512,3,1),(1,8,1,512,8,1),(1,8,1,128,16,1),(1,64,8,512,4,1),(1,8,1,100,1),(1,16,1,512,8,1)]:
    run(*args)
