"""Per-CTA timeline of one decode step from a -DDECATTN_TRACE build (development tool).

DECATTN_LIB=paper_2604_00028_b200/lib/variants/libdecattn_trace.so python scripts/trace_timeline.py
Slots (globaltimer ns): 0 entry, 1 after griddepcontrol.wait, 2+i TMA issued tile i,
10+i tile i landed (consumer), 18+i tile i computed, 32-35 tile 0's QK^T / softmax / V landed /
PV results available, 26 epilogue start, 27 merge done,
29 rank-0 push wait done, 30 CTA end, 63 previous step's end stamp.
"""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2604_00028_b200 as dec
from paper_2604_00028_b200 import _lib as L
import synth

L.LIB.da_trace_fetch.argtypes = [ctypes.c_void_p, ctypes.c_int]
if hasattr(L.LIB, "da_trace_fetch_combine"):
    L.LIB.da_trace_fetch_combine.argtypes = [ctypes.c_void_p, ctypes.c_int]


def trace(b, hq, hkv, lk, policy, forced=0, steps=50, combine=None):
    w = synth.make_inputs(b, hq, hkv, lk, device="cuda", seed=3)
    nbuf = int(os.environ.get("TRACE_NBUF", "64"))
    ks = [w["k"].clone() for _ in range(nbuf)]
    vs = [w["v"].clone() for _ in range(nbuf)]
    plan = dec.make_plan(b, hq, hkv, lk, policy=policy, forced_splits=forced, combine_mode=combine)
    ws = dec.workspace_for(plan, w["q"].device)
    out = torch.empty_like(w["q"])
    lse = torch.empty(b, hq, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(3):
            dec.forward(plan, w["q"], ks[i % nbuf], vs[i % nbuf], None, out=out, lse=lse, workspace=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(steps):
            dec.forward(plan, w["q"], ks[i % nbuf], vs[i % nbuf], None, out=out, lse=lse, workspace=ws)
    for _ in range(3):
        with torch.cuda.stream(st):
            g.replay()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        g.replay()
        e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / steps
    buf = (ctypes.c_ulonglong * (64 * 64))()
    L.LIB.da_trace_fetch(ctypes.addressof(buf), 64 * 64)
    n_cta = plan.grid_x * plan.grid_y * plan.grid_z
    rows = [[buf[c * 64 + j] for j in range(64)] for c in range(min(n_cta, 64))]
    t0 = min(r[63] for r in rows if r[63]) if any(r[63] for r in rows) else min(r[0] for r in rows)
    print(f"\n== B={b} HQ={hq} HKV={hkv} L={lk} {policy} s={plan.num_splits} comb={plan.combine_mode}: "
          f"{us:.2f} us/step (graph); times in ns after the previous step's end stamp")
    names = {0: "entry", 1: "pdl_wait", 26: "epi", 27: "merged", 29: "push_in", 30: "end",
             32: "t0_qk", 33: "t0_p", 34: "t0_v", 35: "t0_pv"}
    for c, r in enumerate(rows[:8]):
        parts = []
        for j in (0, 1):
            parts.append(f"{names[j]}={int(r[j]) - t0}")
        iss = [int(r[2 + i]) - t0 for i in range(8) if r[2 + i]]
        rdy = [int(r[10 + i]) - t0 for i in range(8) if r[10 + i]]
        dn = [int(r[18 + i]) - t0 for i in range(8) if r[18 + i]]
        parts.append(f"issue={iss}")
        parts.append(f"ready={rdy}")
        parts.append(f"done={dn}")
        for j in (32, 33, 34, 35, 26, 40, 41, 42, 27, 29, 44, 45, 46, 47, 30):
            if r[j]:
                parts.append(f"{names.get(j, j)}={int(r[j]) - t0}")
        if r[60] and r[61] and r[30] > r[0]:
            parts.append(f"clk={(int(r[61]) - int(r[60])) / (int(r[30]) - int(r[0])) * 1e3:.0f}MHz")
        print(f"  cta{c}: " + " ".join(parts))
    # spread over every traced CTA (first 64): when each started streaming and when each finished
    def spread(j):
        v = [int(r[j]) - t0 for r in rows if r[j]]
        return (min(v), statistics.median(v), max(v)) if v else None
    print(f"  spread over {len(rows)} CTAs (min / median / max ns): pdl_wait={spread(1)} first_ready={spread(10)} "
          f"epi={spread(26)} end={spread(30)}")
    if plan.combine_mode == L.DA_COMBINE_KERNEL and hasattr(L.LIB, "da_trace_fetch_combine"):
        cb = (ctypes.c_ulonglong * (64 * 4))()
        L.LIB.da_trace_fetch_combine(ctypes.addressof(cb), 64 * 4)
        f0 = min(int(r[0]) for r in rows if r[0])
        fend = max(int(r[30]) for r in rows if r[30])
        print(f"  fwd: first entry 0, last CTA end {fend - f0}")
        for c in range(min(b * hq, 4)):
            print(f"  comb row{c}: entry={int(cb[c * 4]) - f0} waited={int(cb[c * 4 + 1]) - f0} "
                  f"end={int(cb[c * 4 + 2]) - f0}")


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "latency"
    if which == "latency":
        trace(1, 8, 1, 512, "seq_aware_sm")
        trace(1, 64, 8, 512, "seq_aware_sm")
    elif which == "long":
        os.environ.setdefault("TRACE_NBUF", "1")
        trace(1, 64, 8, 131072, "seq_aware_sm", steps=10)
        trace(1, 64, 8, 131072, "seq_aware", steps=10)
        trace(1, 64, 8, 131072, "fixed", 18, steps=10, combine=2)
        trace(1, 8, 1, 131072, "fixed", 64, steps=10, combine=2)
    elif which == "kernel":
        trace(1, 8, 1, 768, "fixed", 16, combine=1)
        trace(1, 8, 1, 768, "fixed", 16, combine=2)
        trace(1, 8, 1, 768, "fixed", 24, combine=2)
        trace(1, 8, 1, 4096, "guarded")
