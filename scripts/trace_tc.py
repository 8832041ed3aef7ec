"""Per-stage timeline of the tcgen05 kernel (DA_PATH_TC) from a -DDECATTN_TRACE build (development
tool): 128-token stages 16..23 of CTAs 0 and 1, globaltimer ns relative to the K TMA issue of stage 16.

DECATTN_LIB=paper_2604_00028_b200/lib/variants/libdecattn_trace.so python scripts/trace_tc.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2604_00028_b200 as dec
from paper_2604_00028_b200 import _lib as L
import synth

L.LIB.da_trace_fetch_tc.argtypes = [ctypes.c_void_p, ctypes.c_int]
if hasattr(L.LIB, "da_trace_fetch_tc_clock"):
    L.LIB.da_trace_fetch_tc_clock.argtypes = [ctypes.c_void_p]


def trace(b, hq, hkv, lk, policy="seq_aware", forced=0):
    w = synth.make_inputs(b, hq, hkv, lk, device="cuda", seed=3)
    plan = dec.make_plan(b, hq, hkv, lk, policy=policy, forced_splits=forced)
    ws = dec.workspace_for(plan, w["q"].device)
    for _ in range(3):
        dec.forward(plan, w["q"], w["k"], w["v"], None, workspace=ws)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (64 * 64))()
    L.LIB.da_trace_fetch_tc(ctypes.addressof(buf), 64 * 64)
    names = ["K_tma", "S_issue", "S_seen", "P_done", "PV_issue", "PVm2_seen", "S_start", "PV_start"]
    print(f"== B={b} HQ={hq} HKV={hkv} L={lk} s={plan.num_splits} path={plan.path}")
    ck = (ctypes.c_ulonglong * 4)()
    if hasattr(L.LIB, "da_trace_fetch_tc_clock") and L.LIB.da_trace_fetch_tc_clock(ctypes.addressof(ck)) == 0 and ck[1] > ck[0]:
        print(f" SM clock over stages 16-23 (CTA 0): {(ck[3] - ck[2]) / (ck[1] - ck[0]) * 1e3:.0f} MHz")
    for c in (0, 1):
        base = buf[c * 64 + 0]
        print(f" cta{c}")
        for k in range(8):
            row = [int(buf[c * 64 + 8 * j + k]) - base if buf[c * 64 + 8 * j + k] else None for j in range(8)]
            print("  stage", 16 + k, " ".join(f"{n}={v}" for n, v in zip(names, row)))


if __name__ == "__main__":
    trace(128, 64, 1, 8192)
    trace(1, 64, 1, 131072)
