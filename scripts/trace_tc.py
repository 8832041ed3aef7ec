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


def trace(b, hq, hkv, lk, policy="seq_aware", forced=0, path=None):
    w = synth.make_inputs(b, hq, hkv, lk, device="cuda", seed=3)
    plan = dec.make_plan(b, hq, hkv, lk, policy=policy, forced_splits=forced, path=path)
    ws = dec.workspace_for(plan, w["q"].device)
    for _ in range(3):
        dec.forward(plan, w["q"], w["k"], w["v"], None, workspace=ws)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (64 * 64))()
    L.LIB.da_trace_fetch_tc(ctypes.addressof(buf), 64 * 64)
    names = ["K_tma", "S_issue", "S_seen", "P_done", "PV_issue", "P_seen_mma", "S_start", "PV_start"]
    print(f"== B={b} HQ={hq} HKV={hkv} L={lk} s={plan.num_splits} path={plan.path}")
    ck = (ctypes.c_ulonglong * 4)()
    if hasattr(L.LIB, "da_trace_fetch_tc_clock") and L.LIB.da_trace_fetch_tc_clock(ctypes.addressof(ck)) == 0 and ck[1] > ck[0]:
        print(f" SM clock over stages 16-23 (CTA 0): {(ck[3] - ck[2]) / (ck[1] - ck[0]) * 1e3:.0f} MHz")
    if hasattr(L.LIB, "da_trace_fetch_tc_cta"):
        L.LIB.da_trace_fetch_tc_cta.argtypes = [ctypes.c_void_p]
        cb = (ctypes.c_ulonglong * (8 * 1024))()
        L.LIB.da_trace_fetch_tc_cta(ctypes.addressof(cb))
        n = min(1024, plan.grid_x * plan.grid_y * plan.grid_z)
        st = [cb[i] for i in range(n)]
        en = [cb[1024 + i] for i in range(n)]
        t0 = min(st)
        dur = sorted((e - s_) / 1e3 for s_, e in zip(st, en))
        ends = sorted((e - t0) / 1e3 for e in en)
        starts = sorted((s_ - t0) / 1e3 for s_ in st)
        q = lambda a, f: a[min(len(a) - 1, int(f * len(a)))]
        print(f" CTAs {n}: start us p0/p50/p100 {starts[0]:.2f}/{q(starts, .5):.2f}/{starts[-1]:.2f}; "
              f"end {ends[0]:.2f}/{q(ends, .1):.2f}/{q(ends, .5):.2f}/{q(ends, .9):.2f}/{ends[-1]:.2f}; "
              f"duration p0/p50/p100 {dur[0]:.2f}/{q(dur, .5):.2f}/{dur[-1]:.2f}")
        med = lambda j: sorted((cb[j * 1024 + i] - cb[3 * 1024 + i]) / 1e3 for i in range(n) if cb[j * 1024 + i])
        for j, nm in ((0, "PDL wait done"), (4, "Q in TMEM"), (5, "first S seen"), (6, "last PV seen"), (1, "end")):
            m = med(j)
            if m:
                print(f"  from entry to {nm:14s} us p50 {q(m, .5):.2f} (p0 {m[0]:.2f}, p100 {m[-1]:.2f})")
        order = sorted(range(n), key=lambda i: en[i])
        print("  slowest CTAs (cta, sm, start, end):",
              [(i, int(cb[2048 + i]), round((st[i] - t0) / 1e3, 2), round((en[i] - t0) / 1e3, 2)) for i in order[-6:]])
        print("  fastest CTAs (cta, sm, start, end):",
              [(i, int(cb[2048 + i]), round((st[i] - t0) / 1e3, 2), round((en[i] - t0) / 1e3, 2)) for i in order[:6]])
    smx = None
    if hasattr(L.LIB, "da_trace_fetch_tc_smx"):
        L.LIB.da_trace_fetch_tc_smx.argtypes = [ctypes.c_void_p]
        sb = (ctypes.c_ulonglong * 32)()
        if L.LIB.da_trace_fetch_tc_smx(ctypes.addressof(sb)) == 0:
            smx = sb
    pw = None
    if hasattr(L.LIB, "da_trace_fetch_tc_pw"):
        L.LIB.da_trace_fetch_tc_pw.argtypes = [ctypes.c_void_p]
        pb = (ctypes.c_ulonglong * 128)()
        if L.LIB.da_trace_fetch_tc_pw(ctypes.addressof(pb)) == 0:
            pw = pb
    for c in (0, 1):
        base = buf[c * 64 + 0]
        if c == 0 and pw is not None:
            for k in range(8):
                print("  P stored per softmax warp, stage", 16 + k, [int(pw[w * 8 + k]) - base if pw[w * 8 + k] else None
                                                                      for w in range(16)])
        if c == 0 and smx is not None:
            for k in range(8):
                print("  softmax warp 0 stage", 16 + k, " ".join(
                    f"{n}={int(smx[j * 8 + k]) - base}" for j, n in enumerate(("S_loaded", "max_done", "P_computed", "P_stored"))))
        print(f" cta{c}")
        for k in range(8):
            row = [int(buf[c * 64 + 8 * j + k]) - base if buf[c * 64 + 8 * j + k] else None for j in range(8)]
            print("  stage", 16 + k, " ".join(f"{n}={v}" for n, v in zip(names, row)))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "mqa":
        trace(128, 64, 1, 8192)
        sys.exit(0)
    trace(4, 64, 1, 8192, "guarded")
    trace(1, 64, 1, 4096, "seq_aware_sm", path=2)
    trace(128, 64, 1, 8192)
    trace(128, 32, 1, 8192)
    trace(32, 64, 1, 32768)
    trace(1, 64, 1, 131072)
