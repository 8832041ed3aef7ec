#!/usr/bin/env python3
"""bench.py - decode-attention benchmark for the B200 path (contract: DESIGN.md §7).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]

One JSON line on rank 0.  A *step* is one pass of the whole hot path (SURVEY
§8(a) rows a1-a8) over one batch: the plan (precomputed per shape, like the
scheduler metadata the paper measures with) and one da_forward call,
i.e. the split-KV kernel plus the LSE combine when s > 1.

Headline (N = 1): the largest single-GPU BASELINE.json config, high-load (configs[3]: B=128
H_Q=64 H_KV=8 d=128 L_K=8192 bf16, 4.3 GB of KV per step), the HBM-bound step whose roofline
fraction is the measure of the kernel.  ``--workload`` selects another config (llama70b =
configs[1], Llama-3.1-70B decode B=1 L_K=512, latency-bound; long_context = configs[4]).
``--policy`` picks the split policy (default: the SM-count-aware sequence-aware policy,
DESIGN.md C-ext-1; ``seq_aware`` = the paper's literal Fig. 3 rule; high-load is saturated, so
every policy gives s = 1 there).  ``value`` = aggregate algorithmic HBM GB/s over all ranks
(K+V+q+out+lse bytes / step time), inputs resident in HBM; ``us_per_step`` the same as time.
Timing: W eager warm-up steps, then K steps captured in ONE CUDA graph ("CUDA Graph
replay") and timed with CUDA events between barrier + synchronize; a GPU-side sleep is queued
before the start event so the host's graph submission is never inside the timed region; the
max over ranks is reported.  L2: inputs larger than L2 (high-load, long-context) or a rotation
of KV buffers totalling > 2x L2, and L2 is scrubbed (256 MB write) before each timed replay.

N > 1: high-load shards the B = 128 batch across the ranks (strong scaling, no collective:
SURVEY §8(e) "shards by batch x KV-head"); ``--workload long_context`` shards the sequence
(fp32 shard partials merged across ranks, over peer memory by default or ``--exchange nccl``:
NCCL all-gather + the combine kernel); latency workloads run one replica per rank (weak).

Extras (N = 1): the policy A/B (guarded / the paper's seq-aware / SM-count-aware / evolved,
interleaved graph replays in random order per round, medians) on Llama-70B and its 8-way
tensor-parallel slice (H_Q=8, H_KV=1) where the paper's rule differs (s = 1 vs 3), the
isolated-step latency of those (one step per launch, no overlap with a preceding step), the
KV-streaming configs with their roofline fractions, and a ragged batch.  ``--impl reference``
times the fp64 CPU oracle instead (the reference arm of this tier; rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import random
import statistics
import subprocess
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
HEAD_DIM = 128
WORKLOADS = {
    "llama70b": dict(synth.CONFIGS["llama70b"]),
    "llama70b_tp8": dict(synth.CONFIGS["llama70b_tp8"]),
    "mqa_tiny": dict(synth.CONFIGS["mqa_tiny"]),
    "high_load": dict(synth.CONFIGS["high_load"]),
    "long_context": dict(synth.CONFIGS["long_context"]),
    # beyond BASELINE.json's configs (all G = 8): MQA with 64 query heads per KV head, the shape
    # the tcgen05 kernel (DA_PATH_TC) exists for; reported in extras only
    "mqa_g64": dict(batch=128, h_q=64, h_kv=1, l_k=8192),
}
FALLBACK_HBM_GBS = 6650.0   # /opt/skills/guides/B200_PROFILING.md fallback (used only if MEASURED_PEAKS.json is absent)


# ----------------------------------------------------------------------------------------------
def alg_bytes(batch, h_q, h_kv, l_k, d=HEAD_DIM):
    """Algorithmic bytes of one step: K+V bf16 + q bf16 + out bf16 + lse fp32."""
    return 4 * batch * l_k * h_kv * d + 2 * batch * h_q * d + 2 * batch * h_q * d + 4 * batch * h_q


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        p = json.load(open(path))
        return float(p["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
    return FALLBACK_HBM_GBS, "fallback 6.65 TB/s (B200_PROFILING.md)"


def traffic_record():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(path):
        try:
            return json.load(open(path))
        except Exception:
            return {}
    return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms while running."""

    FIELDS = ("clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        props = torch.cuda.get_device_properties(device_index)
        self.bus = f"{props.pci_domain_id:08X}:{props.pci_bus_id:02X}:{props.pci_device_id:02X}.0"
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.bus, "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------------------------
class Workload:
    """Device-resident inputs of one config with a rotation of KV buffers (> 2x L2 total)."""

    def __init__(self, cfg, device, seed, l2_bytes, max_rot_bytes=300 << 20, uniform=True):
        self.cfg = cfg
        b, hq, hkv, lk = cfg["batch"], cfg["h_q"], cfg["h_kv"], cfg["l_k"]
        kv_bytes = 4 * b * lk * hkv * HEAD_DIM
        self.nbuf = max(1, min(1024, -(-2 * l2_bytes // kv_bytes))) if kv_bytes < 2 * l2_bytes else 1
        if kv_bytes * self.nbuf > max(max_rot_bytes, 2 * l2_bytes + kv_bytes):
            self.nbuf = max(1, (2 * l2_bytes) // kv_bytes + 1)
        base = synth.make_inputs(b, hq, hkv, lk, device=device, seed=seed)
        self.q = base["q"]
        # one contiguous allocation per K and V: [nbuf, B, L, H_KV, d]
        self.k = base["k"].unsqueeze(0).repeat(self.nbuf, 1, 1, 1, 1) if self.nbuf > 1 else base["k"].unsqueeze(0)
        self.v = base["v"].unsqueeze(0).repeat(self.nbuf, 1, 1, 1, 1) if self.nbuf > 1 else base["v"].unsqueeze(0)
        # uniform lengths (the paper's fixed shapes): cache_seqlens = NULL means L_K for all b
        self.seqlens = None if uniform else base["seqlens"]
        self.out = torch.empty((b, hq, HEAD_DIM), dtype=torch.bfloat16, device=device)
        self.lse = torch.empty((b, hq), dtype=torch.float32, device=device)
        self.bytes = alg_bytes(b, hq, hkv, lk)
        self.kv_total = kv_bytes * self.nbuf

    def l2_note(self, l2_bytes):
        if self.nbuf > 1:
            return (f"rotating {self.nbuf} KV buffers ({self.kv_total / 2**20:.0f} MiB > 2x L2 "
                    f"{l2_bytes / 2**20:.0f} MiB) + 256 MiB L2 scrub before each timed replay")
        return (f"KV {self.kv_total / 2**20:.0f} MiB per step > 2x L2 ({l2_bytes / 2**20:.0f} MiB)"
                " + 256 MiB L2 scrub before each timed replay")


def make_graph(dec, plan, w: Workload, steps: int, stream):
    ws = dec.workspace_for(plan, w.q.device)

    def one(i):
        j = i % w.nbuf
        dec.forward(plan, w.q, w.k[j], w.v[j], w.seqlens, out=w.out, lse=w.lse, workspace=ws)

    with torch.cuda.stream(stream):
        for i in range(3):
            one(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(steps):
            one(i)
    with torch.cuda.stream(stream):
        g.replay()
    torch.cuda.synchronize()
    g.keepalive = ws          # the graph reads the workspace: it must outlive the graph
    return g


# GPU-side sleep queued before a start event (~0.5 ms at 1.9 GHz): the stream is still busy when the
# host has submitted the graph, so the host's submission latency never falls inside the timed region
GUARD_CYCLES = 1_000_000


def guard(stream):
    with torch.cuda.stream(stream):
        torch.cuda._sleep(GUARD_CYCLES)


class Timer:
    def __init__(self, device):
        self.scrub = torch.empty(256 << 20, dtype=torch.uint8, device=device)

    def time_replay(self, g, stream, scrub=True):
        if scrub:
            with torch.cuda.stream(stream):
                self.scrub.fill_(1)
        guard(stream)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            g.replay()
            e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1)  # ms


AB_POLICIES = ("guarded", "seq_aware", "seq_aware_sm", "evolved")


def ab_compare(dec, dev, stream, timer, cfg, steps, rounds, l2, seed, num_sms):
    """Guarded vs the paper's seq-aware (and the SM-count-aware generalisation, the evolved
    Fig. 1 policy), interleaved replays (P:L119 A/B) -> medians in us/step."""
    w = Workload(cfg, dev, seed, l2)
    res = {}
    graphs = {}
    for pol in AB_POLICIES:
        plan = dec.make_plan(cfg["batch"], cfg["h_q"], cfg["h_kv"], cfg["l_k"], policy=pol)
        graphs[pol] = (plan, make_graph(dec, plan, w, steps, stream))
        res[pol] = []
    rng = random.Random(seed)
    for _ in range(rounds):
        order = list(AB_POLICIES)
        rng.shuffle(order)                       # no arm always follows another (order bias)
        for pol in order:
            res[pol].append(timer.time_replay(graphs[pol][1], stream) * 1e3 / steps)
    out = {}
    for pol in AB_POLICIES:
        plan = graphs[pol][0]
        us = statistics.median(res[pol])
        out[pol] = {"num_splits": plan.num_splits, "combine_mode": plan.combine_mode,
                    "ctas": plan.grid_x * plan.grid_y * plan.grid_z,
                    "occupancy_pct": round(100.0 * min(plan.grid_x * plan.grid_y * plan.grid_z, num_sms) / num_sms, 1),
                    "us_per_step": round(us, 3), "p10_us": round(sorted(res[pol])[len(res[pol]) // 10], 3),
                    "p90_us": round(sorted(res[pol])[(9 * len(res[pol])) // 10], 3),
                    "gbs": round(w.bytes / (us * 1e-6) / 1e9, 1)}
    for pol in AB_POLICIES[1:]:
        # median of the per-round paired ratios (guarded time / policy time of the same round)
        out[f"speedup_{pol}_vs_guarded"] = round(statistics.median(
            g / t for g, t in zip(res["guarded"], res[pol])), 4)
    out["config"] = dict(cfg, head_dim=HEAD_DIM)
    out["l2"] = w.l2_note(l2)
    del w, graphs
    torch.cuda.empty_cache()
    return out


def streaming_roofline(dec, dev, stream, timer, cfg, steps, rounds, l2, seed, peak, policy="seq_aware"):
    w = Workload(cfg, dev, seed, l2)
    plan = dec.make_plan(cfg["batch"], cfg["h_q"], cfg["h_kv"], cfg["l_k"], policy=policy)
    g = make_graph(dec, plan, w, steps, stream)
    ts = [timer.time_replay(g, stream) * 1e3 / steps for _ in range(rounds)]
    us = statistics.median(ts)
    gbs = w.bytes / (us * 1e-6) / 1e9
    r = {"config": dict(cfg, head_dim=HEAD_DIM), "policy": policy, "path": plan.path, "num_splits": plan.num_splits,
         "combine_mode": plan.combine_mode, "us_per_step": round(us, 2), "achieved_gbs": round(gbs, 1),
         "frac_of_measured_peak": round(gbs / peak, 4), "frac_of_8tbs_nominal": round(gbs / 8000.0, 4),
         "bytes_per_step": w.bytes, "l2": w.l2_note(l2)}
    del w, g
    torch.cuda.empty_cache()
    return r


RAGGED_AB = dict(batch=16, h_q=64, h_kv=8, l_k=32768)   # one 32768-token sequence + fifteen of 1024


def isolated_latency(dec, dev, stream, timer, cfg, steps, rounds, l2, seed, policies=("guarded", "seq_aware", "seq_aware_sm")):
    """The step's latency when it cannot overlap a preceding step (the paper times "pure kernel
    execution times"): K steps captured as [separator, step] pairs, where the separator is a
    1-element torch fill that does not trigger programmatic dependent launch, so each step's launch,
    prologue and L2 prefetch start only after the previous step has finished; minus a graph of the K
    separators alone.  Interleaved per round in random order (the separator graph included), medians."""
    w = Workload(cfg, dev, seed, l2)
    sep_buf = torch.zeros(1, dtype=torch.int32, device=dev)

    def capture(plan):
        ws = dec.workspace_for(plan, dev) if plan is not None else None
        def body(i):
            sep_buf.fill_(i)
            if plan is not None:
                j = i % w.nbuf
                dec.forward(plan, w.q, w.k[j], w.v[j], w.seqlens, out=w.out, lse=w.lse, workspace=ws)
        with torch.cuda.stream(stream):
            for i in range(3):
                body(i)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for i in range(steps):
                body(i)
        return g

    plans = {p: dec.make_plan(cfg["batch"], cfg["h_q"], cfg["h_kv"], cfg["l_k"], policy=p) for p in policies}
    graphs = {p: capture(plans[p]) for p in policies}
    graphs["_sep"] = capture(None)
    res = {k: [] for k in graphs}
    rng = random.Random(seed)
    for _ in range(rounds):
        order = list(graphs)
        rng.shuffle(order)
        for k in order:
            res[k].append(timer.time_replay(graphs[k], stream) * 1e3 / steps)
    sep = statistics.median(res["_sep"])
    out = {"config": dict(cfg, head_dim=HEAD_DIM), "separator_us": round(sep, 3)}
    for p in policies:
        out[p] = {"num_splits": plans[p].num_splits, "combine_mode": plans[p].combine_mode,
                  "us_per_step": round(statistics.median(res[p]) - sep, 3)}
    for p in policies[1:]:
        out[f"speedup_{p}_vs_guarded"] = round(out[policies[0]]["us_per_step"] / out[p]["us_per_step"], 4)
    out["note"] = ("one step per launch chain: [1-element fill, step] x K minus [fill] x K; no step overlaps "
                   "the previous one (no PDL early launch, no pre-wait prefetch under the previous step)")
    del w, graphs
    torch.cuda.empty_cache()
    return out


def latency_floor(dec, dev, stream, timer, cfg, steps, rounds, l2, seed, us_headline):
    """The latency floor of the headline step on this kernel: the same shape and combine path with
    ONE 64-token tile per CTA (L_K = 64, s = 1), i.e. launch + PDL hop + one TMA round trip + one
    tile + the store.  frac = floor / headline: how close the latency-bound step is to it."""
    fcfg = dict(cfg, l_k=64)
    w = Workload(fcfg, dev, seed, l2)
    plan = dec.make_plan(fcfg["batch"], fcfg["h_q"], fcfg["h_kv"], 64, policy="fixed", forced_splits=1)
    g = make_graph(dec, plan, w, steps, stream)
    us = statistics.median([timer.time_replay(g, stream) * 1e3 / steps for _ in range(rounds)])
    del w, g
    torch.cuda.empty_cache()
    return {"us_per_step": round(us, 3), "config": dict(fcfg, num_splits=1),
            "frac_of_headline": round(us / us_headline, 4),
            "note": "same kernel, one 64-token tile per CTA: launch, PDL hop, one TMA round trip, one tile, store"}


def ragged_ab(dec, dev, stream, timer, steps, rounds, l2, seed):
    """Per-batch dynamic split counts (DA_POLICY_DYNAMIC, DESIGN.md C-ext-2) vs the static policies on
    a skewed ragged batch; the static plans see the cache capacity, the dynamic schedule the lengths."""
    cfg = RAGGED_AB
    lens = [cfg["l_k"]] + [1024] * (cfg["batch"] - 1)
    w = Workload(cfg, dev, seed, l2, uniform=False)
    w.seqlens = torch.tensor(lens, dtype=torch.int32, device=dev)
    pols = ("guarded", "seq_aware_sm", "dynamic", "varlen")
    plans = {p: dec.make_plan(cfg["batch"], cfg["h_q"], cfg["h_kv"], cfg["l_k"], policy=p) for p in pols[:3]}
    plans["varlen"] = dec.make_plan_varlen(cfg["batch"], cfg["h_q"], cfg["h_kv"], cfg["l_k"], lens)
    graphs = {p: make_graph(dec, plans[p], w, steps, stream) for p in pols}
    res = {p: [] for p in pols}
    for _ in range(rounds):
        for p in pols:
            res[p].append(timer.time_replay(graphs[p], stream) * 1e3 / steps)
    byts = 4 * sum(lens) * cfg["h_kv"] * HEAD_DIM + 4 * cfg["batch"] * cfg["h_q"] * HEAD_DIM + 4 * cfg["batch"] * cfg["h_q"]
    out = {"config": dict(cfg, lengths=f"[{cfg['l_k']}] + [1024] x {cfg['batch'] - 1}")}
    for p in pols:
        us = statistics.median(res[p])
        out[p] = {"num_splits": plans[p].num_splits, "combine_mode": plans[p].combine_mode,
                  "us_per_step": round(us, 2), "gbs": round(byts / (us * 1e-6) / 1e9, 1)}
    out["speedup_dynamic_vs_guarded"] = round(out["guarded"]["us_per_step"] / out["dynamic"]["us_per_step"], 3)
    out["speedup_varlen_vs_guarded"] = round(out["guarded"]["us_per_step"] / out["varlen"]["us_per_step"], 3)
    del w, graphs
    torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------------------------
def cpu_baseline(cfg, budget_s=10.0):
    """The fp64 oracle (as it stands) on this host's cores, on a bounded sample of the workload."""
    import numpy as np
    from oracle import attention as OA
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = 1
    scfg = dict(cfg)
    if cfg["batch"] * cfg["h_kv"] * cfg["l_k"] > 8 * 8192:   # bound the sample (fp64 copies of big caches)
        scfg = dict(cfg, batch=1, l_k=min(cfg["l_k"], 8192))
    inp = synth.make_inputs(scfg["batch"], scfg["h_q"], scfg["h_kv"], scfg["l_k"], seed=1000)
    q, k, v, s = (synth.to_f64(inp[n]) for n in ("q", "k", "v", "seqlens"))
    OA.decode_attention(q, k, v, s)     # warm
    n, t0 = 0, time.perf_counter()
    while True:
        OA.decode_attention(q, k, v, s)
        n += 1
        dt = time.perf_counter() - t0
        if dt >= budget_s or n >= 100000:
            break
    step_s = dt / n
    b = alg_bytes(scfg["batch"], scfg["h_q"], scfg["h_kv"], scfg["l_k"])
    # the same oracle with its BLAS limited to one thread (all cores plus a 1-thread
    # figure), on a shorter budget
    single = None
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            n1, t1 = 0, time.perf_counter()
            while True:
                OA.decode_attention(q, k, v, s)
                n1 += 1
                d1 = time.perf_counter() - t1
                if d1 >= max(0.5, budget_s / 5) or n1 >= 100000:
                    break
        single = round(b / (d1 / n1) / 1e9, 6)
    except Exception:
        pass
    what = "full steps of the workload" if scfg == cfg else f"sample steps (batch {scfg['batch']}, L_K {scfg['l_k']})"
    return {"value": round(b / step_s / 1e9, 6), "unit": "GB/s", "cores": int(cores), "kind": "oracle",
            "sample": f"{n} {what} in {dt:.1f} s (fp64 NumPy oracle.attention.decode_attention)",
            "ms_per_step": round(step_s * 1e3, 4), "single_thread_value": single,
            "host_cpus": len(os.sched_getaffinity(0))}


def run_reference(args, rank, world):
    """Reference arm of this tier: the CPU oracle on the same workload / metric."""
    if rank != 0:
        return 0
    cfg = WORKLOADS[args.workload]
    import numpy as np  # noqa: F401
    from oracle import attention as OA
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = 1
    sample_cfg = dict(cfg)
    if cfg["batch"] * cfg["h_kv"] * cfg["l_k"] > 8 * 8192:   # bound a step to a sample (big configs)
        sample_cfg = dict(cfg, batch=1, l_k=min(cfg["l_k"], 8192))
    inp = synth.make_inputs(sample_cfg["batch"], sample_cfg["h_q"], sample_cfg["h_kv"], sample_cfg["l_k"], seed=1000)
    q, k, v, s = (synth.to_f64(inp[n]) for n in ("q", "k", "v", "seqlens"))
    for _ in range(args.warmup):
        OA.decode_attention(q, k, v, s)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        OA.decode_attention(q, k, v, s)
    dt = time.perf_counter() - t0
    b = alg_bytes(sample_cfg["batch"], sample_cfg["h_q"], sample_cfg["h_kv"], sample_cfg["l_k"])
    value = b * args.steps / dt / 1e9
    sample = ("full workload per step" if sample_cfg == cfg else
              f"per step: batch {sample_cfg['batch']} x L_K {sample_cfg['l_k']} of the workload")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt / args.steps * 1e3, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, **cfg, "head_dim": HEAD_DIM},
            "cpu_baseline": {"value": round(value, 6), "unit": "GB/s", "cores": int(cores), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(value, 6), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------------------------
def e2e_measure(dec, L, cfg, dev, stream, steps, warmup, policy="seq_aware_sm", depth=2):
    """Same metric through the C ABI with HOST buffers (da_forward_host): per step da_plan_make,
    then the H2D copies of q/K/V from pinned memory, the forward and the D2H copies of out + lse,
    enqueued on one stream.  depth > 1 pipelines consecutive steps over `depth` streams (each with
    its own device staging and host output buffer, as a serving loop with several requests in
    flight would), so one step's forward and D2H overlap the next step's H2D.  CUDA events around
    the K steps (every stream joined into the end event)."""
    b, hq, hkv, lk = cfg["batch"], cfg["h_q"], cfg["h_kv"], cfg["l_k"]
    inp = synth.make_inputs(b, hq, hkv, lk, seed=2000)
    hq_ = inp["q"].contiguous().pin_memory()
    # the host KV cache as one pinned [2, B, L, H_KV, d] allocation (K then V) and out + lse in one
    # pinned buffer: da_forward_host moves each pair with one DMA
    kv = torch.empty((2,) + tuple(inp["k"].shape), dtype=torch.bfloat16).pin_memory()
    kv[0].copy_(inp["k"])
    kv[1].copy_(inp["v"])
    hk_, hv_ = kv[0], kv[1]
    ob = b * hq * HEAD_DIM * 2
    outs = []
    for _ in range(depth):
        ol = torch.empty(ob + 4 * b * hq, dtype=torch.uint8).pin_memory()
        outs.append((ol[:ob].view(torch.bfloat16).view(b, hq, HEAD_DIM), ol[ob:].view(torch.float32).view(b, hq)))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    streams = [stream] + [torch.cuda.Stream(device=dev) for _ in range(depth - 1)]
    stagings = [dec.HostStaging(dev) for _ in range(depth)]

    def step(j):
        plan = L.da_plan_make(b, hq, hkv, lk, HEAD_DIM, 1, 0, sms, L.POLICIES[policy], 0)
        h_out, h_lse = outs[j % depth]
        dec.forward_host(plan, hq_, hk_, hv_, None, out=h_out, lse=h_lse, staging=stagings[j % depth],
                         stream=streams[j % depth])

    for j in range(max(warmup, depth)):
        step(j)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    for st in streams[1:]:
        st.wait_event(e0)
    for j in range(steps):
        step(j)
    for st in streams[1:]:
        ev = torch.cuda.Event()
        ev.record(st)
        streams[0].wait_event(ev)
    e1.record(streams[0])
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    h2d = sum(t.numel() * t.element_size() for t in (hq_, hk_, hv_))
    d2h = outs[0][0].numel() * outs[0][0].element_size() + outs[0][1].numel() * outs[0][1].element_size()
    return ms, h2d, d2h


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="high_load",
                    help="BASELINE.json config (default: high_load, the largest single-GPU config)")
    ap.add_argument("--no-extras", action="store_true", help="skip the A/B and streaming extras")
    ap.add_argument("--ab-rounds", type=int, default=21)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--seq-shard", action="store_true",
                    help="long_context: take the sequence-sharded path (exchange included) even at N = 1 "
                         "(a one-rank group; checks the sharded step on one GPU)")
    ap.add_argument("--shard-heads", action="store_true",
                    help="N > 1, latency / throughput workloads: split the KV heads (and their query heads) "
                         "across the ranks - the tensor-parallel mapping, e.g. Llama-70B over 8 GPUs = the TP-8 "
                         "slice per rank; strong scaling, no collective")
    ap.add_argument("--exchange", default="p2p", choices=["nccl", "p2p", "p2p-split"],
                    help="long_context with N > 1: the exchange over peer memory (default: one kernel per step, "
                         "LL words over torch symmetric memory with a bounded wait), p2p-split (da_peer_signal + "
                         "da_combine_peers) or nccl (all-gather + da_combine)")
    ap.add_argument("--policy", default="seq_aware_sm",
                    choices=["seq_aware_sm", "seq_aware", "guarded", "evolved"],
                    help="split policy of the headline step (default: the SM-count-aware sequence-aware "
                         "policy, DESIGN.md C-ext-1; the paper's literal Fig. 3 rule is 'seq_aware')")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3          # contract: W >= 3 warm-up steps

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch.distributed as dist
    # DECATTN_BENCH_BACKEND=gloo + DECATTN_BENCH_ONE_GPU=1 run the multi-rank plumbing of the
    # batch-sharded mode as several processes on one GPU (tests only: no kernel of one rank
    # waits on another rank's, and the ranks share the GPU, so the number is not a bench value)
    backend = os.environ.get("DECATTN_BENCH_BACKEND", "nccl")
    gpu_index = 0 if os.environ.get("DECATTN_BENCH_ONE_GPU") == "1" else local_rank
    if world == 1 and args.seq_shard and args.workload == "long_context":
        import socket
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if "MASTER_PORT" not in os.environ:
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
        torch.cuda.set_device(gpu_index)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", gpu_index))
    if world > 1:
        torch.cuda.set_device(gpu_index)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu_index))
        else:
            dist.init_process_group(backend)
    local_rank = gpu_index
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    import paper_2604_00028_b200 as dec
    from paper_2604_00028_b200 import _lib as L

    props = torch.cuda.get_device_properties(dev)
    l2, num_sms = props.L2_cache_size, props.multi_processor_count
    stream = torch.cuda.Stream(device=dev)
    timer = Timer(dev)
    peak, peak_src = peaks()

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local_rank])
            else:
                dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    cfg = WORKLOADS[args.workload]
    long_sharded = args.workload == "long_context" and (world > 1 or args.seq_shard)
    batch_sharded = args.workload == "high_load" and world > 1 and not args.shard_heads
    head_sharded = args.shard_heads and world > 1 and not long_sharded
    if long_sharded:
        from paper_2604_00028_b200.dist import PeerSeqShardedDecode, SeqShardedDecode
        p2p = args.exchange.startswith("p2p")
        if p2p:
            sd = PeerSeqShardedDecode(cfg["batch"], cfg["h_q"], cfg["h_kv"], cfg["l_k"], HEAD_DIM, device=dev,
                                      policy=args.policy, fused=args.exchange == "p2p")
        else:
            sd = SeqShardedDecode(cfg["batch"], cfg["h_q"], cfg["h_kv"], cfg["l_k"], HEAD_DIM, device=dev,
                                  policy=args.policy)
        local_cfg = dict(cfg, l_k=sd.l_local)
        inp = synth.make_inputs(cfg["batch"], cfg["h_q"], cfg["h_kv"], sd.l_local, device=dev, seed=1000 + rank)
        # rotate through shard copies totalling > 2x L2 (a shard of 8 ranks is 67 MB < L2)
        shard_bytes = inp["k"].numel() * inp["k"].element_size() * 2
        nkv = 1 if shard_bytes >= 2 * l2 else -(-2 * l2 // shard_bytes) + 1
        ks = [inp["k"]] + [inp["k"].clone() for _ in range(nkv - 1)]
        vs = [inp["v"]] + [inp["v"].clone() for _ in range(nkv - 1)]
        out = torch.empty((cfg["batch"], cfg["h_q"], HEAD_DIM), dtype=torch.bfloat16, device=dev)
        lse = torch.empty((cfg["batch"], cfg["h_q"]), dtype=torch.float32, device=dev)
        plan = sd.plan
        with torch.cuda.stream(stream):
            for i in range(args.warmup):
                sd.step(inp["q"], ks[i % nkv], vs[i % nkv], None, out, lse)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for i in range(args.steps):
                sd.step(inp["q"], ks[i % nkv], vs[i % nkv], None, out, lse)
        step_bytes_total = alg_bytes(cfg["batch"], cfg["h_q"], cfg["h_kv"], cfg["l_k"])
        # forward (+ workspace combine) + the exchange: fused publish -> pull-combine (1 launch),
        # signal + pull-combine (2), NCCL all-gather (library) + da_combine (1)
        one_kernel = p2p and getattr(sd, "one_kernel", False)
        kernels_per_step = ((2 if plan.combine_mode == L.DA_COMBINE_KERNEL else 1)
                            + (0 if one_kernel else 2 if args.exchange == "p2p-split" else 1))
        scaling = "strong"
        l2_note = f"{nkv} rotating copies of the sequence shard (> 2x L2) + 256 MiB L2 scrub before the timed replay"
        parallelism = {"p2p": (f"seq-sharded sp{world}, one kernel per step: forward + peer-memory publish + cross-rank "
                               f"LSE combine" if one_kernel else
                               f"seq-sharded sp{world} + peer-memory exchange (fused publish + pull-combine)"),
                       "p2p-split": f"seq-sharded sp{world} + peer-memory exchange (signal + pull-combine)",
                       "nccl": f"seq-sharded sp{world} + NCCL all-gather + LSE combine"}[args.exchange]
    else:
        # high-load at N > 1: the B = 128 batch is sharded across ranks (the north star's
        # "sharded by batch x KV-head", total work fixed); other workloads run one replica per rank
        local_cfg = cfg
        if batch_sharded:
            from paper_2604_00028_b200.dist import shard_range
            b0, b1 = shard_range(cfg["batch"], rank, world)
            local_cfg = dict(cfg, batch=b1 - b0)
        elif head_sharded:
            from paper_2604_00028_b200.dist import head_shard
            (k0, k1), (h0, h1) = head_shard(cfg["h_q"], cfg["h_kv"], rank, world)
            local_cfg = dict(cfg, h_q=h1 - h0, h_kv=k1 - k0)
        w = Workload(local_cfg, dev, 1000 + rank, l2)
        plan = dec.make_plan(local_cfg["batch"], local_cfg["h_q"], local_cfg["h_kv"], cfg["l_k"], policy=args.policy)
        with torch.cuda.stream(stream):
            ws = dec.workspace_for(plan, dev)
            for i in range(args.warmup):
                j = i % w.nbuf
                dec.forward(plan, w.q, w.k[j], w.v[j], w.seqlens, out=w.out, lse=w.lse, workspace=ws)
        torch.cuda.synchronize()
        g = make_graph(dec, plan, w, args.steps, stream)
        step_bytes_total = alg_bytes(**cfg) if (batch_sharded or head_sharded) else w.bytes * world
        kernels_per_step = 2 if plan.combine_mode == L.DA_COMBINE_KERNEL else 1
        scaling = "strong" if (batch_sharded or head_sharded) else "weak"
        l2_note = w.l2_note(l2)
        parallelism = (f"batch-sharded dp{world} (B={cfg['batch']} split across ranks, no collective)" if batch_sharded
                       else f"head-sharded tp{world} (H_KV={cfg['h_kv']} split across ranks, no collective)" if head_sharded
                       else f"batch-sharded dp{world} (independent sequences, no collective)" if world > 1
                       else "single GPU")

    # ---- the timed region: exactly K steps (one graph replay), barrier + sync both sides ----
    with ClockSampler(dev.index) as clk:
        t_end = time.time() + 0.6               # keep the GPU busy so clocks settle under load
        while time.time() < t_end:
            with torch.cuda.stream(stream):
                g.replay()
            torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            timer.scrub.fill_(1)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        guard(stream)                            # GPU busy while the host submits the graph
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            g.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        # a few more untimed replays so the sampler sees the steady state around the timed region
        t_end = time.time() + 0.3
        while time.time() < t_end:
            with torch.cuda.stream(stream):
                g.replay()
            torch.cuda.synchronize()
    if long_sharded and hasattr(sd, "check"):
        sd.check()                               # raises if an exchange wait ran past its bound
    ms_max = max_over_ranks(ms)
    us_per_step = ms_max * 1e3 / args.steps
    value = step_bytes_total * args.steps / (ms_max * 1e-3) / 1e9

    # ---- end to end through the public API with host buffers ----
    # (a step that moves > 64 MB over PCIe - high-load's 4.3 GB of K/V - is timed over at most 10 steps)
    e2e_steps = args.steps if alg_bytes(**local_cfg) < (64 << 20) else max(3, min(args.steps, 10))
    e2e_ms, h2d, d2h = e2e_measure(dec, L, local_cfg, dev, stream, e2e_steps, args.warmup, args.policy, depth=2)
    e2e_serial_ms, _, _ = e2e_measure(dec, L, local_cfg, dev, stream, e2e_steps, args.warmup, args.policy, depth=1)
    e2e_ms_max = max_over_ranks(e2e_ms)
    e2e_serial_max = max_over_ranks(e2e_serial_ms)
    e2e_scale = alg_bytes(**local_cfg) * (world if not long_sharded else 1) * e2e_steps / 1e9
    e2e_value = e2e_scale / (e2e_ms_max * 1e-3)

    extras = {}
    if rank == 0 and world == 1 and not args.no_extras:
        lat_steps = 200
        extras["policy_ab"] = {
            "llama70b": ab_compare(dec, dev, stream, timer, WORKLOADS["llama70b"], lat_steps, args.ab_rounds, l2, 1001, num_sms),
            "llama70b_tp8_slice": ab_compare(dec, dev, stream, timer, WORKLOADS["llama70b_tp8"], lat_steps, args.ab_rounds, l2, 1002, num_sms),
        }
        # the paper's headline claim on this box: its literal rule (Fig. 3) vs guarded on the TP-8 slice,
        # where they differ (s = 1 -> 3); the target is >= 1.20x
        extras["paper_rule_tp8_speedup"] = extras["policy_ab"]["llama70b_tp8_slice"]["speedup_seq_aware_vs_guarded"]
        extras["isolated_latency"] = {
            "llama70b": isolated_latency(dec, dev, stream, timer, WORKLOADS["llama70b"], lat_steps, args.ab_rounds, l2, 1007),
            "llama70b_tp8_slice": isolated_latency(dec, dev, stream, timer, WORKLOADS["llama70b_tp8"], lat_steps, args.ab_rounds, l2, 1008),
        }
        extras["roofline_streaming"] = {
            "long_context": streaming_roofline(dec, dev, stream, timer, WORKLOADS["long_context"], 20, 7, l2, 1004, peak),
            "long_context_seq_aware_sm": streaming_roofline(dec, dev, stream, timer, WORKLOADS["long_context"], 20, 7, l2,
                                                            1004, peak, policy="seq_aware_sm"),
            # MQA, G = 64 (not a BASELINE config): the tcgen05 kernel (path 2)
            "mqa_g64_tcgen05": streaming_roofline(dec, dev, stream, timer, WORKLOADS["mqa_g64"], 10, 7, l2, 1007, peak),
        }
        if args.workload != "high_load":
            extras["roofline_streaming"]["high_load"] = streaming_roofline(dec, dev, stream, timer, WORKLOADS["high_load"],
                                                                           5, 5, l2, 1003, peak)
        extras["ragged_ab"] = ragged_ab(dec, dev, stream, timer, 20, 7, l2, 1005)
        extras["latency_floor"] = latency_floor(dec, dev, stream, timer, WORKLOADS["llama70b"], lat_steps, 11, l2, 1006,
                                                extras["policy_ab"]["llama70b"]["seq_aware_sm"]["us_per_step"])
    if world > 1:
        barrier()
    if rank != 0:
        dist.destroy_process_group()
        return 0

    # roofline of the dominant kernel of the headline step (the split-KV forward; with s = 1 it is
    # the only kernel of the step, so its average launch duration is the step time)
    kernel_us = us_per_step
    achieved = alg_bytes(**local_cfg) / (kernel_us * 1e-6) / 1e9
    trec = traffic_record().get(args.workload)
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_max / args.steps, 6),
        "us_per_step": round(us_per_step, 3),
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) bf16 q/K/V, uniform cache_seqlens = L_K)",
        "config": {"workload": args.workload, **cfg, "head_dim": HEAD_DIM, "policy": args.policy,
                   "num_splits": plan.num_splits, "combine_mode": plan.combine_mode,
                   "global_batch": cfg["batch"] * (world if not (long_sharded or batch_sharded or head_sharded) else 1),
                   "parallelism": parallelism, "l2": l2_note, "graph": "K steps in one CUDA graph"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": trec.get("dram_bytes_per_launch") if trec else None,
                     "kernel": "split_kv_fwd_kernel", "peak_source": peak_src,
                     "note": (f"latency-bound config ({alg_bytes(**local_cfg) / 1e6:.2f} MB per step); see "
                              "roofline_streaming for the HBM-bound configs"
                              if alg_bytes(**local_cfg) < (64 << 20) else
                              f"HBM-bound config ({alg_bytes(**local_cfg) / 1e9:.3f} GB per step, one launch per step "
                              "when s = 1); achieved = algorithmic bytes of the step / step time")},
        "cpu_baseline": cpu_baseline(local_cfg, args.cpu_seconds) if world == 1 else None,
        "e2e": {"value": round(e2e_value, 3), "unit": "GB/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms_max / e2e_steps, 6), "steps": e2e_steps,
                "pipeline_depth": 2, "serial_value": round(e2e_scale / (e2e_serial_max * 1e-3), 3),
                "note": "da_forward_host per step (H2D of q/K/V from pinned memory, forward, D2H of out/lse); "
                        "value: two steps in flight on two streams, serial_value: one stream"},
        "gpu_launches": args.steps * kernels_per_step,
        "clocks": clk.summary(),
        "device": {"name": props.name, "sms": num_sms, "l2_bytes": l2},
    }
    line.update(extras)
    print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
