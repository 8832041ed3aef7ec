"""Summarise a round's ncu --set full captures (raw pages exported by scripts/profile_round.sh):
kernel, duration, DRAM bytes per launch vs algorithmic bytes, DRAM throughput, tensor-pipe use,
registers, launch shape, top stall reasons.  Writes profiles/<tag>_ncu_summary.md and
profiles/traffic.json (read by bench.py for the roofline 'traffic' field).

    python scripts/ncu_summary.py r01g gpurun_out/prof_r01g
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402

CONFIGS = {"llama70b": synth.CONFIGS["llama70b"], "llama70b_tp8": synth.CONFIGS["llama70b_tp8"],
           "long_context": synth.CONFIGS["long_context"], "long_context_sm": synth.CONFIGS["long_context"],
           "high_load": synth.CONFIGS["high_load"],
           "mqa_g64": {"batch": 128, "h_q": 64, "h_kv": 1, "l_k": 8192}}   # bench.py WORKLOADS["mqa_g64"]


def alg_bytes(c, d=128):
    b, hq, hkv, lk = c["batch"], c["h_q"], c["h_kv"], c["l_k"]
    return 4 * b * lk * hkv * d + 4 * b * hq * d + 4 * b * hq


def read_raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    return [{h: (v, u) for h, u, v in zip(hdr, units, r)} for r in rows[2:]]


def num(rec, key):
    v, u = rec.get(key, ("", ""))
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    return x * scale.get(u, 1.0)


def main():
    tag, src = sys.argv[1], sys.argv[2]
    lines = [f"# {tag} ncu summary (B200, `ncu --set full --clock-control none`)", "",
             f"Command lines: `TAG={tag} bash scripts/profile_round.sh` (each ncu run follows an identical "
             f"plain run that exited 0).  Raw pages: `{tag}_ncu_raw_<config>.csv`; launch lists (device time "
             f"per launch, cold-cache, serialised): `{tag}_launches_<config>.csv`.", "",
             "| config | kernel | ncu duration (us) | DRAM read+write / launch | algorithmic bytes | DRAM / alg | "
             "DRAM GB/s (vs 8 TB/s) | DRAM % peak | tensor pipe % | CTAs (SMs busy) | achieved occupancy % | "
             "regs | block | cluster |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {"_source": f"ncu --set full --clock-control none ({tag} captures, profiles/{tag}_ncu_raw_*.csv): "
                          "dram__bytes_read.sum + dram__bytes_write.sum of split_kv_fwd_kernel, one launch"}
    stalls_txt = []
    for name, cfg in CONFIGS.items():
        path = os.path.join(src, f"raw_{name}.csv")
        if not os.path.exists(path):
            continue
        recs = [r for r in read_raw(path) if "split_kv" in r.get("Kernel Name", ("", ""))[0]]
        if not recs:
            continue
        r = recs[0]
        kname = r["Kernel Name"][0]
        i0 = kname.find("split_kv_fwd")
        short = kname[i0:kname.find("(")] if "(" in kname else kname[i0:]
        dur = num(r, "gpu__time_duration.sum")
        dram = (num(r, "dram__bytes_read.sum") or 0.0) + (num(r, "dram__bytes_write.sum") or 0.0)
        alg = alg_bytes(cfg)
        thr = num(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
        # tensor pipe busy cycles: HMMA (mma.sync) and tcgen05 (UTCHMMA) both count here
        tens = num(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
        if tens is None:
            tens = num(r, "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active")
        regs = r.get("launch__registers_per_thread", ("?", ""))[0]
        grid = r.get("launch__grid_size", ("?", ""))[0]
        block = r.get("launch__block_size", ("?", ""))[0]
        cl = r.get("launch__cluster_dim_x", ("", ""))[0] or "-"
        occ = num(r, "sm__warps_active.avg.pct_of_peak_sustained_active")
        gbs = dram / (dur * 1e-6) / 1e9 if dur else 0.0
        try:
            busy = min(int(float(grid)), 148)
        except ValueError:
            busy = "?"
        lines.append(f"| {name} (B{cfg['batch']} H_Q{cfg['h_q']} H_KV{cfg['h_kv']} L{cfg['l_k']}) | `{short}` | "
                     f"{dur:.2f} | {dram:,.0f} | {alg:,} | {dram / alg:.3f} | {gbs:,.0f} ({gbs / 8000:.2f}) | "
                     f"{'' if thr is None else f'{thr:.1f}'} | {'' if tens is None else f'{tens:.1f}'} | "
                     f"{grid} ({busy}) | {'' if occ is None else f'{occ:.1f}'} | {regs} | {block} | {cl} |")
        traffic[name] = {"dram_bytes_per_launch": int(dram), "algorithmic_bytes": alg, "kernel": short,
                         "ncu_duration_us": dur}
        st = []
        for k, (v, _u) in r.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        stalls_txt.append(f"* {name}: " + ", ".join(f"{n} {v:.2f}" for v, n in st[:5]))
    lines += ["", "Top warp-stall reasons (cycles per issued instruction):", ""] + stalls_txt
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
