"""Summarise per-SASS-instruction warp-stall samples of an ncu report (development tool).
python scripts/sass_stalls.py <report.ncu-rep> [kernel-index]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
# the page holds one block per kernel: "Kernel Name" line, header, rows
blocks, cur = [], None
for row in csv.reader(io.StringIO(out)):
    if row and row[0] == "Kernel Name":
        cur = {"name": row[1], "rows": []}
        blocks.append(cur)
    elif cur is not None and row:
        cur["rows"].append(row)
for bi, blk in enumerate(blocks):
    hdr = blk["rows"][0]
    idx = {h: i for i, h in enumerate(hdr)}
    data = blk["rows"][1:]
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = Counter()
    samp = lambda r: int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    for r in data:
        for s in stalls:
            tot[s] += int(r[idx[s]] or 0)
    total = sum(samp(r) for r in data)
    print(f"\n=== kernel {bi}: {blk['name'][:100]}  samples={total}")
    print("  by reason:", ", ".join(f"{k[6:]}={v}" for k, v in tot.most_common(10)))
    # cumulative samples along the program (coarse phases)
    top = sorted(data, key=lambda r: -samp(r))[:25]
    for r in top:
        st = sorted(((s[6:], int(r[idx[s]] or 0)) for s in stalls), key=lambda kv: -kv[1])[:3]
        print(f"  {r[idx['Address']][-5:]} {samp(r):5d}  {r[idx['Source']][:58]:58s} {st}")
