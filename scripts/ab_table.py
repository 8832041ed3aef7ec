"""Summarise a probe_variants.py log (development tool): best time per shape and library.

    python scripts/ab_table.py gpurun_out/<log>"""
import re, sys
rows={}
cur=None
for L in open(sys.argv[1]):
    if L.startswith("=="): cur=L.split()[-1]; continue
    m=re.search(r'B=\s*(\d+) HQ=\s*(\d+) HKV=\s*(\d+) L=\s*(\d+) pack=\d (\S+)\s+s=\s*(\d+).*?(?:path=(\d).*)?:\s+([\d.]+) us',L)
    if m:
        k=(m.group(1),m.group(2),m.group(3),m.group(4),m.group(5),m.group(6),'p'+(m.group(7) or '?'))
        rows.setdefault(k,{}).setdefault(cur,[]).append(float(m.group(8)))
for k,v in rows.items():
    print(' '.join(k), {a:round(min(b),2) for a,b in v.items()})
