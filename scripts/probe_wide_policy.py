"""Wide query groups (G >= 32) under the C-ext-1 policy against the efficiency loop's split
(development tool): which plan each policy picks (split count, kernel) and its step time.

    python scripts/probe_wide_policy.py      (on the GPU box)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_timing import bench

if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "wide2":
        # the clause's neighbourhood beyond the calibration grid: H_KV > 1, G = 48 / 96
        for g, hkv in ((48, 1), (96, 1), (32, 2), (64, 2), (32, 4)):
            for b in (2, 4, 8, 16):
                for lk in (2048, 4096, 8192):
                    if b * hkv * lk * 512 > (1 << 30):
                        continue
                    for pol in ("guarded", "seq_aware_sm"):
                        bench(b, g * hkv, hkv, lk, pol, steps=50, reps=5)
        sys.exit(0)
    for g in (64, 32):
        for b in (1, 2, 4, 8, 16, 32):
            for lk in (2048, 4096, 8192, 16384):
                if b * lk * 512 > (1 << 30):
                    continue
                for pol in ("guarded", "seq_aware_sm"):
                    bench(b, g, 1, lk, pol, steps=50, reps=5)
