"""Wide query groups (G >= 32) under the C-ext-1 policy against the efficiency loop's split
(development tool): which plan each policy picks (split count, kernel) and its step time.

    python scripts/probe_wide_policy.py      (on the GPU box)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_timing import bench

if __name__ == "__main__":
    for g in (64, 32):
        for b in (1, 2, 4, 8, 16, 32):
            for lk in (2048, 4096, 8192, 16384):
                if b * lk * 512 > (1 << 30):
                    continue
                for pol in ("guarded", "seq_aware_sm"):
                    bench(b, g, 1, lk, pol, steps=50, reps=5)
