"""C-ext-1 against guarded for 16 < G < 32 at L_K = 4096 (development tool): the B16 shape where the
one-wave cluster fit leaves a 2-CTA split on mma.sync and the efficiency loop's split runs on tcgen05.

    python scripts/probe_g_mid_policy.py      (on the GPU box)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_timing import bench

if __name__ == "__main__":
    for g in (20, 24, 28):
        for b in (4, 8, 16, 32):
            for pol in ("guarded", "seq_aware_sm"):
                bench(b, g, 1, 4096, pol, steps=50, reps=5)
