"""Where the cluster-capped split (s = 16, one wave) stops beating the efficiency loop's
workspace-combine split for few tiles (T = 1, 2, 4) as L_K grows (C-ext-1 regime boundary)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_timing import bench  # noqa: E402

if __name__ == "__main__":
    for hkv in (1, 2, 4):
        for lk in (4096, 8192, 12288, 16384, 32768):
            steps = 100 if lk <= 16384 else 40
            bench(1, 8 * hkv, hkv, lk, "fixed", 16, steps=steps, reps=5)
            bench(1, 8 * hkv, hkv, lk, "guarded", steps=steps, reps=5)
