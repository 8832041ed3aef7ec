"""L_K = 2048, T <= 4: the balanced split s = 11 (3 units per split) vs 12 / 14 / 16 (C-ext-1 v3)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_timing import bench  # noqa: E402

if __name__ == "__main__":
    for hkv in (1, 2, 4):
        for s in (11, 12, 14, 16):
            bench(1, 8 * hkv, hkv, 2048, "fixed", s, steps=200, reps=7, combine=1)
