"""Long context B1 H_KV8 L131072: split count x workspace-kernel configuration (set by DECATTN_LIB)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_timing import bench  # noqa: E402

if __name__ == "__main__":
    for s in (10, 16, 18):
        bench(1, 64, 8, 131072, "fixed", s, steps=20, reps=5, combine=2)
    bench(1, 64, 8, 131072, "fixed", 10, steps=20, reps=5, combine=1)
    bench(128, 64, 8, 8192, "fixed", 1, steps=3, reps=3)
