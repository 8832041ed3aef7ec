"""Long-context T=8: cluster-sized splits vs the efficiency loop's s=16 workspace combine."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_timing import bench  # noqa: E402

if __name__ == "__main__":
    for s in (6, 8, 10, 16):
        bench(1, 64, 8, 131072, "fixed", s, steps=20, reps=7)
    bench(1, 64, 8, 131072, "fixed", 16, steps=20, reps=7, combine=2)
    for s in (8, 10, 16):
        bench(1, 64, 8, 32768, "fixed", s, steps=50, reps=7)
    bench(1, 8, 1, 131072, "fixed", 16, steps=20, reps=7)
    bench(1, 8, 1, 131072, "fixed", 64, steps=20, reps=7)
    bench(1, 8, 1, 131072, "guarded", steps=20, reps=7)
