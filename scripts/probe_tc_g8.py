"""G = 8 streaming shapes forced onto the tcgen05 kernel (development tool): its 224 KB ring per CTA
against the mma.sync kernel's 128 KB (workspace plans) / 192 KB (cluster plans) / 224 KB (s = 1).

    python scripts/probe_tc_g8.py      (on the GPU box)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_timing import bench

if __name__ == "__main__":
    for _ in range(2):
        bench(1, 64, 8, 131072, "fixed", 10, combine=1, steps=20, reps=7)          # the C-ext-1 plan
        bench(1, 64, 8, 131072, "fixed", 16, combine=2, steps=20, reps=7)          # the paper's rule
        for s in (16, 18):
            bench(1, 64, 8, 131072, "fixed", s, combine=2, steps=20, reps=7, path=2)
        bench(128, 64, 8, 8192, "seq_aware", steps=5, reps=5)                       # high-load
        bench(128, 64, 8, 8192, "seq_aware", steps=5, reps=5, path=2)
        bench(4, 32, 4, 65536, "seq_aware", steps=20, reps=7)
        bench(4, 32, 4, 65536, "seq_aware", steps=20, reps=7, path=2)
