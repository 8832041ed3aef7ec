"""DRAM-locality probe (development tool): the same bytes per CTA and the same CTA count, with each
CTA streaming its own contiguous region (H_KV = 1) or the CTAs of one sequence interleaving their
heads over a shared region (H_KV = 8), on both kernels.

    python scripts/probe_locality.py      (on the GPU box)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_timing import bench

if __name__ == "__main__":
    for _ in range(2):
        bench(128, 8, 1, 8192, "seq_aware", steps=10, reps=5)      # mma.sync, 128 CTAs, own regions
        bench(16, 64, 8, 8192, "seq_aware", steps=10, reps=5)      # mma.sync, 128 CTAs, 8 heads share
        bench(128, 64, 1, 8192, "seq_aware", steps=10, reps=5)     # tcgen05, 128 CTAs, own regions
        bench(16, 512, 8, 8192, "seq_aware", steps=10, reps=5)     # tcgen05, 128 CTAs, 8 heads share
        bench(148, 8, 1, 8192, "seq_aware", steps=10, reps=5)      # mma.sync, 148 CTAs, own regions
        bench(1024, 8, 1, 1024, "seq_aware", steps=10, reps=5)     # mma.sync, 1024 CTAs, own 512 KB
        bench(128, 64, 8, 8192, "seq_aware", steps=5, reps=5)      # high-load
