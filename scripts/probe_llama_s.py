"""Llama-70B decode step (B1 H_Q64 H_KV8 L512) at forced split counts and combine modes
(development tool): where the U-curve of the latency shape bottoms out on this kernel.

    python scripts/probe_llama_s.py      (on the GPU box)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_timing import bench

if __name__ == "__main__":
    for _ in range(2):
        bench(1, 64, 8, 512, "seq_aware_sm", steps=200, reps=7)
        for s in (2, 4, 6, 8):
            bench(1, 64, 8, 512, "fixed", s, combine=1, steps=200, reps=7)
        for s in (4, 8):
            bench(1, 64, 8, 512, "fixed", s, combine=2, steps=200, reps=7)
        bench(1, 8, 1, 512, "seq_aware_sm", steps=200, reps=7)
        for s in (4, 8, 12, 16):
            bench(1, 8, 1, 512, "fixed", s, combine=1, steps=200, reps=7)
