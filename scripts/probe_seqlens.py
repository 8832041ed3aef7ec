"""Headline shapes WITH a cache_seqlens tensor (the serving call): the speculative pre-wait prefetch."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_timing import bench  # noqa: E402

if __name__ == "__main__":
    bench(1, 64, 8, 512, "seq_aware_sm", steps=200, reps=7)
    bench(1, 8, 1, 512, "seq_aware_sm", steps=200, reps=7)
    bench(1, 64, 8, 512, "guarded", steps=200, reps=7)
