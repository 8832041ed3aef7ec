"""Scalar (one query row per CTA) path throughput on MHA shapes (G = 1) and unpacked GQA."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_timing import bench  # noqa: E402

if __name__ == "__main__":
    bench(128, 8, 8, 8192, "seq_aware", steps=5, reps=3)             # MHA, 4.3 GB of KV
    bench(16, 32, 32, 8192, "seq_aware", steps=5, reps=3)            # MHA, 2.1 GB
    bench(1, 32, 32, 4096, "seq_aware", steps=50, reps=5)            # MHA latency-ish
    bench(128, 64, 8, 8192, "seq_aware", steps=5, reps=3, pack=False)  # unpacked GQA
    bench(1, 64, 8, 512, "seq_aware", steps=200, reps=5, pack=False)
