"""G = 16: 16-row CTAs vs two 8-row CTAs per KV head (DECATTN_ROWS16 A/B), policy picks."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_timing import bench  # noqa: E402

if __name__ == "__main__":
    for (b, hkv, lk, steps) in ((1, 1, 512, 200), (1, 8, 512, 200), (1, 8, 2048, 200), (1, 2, 4096, 200),
                                (64, 8, 8192, 5), (1, 8, 65536, 20)):
        bench(b, 16 * hkv, hkv, lk, "seq_aware_sm", steps=steps, reps=5)
        bench(b, 16 * hkv, hkv, lk, "guarded", steps=steps, reps=5)
