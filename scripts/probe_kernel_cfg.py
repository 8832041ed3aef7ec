"""Workspace-combine (KERNEL) kernel configuration A/B (DECATTN_KERNEL_STAGES / _WARPS builds via
DECATTN_LIB): the streaming long-context split and latency-regime workspace splits."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_timing import bench  # noqa: E402

if __name__ == "__main__":
    print("==", os.environ.get("DECATTN_LIB", "product"), flush=True)
    bench(1, 64, 8, 131072, "fixed", forced=16, combine=2, steps=20, reps=5)
    bench(1, 64, 8, 131072, "fixed", forced=18, combine=2, steps=20, reps=5)
    bench(1, 64, 8, 131072, "seq_aware_sm", steps=20, reps=5)
    bench(1, 64, 8, 32768, "fixed", forced=18, combine=2, steps=50, reps=5)
    bench(1, 64, 8, 32768, "seq_aware_sm", steps=50, reps=5)
    bench(1, 64, 8, 2048, "guarded", steps=200, reps=5)
    bench(1, 8, 1, 4096, "guarded", steps=200, reps=5)
    bench(1, 64, 8, 512, "evolved", steps=200, reps=5)
    bench(1, 8, 1, 512, "fixed", forced=32, combine=2, steps=200, reps=5)
