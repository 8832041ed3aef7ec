"""G = 16 (the 16-row MMA path): forced splits vs the SM-count-aware pick (its constants were
calibrated at G = 8)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_timing import bench  # noqa: E402
import paper_2604_00028_b200 as dec  # noqa: E402

if __name__ == "__main__":
    for (b, hkv, lk) in ((1, 1, 512), (1, 8, 512), (1, 1, 2048), (1, 8, 2048), (1, 1, 384)):
        pick = dec.make_plan(b, 16 * hkv, hkv, lk, policy="seq_aware_sm").num_splits
        print(f"== B={b} H_KV={hkv} L={lk} G=16: SM-count-aware pick s={pick}", flush=True)
        for s in (1, 2, 4, 6, 8, 12, 16):
            bench(b, 16 * hkv, hkv, lk, "fixed", s, steps=200, reps=5)
