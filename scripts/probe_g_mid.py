"""Query groups between 16 and 32 (development tool): the mma.sync kernel needs two 16-row CTAs per
KV head (K / V read twice) where the tcgen05 kernel's 64-row CTA reads them once.

    python scripts/probe_g_mid.py      (on the GPU box)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_timing import bench

if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "grid":
    pass
elif __name__ == "__main__":
    for _ in range(2):
        for hq, hkv in ((24, 1), (20, 1), (48, 2), (16, 1)):
            for b, lk in ((128, 8192), (16, 8192), (4, 16384)):
                bench(b, hq, hkv, lk, "seq_aware", steps=10, reps=5)
                bench(b, hq, hkv, lk, "seq_aware", steps=10, reps=5, path=2)


def grid():
    """The planner's choice (tcgen05 for G > 16 on >= 4-tile splits with >= U / 2 CTAs) against the
    mma.sync kernel forced, over G 20 / 24 / 28 and a range of batch sizes and lengths."""
    for g in (20, 24, 28):
        for b in (1, 2, 4, 8, 16, 32, 64):
            for lk in (2048, 8192, 32768):
                if b * lk * 512 > (1 << 30):
                    continue
                for pol in ("guarded", "seq_aware_sm"):
                    bench(b, g, 1, lk, pol, steps=20, reps=5)
                    bench(b, g, 1, lk, pol, steps=20, reps=5, path=1)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "grid":
    grid()


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "small":
    # 8 < G <= 16: one 16-row mma.sync CTA per KV head on long splits (two 8-row CTAs on short ones)
    for g, hkv in ((12, 1), (16, 1), (16, 2)):
        for b in (4, 16, 64, 128):
            for lk in (2048, 8192, 32768):
                if b * hkv * lk * 512 > (1 << 30):
                    continue
                bench(b, g * hkv, hkv, lk, "seq_aware", steps=20, reps=5)
                bench(b, g * hkv, hkv, lk, "seq_aware", steps=20, reps=5, path=2)
