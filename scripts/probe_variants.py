"""Build-variant A/B (development tool): the same shapes under the product library and the
variants in paper_2604_00028_b200/lib/variants/libdecattn_<name>.so (DECATTN_LIB), in
interleaved rounds.

    python scripts/probe_variants.py [--set=latency] name1 name2 ...      (on the GPU box)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "one" and sys.argv[2] == "latency":
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        from probe_timing import bench
        for pol in ("guarded", "seq_aware", "seq_aware_sm", "evolved"):
            bench(1, 64, 8, 512, pol, steps=200, reps=7)
            bench(1, 8, 1, 512, pol, steps=200, reps=7)
        for lk in (128, 256, 384):
            bench(1, 8, 1, lk, "guarded", steps=200, reps=7)
        bench(1, 16, 1, 512, "seq_aware_sm", steps=200, reps=7)
        bench(1, 128, 8, 512, "seq_aware_sm", steps=200, reps=7)
        bench(2, 16, 2, 1024, "seq_aware_sm", steps=200, reps=7)
        bench(1, 64, 8, 2048, "seq_aware_sm", steps=200, reps=7)
        bench(1, 8, 1, 4096, "seq_aware_sm", steps=200, reps=7)
        bench(1, 64, 8, 512, "seq_aware", pack=False, steps=200, reps=7)
        sys.exit(0)
    if len(sys.argv) > 2 and sys.argv[1] == "one" and sys.argv[2] == "wide":
        # G > 8: 16-row CTAs (two 8-row MMA blocks per warp) on streaming and latency shapes
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        from probe_timing import bench
        bench(64, 128, 8, 8192, "seq_aware", steps=5, reps=5)      # G = 16, saturated, 2.1 GB
        bench(32, 128, 4, 16384, "seq_aware", steps=5, reps=5)     # G = 32, 2 m-blocks of 16 rows
        bench(128, 64, 8, 8192, "seq_aware", steps=5, reps=5)      # G = 8 reference (high-load)
        bench(1, 128, 8, 131072, "seq_aware_sm", steps=20, reps=5) # G = 16, long context
        bench(1, 128, 8, 131072, "seq_aware", steps=20, reps=5)
        bench(1, 16, 1, 512, "seq_aware_sm", steps=200, reps=7)
        bench(1, 128, 8, 512, "seq_aware_sm", steps=200, reps=7)
        bench(128, 64, 1, 8192, "seq_aware", steps=10, reps=5)     # MQA, G = 64: 4 CTAs per KV head
        bench(32, 64, 1, 32768, "seq_aware", steps=10, reps=5)
        bench(128, 32, 1, 8192, "seq_aware", steps=10, reps=5)     # G = 32
        bench(128, 16, 1, 8192, "seq_aware", steps=10, reps=5)     # G = 16
        bench(128, 8, 1, 8192, "seq_aware", steps=10, reps=5)      # G = 8
        bench(1, 64, 1, 131072, "seq_aware", steps=20, reps=5)     # MQA long context
        sys.exit(0)
    if len(sys.argv) > 2 and sys.argv[1] == "one" and sys.argv[2] == "mqa":
        # wide query groups: the tcgen05 path (G >= 32) against the mma.sync path (variant notc)
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        from probe_timing import bench
        bench(128, 64, 1, 8192, "seq_aware", steps=10, reps=5)
        bench(32, 64, 1, 32768, "seq_aware", steps=10, reps=5)
        bench(128, 32, 1, 8192, "seq_aware", steps=10, reps=5)
        bench(64, 128, 2, 8192, "seq_aware", steps=10, reps=5)
        bench(1, 64, 1, 131072, "seq_aware", steps=20, reps=5)
        bench(1, 64, 1, 131072, "seq_aware_sm", steps=20, reps=5)
        for pol in ("guarded", "seq_aware", "seq_aware_sm"):
            bench(1, 64, 1, 512, pol, steps=200, reps=7)
            bench(1, 32, 1, 512, pol, steps=200, reps=7)
            bench(4, 64, 1, 2048, pol, steps=200, reps=7)
        sys.exit(0)
    if len(sys.argv) > 2 and sys.argv[1] == "one" and sys.argv[2] == "mqa_mid":
        # MQA G = 64 mid-size shapes: where the tcgen05 / mma.sync boundary (kTcMinTiles) should sit
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        from probe_timing import bench
        for shp in ((4, 64, 1, 8192), (8, 64, 1, 4096), (2, 64, 1, 32768), (16, 64, 1, 2048), (1, 64, 1, 16384),
                    (1, 64, 1, 4096), (1, 64, 1, 1024), (32, 64, 1, 1024), (64, 64, 1, 2048)):
            for pol in ("guarded", "seq_aware_sm"):
                bench(*shp, pol, steps=50, reps=5)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        from probe_timing import bench
        bench(1, 64, 8, 131072, "fixed", 10, combine=1, steps=20, reps=7)
        bench(1, 64, 8, 131072, "fixed", 16, combine=2, steps=20, reps=7)
        bench(1, 64, 8, 131072, "fixed", 18, combine=2, steps=20, reps=7)
        bench(4, 32, 4, 65536, "seq_aware", steps=20, reps=7)
        bench(1, 8, 1, 131072, "guarded", steps=40, reps=7)
        bench(128, 64, 8, 8192, "seq_aware", steps=5, reps=5)
        bench(1, 64, 8, 512, "seq_aware_sm", steps=200, reps=7)
        bench(1, 8, 1, 512, "seq_aware", steps=200, reps=7)
        bench(1, 64, 8, 2048, "seq_aware", steps=200, reps=7)
        sys.exit(0)
    args = sys.argv[1:]
    which = []
    if args and args[0].startswith("--set="):
        which, args = [args[0][6:]], args[1:]
    names = [""] + args
    for rnd in range(2):
        for v in names:
            lib = os.path.join(ROOT, "paper_2604_00028_b200", "lib",
                               *(["variants", f"libdecattn_{v}.so"] if v else ["libdecattn.so"]))
            env = dict(os.environ, DECATTN_LIB=lib)
            r = subprocess.run([sys.executable, __file__, "one"] + which, env=env, capture_output=True, text=True)
            print(f"== round {rnd} {v or 'product'}\n{r.stdout}{r.stderr[-2000:] if r.returncode else ''}", flush=True)
