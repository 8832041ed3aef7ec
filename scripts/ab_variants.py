"""A/B the ring-depth / consumer-warp configurations (development tool).
Builds variant libraries locally (python scripts/ab_variants.py build) and times them on the GPU
(python scripts/ab_variants.py run)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VARIANTS = {   # name: (none stages, none warps, cluster stages, cluster warps, kernel stages, kernel warps)
    "n7w7_c6w3_k4w4": (7, 7, 6, 3, 4, 4),
    "n6w3_c6w3_k6w3": (6, 3, 6, 3, 6, 3),
}
SHAPES = [(1, 8, 1, 512, "guarded"), (1, 8, 1, 512, "seq_aware"), (1, 16, 2, 512, "guarded"),
          (1, 16, 2, 512, "seq_aware"), (2, 8, 1, 512, "seq_aware"), (1, 128, 8, 512, "seq_aware"),
          (1, 8, 1, 1024, "seq_aware"), (1, 8, 1, 2048, "seq_aware")]

if sys.argv[1] == "build":
    import importlib.util
    _spec = importlib.util.spec_from_file_location("_decattn_build", os.path.join(ROOT, "paper_2604_00028_b200", "build.py"))
    B = importlib.util.module_from_spec(_spec)
    _spec.loader.exec_module(B)
    for name, (ns, nw, cs, cw, ks, kw) in VARIANTS.items():
        B.build(defines=[f"DECATTN_NONE_STAGES={ns}", f"DECATTN_NONE_WARPS={nw}",
                         f"DECATTN_CLUSTER_STAGES={cs}", f"DECATTN_CLUSTER_WARPS={cw}",
                         f"DECATTN_KERNEL_STAGES={ks}", f"DECATTN_KERNEL_WARPS={kw}"],
                lib=f"{B.PKG}/lib/variants/libdecattn_{name}.so", build_dir=f"{B.PKG}/build/{name}")
    print("built")
elif sys.argv[1] == "run":
    for name in VARIANTS:
        env = dict(os.environ, DECATTN_LIB=f"{ROOT}/paper_2604_00028_b200/lib/variants/libdecattn_{name}.so")
        out = subprocess.run([sys.executable, __file__, "one"], env=env, capture_output=True, text=True)
        print(f"== {name}\n{out.stdout}{out.stderr[-2000:] if out.returncode else ''}", flush=True)
else:
    sys.argv = [sys.argv[0]]
    sys.path.insert(0, os.path.join(ROOT, "scripts"))
    from probe_timing import bench
    import io, contextlib
    res = []
    for b, hq, hkv, lk, pol in SHAPES:
        steps = 5 if b == 128 else (20 if lk > 100000 else 200)
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            us = bench(b, hq, hkv, lk, pol, steps=steps, reps=5 if b < 128 else 3)
        res.append(f"{b}x{hq}x{hkv}x{lk}:{pol[:3]}={us:.2f}")
    print("  " + "  ".join(res))
