"""Rebuild the development variants of the library (debug asserts, per-CTA trace) in-tree, so a
GPU box that receives the snapshot finds them current (tests/test_gpu_debug_build.py builds the
debug variant itself when stale)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2604_00028_b200"))
import build as B  # noqa: E402

if __name__ == "__main__":
    for name, define in (("debug", "DECATTN_DEBUG=1"), ("trace", "DECATTN_TRACE=1")):
        print(B.build(defines=[define], lib=os.path.join(B.PKG, "lib", "variants", f"libdecattn_{name}.so"),
                      build_dir=os.path.join(B.PKG, "build", name), force=True))
