"""A/B of the latency shapes across source trees (development tool): each tree (the repo and
git worktrees of older commits under build/wt_<sha>, each built in place) runs the same shapes in
its own process, in interleaved rounds on one box.

    python scripts/ab_trees.py build/wt_<sha> ...      (on the GPU box)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = """
import sys
sys.path.insert(0, 'scripts')
from probe_timing import bench
bench(1, 8, 1, 512, 'seq_aware_sm', steps=200, reps=7)
bench(1, 8, 1, 512, 'seq_aware', steps=200, reps=7)
bench(1, 64, 8, 512, 'seq_aware_sm', steps=200, reps=7)
bench(1, 16, 2, 384, 'seq_aware_sm', steps=200, reps=7)
bench(1, 8, 1, 512, 'guarded', steps=200, reps=7)
bench(1, 64, 8, 512, 'guarded', steps=200, reps=7)
"""

STREAM = """
import sys
sys.path.insert(0, 'scripts')
from probe_timing import bench
bench(128, 64, 8, 8192, 'seq_aware', steps=5, reps=5)
bench(1, 64, 8, 131072, 'seq_aware_sm', steps=20, reps=7)
bench(1, 64, 8, 131072, 'seq_aware', steps=20, reps=7)
bench(4, 32, 4, 65536, 'seq_aware', steps=20, reps=7)
"""

MQA = """
import sys
sys.path.insert(0, 'scripts')
from probe_timing import bench
for shp in ((4, 64, 1, 8192), (8, 64, 1, 4096), (2, 64, 1, 32768), (16, 64, 1, 2048), (32, 64, 1, 1024), (64, 64, 1, 2048)):
    bench(*shp, 'guarded', steps=50, reps=5)
bench(128, 64, 1, 8192, 'seq_aware', steps=10, reps=5)
"""

if __name__ == "__main__":
    if os.environ.get("AB_SET") == "stream":
        CODE = STREAM
    if os.environ.get("AB_SET") == "mqa":
        CODE = MQA
    trees = [ROOT] + [os.path.join(ROOT, t) for t in sys.argv[1:]]
    env = dict(os.environ)
    env.pop("DECATTN_LIB", None)
    for rnd in range(3):
        for t in trees:
            print(f"== round {rnd} {os.path.basename(t) if t != ROOT else 'HEAD'}", flush=True)
            r = subprocess.run([sys.executable, "-c", CODE], cwd=t, env=env, capture_output=True, text=True)
            print(r.stdout.strip() or r.stderr[-2000:], flush=True)
