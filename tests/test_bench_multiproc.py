"""bench.py's multi-rank plumbing (weak scaling by batch: barrier, max-over-ranks timing,
rank-0 JSON) with world_size 2 as two processes sharing one GPU over gloo.  Kernels of one
rank never wait on the other's (no data-path collective in this mode)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_two_ranks_batch_sharded():
    env = dict(os.environ, DECATTN_BENCH_BACKEND="gloo", DECATTN_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--workload", "llama70b", "--steps", "20", "--warmup", "3"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout              # rank 0 alone prints one JSON line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["config"]["global_batch"] == 2
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] == 20


@pytest.mark.gpu
@pytest.mark.parametrize("exchange,launches", [("p2p", 1), ("p2p-split", 3), ("nccl", 2)])
def test_bench_sequence_sharded_step_one_rank(exchange, launches):
    # the long-context sequence-sharded step (forward + exchange + combine) through bench.py on a
    # one-rank group: the same code path the N-GPU run takes, every exchange flavour
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "long_context", "--seq-shard",
           "--exchange", exchange, "--steps", "5", "--warmup", "3", "--no-extras", "--cpu-seconds", "0.5"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["scaling"] == "strong" and d["config"]["workload"] == "long_context"
    assert d["value"] > 1000 and d["gpu_launches"] == 5 * launches


@pytest.mark.gpu
def test_bench_two_ranks_high_load_batch_split():
    # high-load at N > 1 splits the B = 128 batch across ranks (strong scaling, no collective)
    env = dict(os.environ, DECATTN_BENCH_BACKEND="gloo", DECATTN_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29519", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--workload", "high_load", "--steps", "3", "--warmup", "3"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["global_batch"] == 128
    assert d["value"] > 0 and d["gpu_launches"] == 3


@pytest.mark.gpu
def test_bench_two_ranks_head_sharded():
    # Llama-70B with the KV heads split across ranks (the tensor-parallel mapping): strong scaling
    env = dict(os.environ, DECATTN_BENCH_BACKEND="gloo", DECATTN_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29521", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--workload", "llama70b", "--shard-heads", "--steps", "20", "--warmup", "3"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["scaling"] == "strong" and d["config"]["global_batch"] == 1 and "head-sharded" in d["config"]["parallelism"]
    assert d["value"] > 0 and d["gpu_launches"] == 20
