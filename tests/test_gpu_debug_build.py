"""Memory-safety substitute for compute-sanitizer (closed on the GPU pool): build the library
with -DDECATTN_DEBUG (device asserts on every computed global / shared-memory index, see
csrc/ptx.cuh DA_DASSERT) and run a cross-section of the GPU parity tests against it in a
subprocess (DECATTN_LIB selects the variant).  A failed assert aborts the kernel and fails
the run."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_parity_subset_under_debug_asserts():
    sys.path.insert(0, ROOT)
    import importlib.util
    _spec = importlib.util.spec_from_file_location("_decattn_build", os.path.join(ROOT, "paper_2604_00028_b200", "build.py"))
    B = importlib.util.module_from_spec(_spec)
    _spec.loader.exec_module(B)
    lib = B.build(defines=["DECATTN_DEBUG=1"], lib=os.path.join(B.PKG, "lib", "variants", "libdecattn_debug.so"),
                  build_dir=os.path.join(B.PKG, "build", "debug"))
    env = dict(os.environ, DECATTN_LIB=lib)
    sel = ("baseline_configs or cluster_combine or kernel_combine_partials or scalar_path or lcap_larger "
           "or short_sequences or combine_kernel_direct or variants or group_sizes or strided "
           "or dynamic_splits or paged or seq_aware_sm_fit or forward_host")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                        "-m", "gpu", "-x", "-q", "-k", sel], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    # the fused peer publish instantiations (da_forward_peer) and the peer exchange kernels
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_peer_exchange.py"),
                        "-m", "gpu", "-x", "-q"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
