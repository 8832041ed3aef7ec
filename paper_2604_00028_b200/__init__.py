"""paper_2604_00028_b200 - B200-native (sm_100a) split-KV decode attention with the
sequence-aware split policy of arxiv/paper_2604_00028.

Layers:
  include/decattn.h + csrc/  C ABI library libdecattn.so (planner, kernels)
  _lib                       ctypes binding, same names as the C entry points
  api                        torch convenience: make_plan / forward / combine
  dist                       multi-GPU layer (batch / head / sequence sharding)

The product path never imports the CPU oracle (oracle/, test infrastructure)
and has no CPU fallback: importing this package fails if libdecattn.so is
missing.
"""

from . import _lib  # noqa: F401  (raises ImportError if libdecattn.so is missing)
from ._lib import (DA_BF16, DA_COMBINE_CLUSTER, DA_COMBINE_KERNEL, DA_COMBINE_NONE, DA_F32,  # noqa: F401
                   DA_ERR_TIMEOUT, DA_PATH_MMA, DA_PATH_SCALAR, DA_PATH_TC, DA_POLICY_FIXED, DA_POLICY_GUARDED,
                   DA_POLICY_SEQ_AWARE, DecAttnError, da_abi_version, da_combine, da_combine_peers, da_forward,
                   da_forward_host, da_forward_host_bytes, da_forward_paged, da_forward_peer, da_peer_signal,
                   da_plan, da_plan_make, da_plan_make_varlen, da_plan_set_combine, da_plan_set_path, da_plan_set_seq_offset, da_query_residency,
                   da_status_string)
from .api import (HostStaging, combine, decode_attention, forward, forward_host, forward_paged,  # noqa: F401
                  forward_peer, forward_peer_combine, make_plan, make_plan_varlen, workspace_for)

__all__ = ["da_plan_make", "da_plan_make_varlen", "da_plan_set_combine", "da_plan_set_path", "da_plan_set_seq_offset", "da_forward", "da_forward_paged", "da_forward_host",
           "da_forward_host_bytes", "da_combine", "da_status_string", "da_abi_version", "make_plan", "forward",
           "forward_paged", "forward_host", "HostStaging", "combine", "decode_attention",
           "make_plan_varlen", "da_peer_signal", "da_combine_peers", "da_forward_peer", "forward_peer",
           "forward_peer_combine", "da_query_residency"]
