"""ctypes binding of libdecattn.so (include/decattn.h) - argument marshalling only.

Every function here has the name of the C entry point it calls and does
nothing but turn torch tensors into (pointer, stride) arguments, pick the
current CUDA stream, and raise on a non-zero da_status.  All computation runs
in the library's kernels; there is no fallback: if the shared library is
missing this module fails to import.
"""

from __future__ import annotations

import ctypes
import os

import torch

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# DECATTN_LIB selects a development build variant (scripts/ A/B experiments only).
LIB_PATH = os.environ.get("DECATTN_LIB") or os.path.join(PKG_DIR, "lib", "libdecattn.so")

# ---- constants mirrored from include/decattn.h ----------------------------
DA_OK, DA_ERR_INVALID_ARG, DA_ERR_UNSUPPORTED, DA_ERR_ALIGNMENT, DA_ERR_WORKSPACE, DA_ERR_CUDA, DA_ERR_TIMEOUT = range(7)
(DA_POLICY_GUARDED, DA_POLICY_SEQ_AWARE, DA_POLICY_FIXED, DA_POLICY_EVOLVED, DA_POLICY_SEQ_AWARE_SM,
 DA_POLICY_DYNAMIC) = range(6)
(DA_RULE_SATURATED, DA_RULE_GUARD_NBLK4, DA_RULE_GUARD1, DA_RULE_GUARD2, DA_RULE_LOW_TILE,
 DA_RULE_EFF_LOOP, DA_RULE_FORCED, DA_RULE_EVOLVED, DA_RULE_SM_SHORT, DA_RULE_SM_SPLIT,
 DA_RULE_SM_FIT, DA_RULE_DYNAMIC) = range(12)
DA_BF16, DA_F32 = 0, 1
DA_COMBINE_NONE, DA_COMBINE_CLUSTER, DA_COMBINE_KERNEL = range(3)
DA_PATH_SCALAR, DA_PATH_MMA, DA_PATH_TC = 0, 1, 2
DA_ABI_VERSION = 7

POLICIES = {"guarded": DA_POLICY_GUARDED, "seq_aware": DA_POLICY_SEQ_AWARE, "fixed": DA_POLICY_FIXED,
            "evolved": DA_POLICY_EVOLVED, "seq_aware_sm": DA_POLICY_SEQ_AWARE_SM, "dynamic": DA_POLICY_DYNAMIC}
RULE_NAMES = {DA_RULE_SATURATED: "saturated", DA_RULE_GUARD_NBLK4: "guard_nblk4",
              DA_RULE_GUARD1: "guard1", DA_RULE_GUARD2: "guard2", DA_RULE_LOW_TILE: "low_tile",
              DA_RULE_EFF_LOOP: "efficiency_loop", DA_RULE_FORCED: "forced", DA_RULE_EVOLVED: "evolved",
              DA_RULE_SM_SHORT: "sm_short", DA_RULE_SM_SPLIT: "sm_split",
              DA_RULE_SM_FIT: "sm_fit", DA_RULE_DYNAMIC: "dynamic"}


class da_plan(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "batch", "h_q", "h_kv", "l_k", "head_dim", "pack_gqa", "sm_margin", "num_sms",
        "policy", "forced_splits", "usable_sms", "block_n", "num_n_blocks", "num_m_blocks",
        "total_mblocks", "num_splits", "nonempty_splits", "rule", "split_unit", "path",
        "rows_per_cta", "combine_mode", "grid_x", "grid_y", "grid_z", "block_threads",
        "cluster_x", "smem_bytes")] + [("workspace_bytes", ctypes.c_int64), ("seq_offset", ctypes.c_int32),
                                      ("path_override", ctypes.c_int32)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}

    def __repr__(self):
        d = self.as_dict()
        return "da_plan(" + ", ".join(f"{k}={v}" for k, v in d.items()) + ")"


class DecAttnError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: {da_status_string(status)} (status {status})")
        self.status = status


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`python paper_2604_00028_b200/build.py` (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    i32, i64, vp, f32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_float
    lib.da_plan_make.argtypes = [i32] * 10 + [ctypes.POINTER(da_plan)]
    lib.da_plan_make.restype = i32
    lib.da_plan_make_varlen.argtypes = [i32] * 8 + [vp, ctypes.POINTER(da_plan)]
    lib.da_plan_make_varlen.restype = i32
    lib.da_plan_set_combine.argtypes = [ctypes.POINTER(da_plan), i32]
    lib.da_plan_set_combine.restype = i32
    lib.da_plan_set_seq_offset.argtypes = [ctypes.POINTER(da_plan), i32]
    lib.da_plan_set_seq_offset.restype = i32
    lib.da_plan_set_path.argtypes = [ctypes.POINTER(da_plan), i32]
    lib.da_plan_set_path.restype = i32
    lib.da_forward.argtypes = [ctypes.POINTER(da_plan), vp, vp, vp, i32, vp, vp, f32, i32, vp, vp,
                               vp, i64, vp]
    lib.da_forward.restype = i32
    lib.da_forward_paged.argtypes = [ctypes.POINTER(da_plan), vp, vp, vp, i32, i32, vp, i64, i32, vp, vp, f32,
                                     i32, vp, vp, vp, i64, vp]
    lib.da_forward_paged.restype = i32
    lib.da_forward_host_bytes.argtypes = [ctypes.POINTER(da_plan), i32, i32, i32]
    lib.da_forward_host_bytes.restype = i64
    lib.da_forward_host.argtypes = [ctypes.POINTER(da_plan), vp, vp, vp, i32, vp, f32, i32, vp, vp, vp, i64, vp]
    lib.da_forward_host.restype = i32
    lib.da_peer_signal.argtypes = [i32, i32, vp, vp, vp, i32, i32, i32, i64, i64, i64, vp, vp]
    lib.da_peer_signal.restype = i32
    lib.da_combine_peers.argtypes = [i32, i32, vp, i64, i64, i64, vp, i32, i32, i32, i32, vp, vp, vp, i64, vp]
    lib.da_combine_peers.restype = i32
    lib.da_forward_peer.argtypes = [ctypes.POINTER(da_plan), vp, vp, vp, i32, vp, vp, f32, i32, i32, vp, i64, i64,
                                    i64, vp, vp, vp, i64, vp]
    lib.da_forward_peer.restype = i32
    lib.da_forward_peer_combine.argtypes = [ctypes.POINTER(da_plan), vp, vp, vp, i32, vp, vp, f32, i32, i32, vp,
                                            i64, i64, vp, vp, i32, vp, vp, vp, i64, vp, i64, vp]
    lib.da_forward_peer_combine.restype = i32
    lib.da_query_residency.argtypes = [ctypes.POINTER(da_plan), i32, i32, ctypes.POINTER(i32)]
    lib.da_query_residency.restype = i32
    lib.da_combine.argtypes = [i32, i32, i32, i32, vp, i64, vp, i64, i32, vp, vp, vp]
    lib.da_combine.restype = i32
    lib.da_status_string.argtypes = [i32]
    lib.da_status_string.restype = ctypes.c_char_p
    lib.da_abi_version.argtypes = []
    lib.da_abi_version.restype = i32
    if lib.da_abi_version() != DA_ABI_VERSION:
        raise ImportError("libdecattn.so ABI version mismatch")
    return lib


LIB = _load()

EXPORTED = ("da_plan_make", "da_plan_make_varlen", "da_plan_set_combine", "da_plan_set_seq_offset", "da_plan_set_path", "da_forward", "da_forward_paged",
            "da_forward_host_bytes", "da_forward_host", "da_combine", "da_peer_signal", "da_combine_peers",
            "da_forward_peer", "da_forward_peer_combine", "da_query_residency", "da_status_string",
            "da_abi_version")


def da_status_string(status: int) -> str:
    return LIB.da_status_string(int(status)).decode()


def da_abi_version() -> int:
    return int(LIB.da_abi_version())


def da_plan_make(batch, h_q, h_kv, l_k, head_dim=128, pack_gqa=1, sm_margin=0, num_sms=148,
                 policy=DA_POLICY_SEQ_AWARE, forced_splits=0) -> da_plan:
    if isinstance(policy, str):
        policy = POLICIES[policy]
    p = da_plan()
    st = LIB.da_plan_make(int(batch), int(h_q), int(h_kv), int(l_k), int(head_dim), int(pack_gqa),
                          int(sm_margin), int(num_sms), int(policy), int(forced_splits),
                          ctypes.byref(p))
    if st != DA_OK:
        raise DecAttnError(st, "da_plan_make")
    return p


def da_plan_make_varlen(batch, h_q, h_kv, l_cap, head_dim, pack_gqa, sm_margin, num_sms, host_seqlens) -> da_plan:
    """host_seqlens: a sequence of ints (copied into a host int32 array)."""
    lens = [int(x) for x in host_seqlens]
    if len(lens) != int(batch):
        raise DecAttnError(DA_ERR_INVALID_ARG, "da_plan_make_varlen: len(host_seqlens) != batch")
    arr = (ctypes.c_int32 * max(1, len(lens)))(*lens)
    p = da_plan()
    st = LIB.da_plan_make_varlen(int(batch), int(h_q), int(h_kv), int(l_cap), int(head_dim), int(pack_gqa),
                                 int(sm_margin), int(num_sms), ctypes.cast(arr, ctypes.c_void_p), ctypes.byref(p))
    if st != DA_OK:
        raise DecAttnError(st, "da_plan_make_varlen")
    return p


def da_plan_set_path(plan: da_plan, path: int) -> da_plan:
    st = LIB.da_plan_set_path(ctypes.byref(plan), int(path))
    if st != DA_OK:
        raise DecAttnError(st, "da_plan_set_path")
    return plan


def da_plan_set_seq_offset(plan: da_plan, seq_offset: int) -> da_plan:
    st = LIB.da_plan_set_seq_offset(ctypes.byref(plan), int(seq_offset))
    if st != DA_OK:
        raise DecAttnError(st, "da_plan_set_seq_offset")
    return plan


def da_plan_set_combine(plan: da_plan, combine_mode: int) -> da_plan:
    st = LIB.da_plan_set_combine(ctypes.byref(plan), int(combine_mode))
    if st != DA_OK:
        raise DecAttnError(st, "da_plan_set_combine")
    return plan


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream_handle(stream):
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def da_forward(plan: da_plan, q, k_cache, v_cache, l_cap, cache_seqlens, strides, softmax_scale,
               out_dtype, out, lse, workspace, workspace_bytes, stream=None) -> None:
    """Marshal to ``da_forward``.  Tensor arguments may be torch tensors or raw
    device pointers (ints); ``strides`` is a sequence of 8 ints or None."""
    sarr = None
    if strides is not None:
        sarr = (ctypes.c_int64 * 8)(*[int(x) for x in strides])
    st = LIB.da_forward(ctypes.byref(plan), _ptr(q), _ptr(k_cache), _ptr(v_cache), int(l_cap),
                        _ptr(cache_seqlens), sarr, float(softmax_scale), int(out_dtype), _ptr(out),
                        _ptr(lse), _ptr(workspace), int(workspace_bytes), _stream_handle(stream))
    if st != DA_OK:
        raise DecAttnError(st, "da_forward")


def da_forward_paged(plan: da_plan, q, k_pages, v_pages, num_pages, page_size, block_table,
                     block_table_stride, max_pages_per_seq, cache_seqlens, strides, softmax_scale,
                     out_dtype, out, lse, workspace, workspace_bytes, stream=None) -> None:
    """Marshal to ``da_forward_paged`` (paged KV cache with a block table)."""
    sarr = None
    if strides is not None:
        sarr = (ctypes.c_int64 * 8)(*[int(x) for x in strides])
    st = LIB.da_forward_paged(ctypes.byref(plan), _ptr(q), _ptr(k_pages), _ptr(v_pages), int(num_pages),
                              int(page_size), _ptr(block_table), int(block_table_stride),
                              int(max_pages_per_seq), _ptr(cache_seqlens), sarr, float(softmax_scale),
                              int(out_dtype), _ptr(out), _ptr(lse), _ptr(workspace), int(workspace_bytes),
                              _stream_handle(stream))
    if st != DA_OK:
        raise DecAttnError(st, "da_forward_paged")


def da_forward_host_bytes(plan: da_plan, l_cap, with_seqlens, out_dtype) -> int:
    n = int(LIB.da_forward_host_bytes(ctypes.byref(plan), int(l_cap), int(bool(with_seqlens)), int(out_dtype)))
    if n < 0:
        raise DecAttnError(DA_ERR_INVALID_ARG, "da_forward_host_bytes")
    return n


def da_forward_host(plan: da_plan, q, k_cache, v_cache, l_cap, cache_seqlens, softmax_scale, out_dtype,
                    out, lse, device_buffer, device_buffer_bytes, stream=None) -> None:
    """Marshal to ``da_forward_host``: q / k_cache / v_cache / cache_seqlens / out / lse are HOST
    tensors (or host addresses); device_buffer is device scratch."""
    st = LIB.da_forward_host(ctypes.byref(plan), _ptr(q), _ptr(k_cache), _ptr(v_cache), int(l_cap),
                             _ptr(cache_seqlens), float(softmax_scale), int(out_dtype), _ptr(out), _ptr(lse),
                             _ptr(device_buffer), int(device_buffer_bytes), _stream_handle(stream))
    if st != DA_OK:
        raise DecAttnError(st, "da_forward_host")


def da_peer_signal(world, rank, peer_bases, o_local, lse_local, batch, h_q, head_dim, slot_bytes, lse_offset,
                   flag_offset, epoch, stream=None) -> None:
    st = LIB.da_peer_signal(int(world), int(rank), _ptr(peer_bases), _ptr(o_local), _ptr(lse_local), int(batch),
                            int(h_q), int(head_dim), int(slot_bytes), int(lse_offset), int(flag_offset), _ptr(epoch),
                            _stream_handle(stream))
    if st != DA_OK:
        raise DecAttnError(st, "da_peer_signal")


def da_combine_peers(world, rank, peer_bases, slot_bytes, lse_offset, flag_offset, epoch, batch, h_q, head_dim,
                     out_dtype, out, lse, status, timeout_ns=0, stream=None) -> None:
    st = LIB.da_combine_peers(int(world), int(rank), _ptr(peer_bases), int(slot_bytes), int(lse_offset),
                              int(flag_offset), _ptr(epoch), int(batch), int(h_q), int(head_dim), int(out_dtype),
                              _ptr(out), _ptr(lse), _ptr(status), int(timeout_ns), _stream_handle(stream))
    if st != DA_OK:
        raise DecAttnError(st, "da_combine_peers")


def da_forward_peer(plan: da_plan, q, k_cache, v_cache, l_cap, cache_seqlens, strides, softmax_scale, world, rank,
                    peer_bases, slot_bytes, lse_offset, flag_offset, epoch, counter, workspace, workspace_bytes,
                    stream=None) -> None:
    sarr = None
    if strides is not None:
        sarr = (ctypes.c_int64 * 8)(*[int(x) for x in strides])
    st = LIB.da_forward_peer(ctypes.byref(plan), _ptr(q), _ptr(k_cache), _ptr(v_cache), int(l_cap),
                             _ptr(cache_seqlens), sarr, float(softmax_scale), int(world), int(rank), _ptr(peer_bases),
                             int(slot_bytes), int(lse_offset), int(flag_offset), _ptr(epoch), _ptr(counter),
                             _ptr(workspace), int(workspace_bytes), _stream_handle(stream))
    if st != DA_OK:
        raise DecAttnError(st, "da_forward_peer")


def da_forward_peer_combine(plan: da_plan, q, k_cache, v_cache, l_cap, cache_seqlens, strides, softmax_scale, world,
                            rank, peer_bases, ll_offset, ll_slot_bytes, epoch, counter, out_dtype, out, lse,
                            status, timeout_ns=0, workspace=None, workspace_bytes=0, stream=None) -> None:
    sarr = None
    if strides is not None:
        sarr = (ctypes.c_int64 * 8)(*[int(x) for x in strides])
    st = LIB.da_forward_peer_combine(ctypes.byref(plan), _ptr(q), _ptr(k_cache), _ptr(v_cache), int(l_cap),
                                     _ptr(cache_seqlens), sarr, float(softmax_scale), int(world), int(rank),
                                     _ptr(peer_bases), int(ll_offset), int(ll_slot_bytes), _ptr(epoch), _ptr(counter),
                                     int(out_dtype), _ptr(out), _ptr(lse), _ptr(status), int(timeout_ns),
                                     _ptr(workspace), int(workspace_bytes), _stream_handle(stream))
    if st != DA_OK:
        raise DecAttnError(st, "da_forward_peer_combine")


def da_query_residency(plan: da_plan, kernel: int, exchange: int = 0) -> int:
    """Co-resident launch units of the plan's forward (kernel 0; clusters for CLUSTER plans, else
    CTAs) or of the combine kernel (kernel 1) on the current device."""
    n = ctypes.c_int32(0)
    st = LIB.da_query_residency(ctypes.byref(plan), int(kernel), int(exchange), ctypes.byref(n))
    if st != DA_OK:
        raise DecAttnError(st, "da_query_residency")
    return int(n.value)


def da_combine(num_splits, batch, h_q, head_dim, o_partial, o_split_stride, lse_partial,
               lse_split_stride, out_dtype, out, lse, stream=None) -> None:
    st = LIB.da_combine(int(num_splits), int(batch), int(h_q), int(head_dim), _ptr(o_partial),
                        int(o_split_stride), _ptr(lse_partial), int(lse_split_stride),
                        int(out_dtype), _ptr(out), _ptr(lse), _stream_handle(stream))
    if st != DA_OK:
        raise DecAttnError(st, "da_combine")
