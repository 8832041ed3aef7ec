"""Torch-facing convenience over the C ABI (allocation + marshalling only).

    plan = make_plan(batch, h_q, h_kv, l_k, policy="seq_aware")
    out, lse = forward(plan, q, k_cache, v_cache, cache_seqlens)

``make_plan`` caches plans per shape (the precomputed-metadata deployment
path the paper measures, §5.1: the split is decided once per shape,
off the timed path).  ``forward`` allocates out / lse / workspace when not
given and calls ``da_forward`` on the current stream.  Nothing here computes
attention: every step of the path runs in libdecattn.so's kernels.
"""

from __future__ import annotations

import functools

import torch

from . import _lib as L


def _check_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("decattn: tensors must be CUDA tensors (there is no CPU path)")


@functools.lru_cache(maxsize=None)
def num_sms(device_index: int = 0) -> int:
    return torch.cuda.get_device_properties(device_index).multi_processor_count


@functools.lru_cache(maxsize=4096)
def _plan_cached(batch, h_q, h_kv, l_k, head_dim, pack_gqa, sm_margin, sms, policy, forced,
                 combine_mode, seq_offset=0, path=None):
    p = L.da_plan_make(batch, h_q, h_kv, l_k, head_dim, pack_gqa, sm_margin, sms, policy, forced)
    if path is not None:
        L.da_plan_set_path(p, path)
    if combine_mode is not None and combine_mode != p.combine_mode:
        L.da_plan_set_combine(p, combine_mode)
    if seq_offset:
        L.da_plan_set_seq_offset(p, seq_offset)
    return p


def make_plan(batch, h_q, h_kv, l_k, head_dim=128, pack_gqa=True, sm_margin=0, num_sms_=None,
              policy="seq_aware", forced_splits=0, combine_mode=None, seq_offset=0, path=None) -> L.da_plan:
    """da_plan_make (+ da_plan_set_combine when combine_mode is given, + da_plan_set_seq_offset for
    the shard of a sequence-sharded cache that starts at token seq_offset: cache_seqlens are then
    whole-sequence lengths; + da_plan_set_path when path is given: DA_PATH_MMA / DA_PATH_TC).  The
    returned plan is shared through a cache: copy it before editing."""
    if isinstance(policy, str):
        policy = L.POLICIES[policy]
    sms = num_sms_ if num_sms_ is not None else num_sms(torch.cuda.current_device())
    return _plan_cached(int(batch), int(h_q), int(h_kv), int(l_k), int(head_dim), int(bool(pack_gqa)),
                        int(sm_margin), int(sms), int(policy), int(forced_splits), combine_mode, int(seq_offset),
                        None if path is None else int(path))


def make_plan_varlen(batch, h_q, h_kv, l_cap, host_seqlens, head_dim=128, pack_gqa=True, sm_margin=0,
                     num_sms_=None) -> L.da_plan:
    """da_plan_make_varlen: the plan for a ragged batch whose lengths are known on the host
    (static SM-count-aware unless the lengths are skewed enough for the dynamic schedule)."""
    sms = num_sms_ if num_sms_ is not None else num_sms(torch.cuda.current_device())
    return L.da_plan_make_varlen(int(batch), int(h_q), int(h_kv), int(l_cap), int(head_dim),
                                 int(bool(pack_gqa)), int(sm_margin), int(sms), host_seqlens)


def _kv_strides(q, k, v):
    if q.stride(-1) != 1 or k.stride(-1) != 1 or v.stride(-1) != 1:
        raise ValueError("innermost (head_dim) dimension must be contiguous")
    return (q.stride(0), q.stride(1), k.stride(0), k.stride(1), k.stride(2),
            v.stride(0), v.stride(1), v.stride(2))


def _check_shapes(plan: L.da_plan, q, k, v, cache_seqlens=None, out=None, lse=None, paged=False):
    """The tensors against the plan's shape (the C ABI takes bare pointers, so a mismatch would
    read or write out of bounds): q [B, H_Q, d]; dense k / v [B, L_cap >= L_K, H_KV, d], paged
    [num_pages, page_size, H_KV, d]; cache_seqlens [B]; out [B, H_Q, d]; lse [B, H_Q]."""
    B, HQ, HKV, D = plan.batch, plan.h_q, plan.h_kv, plan.head_dim
    if tuple(q.shape) != (B, HQ, D):
        raise ValueError(f"q shape {tuple(q.shape)} != plan (batch, h_q, head_dim) {(B, HQ, D)}")
    for name, t in (("k_cache", k), ("v_cache", v)):
        if t.dim() != 4 or t.shape[2] != HKV or t.shape[3] != D or (not paged and (t.shape[0] != B or t.shape[1] < plan.l_k)):
            raise ValueError(f"{name} shape {tuple(t.shape)} does not match the plan (batch {B}, l_k {plan.l_k}, "
                             f"h_kv {HKV}, head_dim {D})")
    if cache_seqlens is not None and tuple(cache_seqlens.shape) != (B,):
        raise ValueError(f"cache_seqlens shape {tuple(cache_seqlens.shape)} != ({B},)")
    if out is not None and tuple(out.shape) != (B, HQ, D):
        raise ValueError(f"out shape {tuple(out.shape)} != {(B, HQ, D)}")
    if lse is not None and tuple(lse.shape) != (B, HQ):
        raise ValueError(f"lse shape {tuple(lse.shape)} != {(B, HQ)}")


def workspace_for(plan: L.da_plan, device) -> torch.Tensor | None:
    if plan.combine_mode != L.DA_COMBINE_KERNEL:
        return None
    return torch.empty(plan.workspace_bytes // 4, dtype=torch.float32, device=device)


def forward(plan: L.da_plan, q, k_cache, v_cache, cache_seqlens=None, *, out=None, lse=None,
            workspace=None, softmax_scale=0.0, out_dtype=torch.bfloat16, stream=None):
    """Decode attention via da_forward.  q [B, H_Q, d] bf16; k/v [B, L_cap, H_KV, d] bf16;
    cache_seqlens int32 [B] or None.  Returns (out [B, H_Q, d], lse [B, H_Q] fp32)."""
    _check_cuda(q, k_cache, v_cache, cache_seqlens)
    if q.dtype != torch.bfloat16 or k_cache.dtype != torch.bfloat16 or v_cache.dtype != torch.bfloat16:
        raise ValueError("q, k_cache, v_cache must be bfloat16")
    if cache_seqlens is not None and cache_seqlens.dtype != torch.int32:
        raise ValueError("cache_seqlens must be int32")
    _check_shapes(plan, q, k_cache, v_cache, cache_seqlens, out, lse)
    B, HQ, D = q.shape
    if out is None:
        out = torch.empty((B, HQ, D), dtype=out_dtype, device=q.device)
    if lse is None:
        lse = torch.empty((B, HQ), dtype=torch.float32, device=q.device)
    if workspace is None:
        workspace = workspace_for(plan, q.device)
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    dt = L.DA_F32 if out.dtype == torch.float32 else L.DA_BF16
    L.da_forward(plan, q, k_cache, v_cache, k_cache.shape[1], cache_seqlens,
                 _kv_strides(q, k_cache, v_cache), softmax_scale, dt, out, lse, workspace, ws_bytes,
                 stream)
    return out, lse


def forward_peer(plan: L.da_plan, q, k_cache, v_cache, cache_seqlens, world, rank, peer_bases, slot_bytes,
                 lse_offset, flag_offset, epoch, counter, *, workspace=None, softmax_scale=0.0, stream=None):
    """Forward + peer publish via da_forward_peer: this rank's fp32 partial (out, lse) lands in slot
    epoch & 1 of its exchange buffer and every rank's flag `rank` is released (dist.py
    PeerSeqShardedDecode).  peer_bases int64 [world], epoch / counter int32 [1], all on the device."""
    _check_cuda(q, k_cache, v_cache, cache_seqlens, peer_bases, epoch, counter)
    if q.dtype != torch.bfloat16 or k_cache.dtype != torch.bfloat16 or v_cache.dtype != torch.bfloat16:
        raise ValueError("q, k_cache, v_cache must be bfloat16")
    if cache_seqlens is not None and cache_seqlens.dtype != torch.int32:
        raise ValueError("cache_seqlens must be int32")
    _check_shapes(plan, q, k_cache, v_cache, cache_seqlens)
    if workspace is None:
        workspace = workspace_for(plan, q.device)
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    L.da_forward_peer(plan, q, k_cache, v_cache, k_cache.shape[1], cache_seqlens, _kv_strides(q, k_cache, v_cache),
                      softmax_scale, world, rank, peer_bases, slot_bytes, lse_offset, flag_offset, epoch, counter,
                      workspace, ws_bytes, stream)


def one_kernel_exchange_ok(plan: L.da_plan) -> bool:
    """da_forward_peer_combine's condition: the kernel that writes the final rows keeps its whole grid
    resident on the current device - the forward's CTAs (NONE) or clusters (CLUSTER), or the combine
    kernel's one CTA per row (workspace plans) - by the occupancy API's answer for that exact kernel
    (da_query_residency), scaled to the plan's usable SMs."""
    kernel_ws = plan.combine_mode == L.DA_COMBINE_KERNEL
    if plan.path == L.DA_PATH_TC and not kernel_ws:
        return False                  # the tcgen05 forward does not publish (da_forward_peer* reject it)
    units = L.da_query_residency(plan, 1 if kernel_ws else 0, 2)
    fit = units * plan.usable_sms // max(plan.num_sms, 1)
    if kernel_ws:
        need = plan.batch * plan.h_q
    elif plan.combine_mode == L.DA_COMBINE_CLUSTER:
        need = plan.grid_y * plan.grid_z
    else:
        need = plan.grid_x * plan.grid_y * plan.grid_z
    return need <= fit


def forward_peer_combine(plan: L.da_plan, q, k_cache, v_cache, cache_seqlens, world, rank, peer_bases, ll_offset,
                         ll_slot_bytes, epoch, counter, status, *, timeout_ns=0, out=None, lse=None, workspace=None,
                         softmax_scale=0.0, out_dtype=torch.bfloat16, stream=None):
    """The sequence-sharded step in one kernel via da_forward_peer_combine: the forward publishes
    this rank's partial, waits for every rank's, and LSE-merges them into (out, lse).  status: device
    int32 [1], set to DA_ERR_TIMEOUT if a peer's words did not arrive within timeout_ns."""
    _check_cuda(q, k_cache, v_cache, cache_seqlens, peer_bases, epoch, counter, status, out, lse)
    if q.dtype != torch.bfloat16 or k_cache.dtype != torch.bfloat16 or v_cache.dtype != torch.bfloat16:
        raise ValueError("q, k_cache, v_cache must be bfloat16")
    if cache_seqlens is not None and cache_seqlens.dtype != torch.int32:
        raise ValueError("cache_seqlens must be int32")
    _check_shapes(plan, q, k_cache, v_cache, cache_seqlens, out, lse)
    B, HQ, D = q.shape
    if out is None:
        out = torch.empty((B, HQ, D), dtype=out_dtype, device=q.device)
    if lse is None:
        lse = torch.empty((B, HQ), dtype=torch.float32, device=q.device)
    dt = L.DA_F32 if out.dtype == torch.float32 else L.DA_BF16
    if workspace is None:
        workspace = workspace_for(plan, q.device)
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    L.da_forward_peer_combine(plan, q, k_cache, v_cache, k_cache.shape[1], cache_seqlens,
                              _kv_strides(q, k_cache, v_cache), softmax_scale, world, rank, peer_bases, ll_offset,
                              ll_slot_bytes, epoch, counter, dt, out, lse, status, timeout_ns, workspace, ws_bytes,
                              stream)
    return out, lse


def forward_paged(plan: L.da_plan, q, k_pages, v_pages, block_table, cache_seqlens=None, *, out=None,
                  lse=None, workspace=None, softmax_scale=0.0, out_dtype=torch.bfloat16, stream=None):
    """Decode attention over a paged cache via da_forward_paged.  k/v_pages [num_pages, page_size,
    H_KV, d] bf16; block_table int32 [B, max_pages_per_seq]; page_size a multiple of 64."""
    _check_cuda(q, k_pages, v_pages, block_table, cache_seqlens)
    if block_table.dtype != torch.int32 or block_table.dim() != 2 or block_table.stride(1) != 1:
        raise ValueError("block_table must be a row-major int32 [B, max_pages] tensor")
    _check_shapes(plan, q, k_pages, v_pages, cache_seqlens, out, lse, paged=True)
    if block_table.shape[0] != plan.batch:
        raise ValueError(f"block_table rows {block_table.shape[0]} != batch {plan.batch}")
    B, HQ, D = q.shape
    if out is None:
        out = torch.empty((B, HQ, D), dtype=out_dtype, device=q.device)
    if lse is None:
        lse = torch.empty((B, HQ), dtype=torch.float32, device=q.device)
    if workspace is None:
        workspace = workspace_for(plan, q.device)
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    dt = L.DA_F32 if out.dtype == torch.float32 else L.DA_BF16
    L.da_forward_paged(plan, q, k_pages, v_pages, k_pages.shape[0], k_pages.shape[1], block_table,
                       block_table.stride(0), block_table.shape[1], cache_seqlens,
                       _kv_strides(q, k_pages, v_pages), softmax_scale, dt, out, lse, workspace, ws_bytes,
                       stream)
    return out, lse


class HostStaging:
    """Device scratch for ``forward_host`` (da_forward_host_bytes of the plan), reused across
    steps; grows when a larger plan needs more."""

    def __init__(self, device=None):
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.buf = None

    def get(self, nbytes: int) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        return self.buf


def forward_host(plan: L.da_plan, q, k_cache, v_cache, cache_seqlens=None, *, out=None, lse=None,
                 staging: HostStaging | None = None, softmax_scale=0.0, out_dtype=torch.bfloat16,
                 stream=None):
    """Decode attention on HOST tensors via da_forward_host: the H2D copies, the forward and the
    D2H copies of out / lse are enqueued on ``stream``; out / lse are valid after it synchronises.
    Pass pinned (page-locked) tensors for asynchronous copies."""
    for t in (q, k_cache, v_cache, cache_seqlens, out, lse):
        if t is not None and (t.is_cuda or not t.is_contiguous()):
            raise ValueError("forward_host takes contiguous host tensors")
    if q.dtype != torch.bfloat16 or k_cache.dtype != torch.bfloat16 or v_cache.dtype != torch.bfloat16:
        raise ValueError("q, k_cache, v_cache must be bfloat16")
    if cache_seqlens is not None and cache_seqlens.dtype != torch.int32:
        raise ValueError("cache_seqlens must be int32")
    _check_shapes(plan, q, k_cache, v_cache, cache_seqlens, out, lse)
    B, HQ, D = q.shape
    if out is None:
        out = torch.empty((B, HQ, D), dtype=out_dtype).pin_memory()
    if lse is None:
        lse = torch.empty((B, HQ), dtype=torch.float32).pin_memory()
    dt = L.DA_F32 if out.dtype == torch.float32 else L.DA_BF16
    l_cap = k_cache.shape[1]
    nbytes = L.da_forward_host_bytes(plan, l_cap, cache_seqlens is not None, dt)
    buf = (staging or HostStaging()).get(nbytes)
    L.da_forward_host(plan, q, k_cache, v_cache, l_cap, cache_seqlens, softmax_scale, dt, out, lse, buf,
                      buf.numel(), stream)
    return out, lse


def combine(o_partial, lse_partial, *, out=None, lse=None, out_dtype=torch.bfloat16, stream=None):
    """da_combine over o_partial [s, B, H_Q, d] fp32 and lse_partial [s, B, H_Q] fp32
    (split strides taken from the tensors)."""
    _check_cuda(o_partial, lse_partial)
    s, B, HQ, D = o_partial.shape
    if out is None:
        out = torch.empty((B, HQ, D), dtype=out_dtype, device=o_partial.device)
    if lse is None:
        lse = torch.empty((B, HQ), dtype=torch.float32, device=o_partial.device)
    dt = L.DA_F32 if out.dtype == torch.float32 else L.DA_BF16
    L.da_combine(s, B, HQ, D, o_partial, o_partial.stride(0), lse_partial, lse_partial.stride(0), dt,
                 out, lse, stream)
    return out, lse


def decode_attention(q, k_cache, v_cache, cache_seqlens=None, *, policy="seq_aware", pack_gqa=True,
                     sm_margin=0, forced_splits=0, l_k=None, softmax_scale=0.0,
                     out_dtype=torch.bfloat16):
    """One-call decode attention: plan (cached per shape) + forward."""
    B, HQ, D = q.shape
    HKV = k_cache.shape[2]
    lk = int(l_k) if l_k is not None else k_cache.shape[1]
    plan = make_plan(B, HQ, HKV, lk, D, pack_gqa, sm_margin, None, policy, forced_splits)
    return forward(plan, q, k_cache, v_cache, cache_seqlens, softmax_scale=softmax_scale,
                   out_dtype=out_dtype)
