"""Seeded synthetic inputs shared by the tests, bench.py and smoke().

This module holds NONE of the method's arithmetic: it only draws the bf16
query / KV-cache tensors and the per-batch cache lengths that both the CUDA
path and the CPU oracle then consume.  The recipe:

* q, k, v  i.i.d. N(0, 1) drawn in fp32 by a seeded ``torch.Generator`` and
  rounded to bf16 (the paper gives no distributions; inputs were frozen,
  P:L40).  ``peaked`` multiplies q by 8 before rounding (a sharp softmax that
  exercises the running-max rescale).
* cache_seqlens = L_K for every batch (the paper's fixed shapes),
  or, for ``ragged``, U[0, L_K] with batch 0 forced to 0 and batch 1 to 1
  when B allows (empty sequences and single keys).
* KV layout [B, L_cap, H_KV, d] contiguous, L_cap = L_K unless given.
* seed = 1000 + config index by convention.
"""

from __future__ import annotations

import torch


def make_inputs(batch: int, h_q: int, h_kv: int, l_k: int, head_dim: int = 128, *,
                l_cap: int | None = None, seed: int = 1000, variant: str = "normal",
                device: str | torch.device = "cpu") -> dict:
    """Return dict(q, k, v, seqlens, l_k, l_cap) of tensors on ``device``.

    q [B, H_Q, d] bf16, k/v [B, L_cap, H_KV, d] bf16, seqlens [B] int32.
    Values are drawn on ``device`` (CPU and CUDA generators give different
    streams; timing does not depend on values, parity tests use one device's
    draw for both sides).
    """
    if l_cap is None:
        l_cap = l_k
    if l_cap < l_k:
        raise ValueError("l_cap must be >= l_k")
    device = torch.device(device)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    qscale = 8.0 if variant == "peaked" else 1.0
    q = (torch.randn((batch, h_q, head_dim), generator=gen, device=device,
                     dtype=torch.float32) * qscale).to(torch.bfloat16)
    k = torch.randn((batch, l_cap, h_kv, head_dim), generator=gen, device=device,
                    dtype=torch.float32).to(torch.bfloat16)
    v = torch.randn((batch, l_cap, h_kv, head_dim), generator=gen, device=device,
                    dtype=torch.float32).to(torch.bfloat16)
    if variant == "ragged":
        seqlens = torch.randint(0, l_k + 1, (batch,), generator=gen, device=device,
                                dtype=torch.int32)
        if batch >= 1:
            seqlens[0] = 0
        if batch >= 2:
            seqlens[1] = 1
    elif variant in ("normal", "peaked"):
        seqlens = torch.full((batch,), l_k, dtype=torch.int32, device=device)
    else:
        raise ValueError(f"unknown variant {variant!r}")
    return {"q": q, "k": k, "v": v, "seqlens": seqlens, "l_k": l_k, "l_cap": l_cap}


def to_f64(t: torch.Tensor):
    """bf16/int tensor -> NumPy (float64 for floating types; exact for bf16)."""
    t = t.detach().cpu()
    if t.is_floating_point():
        return t.to(torch.float64).numpy()
    return t.numpy()


# The BASELINE.json configurations, index = seed offset.
CONFIGS = {
    "mqa_tiny": dict(batch=1, h_q=8, h_kv=1, l_k=128),
    "llama70b": dict(batch=1, h_q=64, h_kv=8, l_k=512),
    "llama70b_tp8": dict(batch=1, h_q=8, h_kv=1, l_k=512),
    "high_load": dict(batch=128, h_q=64, h_kv=8, l_k=8192),
    "long_context": dict(batch=1, h_q=64, h_kv=8, l_k=131072),
}


def low_head_sweep():
    """configs[2]: B in {1,2,4,8} x H_KV in {1,2,8} x L_K in {64,128,256,512},
    H_Q = 8 H_KV (48 shapes)."""
    out = []
    for b in (1, 2, 4, 8):
        for hkv in (1, 2, 8):
            for lk in (64, 128, 256, 512):
                out.append(dict(batch=b, h_q=8 * hkv, h_kv=hkv, l_k=lk))
    return out
