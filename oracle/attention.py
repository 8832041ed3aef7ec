"""fp64 decode-attention oracle: C-att, C-part, C-comb of SURVEY.md §8(c).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain NumPy, float64,
no blocking, fusion or reordering beyond the definitions below.

What the paper fixes
--------------------
* The operation is decode-step attention, "a memory-bound reduction over the
  sequence dimension" with L_Q = 1 (§2.1) over the keys/values of
  prior tokens (§1), for MQA / GQA (H_Q a multiple of H_KV, P:L10,
  P:L37 "Llama 70B uses an 8:1 Key-Value ratio").
* Splitting the sequence (num_splits, "sequence-level parallelization",
  P:L36, §3.1) must not change the result: the search froze "variables
  defining model semantics" so only scheduling changes (§3.1).  The
  split partials are merged by the log-sum-exp identity implemented in
  ``lse_combine`` (the "final reductions" of P:L38 / "combination" of
  P:L179).

Readings where the paper is silent: softmax scale 1/sqrt(d)
(C-amb-9); lse in natural log, fp32, [B, H_Q] (C-amb-10); GQA head mapping
g = floor(h / G) (C-amb-11); empty sequence -> out = 0, lse = -inf
(C-amb-12).

Array conventions (all float64 NumPy; the caller upcasts the bf16 inputs,
which is exact):
  q        [B, H_Q, d]
  k, v     [B, L_cap, H_KV, d]          (token-major "BSHD" cache layout)
  seqlens  [B] integers, 0 <= n_b <= L_cap
  out      [B, H_Q, d]
  lse      [B, H_Q]
"""

from __future__ import annotations

import math

import numpy as np


def default_scale(head_dim: int) -> float:
    """C-amb-9: the softmax scale is unstated by the paper; FA's default."""
    return 1.0 / math.sqrt(head_dim)


def _check(q, k, v, seqlens):
    B, HQ, d = q.shape
    Bk, L_cap, HKV, dk = k.shape
    if k.shape != v.shape or Bk != B or dk != d:
        raise ValueError("shape mismatch between q, k, v")
    if HQ % HKV != 0:  # S:L32 "h_q is a positive multiple of h_kv"
        raise ValueError("h_q must be a multiple of h_kv")
    seqlens = np.asarray(seqlens, dtype=np.int64)
    if seqlens.shape != (B,) or (seqlens < 0).any() or (seqlens > L_cap).any():
        raise ValueError("seqlens must be [B] with 0 <= n_b <= L_cap")
    return B, HQ, HKV, d, seqlens


def decode_attention(q, k, v, seqlens, scale=None):
    """C-att.  For each b and query head h, with g = floor(h / G) and
    n = seqlens[b]:

        s_j   = scale * sum_c q[b,h,c] * k[b,j,g,c]          j < n
        m     = max_j s_j,   l = sum_j exp(s_j - m)
        out   = sum_j exp(s_j - m) * v[b,j,g,:] / l
        lse   = m + ln l

    The G query heads sharing KV head g are evaluated together as one
    [G, d] x [d, n] product (a matmul used as a step; the definition per row
    is unchanged).  n = 0 gives out = 0, lse = -inf (C-amb-12).
    """
    B, HQ, HKV, d, seqlens = _check(q, k, v, seqlens)
    G = HQ // HKV
    if scale is None or scale <= 0:
        scale = default_scale(d)
    out = np.zeros((B, HQ, d), dtype=np.float64)
    lse = np.full((B, HQ), -np.inf, dtype=np.float64)
    for b in range(B):
        n = int(seqlens[b])
        if n == 0:
            continue
        for g in range(HKV):
            rows = slice(g * G, (g + 1) * G)
            kk = k[b, :n, g, :]                      # [n, d]
            vv = v[b, :n, g, :]                      # [n, d]
            s = scale * (q[b, rows, :] @ kk.T)       # [G, n]
            m = s.max(axis=1, keepdims=True)         # [G, 1]
            e = np.exp(s - m)                        # [G, n]
            l = e.sum(axis=1, keepdims=True)         # [G, 1]
            out[b, rows, :] = (e @ vv) / l
            lse[b, rows] = (m + np.log(l))[:, 0]
    return out, lse


def split_partials(q, k, v, seqlens, ranges, scale=None):
    """C-part.  ``ranges[b]`` is the list of s token ranges (t0, t1) of batch
    b (same s for every b).  Split i is C-att restricted to tokens
    [t0, t1): o_i normalised by its own l_i, lse_i = m_i + ln l_i; an empty
    range gives o_i = 0, lse_i = -inf.

    Returns o [s, B, H_Q, d], lse [s, B, H_Q].
    """
    B, HQ, HKV, d, seqlens = _check(q, k, v, seqlens)
    s_count = len(ranges[0])
    if any(len(r) != s_count for r in ranges) or len(ranges) != B:
        raise ValueError("ranges must list the same number of splits per batch")
    o = np.zeros((s_count, B, HQ, d), dtype=np.float64)
    lse = np.full((s_count, B, HQ), -np.inf, dtype=np.float64)
    for b in range(B):
        for i, (t0, t1) in enumerate(ranges[b]):
            t0, t1 = int(t0), int(t1)
            if not (0 <= t0 <= t1 <= int(seqlens[b])):
                raise ValueError("split range outside [0, seqlens[b]]")
            if t1 == t0:
                continue
            # C-att on the sub-sequence [t0, t1) of batch b.
            ob, lb = decode_attention(q[b:b + 1], k[b:b + 1, t0:t1], v[b:b + 1, t0:t1],
                                      [t1 - t0], scale)
            o[i, b] = ob[0]
            lse[i, b] = lb[0]
    return o, lse


def lse_combine(o_parts, lse_parts):
    """C-comb.  Given s partials o_i [..., d] and lse_i [...]:

        M   = max_i lse_i                  (M := 0 if every lse_i = -inf)
        lse = M + ln sum_i exp(lse_i - M)
        out = sum_i exp(lse_i - lse) * o_i
        all splits empty -> out = 0, lse = -inf.

    This is the identity that makes "s > 1 combined afterward"
    equal the unsplit result; the paper counts its cost as the split
    overhead.
    """
    o_parts = np.asarray(o_parts, dtype=np.float64)
    lse_parts = np.asarray(lse_parts, dtype=np.float64)
    M = lse_parts.max(axis=0)
    all_empty = np.isneginf(M)
    M = np.where(all_empty, 0.0, M)
    w = np.exp(lse_parts - M[None])                    # exp(-inf) = 0 for empty splits
    total = w.sum(axis=0)
    with np.errstate(divide="ignore"):
        lse = M + np.log(total)                        # -inf when all empty
    scale = np.where(all_empty[None], 0.0, w / np.where(total == 0, 1.0, total)[None])
    out = (scale[..., None] * o_parts).sum(axis=0)
    return out, lse


def partition(n_b: int, num_splits: int, split_unit: int):
    """C-pol item 6: the token ranges of batch b's s splits.

    n_u = ceil(n_b / split_unit) units; split i covers units
    [floor(i n_u / s), floor((i+1) n_u / s)), clipped to n_b.  Balanced;
    empty only when s > n_u (C-amb-6).  Outputs do not depend on the
    partition (the LSE identity); the kernel must nevertheless use exactly
    this one so that per-split partials can be compared.
    """
    if num_splits < 1 or split_unit < 1 or n_b < 0:
        raise ValueError("bad partition arguments")
    n_u = -(-n_b // split_unit)
    out = []
    for i in range(num_splits):
        u0 = (i * n_u) // num_splits
        u1 = ((i + 1) * n_u) // num_splits
        out.append((min(u0 * split_unit, n_b), min(u1 * split_unit, n_b)))
    return out


def gather_pages(pages, block_table, seqlens, page_size):
    """Paged KV cache -> dense [B, L, H_KV, d] cache (vLLM-style block tables).

    pages [num_pages, page_size, H_KV, d]; block_table[b][j] = page holding tokens
    [j page_size, (j+1) page_size) of sequence b.  Dense L = max_b ceil(n_b / page_size)
    page_size; token t of sequence b is pages[block_table[b][t // page_size], t % page_size].
    Tokens past n_b are filled with zeros (never read by decode_attention)."""
    pages = np.asarray(pages)
    seqlens = np.asarray(seqlens, dtype=np.int64)
    B = len(seqlens)
    n_pages = int(max((-(-int(n) // page_size) for n in seqlens), default=0))
    L = max(n_pages * page_size, 1)
    out = np.zeros((B, L) + pages.shape[2:], dtype=pages.dtype)
    for b in range(B):
        for t in range(int(seqlens[b])):
            out[b, t] = pages[int(block_table[b][t // page_size]), t % page_size]
    return out


def decode_attention_paged(q, k_pages, v_pages, block_table, seqlens, page_size, scale=None):
    """C-att over a paged cache: gather the pages in sequence order, then decode_attention."""
    k = gather_pages(k_pages, block_table, seqlens, page_size)
    v = gather_pages(v_pages, block_table, seqlens, page_size)
    return decode_attention(q, k, v, seqlens, scale)


def bf16_round(x):
    """Round float64 values to the nearest bfloat16 (ties to even) and return
    them as float64.  C-amb-13: the kernel rounds its fp32 result to bf16 once
    at the end; tests use this to state the bf16 representation error of the
    exact answer."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    r = r.astype(np.uint32)
    nan = np.isnan(f)
    r = np.where(nan, np.uint32(0x7FC00000), r)
    return r.view(np.float32).astype(np.float64)
