"""Split-count policies (C-pol of SURVEY.md §8(c)) in pure Python integers.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Steps follow the paper's order and notation:

* Geometry (§4, Fig. 3 comment):
  nblk = num_n_blocks = ceil(L_K / 128)    (128-token accounting, C-amb-1:
         "L_K <= 512" <=> "nblk <= 4"; "L_K <= 384" <=> "nblk <= 3")
  num_m_blocks = ceil(L_Q * G / 64)        (L_Q = 1; = 1 for every G <= 64)
  total_mblocks T = Batch * H_KV * num_m_blocks   ("reduces to
         batch_size * num_heads_kv")
  usable SMs U = num_SMs - sm_margin       (C-amb-8)
* Guarded (the FA3 default the paper patches, §2.2, §4.2):
  saturation guard, then "returns s = 1 if ... L_K <= 512" (nblk <= 4),
  else the efficiency loop.
* Sequence-aware (Fig. 3), in this order:
  Guard 1  nblk <= 3                  -> 1
  Guard 2  nblk <= 4 and T >= 4       -> 1
  Low-tile nblk == 4 and T < 4        -> 3  ("s=3 on the current stack")
  else     "existing efficiency loop runs (unchanged)"
* The efficiency loop is referenced but never
  defined by the paper; ``efficiency_loop`` is the reconstruction stated in
  DESIGN.md §3 (C-amb-2..4).  Its single-wave closed form is pinned by tests;
  beyond that it is "parity unpinned" by the paper.

All comparisons are exact integer cross-multiplications (C-amb-3): there is
no floating point anywhere in this module.

Policies beyond the paper's pair: the evolved
Python fragment of Fig. 1 as a planner mode, and the SM-count-aware
generalisation (C-ext-1) whose constants are calibrated on B200 - "parity
unpinned" by the paper for the latter's constants (its structural properties
are pinned in tests/test_oracle_policy.py) - and per-batch dynamic split counts
for ragged batches (C-ext-2, ``dynamic_schedule``; parity unpinned by the paper,
which names only the metadata role; invariants pinned).
"""

from __future__ import annotations

BLOCK_N = 128            # tokens per policy block (C-amb-1)
BLOCK_M = 64             # query rows per m-block for the tile count
LOW_TILE_SPLITS = 3      # Fig. 3 "return 3", C-amb-5
EFF_MAX_SPLITS = 128     # efficiency-loop candidate cap (C-amb-2)
MAX_FORCED_SPLITS = 256  # S:L98 max_splits default
SPLIT_UNIT = 64          # partition unit in tokens (C-pol item 6)

GUARDED, SEQ_AWARE, FIXED, EVOLVED, SEQ_AWARE_SM, DYNAMIC = 0, 1, 2, 3, 4, 5
POLICY_NAMES = {"guarded": GUARDED, "seq_aware": SEQ_AWARE, "fixed": FIXED, "evolved": EVOLVED,
                "seq_aware_sm": SEQ_AWARE_SM, "dynamic": DYNAMIC}

# Which step of the cascade decided s (mirrors SPEC's SplitDecision.source).
RULE_SATURATED = 0
RULE_GUARD_NBLK4 = 1
RULE_GUARD1 = 2
RULE_GUARD2 = 3
RULE_LOW_TILE = 4
RULE_EFF_LOOP = 5
RULE_FORCED = 6
RULE_EVOLVED = 7      # Fig. 1 fragment
RULE_SM_SHORT = 8     # SM-count-aware generalisation: too few 64-token units to split
RULE_SM_SPLIT = 9     # SM-count-aware generalisation: split count from units, tiles and SMs
RULE_SM_FIT = 10      # SM-count-aware generalisation: efficiency-loop split moved to one wave
RULE_DYNAMIC = 11     # per-batch split counts from the lengths on the device (dynamic_schedule)

# SM-count-aware generalisation of the sequence-aware rule (DESIGN.md §3,
# C-ext-1).  The paper leaves "extending the benefit to lower L_K values and learning more
# configuration-specific split counts" to future work and calls its
# own constant stack-specific ("s=3 on the current stack").  These constants are
# calibrated from the B200 U-curves of the current kernel (profiles/r01h_ugrid.csv,
# r01h_ugrid2.csv, r01h_ugrid3.csv, measured with the pre-wait L2 prefetch of short splits, and
# the 48-shape low-head sweep of BASELINE configs[2], profiles/r01i_lowhead.csv;
# long-context boundary from scripts/probe_regime.py and probe_long.py; s = 11 vs 12 from
# scripts/probe_s11.py) and frozen:
SM_UNIT = 64          # tokens per split unit of the B200 kernel
SM_MIN_UNITS = 5      # fewer units (L_K <= 256): every split loses or ties on B200
SM_MIN_SPLITS = 3     # guard region: a 2-way split (only 2-CTA clusters fit, T = 46..74) loses
SM_MIN_UNITS_WIDE = 8  # with T > SM_WIDE_T tiles, fewer units (L_K <= 448) do not pay either
SM_WIDE_T = 16
SM_NARROW_T = 4       # T <= 4 tiles: the plateau extends to s = 8 ...
SM_NARROW_SPLITS = 8
SM_MAX_SPLITS = 4     # ... otherwise the measured plateau starts at s = 4
SM_STREAM_UNITS = 16  # efficiency region: cap to the one-wave cluster split while each split
                      # holds <= 16 units (1024 tokens) or the capped launch still has >= U/2 CTAs
SM_MID_T = 8          # efficiency region, <= 64 units (latency regime): at most 4 splits for T > 8,
SM_MID_UNITS = 64
SM_CLUSTER_CAP = 12   # at most 12 otherwise (clusters of 13..16 measured slower than 12)
# wide query groups (round 2, profiles/r02zz4_wide_group_policy.log, 48 MQA shapes G = 32 / 64, and
# r02zz33_g17_31_policy.log, G = 20 / 24 / 28 at L_K = 4096, where the same B16 loss appears):
# where the one-wave cluster fit leaves only a 2-CTA cluster split, the efficiency loop's split
# runs on the tcgen05 kernel (64 query rows per CTA, workspace combine) and is faster, provided
# each of its splits holds >= SM_TC_MIN_TILES 64-token tiles, its 64-row grid has >= U / 2 CTAs and
# the sequence has >= SM_TC_UNITS units (B8 G64 L4096: 13.7 -> 9.9 us; B16 G32 L4096: 13.9 ->
# 11.5 us; at 32 units, B16 G32 L2048, the 2-split mma.sync plan stays ahead)
SM_TC_MIN_G = 17      # the tcgen05 kernel's group sizes (config.h kTcMinG: G > 16)
SM_TC_MIN_TILES = 4   # tiles per split it needs (config.h kTcMinTiles)
SM_TC_ROWS = 64       # its query rows per CTA (config.h kTcRows)
SM_TC_MAX_FIT = 2     # the cluster split it replaces: a 2-CTA cluster at most
SM_TC_UNITS = 64
# Clusters of s CTAs (one per split, s = 1..16) that are co-resident in one wave on a 148-SM
# B200 with the cluster-combine kernel configuration: a HARDWARE MEASUREMENT, not a paper value -
# the CUDA occupancy API's answer for the exact cluster kernels, recorded by
# scripts/measure_residency.py in profiles/cluster_fit_b200.json (the one source: this module loads
# it, tests/test_abi_cpu.py checks the planner's copy in config.h against it, and
# tests/test_gpu_residency.py checks both against the live device).  Index 0 unused, index 1 = one
# CTA per SM.  Scaled by U / 148.
def _load_cluster_fit():
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "cluster_fit_b200.json")
    with open(path) as f:
        rec = json.load(f)
    if rec["sms"] != 148 or len(rec["max_active_clusters"]) != 17:
        raise ValueError("profiles/cluster_fit_b200.json is not a 148-SM B200 record")
    return tuple(int(x) for x in rec["max_active_clusters"])


CLUSTER_FIT_B200 = _load_cluster_fit()
CLUSTER_MAX_SPLITS = 16
# Per-batch dynamic split counts (the scheduler-metadata role of P:L125):
DYN_MAX_SPLITS = 128  # per-sequence cap (the efficiency loop's candidate cap, C-amb-2)
VARLEN_MIN_UNITS = 32  # C-ext-3: the dynamic path pays off only for splits of >= 2048 tokens

def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def geometry(batch: int, h_q: int, h_kv: int, l_k: int, num_sms: int, sm_margin: int,
             l_q: int = 1) -> dict:
    """Tile geometry."""
    for name, val in (("batch", batch), ("h_q", h_q), ("h_kv", h_kv), ("l_k", l_k),
                      ("num_sms", num_sms), ("l_q", l_q)):
        if int(val) != val or val < 1:
            raise ValueError(f"{name} must be a positive integer")
    if h_q % h_kv:
        raise ValueError("h_q must be a multiple of h_kv (S:L32)")
    if sm_margin < 0 or sm_margin >= num_sms:
        raise ValueError("0 <= sm_margin < num_sms (S:L39)")
    G = h_q // h_kv
    nblk = ceil_div(l_k, BLOCK_N)
    num_m_blocks = ceil_div(l_q * G, BLOCK_M)
    T = batch * h_kv * num_m_blocks
    U = num_sms - sm_margin
    return {"G": G, "nblk": nblk, "num_m_blocks": num_m_blocks, "T": T, "U": U}


def occupancy_fraction(active_ctas: int, usable_sms: int):
    """S:L61-69 / P:L20: occupancy = min(CTAs, U) / U as an exact
    (numerator, denominator) pair; 8 CTAs on 132 SMs ~ 6 %."""
    if active_ctas < 1 or usable_sms < 1:
        raise ValueError("active_ctas and usable_sms must be >= 1")
    return (min(active_ctas, usable_sms), usable_sms)


def saturated(T: int, U: int) -> bool:
    """FA3 first guard (C-amb-4): total_mblocks >= 0.8 * SMs, as 5T >= 4U."""
    return 5 * T >= 4 * U


def efficiency_loop(T: int, U: int, nblk: int) -> int:
    """C-amb-2 reconstruction of the loop the paper leaves unchanged.

    Candidates s = 1 .. smax with smax = min(128, U, nblk).  Waves
    w_s = ceil(T s / U); efficiency(s) = (T s) / (U w_s).  Return the smallest
    s with efficiency(s) >= 0.85 * max_s efficiency(s), i.e. with s* any
    maximiser of s / w_s:   20 s w_{s*} >= 17 s* w_s   (T and U cancel).
    """
    smax = min(EFF_MAX_SPLITS, U, nblk)
    waves = [ceil_div(T * s, U) for s in range(1, smax + 1)]
    best_s, best_w = 1, waves[0]
    for s in range(2, smax + 1):
        w = waves[s - 1]
        if s * best_w > best_s * w:          # s / w > best_s / best_w
            best_s, best_w = s, w
    for s in range(1, smax + 1):
        if 20 * s * best_w >= 17 * best_s * waves[s - 1]:
            return s
    return 1  # unreachable: s = best_s satisfies the test


def guarded_splits(geo: dict):
    """FA3-style default: saturation guard, then the static L_K <= 512 guard
    ("returns s=1 if the sequence length L_K <= 512"; "strictly
    enforced s=1 when num_n_blocks <= 4"), else the efficiency loop."""
    T, U, nblk = geo["T"], geo["U"], geo["nblk"]
    if saturated(T, U):
        return 1, RULE_SATURATED
    if nblk <= 4:
        return 1, RULE_GUARD_NBLK4
    return efficiency_loop(T, U, nblk), RULE_EFF_LOOP


def seq_aware_splits(geo: dict):
    """The paper's policy, Fig. 3, after the unchanged
    saturation guard (C-c item 4.1)."""
    T, U, nblk = geo["T"], geo["U"], geo["nblk"]
    if saturated(T, U):
        return 1, RULE_SATURATED
    if nblk <= 3:                                   # P:L96  Guard 1
        return 1, RULE_GUARD1
    if nblk <= 4 and T >= 4:                        # P:L101 Guard 2
        return 1, RULE_GUARD2
    if nblk == 4 and T < 4:                         # P:L104 low-tile override
        return LOW_TILE_SPLITS, RULE_LOW_TILE
    return efficiency_loop(T, U, nblk), RULE_EFF_LOOP


def rows_per_cta(G: int, l_k: int) -> int:
    """BUILDER SPECIFICATION (C-ext-1's launch geometry), not a reading of the paper: the paper has
    no B200 kernel.  Pinned by its hand-checked cases in tests/test_oracle_policy.py.
    Query rows one CTA of the tensor-core path computes: 8, or 16 for G > 8 on
    long sequences (> 64 units).  Short sequences with G > 8 run two 8-row CTAs per 16 rows: the
    16-row kernel is twice the MMA work per warp and past the instruction cache, which costs
    the latency regime 25-40 % (scripts/probe_g16b.py), while on streaming lengths the 8-row split
    would read every KV tile twice."""
    return 8 if G <= 8 or ceil_div(l_k, SM_UNIT) <= SM_MID_UNITS else 16


def launch_rows(batch: int, G: int, h_kv: int, l_k: int, s: int, U: int) -> int:
    """BUILDER SPECIFICATION (launch geometry of the B200 kernel), not a reading of the paper.
    Rows per CTA the plan launches with s splits: rows_per_cta(G, L_K), except
    that 8-row CTAs for G > 8 need their whole grid, Batch x H_KV x ceil(G / 8) x s CTAs, in one
    wave of U SMs -- past it, the doubled CTA count costs a second wave and 16-row CTAs stand."""
    rows = rows_per_cta(G, l_k)
    if rows == 8 and G > 8 and batch * h_kv * ceil_div(G, 8) * s > U:
        rows = 16
    return rows


def cluster_fit_splits(T: int, U: int) -> int:
    """BUILDER SPECIFICATION (C-ext-1), not a reading of the paper; the table is a hardware
    measurement (CLUSTER_FIT_B200, loaded from profiles/cluster_fit_b200.json).
    Largest s in 1..16 whose T clusters of s CTAs are co-resident in one wave:
    T <= floor(CLUSTER_FIT_B200[s] * U / 148); s = 1 (one CTA per tile) always qualifies."""
    best = 1
    for s in range(2, CLUSTER_MAX_SPLITS + 1):
        if T <= CLUSTER_FIT_B200[s] * U // 148:
            best = s
    return best


def seq_aware_sm_splits(geo: dict, l_k: int):
    """BUILDER SPECIFICATION (C-ext-1, the SM-count-aware generalisation the paper leaves to future
    work), not a reading of the paper: its constants are B200 calibrations.
    Pinned by structure (tests/test_oracle_policy.py::test_seq_aware_sm_structure) and against the
    measurements it was calibrated on; the paper pins only that it splits where Fig. 3 splits.
    C-ext-1, in this order (n_u = ceil(L_K / 64) units; T_k = Batch x H_KV x ceil(G / rows),
    rows = rows_per_cta(G, L_K), the CTA groups the kernel launches per split (= T for G <= 8);
    f = cluster_fit_splits(T_k, U); c = 8 if T_k <= 4 else 4):
      saturated (5T >= 4U)                      -> 1                      (unchanged FA3 guard)
      nblk <= 4 (the paper's guard region):
        n_u < 5, or n_u < 8 with T_k > 16       -> 1                      (short: splitting loses)
        s = min(n_u, c, f);  s < 3 -> 1
      nblk >= 5 (efficiency region), e = the unchanged efficiency loop:
        e <= f                                  -> s = max(e, min(c, n_u, f))
        e > f >= 2, 8-row CTAs and (n_u <= 16 f or 2 T_k f >= U) -> s = f
        else                                    -> e (streaming: returned as is)
        then, for short sequences (n_u <= 64): s = min(s, 4) if T_k > 8, and s = min(s, 12)
        wide groups (round 2): G > 16, s <= 2, n_u >= 64, n_u >= 4 e and
          2 Batch H_KV ceil(G / 64) e >= U              -> e       (the tcgen05 kernel's split)
    The split count depends on the CTA groups T_k versus the usable SMs U through f, the largest
    split whose clusters all fit one wave, not on a static L_K guard.  The wide-group clause is a
    launch-geometry statement about the packed layout (pack_gqa = 1, the default), like rows."""
    T, U, nblk = geo["T"], geo["U"], geo["nblk"]
    if saturated(T, U):
        return 1, RULE_SATURATED
    n_u = ceil_div(l_k, SM_UNIT)
    rows = rows_per_cta(geo["G"], l_k)
    Tk = T // geo["num_m_blocks"] * ceil_div(geo["G"], rows)
    f = cluster_fit_splits(Tk, U)
    c = SM_NARROW_SPLITS if Tk <= SM_NARROW_T else SM_MAX_SPLITS
    if nblk <= 4:
        if n_u < SM_MIN_UNITS or (n_u < SM_MIN_UNITS_WIDE and Tk > SM_WIDE_T):
            return 1, RULE_SM_SHORT
        s = min(n_u, c, f)
        if s < SM_MIN_SPLITS:
            return 1, RULE_SM_SHORT
        return s, RULE_SM_SPLIT
    e = efficiency_loop(T, U, nblk)
    if e <= f:
        s = max(e, min(c, n_u, f))
    elif f >= 2 and rows == 8 and (n_u <= SM_STREAM_UNITS * f or 2 * Tk * f >= U):
        s = f
    else:
        return e, RULE_EFF_LOOP
    if n_u <= SM_MID_UNITS:
        s = min(s, SM_MAX_SPLITS if Tk > SM_MID_T else SM_CLUSTER_CAP)
    G = geo["G"]
    if (G >= SM_TC_MIN_G and s <= SM_TC_MAX_FIT and n_u >= SM_TC_UNITS and n_u >= SM_TC_MIN_TILES * e
            and 2 * (T // geo["num_m_blocks"]) * ceil_div(G, SM_TC_ROWS) * e >= U):
        return e, RULE_EFF_LOOP
    return s, (RULE_EFF_LOOP if s == e else RULE_SM_FIT)


def dynamic_cap(l_k: int) -> int:
    """BUILDER SPECIFICATION (C-ext-2), not a reading of the paper.
    DA_POLICY_DYNAMIC's per-sequence split cap: no more splits than 64-token units of the
    longest sequence, and at most DYN_MAX_SPLITS."""
    return max(1, min(DYN_MAX_SPLITS, ceil_div(l_k, SPLIT_UNIT)))


def dynamic_slots(batch: int, tiles_per_batch: int, U: int, s_cap: int) -> int:
    """BUILDER SPECIFICATION (C-ext-2), not a reading of the paper.
    Slots (split CTAs per head group) a dynamic launch provides: enough for any lengths,
    because s_b <= n_u_b / W, or s_b = 1 where that rounds to 0, so sum_b s_b <=
    sum_b n_u_b / W + batch <= U / tiles_per_batch + batch."""
    return min(batch * s_cap, ceil_div(U, tiles_per_batch) + batch)


def dynamic_schedule(seqlens, tiles_per_batch: int, U: int, s_cap: int):
    """BUILDER SPECIFICATION (C-ext-2: the paper names the scheduler-metadata role, not a
    rule), not a reading of the paper; invariants and hand-computed cases pinned.
    Per-batch split counts for one ragged batch, in this order:
      n_u_b = ceil(n_b / 64)                      (units of each sequence, n_b already clamped)
      W     = max(1, ceil(sum_b n_u_b * tiles_per_batch / U))   (units per CTA for one wave)
      s_b   = min(s_cap, max(1, floor(n_u_b / W)))
      P_b   = s_0 + ... + s_{b-1}                 (first slot of sequence b)
    Sequence b then uses the standard partition (``partition``) with s_b splits.  Rounding s_b
    down keeps sum_b s_b * tiles_per_batch <= U except where a short sequence is lifted to one
    split: a single sequence never spills into a second wave (ceil would give 19 x 8 = 152 CTAs
    on 148 SMs at L_K = 131072, H_KV = 8), and a long sequence in a batch of short ones gets
    proportionally more splits.  Returns (W, s, P)."""
    n_u = [ceil_div(int(n), SPLIT_UNIT) for n in seqlens]
    W = max(1, ceil_div(sum(n_u) * tiles_per_batch, U))
    s = [min(s_cap, max(1, u // W)) for u in n_u]
    P, acc = [], 0
    for v in s:
        P.append(acc)
        acc += v
    return W, s, P


def varlen_policy(batch: int, h_q: int, h_kv: int, l_cap: int, num_sms: int, sm_margin: int, seqlens):
    """BUILDER SPECIFICATION (C-ext-3), not a reading of the paper.
    C-ext-3, the plan for a ragged batch whose lengths are known on the host (the
    scheduler-metadata path of P:L125): the static SM-count-aware plan (C-ext-1) for the cache
    capacity, unless its longest split would hold more than twice the balanced per-CTA work W
    of dynamic_schedule and at least VARLEN_MIN_UNITS units (below that the step is latency-bound
    and the workspace combine of the dynamic path costs more than the imbalance), in which case
    the per-batch dynamic counts (C-ext-2):
        s_st = seq_aware_sm(batch, h_q, h_kv, l_cap);  u_max = ceil(max_b n_b / 64)
        W    = dynamic_schedule's W;  c = ceil(u_max / s_st);  dynamic iff c > 2 W and c >= 32
    Returns the policy code (SEQ_AWARE_SM or DYNAMIC)."""
    geo = geometry(batch, h_q, h_kv, l_cap, num_sms, sm_margin)
    s_st, _ = seq_aware_sm_splits(geo, l_cap)
    lens = [min(max(int(n), 0), l_cap) for n in seqlens]
    u_max = ceil_div(max(lens), SPLIT_UNIT) if lens else 0
    W, _, _ = dynamic_schedule(lens, h_kv * geo["num_m_blocks"], geo["U"], dynamic_cap(l_cap))
    c = ceil_div(u_max, s_st)
    return DYNAMIC if (c > 2 * W and c >= VARLEN_MIN_UNITS) else SEQ_AWARE_SM


def evolved_policy_splits(geo: dict, batch: int, l_k: int):
    """Fig. 1 as a policy: batch == 1 -> s = 12, or 16 when L_K < 256 (literal,
    no clamp: s > nblk gives empty splits, as in the paper's s = 1..64 sweep).  The
    fragment does not show the batch != 1 branch; it falls back to the guarded default
    (SPEC's reading)."""
    ev = evolved_splits(batch, l_k)
    if ev is None:
        return guarded_splits(geo)
    return ev[0], RULE_EVOLVED


def num_splits(batch: int, h_q: int, h_kv: int, l_k: int, num_sms: int, sm_margin: int,
               policy, forced_splits: int = 0):
    """Decision (s, rule) for one shape under ``policy`` (name or code)."""
    if isinstance(policy, str):
        policy = POLICY_NAMES[policy]
    geo = geometry(batch, h_q, h_kv, l_k, num_sms, sm_margin)
    if policy == GUARDED:
        return guarded_splits(geo)
    if policy == SEQ_AWARE:
        return seq_aware_splits(geo)
    if policy == FIXED:
        if not (1 <= forced_splits <= MAX_FORCED_SPLITS):
            raise ValueError("forced_splits must be in [1, 256] (S:L98)")
        return forced_splits, RULE_FORCED
    if policy == EVOLVED:
        return evolved_policy_splits(geo, batch, l_k)
    if policy == SEQ_AWARE_SM:
        return seq_aware_sm_splits(geo, l_k)
    if policy == DYNAMIC:                 # the cap; the per-batch counts come from dynamic_schedule
        return dynamic_cap(l_k), RULE_DYNAMIC
    raise ValueError("unknown policy")


def evolved_splits(batch: int, l_k: int):
    """Fig. 1, the evolved Python fragment, for reference only
    (the paper treats it as evidence, not policy).  Returns
    (num_splits, pack_gqa, sm_margin) or None for the batch != 1 branch the
    fragment does not show."""
    if batch == 1:
        s = 12
        if l_k < 256:
            s = 16
        return s, True, 0
    return None
