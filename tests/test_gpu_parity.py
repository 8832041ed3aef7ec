"""GPU parity: the CUDA path (through the C ABI) vs the fp64 CPU oracle, element
by element, on seeded synthetic inputs (SURVEY §8(c) parity matrix, item 2)."""

import numpy as np
import pytest
import torch

import synth
from oracle import attention as OA
from oracle import policy as OP
from tests.helpers import assert_lse_close, assert_out_close

pytestmark = pytest.mark.gpu


def _dec():
    import paper_2604_00028_b200 as dec
    return dec


def run_and_check(batch, h_q, h_kv, l_k, *, policy="seq_aware", forced=0, pack_gqa=True,
                  variant="normal", l_cap=None, seed=1000, combine_mode=None, out_f32=False,
                  check_partials=False, nan_tail=False, path=None):
    dec = _dec()
    inp = synth.make_inputs(batch, h_q, h_kv, l_k, l_cap=l_cap, seed=seed, variant=variant,
                            device="cuda")
    q, k, v, seq = inp["q"], inp["k"], inp["v"], inp["seqlens"]
    if nan_tail:  # cache slots past each sequence hold garbage: must not leak into the result
        for b in range(batch):
            n = int(seq[b])
            k[b, n:] = float("nan")
            v[b, n:] = float("nan")
    plan = dec.make_plan(batch, h_q, h_kv, l_k, pack_gqa=pack_gqa, policy=policy,
                         forced_splits=forced, combine_mode=combine_mode, path=path)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    # the planner's split count is the oracle's, bit for bit
    s_ref, rule_ref = OP.num_splits(batch, h_q, h_kv, l_k, sms, 0, policy, forced)
    assert (plan.num_splits, plan.rule) == (s_ref, rule_ref)
    ws = dec.workspace_for(plan, q.device)
    out, lse = dec.forward(plan, q, k, v, seq, workspace=ws,
                           out_dtype=torch.float32 if out_f32 else torch.bfloat16)
    torch.cuda.synchronize()
    qn, kn, vn, sn = (synth.to_f64(t) for t in (q, k, v, seq))
    if nan_tail:
        kn = np.nan_to_num(kn, nan=0.0)
        vn = np.nan_to_num(vn, nan=0.0)
    ref_o, ref_l = OA.decode_attention(qn, kn, vn, sn)
    assert_out_close(synth.to_f64(out), ref_o)
    assert_lse_close(synth.to_f64(lse), ref_l)
    if check_partials:
        assert plan.combine_mode == dec.DA_COMBINE_KERNEL
        s = plan.num_splits
        nrow = batch * h_q * 128
        ws_o = ws[: s * nrow].view(s, batch, h_q, 128)
        ws_l = ws[s * nrow: s * nrow + s * batch * h_q].view(s, batch, h_q)
        ranges = [OA.partition(int(n), s, OP.SPLIT_UNIT) for n in sn]
        po, pl = OA.split_partials(qn, kn, vn, sn, ranges)
        assert_out_close(synth.to_f64(ws_o), po, "partial o")
        assert_lse_close(synth.to_f64(ws_l), pl, "partial lse")
    return plan, out, lse


# ---- BASELINE.json configurations -----------------------------------------
@pytest.mark.parametrize("policy", ["guarded", "seq_aware", "seq_aware_sm", "evolved"])
@pytest.mark.parametrize("name", ["mqa_tiny", "llama70b", "llama70b_tp8"])
def test_baseline_configs(name, policy):
    cfg = synth.CONFIGS[name]
    plan, _, _ = run_and_check(**cfg, policy=policy)
    if name == "llama70b_tp8":
        assert plan.num_splits == {"guarded": 1, "seq_aware": 3, "seq_aware_sm": 8, "evolved": 12}[policy]


@pytest.mark.parametrize("cfg", synth.low_head_sweep(),
                         ids=lambda c: f"B{c['batch']}_hkv{c['h_kv']}_L{c['l_k']}")
def test_low_head_sweep(cfg):
    for policy in ("guarded", "seq_aware"):
        run_and_check(**cfg, policy=policy, seed=1002)


# ---- forced split counts (the U-curve sweep shapes) ------------------
@pytest.mark.parametrize("s", [1, 2, 3, 4, 5, 8, 16, 64])
def test_forced_splits_tp8_slice(s):
    run_and_check(1, 8, 1, 512, policy="fixed", forced=s)


@pytest.mark.parametrize("s", [2, 3, 5, 16, 64])
def test_forced_splits_kernel_combine_partials(s):
    run_and_check(2, 16, 2, 700, policy="fixed", forced=s, combine_mode=2, check_partials=True,
                  variant="ragged", seed=7)


@pytest.mark.parametrize("s", [2, 3, 7, 8, 9, 12, 16])
def test_cluster_combine(s):
    run_and_check(2, 8, 1, 1000, policy="fixed", forced=s, combine_mode=1, seed=11)


# ---- tail balancing of cluster plans: splits of >= 32 tiles stream the head of their
#      range and share the pooled tails through a ticket counter in rank 0's shared memory ----------
@pytest.mark.parametrize("batch,h_q,h_kv,l_k,s,pack,variant", [
    (1, 8, 1, 16384, 8, True, "normal"),      # 32 tiles per split: the smallest balanced split
    (1, 8, 1, 16448, 8, True, "normal"),      # a ragged last tile (16448 = 257 tiles)
    (4, 16, 2, 20000, 5, True, "ragged"),     # balanced and static clusters in one launch
    (2, 16, 2, 20000, 7, True, "peaked"),
    (1, 32, 2, 40000, 9, True, "normal"),     # 16-row CTAs
    (2, 4, 2, 9000, 4, False, "ragged"),      # scalar path
    (1, 64, 8, 131072, 10, True, "normal"),   # the long-context C-ext-1 plan
])
def test_cluster_tail_balancing(batch, h_q, h_kv, l_k, s, pack, variant):
    dec = _dec()
    for _ in range(2):        # the tickets live in shared memory: nothing carries over between calls
        plan, _, _ = run_and_check(batch, h_q, h_kv, l_k, policy="fixed", forced=s, combine_mode=1,
                                   pack_gqa=pack, variant=variant, seed=31)
        assert plan.combine_mode == dec.DA_COMBINE_CLUSTER


@pytest.mark.parametrize("s", [5, 11, 15, 16])
def test_cluster_combine_16_rows(s):
    # G = 16 query rows per CTA (L_K > 64 units): the largest push-slot use (s ceil(16 / s) rows
    # per owner)
    plan, _, _ = run_and_check(1, 32, 2, 4500, policy="fixed", forced=s, combine_mode=1, seed=13,
                               variant="ragged")
    assert plan.rows_per_cta == 16


# ---- head grouping / paths ----------------------------------------------------
@pytest.mark.parametrize("h_q,h_kv", [(8, 8), (16, 2), (8, 2), (24, 2), (64, 2), (32, 1), (64, 1),
                                      (32, 32), (12, 1)])
def test_group_sizes_mma_path(h_q, h_kv):
    run_and_check(2, h_q, h_kv, 300, seed=21)


@pytest.mark.parametrize("h_q,h_kv", [(32, 2), (24, 2), (16, 1), (12, 1)])
def test_group_sizes_16_row_ctas(h_q, h_kv):
    # G > 8 beyond 64 units: 16 query rows per CTA, incl. ragged G = 12 / 24
    plan, _, _ = run_and_check(1, h_q, h_kv, 4500, seed=22, variant="ragged")
    assert plan.rows_per_cta == 16


@pytest.mark.parametrize("batch,h_q,h_kv,l_k,policy", [(1, 128, 1, 1000, "seq_aware"), (2, 256, 2, 700, "seq_aware_sm"),
                                                       (1, 128, 1, 3000, "dynamic"), (1, 128, 1, 4500, "seq_aware_sm"),
                                                       (2, 128, 1, 5000, "dynamic")])
def test_many_query_rows_per_kv_head(batch, h_q, h_kv, l_k, policy):
    # G = 128: two policy m-blocks (T = 2 B H_KV) and sixteen 8-row (<= 64 units, one-wave grid) or
    # eight 16-row CTAs per KV head on the MMA path
    plan, _, _ = run_and_check(batch, h_q, h_kv, l_k, policy=policy, variant="ragged", seed=1500)
    assert plan.num_m_blocks == 2
    if plan.path == 2:        # G >= 32 with >= 16 tiles per split: tcgen05, 64 rows, two CTAs per KV head
        assert policy != "dynamic" and -(-l_k // 64) >= 4 * plan.num_splits
        assert (plan.rows_per_cta, plan.grid_y) == (64, 2 * h_kv)
    else:                     # short splits and the dynamic schedule: the mma.sync kernel
        assert plan.rows_per_cta == OP.launch_rows(batch, h_q // h_kv, h_kv, l_k, plan.num_splits, plan.usable_sms)
        assert plan.rows_per_cta == 16 or l_k <= 4096


def test_large_batch_small_cache():
    plan, _, _ = run_and_check(2000, 8, 1, 64, policy="seq_aware_sm", variant="ragged", seed=1510)
    assert plan.grid_z == 2000


@pytest.mark.parametrize("h_q,h_kv", [(8, 1), (16, 2), (8, 8)])
def test_scalar_path_unpacked(h_q, h_kv):
    plan, _, _ = run_and_check(2, h_q, h_kv, 333, pack_gqa=False, seed=31)
    assert plan.path == _dec().DA_PATH_SCALAR


@pytest.mark.parametrize("pack", [True, False])
@pytest.mark.parametrize("variant", ["peaked", "ragged"])
def test_variants(variant, pack):
    run_and_check(5, 16, 2, 777, variant=variant, pack_gqa=pack, seed=41, policy="fixed", forced=4)


@pytest.mark.parametrize("pack", [True, False])
def test_lcap_larger_and_nan_tail(pack):
    run_and_check(3, 16, 2, 200, l_cap=400, variant="ragged", pack_gqa=pack, seed=51,
                  nan_tail=True, policy="fixed", forced=3)


@pytest.mark.parametrize("l_k", [2, 3, 4, 6, 8, 16, 64, 512])
@pytest.mark.parametrize("variant", ["normal", "peaked"])
def test_pv_precision_short_and_peaked(l_k, variant):
    # the cases where a single-bf16 P in the PV product misses the per-element bound
    # (scripts/emulate_p_precision.py: err/bound up to 1.4): 8 batches x 64 query rows each
    run_and_check(8, 64, 8, l_k, variant=variant, seed=1400 + l_k, policy="seq_aware_sm")


def test_out_f32():
    run_and_check(2, 16, 2, 513, out_f32=True, policy="fixed", forced=5, seed=61)


def test_short_sequences_edge():
    for lk in (1, 2, 63, 64, 65, 127, 129):
        run_and_check(2, 8, 1, lk, seed=70 + lk)
        run_and_check(1, 8, 1, lk, pack_gqa=False, seed=70 + lk)


def test_strided_inputs():
    dec = _dec()
    torch.manual_seed(0)
    B, HQ, HKV, L, D = 2, 16, 2, 300, 128
    qbig = torch.randn(B, HQ, 2 * D, device="cuda").to(torch.bfloat16)
    q = qbig[:, :, :D]                                    # q row stride 256 elements
    kv = torch.randn(B, L, 2, HKV, D, device="cuda").to(torch.bfloat16)
    k, v = kv[:, :, 0], kv[:, :, 1]                       # interleaved K/V cache
    seq = torch.tensor([300, 123], dtype=torch.int32, device="cuda")
    plan = dec.make_plan(B, HQ, HKV, L, policy="fixed", forced_splits=3)
    out, lse = dec.forward(plan, q, k, v, seq)
    torch.cuda.synchronize()
    ref_o, ref_l = OA.decode_attention(*(synth.to_f64(t) for t in (q, k, v, seq)))
    assert_out_close(synth.to_f64(out), ref_o)
    assert_lse_close(synth.to_f64(lse), ref_l)


def test_combine_kernel_direct():
    dec = _dec()
    rng = np.random.default_rng(3)
    for s in (1, 2, 5, 33, 100):
        o = rng.standard_normal((s, 3, 8, 128))
        l = rng.standard_normal((s, 3, 8)) * 3
        l[rng.random((s, 3, 8)) < 0.2] = -np.inf
        l[:, 0, 0] = -np.inf                               # one row with every split empty
        o[np.isneginf(l)] = 0.0
        ot = torch.tensor(o, dtype=torch.float32, device="cuda")
        lt = torch.tensor(l, dtype=torch.float32, device="cuda")
        for dt in (torch.bfloat16, torch.float32):
            out, lse = dec.combine(ot, lt, out_dtype=dt)
            torch.cuda.synchronize()
            ref_o, ref_l = OA.lse_combine(synth.to_f64(ot), synth.to_f64(lt))
            assert_out_close(synth.to_f64(out), ref_o)
            assert_lse_close(synth.to_f64(lse), ref_l)


def test_combine_kernel_padded_split_stride():
    # da_combine with split strides larger than a split's rows (the NCCL all-gather buffer [P][o | lse]
    # padded to 16 bytes, dist.SeqShardedDecode): partials read through a non-contiguous view
    dec = _dec()
    from paper_2604_00028_b200 import _lib as L
    rng = np.random.default_rng(4)
    for s, B, HQ in ((2, 1, 64), (8, 3, 24), (5, 2, 8)):
        rows = B * HQ
        chunk = -(-(rows * 129) // 4) * 4 + 4 * int(rng.integers(0, 5))   # padded (+ up to 16 extra floats)
        buf = torch.full((s, chunk), float("nan"), dtype=torch.float32, device="cuda")
        o = rng.standard_normal((s, B, HQ, 128))
        l = rng.standard_normal((s, B, HQ)) * 2
        l[rng.random((s, B, HQ)) < 0.25] = -np.inf
        o[np.isneginf(l)] = 0.0
        buf[:, : rows * 128] = torch.tensor(o.reshape(s, -1), dtype=torch.float32, device="cuda")
        buf[:, rows * 128: rows * 129] = torch.tensor(l.reshape(s, -1), dtype=torch.float32, device="cuda")
        o_view = buf[:, : rows * 128]
        l_view = buf[:, rows * 128: rows * 129]
        for dt in (L.DA_BF16, L.DA_F32):
            out = torch.empty((B, HQ, 128), dtype=torch.float32 if dt == L.DA_F32 else torch.bfloat16, device="cuda")
            lse = torch.empty((B, HQ), dtype=torch.float32, device="cuda")
            L.da_combine(s, B, HQ, 128, o_view, chunk, l_view, chunk, dt, out, lse)
            torch.cuda.synchronize()
            ref_o, ref_l = OA.lse_combine(o, l)
            assert_out_close(synth.to_f64(out), ref_o)
            assert_lse_close(synth.to_f64(lse), ref_l)


def test_deterministic_replay():
    dec = _dec()
    inp = synth.make_inputs(1, 8, 1, 512, device="cuda", seed=5)
    plan = dec.make_plan(1, 8, 1, 512)
    a, la = dec.forward(plan, inp["q"], inp["k"], inp["v"], inp["seqlens"])
    b, lb = dec.forward(plan, inp["q"], inp["k"], inp["v"], inp["seqlens"])
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(la, lb)


# ---- BASELINE.json full sizes, in bench.py's launch configuration (cache_seqlens = NULL, plan
#      cached per shape); EVERY (b, kv-head) group checked against the fp64 oracle, one group at a
#      time (the oracle's fp64 copy of one group is 2 x L_K x 128 x 8 bytes) -------------------------
def _check_full(cfg, policy, seed, variant="normal", picks=None):
    dec = _dec()
    B, HQ, HKV, L = cfg["batch"], cfg["h_q"], cfg["h_kv"], cfg["l_k"]
    inp = synth.make_inputs(B, HQ, HKV, L, device="cuda", seed=seed, variant=variant)
    plan = dec.make_plan(B, HQ, HKV, L, policy=policy)
    seq = None if variant == "normal" else inp["seqlens"]
    out, lse = dec.forward(plan, inp["q"], inp["k"], inp["v"], seq)
    torch.cuda.synchronize()
    G = HQ // HKV
    out_h, lse_h = synth.to_f64(out), synth.to_f64(lse)
    q_h = synth.to_f64(inp["q"])
    seq_h = None if seq is None else seq.cpu().tolist()
    del out, lse
    groups = picks if picks is not None else [(b, g) for b in range(B) for g in range(HKV)]
    for b in sorted({b for b, _ in groups}):
        kb, vb = inp["k"][b].cpu(), inp["v"][b].cpu()          # one sequence's cache on the host (bf16)
        for g in [g for bb, g in groups if bb == b]:
            rows = slice(g * G, (g + 1) * G)
            n = L if seq_h is None else int(seq_h[b])
            k = synth.to_f64(kb[None, :n, g:g + 1])
            v = synth.to_f64(vb[None, :n, g:g + 1])
            ref_o, ref_l = OA.decode_attention(q_h[b:b + 1, rows], k, v, [n])
            assert_out_close(out_h[b:b + 1, rows], ref_o, f"out[b={b}, g={g}]")
            assert_lse_close(lse_h[b:b + 1, rows], ref_l, f"lse[b={b}, g={g}]")
    return plan


def test_full_size_high_load_every_group():
    cfg = synth.CONFIGS["high_load"]               # B=128 H_Q=64 H_KV=8 L_K=8192 (4.3 GB of KV), 1024 groups
    plan = _check_full(cfg, "seq_aware", 1003)
    assert plan.num_splits == 1


@pytest.mark.parametrize("policy,s,mode", [("seq_aware", 16, 2), ("seq_aware_sm", 10, 1)])
def test_full_size_long_context_every_group(policy, s, mode):
    # B=1 H_Q=64 H_KV=8 L_K=131072: the paper's rule gives s = 16 (workspace combine), C-ext-1 moves it
    # to the one-wave cluster split (s = 10, 8 clusters)
    plan = _check_full(synth.CONFIGS["long_context"], policy, 1004)
    assert plan.num_splits == s and plan.combine_mode == mode


def test_full_size_mqa_tcgen05_every_group():
    # bench.py's mqa_g64 workload (B=128 H_Q=64 H_KV=1 L_K=8192, 512 MiB of KV) in the plan the bench
    # times: the tcgen05 kernel, one 64-row CTA per sequence, s = 1
    plan = _check_full(dict(batch=128, h_q=64, h_kv=1, l_k=8192), "seq_aware", 1006)
    assert plan.num_splits == 1 and plan.path == 2


def test_full_size_long_context_ragged_every_group():
    # ragged lengths at the long-context size: batch of 3 with 0 / 1 / random tokens
    cfg = dict(synth.CONFIGS["long_context"], batch=3)
    _check_full(cfg, "seq_aware", 1005, variant="ragged")


@pytest.mark.parametrize("policy,forced", [("seq_aware", 0), ("seq_aware_sm", 0), ("fixed", 3), ("fixed", 5),
                                           ("fixed", 20), ("dynamic", 0)])
def test_seqlens_past_plan_length(policy, forced):
    # cache_seqlens in (L_K, L_cap]: the plan is made for L_K = 512, the lengths reach the capacity
    # 1024 (decattn.h: cache_seqlens is clamped to [0, l_cap] on the device, the split range follows
    # the real length); one value past l_cap is clamped to it
    dec = _dec()
    B, HQ, HKV, LK, LCAP = 5, 16, 2, 512, 1024
    inp = synth.make_inputs(B, HQ, HKV, LK, l_cap=LCAP, seed=1040, device="cuda")
    seq = torch.tensor([700, 1024, 513, 200, 5000], dtype=torch.int32, device="cuda")
    plan = dec.make_plan(B, HQ, HKV, LK, policy=policy, forced_splits=forced)
    for dt in (torch.bfloat16, torch.float32):
        out, lse = dec.forward(plan, inp["q"], inp["k"], inp["v"], seq, out_dtype=dt)
        torch.cuda.synchronize()
        ref_o, ref_l = OA.decode_attention(synth.to_f64(inp["q"]), synth.to_f64(inp["k"]), synth.to_f64(inp["v"]),
                                           [700, 1024, 513, 200, 1024])
        assert_out_close(synth.to_f64(out), ref_o)
        assert_lse_close(synth.to_f64(lse), ref_l)


# ---- SM-count-aware policy (C-ext-1): the efficiency-region one-wave cluster splits -----------
@pytest.mark.parametrize("batch,h_q,h_kv,l_k", [(1, 8, 1, 4096), (1, 64, 8, 2048), (2, 64, 8, 2048),
                                                (1, 16, 2, 700), (3, 24, 3, 1500)])
@pytest.mark.parametrize("variant", ["normal", "ragged"])
def test_seq_aware_sm_fit(batch, h_q, h_kv, l_k, variant):
    plan, _, _ = run_and_check(batch, h_q, h_kv, l_k, policy="seq_aware_sm", variant=variant, seed=1100)
    if plan.num_splits > 1 and plan.num_splits <= 16:
        assert plan.combine_mode == _dec().DA_COMBINE_CLUSTER


# ---- paged KV cache (da_forward_paged) --------------------------------------
def run_paged(batch, h_q, h_kv, l_k, page_size, *, policy="seq_aware", forced=0, pack=True, seed=90,
              variant="ragged", combine_mode=None, path=None):
    dec = _dec()
    inp = synth.make_inputs(batch, h_q, h_kv, l_k, seed=seed, variant=variant, device="cuda")
    q, k, v, seq = inp["q"], inp["k"], inp["v"], inp["seqlens"]
    P = -(-l_k // page_size)                                  # pages per sequence
    extra = 3
    n_pages = batch * P + extra
    g = torch.Generator(device="cpu").manual_seed(seed)
    perm = torch.randperm(n_pages, generator=g)
    kp = torch.full((n_pages, page_size, h_kv, 128), float("nan"), dtype=torch.bfloat16, device="cuda")
    vp = torch.full_like(kp, float("nan"))                    # unused slots / pages hold garbage
    table = torch.full((batch, P + 1), -1, dtype=torch.int32)  # entries past a sequence: invalid
    for b in range(batch):
        n = int(seq[b])
        for j in range(-(-n // page_size)):
            pg = int(perm[b * P + j])
            table[b, j] = pg
            lo, hi = j * page_size, min((j + 1) * page_size, n)
            kp[pg, : hi - lo] = k[b, lo:hi]
            vp[pg, : hi - lo] = v[b, lo:hi]
    table = table.to("cuda")
    plan = dec.make_plan(batch, h_q, h_kv, l_k, pack_gqa=pack, policy=policy, forced_splits=forced,
                         combine_mode=combine_mode, path=path)
    out, lse = dec.forward_paged(plan, q, kp, vp, table, seq)
    torch.cuda.synchronize()
    ref_o, ref_l = OA.decode_attention(*(synth.to_f64(t) for t in (q, k, v, seq)))
    assert_out_close(synth.to_f64(out), ref_o)
    assert_lse_close(synth.to_f64(lse), ref_l)
    return plan


@pytest.mark.parametrize("page_size", [64, 128, 256])
@pytest.mark.parametrize("policy,forced,combine", [("seq_aware", 0, None), ("fixed", 3, 1), ("fixed", 12, 2)])
def test_paged_matches_dense(page_size, policy, forced, combine):
    run_paged(4, 16, 2, 700, page_size, policy=policy, forced=forced, combine_mode=combine, seed=91)


@pytest.mark.parametrize("pack", [True, False])
def test_paged_paths_and_uniform_lengths(pack):
    run_paged(2, 8, 1, 512, 64, pack=pack, variant="normal", seed=92)
    run_paged(3, 64, 8, 1024, 128, pack=pack, variant="ragged", seed=93)


def test_paged_rejects_unsupported_page_size():
    dec = _dec()
    plan = dec.make_plan(1, 8, 1, 128)
    q = torch.zeros(1, 8, 128, dtype=torch.bfloat16, device="cuda")
    kp = torch.zeros(4, 32, 1, 128, dtype=torch.bfloat16, device="cuda")
    table = torch.zeros(1, 4, dtype=torch.int32, device="cuda")
    with pytest.raises(dec.DecAttnError) as e:
        dec.forward_paged(plan, q, kp, kp, table)
    assert e.value.status == dec._lib.DA_ERR_UNSUPPORTED


# ---- host-buffer entry point (da_forward_host: H2D + forward + D2H on one stream) -----------
@pytest.mark.parametrize("batch,h_q,h_kv,l_k,policy,forced,seqlens,f32",
                         [(1, 64, 8, 512, "seq_aware_sm", 0, False, False),
                          (3, 24, 3, 1500, "fixed", 40, True, False),     # workspace combine
                          (2, 8, 1, 700, "seq_aware", 0, True, True),
                          (1, 8, 8, 130, "guarded", 0, False, False),     # scalar path
                          (4, 32, 4, 3000, "dynamic", 0, True, False)])   # dynamic: schedule in staging
def test_forward_host_matches_oracle(batch, h_q, h_kv, l_k, policy, forced, seqlens, f32):
    dec = _dec()
    inp = synth.make_inputs(batch, h_q, h_kv, l_k, seed=1200, variant="ragged" if seqlens else "normal")
    q, k, v = (inp[n].contiguous().pin_memory() for n in ("q", "k", "v"))
    seq = inp["seqlens"].to(torch.int32).pin_memory() if seqlens else None
    plan = dec.make_plan(batch, h_q, h_kv, l_k, policy=policy, forced_splits=forced)
    stream = torch.cuda.Stream()
    staging = dec.HostStaging()
    out, lse = dec.forward_host(plan, q, k, v, seq, staging=staging, stream=stream,
                                out_dtype=torch.float32 if f32 else torch.bfloat16)
    stream.synchronize()
    assert not out.is_cuda and not lse.is_cuda
    n = inp["seqlens"] if seqlens else torch.full((batch,), l_k, dtype=torch.int32)
    ref_o, ref_l = OA.decode_attention(*(synth.to_f64(t) for t in (inp["q"], inp["k"], inp["v"], n)))
    assert_out_close(synth.to_f64(out), ref_o)
    assert_lse_close(synth.to_f64(lse), ref_l)
    # one [2, ...] host KV allocation (K and V in one DMA), an adjacent out | lse buffer (one DMA back),
    # and separately pinned K / V that merely sit back to back (two DMAs) give the same bytes
    odt = torch.float32 if f32 else torch.bfloat16
    kv = torch.empty((2,) + tuple(k.shape), dtype=torch.bfloat16).pin_memory()
    kv[0].copy_(k)
    kv[1].copy_(v)
    ob = batch * h_q * 128 * (4 if f32 else 2)
    ol = torch.empty(ob + 4 * batch * h_q, dtype=torch.uint8).pin_memory()
    out3, lse3 = ol[:ob].view(odt).view(batch, h_q, 128), ol[ob:].view(torch.float32).view(batch, h_q)
    dec.forward_host(plan, q, kv[0], kv[1], seq, out=out3, lse=lse3, staging=staging, stream=stream)
    stream.synchronize()
    assert torch.equal(out, out3) and torch.equal(lse, lse3)
    # a second call reuses the staging buffer and returns the same bytes
    out2, lse2 = dec.forward_host(plan, q, k, v, seq, staging=staging, stream=stream,
                                  out_dtype=torch.float32 if f32 else torch.bfloat16)
    stream.synchronize()
    assert torch.equal(out, out2) and torch.equal(lse, lse2)


# ---- per-batch dynamic split counts (DA_POLICY_DYNAMIC, C-ext-2) ----------------
def _dyn_lengths(kind, batch, l_k, seed):
    g = torch.Generator().manual_seed(seed)
    if kind == "skewed":        # one long sequence among short ones
        n = torch.randint(1, max(2, l_k // 16), (batch,), generator=g)
        n[batch // 2] = l_k
    elif kind == "uniform":
        n = torch.full((batch,), l_k)
    elif kind == "empty":
        n = torch.zeros(batch, dtype=torch.int64)
        n[-1] = 3
    else:                       # ragged: U[0, l_k] with an empty and a single-token sequence
        n = torch.randint(0, l_k + 1, (batch,), generator=g)
        n[0] = 0
        if batch > 1:
            n[1] = 1
    return n.to(torch.int32)


@pytest.mark.parametrize("batch,h_q,h_kv,l_k,kind", [
    (8, 64, 8, 4096, "skewed"), (16, 8, 1, 8192, "skewed"), (5, 24, 3, 1500, "ragged"),
    (3, 16, 16, 700, "ragged"), (40, 8, 1, 2048, "ragged"), (2, 8, 2, 1024, "uniform"),
    (4, 8, 1, 600, "empty"), (1, 64, 8, 20000, "uniform"), (70, 16, 2, 300, "ragged")])
def test_dynamic_splits_match_oracle(batch, h_q, h_kv, l_k, kind):
    dec = _dec()
    inp = synth.make_inputs(batch, h_q, h_kv, l_k, seed=1300, device="cuda")
    seq = _dyn_lengths(kind, batch, l_k, 1301).to("cuda")
    plan = dec.make_plan(batch, h_q, h_kv, l_k, policy="dynamic")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    assert (plan.num_splits, plan.rule) == OP.num_splits(batch, h_q, h_kv, l_k, sms, 0, "dynamic")
    ws = dec.workspace_for(plan, inp["q"].device)
    out, lse = dec.forward(plan, inp["q"], inp["k"], inp["v"], seq, workspace=ws)
    torch.cuda.synchronize()
    qn, kn, vn, sn = (synth.to_f64(t) for t in (inp["q"], inp["k"], inp["v"], seq))
    ref_o, ref_l = OA.decode_attention(qn, kn, vn, sn)
    assert_out_close(synth.to_f64(out), ref_o)
    assert_lse_close(synth.to_f64(lse), ref_l)
    if plan.num_splits > 1:
        # the schedule the kernel recorded equals the oracle's, bit for bit
        prows = plan.grid_y * h_q
        meta = ws.view(torch.int32)[prows * 129: prows * 129 + 2 * batch].cpu().tolist()
        tiles = h_kv * plan.num_m_blocks
        W, s_ref, P_ref = OP.dynamic_schedule([int(n) for n in sn], tiles, plan.usable_sms, plan.num_splits)
        assert meta[:batch] == P_ref and meta[batch:] == s_ref
        assert sum(s_ref) <= plan.grid_y
        # per-split partials of the longest sequence vs C-part with its own partition (a sequence
        # with one split writes its final row directly and leaves no partial)
        b = int(np.argmax(sn))
        if s_ref[b] == 1:
            return
        ranges = [OA.partition(int(sn[b]), s_ref[b], OP.SPLIT_UNIT)]
        po, pl = OA.split_partials(qn[b:b + 1], kn[b:b + 1], vn[b:b + 1], sn[b:b + 1], ranges)
        wo = ws[: prows * 128].view(plan.grid_y, h_q, 128)[P_ref[b]: P_ref[b] + s_ref[b]]
        wl = ws[prows * 128: prows * 129].view(plan.grid_y, h_q)[P_ref[b]: P_ref[b] + s_ref[b]]
        assert_out_close(synth.to_f64(wo), po[:, 0], "dynamic partial o")
        assert_lse_close(synth.to_f64(wl), pl[:, 0], "dynamic partial lse")


def test_dynamic_splits_without_seqlens_and_paged():
    # cache_seqlens = NULL (uniform plan length) and the paged cache go through the same schedule
    dec = _dec()
    inp = synth.make_inputs(2, 16, 2, 3000, seed=1310, device="cuda")
    plan = dec.make_plan(2, 16, 2, 3000, policy="dynamic")
    out, lse = dec.forward(plan, inp["q"], inp["k"], inp["v"], None)
    torch.cuda.synchronize()
    ref_o, ref_l = OA.decode_attention(*(synth.to_f64(t) for t in (inp["q"], inp["k"], inp["v"])),
                                       [3000, 3000])
    assert_out_close(synth.to_f64(out), ref_o)
    assert_lse_close(synth.to_f64(lse), ref_l)
    run_paged(6, 32, 4, 2500, 128, policy="dynamic")


# ---- sequence shards (da_plan_set_seq_offset): cache_seqlens are whole-sequence lengths and the
#      cache holds tokens [t0, t0 + L) of each sequence -------------------------------------------
@pytest.mark.parametrize("batch,h_q,h_kv,l_local,t0,policy,forced,combine", [
    (4, 16, 2, 700, 500, "seq_aware", 0, None),
    (4, 16, 2, 700, 500, "fixed", 5, 1),
    (4, 16, 2, 700, 500, "fixed", 20, 2),
    (6, 32, 4, 3000, 2000, "dynamic", 0, None),
    (3, 8, 1, 20000, 16384, "fixed", 5, 1),          # balanced cluster splits
    (2, 8, 8, 300, 1000, "guarded", 0, None),       # scalar path
])
def test_seq_offset_shard(batch, h_q, h_kv, l_local, t0, policy, forced, combine):
    dec = _dec()
    from paper_2604_00028_b200.dist import local_seqlens
    inp = synth.make_inputs(batch, h_q, h_kv, l_local, seed=1300, device="cuda")
    g = torch.Generator(device="cpu").manual_seed(1301)
    # whole-sequence lengths: before the shard, inside it, past it
    glob = torch.randint(0, t0 + l_local + 300, (batch,), generator=g, dtype=torch.int32)
    glob[0] = max(t0 - 1, 0)
    glob[1] = t0 + l_local + 17
    glob = glob.to("cuda")
    plan = dec.make_plan(batch, h_q, h_kv, l_local, policy=policy, forced_splits=forced, combine_mode=combine,
                         seq_offset=t0)
    assert plan.seq_offset == t0
    ws = dec.workspace_for(plan, inp["q"].device)
    out, lse = dec.forward(plan, inp["q"], inp["k"], inp["v"], glob, workspace=ws)
    torch.cuda.synchronize()
    loc = local_seqlens(glob.cpu(), t0, l_local)
    assert int(loc[0]) == 0 and int(loc[1]) == l_local
    ref_o, ref_l = OA.decode_attention(*(synth.to_f64(t) for t in (inp["q"], inp["k"], inp["v"], loc)))
    assert_out_close(synth.to_f64(out), ref_o)
    assert_lse_close(synth.to_f64(lse), ref_l)
    # without cache_seqlens the offset does not apply: every sequence is the plan's l_k long
    out2, lse2 = dec.forward(plan, inp["q"], inp["k"], inp["v"], None, workspace=ws)
    torch.cuda.synchronize()
    ref_o, ref_l = OA.decode_attention(*(synth.to_f64(t) for t in (inp["q"], inp["k"], inp["v"])),
                                       np.full(batch, l_local))
    assert_out_close(synth.to_f64(out2), ref_o)
    assert_lse_close(synth.to_f64(lse2), ref_l)


# ---- DA_PATH_TC: the tcgen05 kernel for G >= 32 (fwd_tc.cu): 64 query rows per CTA on TMEM ----
@pytest.mark.parametrize("batch,h_q,h_kv,l_k,policy,forced,variant", [
    (1, 64, 1, 1024, "fixed", 1, "normal"),          # MQA G = 64, one CTA per KV head, 16 tiles
    (4, 64, 1, 3000, "fixed", 1, "ragged"),          # an empty and a one-token sequence
    (4, 64, 1, 3000, "fixed", 2, "ragged"),          # + empty splits of the short sequences
    (2, 32, 1, 5000, "fixed", 2, "peaked"),          # G = 32: rows 32-63 of the CTA are padding
    (3, 96, 2, 2000, "fixed", 1, "ragged"),          # G = 48
    (1, 128, 1, 9000, "fixed", 4, "normal"),         # G = 128: two 64-row CTAs per KV head
    (2, 64, 1, 4500, "fixed", 4, "peaked"),          # workspace partials
    (8, 64, 2, 1100, "fixed", 1, "normal"),          # a partial last tile (1100 = 17 x 64 + 12)
    (1, 64, 1, 131072, "seq_aware", 0, "normal"),    # the paper's long context as MQA-64 (s = 109)
    (2, 8, 1, 3000, "fixed", 2, "ragged"),           # G = 8 forced onto tcgen05: 56 padding rows
    (1, 16, 2, 700, "fixed", 3, "peaked"),           # short splits (4 tiles) on tcgen05
])
def test_tc_path_matches_oracle(batch, h_q, h_kv, l_k, policy, forced, variant):
    dec = _dec()
    plan, _, _ = run_and_check(batch, h_q, h_kv, l_k, policy=policy, forced=forced, variant=variant, seed=1700,
                               check_partials=forced > 1, path=dec.DA_PATH_TC)
    assert (plan.path, plan.rows_per_cta, plan.cluster_x) == (dec.DA_PATH_TC, 64, 1)
    assert plan.combine_mode == (dec.DA_COMBINE_NONE if plan.num_splits == 1 else dec.DA_COMBINE_KERNEL)


@pytest.mark.parametrize("pack", [True])
def test_tc_path_edges(pack):
    # NaN past each sequence, l_cap > l_k, fp32 output, cache_seqlens past the plan's length
    dec = _dec()
    for kw in (dict(batch=3, l_k=1500, l_cap=1700, variant="ragged", nan_tail=True, forced=1),
               dict(batch=2, l_k=1100, out_f32=True, forced=1),
               dict(batch=2, l_k=3000, out_f32=True, forced=2, check_partials=True)):
        b_ = kw.pop("batch")
        plan, _, _ = run_and_check(b_, 64, 1, policy="fixed", seed=1701, path=dec.DA_PATH_TC, **kw)
        assert plan.path == dec.DA_PATH_TC
    # the planner's choice: short / few splits stay on the mma.sync kernel (and its cluster combine),
    # many CTAs with >= 4 tiles each take tcgen05
    plan, _, _ = run_and_check(1, 64, 1, 512, policy="seq_aware_sm", seed=1704)
    assert plan.path == dec.DA_PATH_MMA
    plan, _, _ = run_and_check(80, 64, 1, 300, policy="guarded", seed=1705, variant="ragged")
    assert (plan.num_splits, plan.path) == (1, dec.DA_PATH_TC)


@pytest.mark.parametrize("batch,h_q,h_kv,l_k,policy,path", [
    (16, 24, 1, 4096, "seq_aware_sm", 2),   # G = 24: C-ext-1's wide-group clause, s = 8 on tcgen05
    (8, 40, 2, 8192, "guarded", 2),         # G = 20, two KV heads
    (4, 28, 1, 16384, "seq_aware", 2),      # G = 28, s = 32
    (16, 12, 1, 8192, "seq_aware", 1),      # G = 12 stays on mma.sync (one 16-row CTA per head)
])
def test_planner_picks_tcgen05_for_groups_above_16(batch, h_q, h_kv, l_k, policy, path):
    # 16 < G < 32: the mma.sync kernel would read K / V twice (two 16-row CTAs per KV head), so the
    # planner's own rule takes the tcgen05 kernel (kernel choice); ragged lengths
    plan, _, _ = run_and_check(batch, h_q, h_kv, l_k, policy=policy, variant="ragged", seed=1720)
    assert plan.path == path


def test_tc_path_rescales_when_the_maximum_grows():
    # scores that climb by ~16 (log2 units) every 64-token tile: the running reference moves and
    # the O rows in TMEM are rescaled on every tile (the path that is rare on N(0, 1) inputs)
    dec = _dec()
    batch, h_q, h_kv, l_k = 2, 64, 1, 1024
    g = torch.Generator(device="cpu").manual_seed(1710)
    base = torch.randn(128, generator=g)
    q = (base + 0.05 * torch.randn(batch, h_q, 128, generator=g)).to(torch.bfloat16)
    ramp = torch.arange(l_k, dtype=torch.float32) / 64.0 * 1.3
    k = (ramp[None, :, None, None] * base[None, None, None, :] / base.norm() * 11.3
         + 0.3 * torch.randn(batch, l_k, h_kv, 128, generator=g)).to(torch.bfloat16)
    v = torch.randn(batch, l_k, h_kv, 128, generator=g).to(torch.bfloat16)
    seq = torch.tensor([l_k, 700], dtype=torch.int32)
    plan = dec.make_plan(batch, h_q, h_kv, l_k, policy="fixed", forced_splits=1, path=2)   # one CTA: 16 tiles
    assert plan.path == dec.DA_PATH_TC and plan.num_splits == 1
    out, lse = dec.forward(plan, q.cuda(), k.cuda(), v.cuda(), seq.cuda())
    torch.cuda.synchronize()
    ref_o, ref_l = OA.decode_attention(*(synth.to_f64(t) for t in (q, k, v, seq)))
    assert (np.diff(ref_l) != 0).any()
    assert_out_close(synth.to_f64(out), ref_o)
    assert_lse_close(synth.to_f64(lse), ref_l)


def test_tc_path_paged_offset_and_graph():
    dec = _dec()
    assert run_paged(3, 64, 1, 2500, 128, policy="fixed", forced=1, seed=1720, path=2).path == dec.DA_PATH_TC
    assert run_paged(2, 128, 2, 2600, 256, policy="fixed", forced=2, seed=1721, path=2).path == dec.DA_PATH_TC
    assert run_paged(3, 64, 1, 2500, 64, policy="fixed", forced=1, seed=1723, path=2).path == dec.DA_PATH_TC
    # a sequence shard (seq_offset) and CUDA-graph replays of the tcgen05 kernel
    batch, h_q, h_kv, l_local, t0 = 3, 64, 1, 2000, 777
    from paper_2604_00028_b200.dist import local_seqlens
    inp = synth.make_inputs(batch, h_q, h_kv, l_local, seed=1722, device="cuda")
    glob = torch.tensor([100, t0 + l_local + 5, t0 + 900], dtype=torch.int32, device="cuda")
    plan = dec.make_plan(batch, h_q, h_kv, l_local, policy="fixed", forced_splits=2, seq_offset=t0, path=2)
    assert plan.path == dec.DA_PATH_TC
    ws = dec.workspace_for(plan, inp["q"].device)
    out = torch.empty((batch, h_q, 128), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((batch, h_q), dtype=torch.float32, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        dec.forward(plan, inp["q"], inp["k"], inp["v"], glob, out=out, lse=lse, workspace=ws)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        for _ in range(3):
            dec.forward(plan, inp["q"], inp["k"], inp["v"], glob, out=out, lse=lse, workspace=ws)
    out.zero_()
    gr.replay()
    torch.cuda.synchronize()
    loc = local_seqlens(glob.cpu(), t0, l_local)
    ref_o, ref_l = OA.decode_attention(*(synth.to_f64(t) for t in (inp["q"], inp["k"], inp["v"], loc)))
    assert_out_close(synth.to_f64(out), ref_o)
    assert_lse_close(synth.to_f64(lse), ref_l)
