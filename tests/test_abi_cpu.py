"""Host-side checks of the C ABI that need no GPU: the library loads, exports
every symbol include/decattn.h declares, the planner matches the CPU oracle
bit for bit, and argument validation returns the documented status codes
before any CUDA call."""

import itertools
import os
import random
import re

import pytest

from oracle import policy as OP

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2604_00028_b200 import _lib
    return _lib


def test_library_exports_every_header_symbol(L):
    with open(os.path.join(ROOT, "include", "decattn.h")) as f:
        hdr = f.read()
    declared = re.findall(r"DA_API\s+[\w\s\*]+?\b(da_\w+)\s*\(", hdr)
    assert set(declared) == set(L.EXPORTED)
    for name in declared:
        assert hasattr(L.LIB, name), name
    assert L.da_abi_version() == L.DA_ABI_VERSION
    for code in range(-1, 8):
        assert isinstance(L.da_status_string(code), str)


def test_plan_struct_layout(L):
    import ctypes
    # 28 int32 fields + one int64 + two int32 = 128 bytes (no implicit padding)
    assert ctypes.sizeof(L.da_plan) == 128
    assert L.da_plan.workspace_bytes.offset == 112 and L.da_plan.seq_offset.offset == 120
    with open(os.path.join(ROOT, "include", "decattn.h")) as f:
        hdr = f.read()
    body = hdr[hdr.index("typedef struct da_plan"):hdr.index("} da_plan;")]
    names = re.findall(r"\b([a-z_]+)(?=\s*[,;])", re.sub(r"/\*.*?\*/", "", body, flags=re.S))
    assert names == [n for n, _ in L.da_plan._fields_]


def _tc(b, hq, hkv, lk, pack, s, U, dynamic=False):
    # the planner's kernel choice: tcgen05 for G > 16 when every split holds >= 4
    # tiles and the 64-row grid has >= U / 2 CTAs (static plans)
    G = hq // hkv
    return bool(pack) and G >= 17 and not dynamic and -(-lk // 64) >= 4 * s and 2 * b * hkv * -(-G // 64) * s >= U


def _expected_launch(b, hq, hkv, lk, pack, s, U, dynamic=False):
    G = hq // hkv
    mma = bool(pack) and G >= 2
    if _tc(b, hq, hkv, lk, pack, s, U, dynamic):   # DA_PATH_TC (fwd_tc.cu): 64 rows per CTA
        return 2, 64, (s, hkv * -(-G // 64), b)
    rows = OP.launch_rows(b, G, hkv, lk, s, U) if mma else 1
    gy = hkv * -(-G // rows) if mma else hq
    return (1 if mma else 0), rows, (s, gy, b)


# cluster combine when every cluster of the launch is co-resident in one wave
# (the measured B200 record of cudaOccupancyMaxActiveClusters for the cluster kernels, loaded by the
# oracle from profiles/cluster_fit_b200.json).
_FIT = list(OP.CLUSTER_FIT_B200)


def test_cluster_fit_table_single_source():
    # the planner's compiled-in copy (config.h kMaxActiveClustersB200) equals the measured record
    import json
    with open(os.path.join(ROOT, "paper_2604_00028_b200", "csrc", "config.h")) as f:
        src = f.read()
    m = re.search(r"kMaxActiveClustersB200\[17\]\s*=\s*\{([^}]*)\}", src)
    table = [int(x) for x in m.group(1).split(",")]
    with open(os.path.join(ROOT, "profiles", "cluster_fit_b200.json")) as f:
        rec = json.load(f)
    assert rec["device"].startswith("NVIDIA B200") and rec["sms"] == 148 and rec["variants_agree"]
    assert table[1:] == rec["max_active_clusters"][1:]
    assert list(OP.CLUSTER_FIT_B200) == rec["max_active_clusters"]


def _expected_combine(b, hq, hkv, lk, pack, sms, s, U):
    if s == 1:
        return 0
    if s > 16 or _tc(b, hq, hkv, lk, pack, s, U):   # > 16 splits or the tcgen05 path: no cluster combine
        return 2
    _, _, (_, gy, gz) = _expected_launch(b, hq, hkv, lk, pack, s, U)
    return 1 if gy * gz <= _FIT[s] * sms // 148 else 2


def _check_plan(L, b, hq, hkv, lk, pack, margin, sms, pol, forced=0):
    p = L.da_plan_make(b, hq, hkv, lk, 128, pack, margin, sms, pol, forced)
    s, rule = OP.num_splits(b, hq, hkv, lk, sms, margin, pol, forced)
    assert (p.num_splits, p.rule) == (s, rule), (b, hq, hkv, lk, margin, sms, pol)
    geo = OP.geometry(b, hq, hkv, lk, sms, margin)
    assert (p.num_n_blocks, p.num_m_blocks, p.total_mblocks, p.usable_sms) == (
        geo["nblk"], geo["num_m_blocks"], geo["T"], geo["U"])
    path, rows, grid = _expected_launch(b, hq, hkv, lk, pack, s, geo["U"], dynamic=pol == "dynamic" and s > 1)
    if pol == "dynamic" and s > 1:      # C-ext-2: split slots decided on the device, workspace combine
        slots = OP.dynamic_slots(b, hkv * geo["num_m_blocks"], geo["U"], s)
        grid = (grid[1], slots, 1)                      # head groups innermost, then split slots
        assert p.workspace_bytes == slots * hq * 129 * 4 + 8 * b
        assert p.combine_mode == 2
    else:
        assert p.workspace_bytes == (s * b * hq * 129 * 4 if s > 1 else 0)
        assert p.combine_mode == _expected_combine(b, hq, hkv, lk, pack, sms, s, geo["U"])
    assert (p.path, p.rows_per_cta, (p.grid_x, p.grid_y, p.grid_z)) == (path, rows, grid)
    assert p.nonempty_splits == min(s, -(-lk // 64))


def test_plan_matches_oracle_dense_lk(L):
    # every L_K up to 4096 at the BASELINE head shapes, both SM counts, both policies
    for sms in (132, 148):
        for (b, hkv) in ((1, 1), (1, 2), (2, 1), (1, 8), (8, 8), (4, 32)):
            for lk in range(1, 4097):
                for pol in ("guarded", "seq_aware", "evolved", "seq_aware_sm", "dynamic"):
                    _check_plan(L, b, 8 * hkv, hkv, lk, 1, 0, sms, pol)


def test_plan_matches_oracle_grid(L):
    Bs = list(range(1, 17)) + [24, 32, 64, 100, 128, 200, 256]
    HKVs = (1, 2, 4, 8, 16, 32)
    LKs = sorted({1, 2, 63, 64, 65, 127, 128, 129, 384, 385, 511, 512, 513, 640, 1000, 2047, 2048,
                  2432, 2433, 2560, 4095, 4096, 8192, 16384, 32768, 65536, 131072, 262144}
                 | {2 ** k + d for k in range(1, 19) for d in (-1, 0, 1)})
    for sms in (132, 148):
        for margin in (0, 4, 16, sms - 1):
            for b, hkv, G in itertools.product(Bs, HKVs, (1, 8)):
                for lk in LKs:
                    for pol in ("guarded", "seq_aware", "seq_aware_sm", "dynamic"):
                        _check_plan(L, b, G * hkv, hkv, lk, 1, margin, sms, pol)


def test_plan_matches_oracle_wide_groups(L):
    # G > 8 at latency sizes: the policy's T_k and the launch's rows per CTA (8 within one wave
    # for <= 64 units, else 16) across the short / long boundary
    LKs = (64, 320, 512, 513, 1024, 2048, 4095, 4096, 4097, 4160, 4161, 8192, 65536)
    # (and G >= 32 where the one-wave cluster fit leaves a 2-CTA split: the tcgen05 clause, B = 16)
    for b, hkv, G in itertools.product((1, 2, 3, 8, 16), (1, 2, 8), (12, 16, 32, 64, 128)):
        for lk in LKs:
            for pol in ("guarded", "seq_aware", "seq_aware_sm", "dynamic", "evolved"):
                _check_plan(L, b, G * hkv, hkv, lk, 1, 0, 148, pol)


def test_plan_float_tie_regression(L):
    # C-amb-3: FA3's float comparison gives 18 at (U=132, T=1, nblk=20); exact integers give 17.
    for lk in (2433, 2500, 2560):
        p = L.da_plan_make(1, 8, 1, lk, 128, 1, 0, 132, "guarded", 0)
        assert p.num_splits == 17
        assert OP.num_splits(1, 8, 1, lk, 132, 0, "guarded")[0] == 17


def test_plan_random_shapes_and_fixed(L):
    rng = random.Random(11)
    for _ in range(20000):
        hkv = rng.choice([1, 2, 3, 4, 8, 16, 32, 64])
        G = rng.choice([1, 2, 3, 4, 5, 8, 12, 16, 32, 64, 128])
        b = rng.randint(1, 300)
        lk = rng.randint(1, 300000)
        sms = rng.choice([132, 148, 7, 2, 1])
        margin = rng.randint(0, sms - 1)
        pack = rng.randint(0, 1)
        pol = rng.choice(["guarded", "seq_aware", "fixed", "evolved", "seq_aware_sm", "dynamic"])
        forced = rng.randint(1, 256) if pol == "fixed" else 0
        _check_plan(L, b, G * hkv, hkv, lk, pack, margin, sms, pol, forced)


def test_paper_decisions_through_abi(L):
    # Table 1 bold rows and Guard 2 at both SM counts.
    for sms in (132, 148):
        for hkv in (1, 2):
            p = L.da_plan_make(1, 8 * hkv, hkv, 512, 128, 1, 0, sms, "seq_aware", 0)
            assert (p.num_splits, p.rule) == (3, L.DA_RULE_LOW_TILE)
            assert p.grid_x * p.grid_y * p.grid_z == 3 * hkv        # 3x the CTAs of s=1
            g = L.da_plan_make(1, 8 * hkv, hkv, 512, 128, 1, 0, sms, "guarded", 0)
            assert (g.num_splits, g.rule) == (1, L.DA_RULE_GUARD_NBLK4)
        p = L.da_plan_make(1, 64, 8, 512, 128, 1, 0, sms, "seq_aware", 0)
        assert (p.num_splits, p.rule) == (1, L.DA_RULE_GUARD2)


@pytest.mark.parametrize("args", [
    (0, 8, 1, 512), (1, 0, 1, 512), (1, 8, 0, 512), (1, 8, 1, 0), (1, 6, 4, 512)])
def test_plan_invalid_shapes(L, args):
    with pytest.raises(L.DecAttnError) as e:
        L.da_plan_make(*args, 128, 1, 0, 148, "seq_aware", 0)
    assert e.value.status == L.DA_ERR_INVALID_ARG


def test_plan_invalid_knobs(L):
    bad = [dict(sm_margin=148), dict(sm_margin=-1), dict(num_sms=0), dict(pack_gqa=2),
           dict(policy=6), dict(policy=-1), dict(policy=L.DA_POLICY_FIXED, forced_splits=0),
           dict(policy=L.DA_POLICY_FIXED, forced_splits=257)]
    for kw in bad:
        args = dict(batch=1, h_q=8, h_kv=1, l_k=512, head_dim=128, pack_gqa=1, sm_margin=0,
                    num_sms=148, policy=1, forced_splits=0)
        args.update(kw)
        with pytest.raises(L.DecAttnError) as e:
            L.da_plan_make(**args)
        assert e.value.status == L.DA_ERR_INVALID_ARG, kw
    with pytest.raises(L.DecAttnError) as e:
        L.da_plan_make(1, 8, 1, 512, 64, 1, 0, 148, 1, 0)
    assert e.value.status == L.DA_ERR_UNSUPPORTED


def test_set_seq_offset(L):
    p = L.da_plan_make(2, 16, 2, 4096, 128, 1, 0, 148, "seq_aware", 0)
    assert p.seq_offset == 0 and p.path_override == 0
    q = L.da_plan.from_buffer_copy(p)
    L.da_plan_set_seq_offset(q, 65536)
    assert q.seq_offset == 65536
    assert {f: getattr(q, f) for f, _ in q._fields_ if f != "seq_offset"} == \
        {f: getattr(p, f) for f, _ in p._fields_ if f != "seq_offset"}      # the launch is unchanged
    with pytest.raises(L.DecAttnError):
        L.da_plan_set_seq_offset(q, -1)
    bad = L.da_plan.from_buffer_copy(p)
    bad.seq_offset = -5                              # hand-edited: rejected by the forwards' checks
    assert _fwd(L, bad) == L.DA_ERR_INVALID_ARG
    bad = L.da_plan.from_buffer_copy(p)
    bad.path_override = 5
    assert _fwd(L, bad) == L.DA_ERR_INVALID_ARG


def test_set_path(L):
    # MQA G = 64, B = 4, L = 8192 under guarded: s = 32, 4 tiles per split, 128 tcgen05 CTAs -> TC
    p = L.da_plan_make(4, 64, 1, 8192, 128, 1, 0, 148, "guarded", 0)
    assert (p.num_splits, p.path, p.rows_per_cta, p.grid_y, p.combine_mode) == (32, L.DA_PATH_TC, 64, 1, 2)
    assert (p.block_threads, p.smem_bytes) == (320, 7 * 32768 + 1024)
    q = L.da_plan.from_buffer_copy(p)
    L.da_plan_set_path(q, L.DA_PATH_MMA)                      # the mma.sync kernel: 16-row CTAs
    assert (q.path, q.rows_per_cta, q.grid_y, q.path_override) == (L.DA_PATH_MMA, 16, 4, L.DA_PATH_MMA)
    L.da_plan_set_path(q, -1)                                 # back to the planner's choice
    assert q.as_dict() == p.as_dict()
    # a short TP-8 slice forced onto tcgen05 (G = 8 rows of the 64); its cluster combine becomes KERNEL
    t = L.da_plan_make(1, 8, 1, 512, 128, 1, 0, 148, "seq_aware", 0)
    assert (t.path, t.combine_mode) == (L.DA_PATH_MMA, L.DA_COMBINE_CLUSTER)
    L.da_plan_set_path(t, L.DA_PATH_TC)
    assert (t.path, t.rows_per_cta, t.combine_mode, t.cluster_x) == (L.DA_PATH_TC, 64, L.DA_COMBINE_KERNEL, 1)
    L.da_plan_set_path(t, L.DA_PATH_MMA)
    assert (t.path, t.combine_mode) == (L.DA_PATH_MMA, L.DA_COMBINE_CLUSTER)
    with pytest.raises(L.DecAttnError):
        L.da_plan_set_combine(L.da_plan_set_path(t, L.DA_PATH_TC), L.DA_COMBINE_CLUSTER)
    for bad in (L.da_plan_make(1, 8, 8, 512, 128, 1, 0, 148, "guarded", 0),    # G = 1: scalar only
                L.da_plan_make(1, 64, 1, 512, 128, 0, 0, 148, "guarded", 0)):   # pack_gqa = 0
        with pytest.raises(L.DecAttnError):
            L.da_plan_set_path(bad, L.DA_PATH_TC)
    d = L.da_plan_make(4, 64, 1, 3000, 128, 1, 0, 148, "dynamic", 0)
    with pytest.raises(L.DecAttnError):
        L.da_plan_set_path(d, L.DA_PATH_TC)                   # the dynamic schedule is mma.sync only
    with pytest.raises(L.DecAttnError):
        L.da_plan_set_path(p, 7)


def test_set_combine_rules(L):
    p = L.da_plan_make(1, 8, 1, 512, 128, 1, 0, 148, "seq_aware", 0)
    assert p.combine_mode == L.DA_COMBINE_CLUSTER and p.cluster_x == 3
    L.da_plan_set_combine(p, L.DA_COMBINE_KERNEL)
    assert p.cluster_x == 1 and p.workspace_bytes == 3 * 8 * 129 * 4
    with pytest.raises(L.DecAttnError):
        L.da_plan_set_combine(p, L.DA_COMBINE_NONE)          # s = 3 needs a combine
    q = L.da_plan_make(1, 8, 1, 512, 128, 1, 0, 148, "fixed", 17)
    assert q.combine_mode == L.DA_COMBINE_KERNEL
    with pytest.raises(L.DecAttnError):
        L.da_plan_set_combine(q, L.DA_COMBINE_CLUSTER)       # cluster only for s <= 16
    q = L.da_plan_make(1, 8, 1, 512, 128, 1, 0, 148, "fixed", 12)
    assert q.combine_mode == L.DA_COMBINE_CLUSTER and q.cluster_x == 12
    q = L.da_plan_make(16, 64, 8, 4096, 128, 1, 0, 148, "fixed", 8)   # 128 clusters of 8 > 15
    assert q.combine_mode == L.DA_COMBINE_KERNEL
    d = L.da_plan_make(4, 32, 4, 4096, 128, 1, 0, 148, "dynamic", 0)  # per-batch counts: workspace only
    assert d.combine_mode == L.DA_COMBINE_KERNEL and d.grid_z == 1
    with pytest.raises(L.DecAttnError):
        L.da_plan_set_combine(d, L.DA_COMBINE_CLUSTER)


# ---- da_forward / da_combine validation (fake device pointers: every check below
#      returns before the library touches CUDA) -------------------------------------
A = 1 << 20          # a 16-byte aligned fake address


def _fwd(L, plan, **kw):
    args = dict(q=A, k_cache=2 * A, v_cache=3 * A, l_cap=plan.l_k, cache_seqlens=None,
                strides=None, softmax_scale=0.0, out_dtype=L.DA_BF16, out=4 * A, lse=5 * A,
                workspace=None, workspace_bytes=0, stream=0)
    args.update(kw)
    with pytest.raises(L.DecAttnError) as e:
        L.da_forward(plan, **args)
    return e.value.status


def test_forward_validation(L):
    p = L.da_plan_make(1, 8, 1, 512, 128, 1, 0, 148, "fixed", 20)   # KERNEL combine
    assert _fwd(L, p, q=None) == L.DA_ERR_INVALID_ARG
    assert _fwd(L, p, out=None) == L.DA_ERR_INVALID_ARG
    assert _fwd(L, p, l_cap=511) == L.DA_ERR_INVALID_ARG
    assert _fwd(L, p, out_dtype=5) == L.DA_ERR_INVALID_ARG
    assert _fwd(L, p, q=A + 2) == L.DA_ERR_ALIGNMENT
    assert _fwd(L, p, k_cache=2 * A + 8) == L.DA_ERR_ALIGNMENT
    assert _fwd(L, p, strides=(1024, 128, 65536, 128, 129, 65536, 128, 128)) == L.DA_ERR_ALIGNMENT
    assert _fwd(L, p) == L.DA_ERR_WORKSPACE
    assert _fwd(L, p, workspace=6 * A, workspace_bytes=p.workspace_bytes - 4) == L.DA_ERR_WORKSPACE
    bad = L.da_plan.from_buffer_copy(p)
    bad.grid_x = 3                                   # inconsistent with num_splits
    assert _fwd(L, bad) == L.DA_ERR_INVALID_ARG
    bad = L.da_plan.from_buffer_copy(p)
    bad.head_dim = 64
    assert _fwd(L, bad) == L.DA_ERR_UNSUPPORTED
    bad = L.da_plan.from_buffer_copy(p)
    bad.combine_mode = L.DA_COMBINE_NONE             # s = 20 cannot skip the combine
    assert _fwd(L, bad) == L.DA_ERR_INVALID_ARG


def test_forward_rejects_oversized_grid(L):
    p = L.da_plan_make(70000, 8, 1, 64, 128, 1, 0, 148, "guarded", 0)   # grid_z = 70000 > 65535
    assert _fwd(L, p) == L.DA_ERR_UNSUPPORTED


def test_combine_validation(L):
    def st(**kw):
        args = dict(num_splits=3, batch=1, h_q=8, head_dim=128, o_partial=A, o_split_stride=1024,
                    lse_partial=2 * A, lse_split_stride=8, out_dtype=L.DA_BF16, out=3 * A, lse=4 * A,
                    stream=0)
        args.update(kw)
        with pytest.raises(L.DecAttnError) as e:
            L.da_combine(**args)
        return e.value.status
    assert st(num_splits=0) == L.DA_ERR_INVALID_ARG
    assert st(o_partial=None) == L.DA_ERR_INVALID_ARG
    assert st(head_dim=64) == L.DA_ERR_UNSUPPORTED
    assert st(o_split_stride=1000) == L.DA_ERR_INVALID_ARG        # < B*H_Q*d
    assert st(o_partial=A + 4) == L.DA_ERR_ALIGNMENT


def test_forward_paged_validation(L):
    p = L.da_plan_make(2, 16, 2, 700, 128, 1, 0, 148, "seq_aware", 0)

    def st(**kw):
        args = dict(q=A, k_pages=2 * A, v_pages=3 * A, num_pages=40, page_size=64, block_table=7 * A,
                    block_table_stride=11, max_pages_per_seq=11, cache_seqlens=None, strides=None,
                    softmax_scale=0.0, out_dtype=L.DA_BF16, out=4 * A, lse=5 * A, workspace=None,
                    workspace_bytes=0, stream=0)
        args.update(kw)
        with pytest.raises(L.DecAttnError) as e:
            L.da_forward_paged(p, **args)
        return e.value.status
    assert st(block_table=None) == L.DA_ERR_INVALID_ARG
    assert st(num_pages=0) == L.DA_ERR_INVALID_ARG
    assert st(page_size=32) == L.DA_ERR_UNSUPPORTED           # not a multiple of the 64-token tile
    assert st(page_size=96) == L.DA_ERR_UNSUPPORTED
    assert st(block_table_stride=10) == L.DA_ERR_INVALID_ARG  # row stride < pages per sequence
    assert st(max_pages_per_seq=10) == L.DA_ERR_INVALID_ARG   # 10 * 64 < l_k = 700
    assert st(block_table=7 * A + 2) == L.DA_ERR_ALIGNMENT
    assert st(q=A + 8) == L.DA_ERR_ALIGNMENT
    assert st(page_size=(1 << 18) + 64) == L.DA_ERR_UNSUPPORTED   # tiles per page must stay < 2^13


def _align256(x):
    return (x + 255) // 256 * 256


@pytest.mark.parametrize("shape,policy,forced", [((1, 64, 8, 512), "seq_aware_sm", 0),
                                                 ((3, 24, 3, 1500), "fixed", 40),
                                                 ((2, 8, 1, 100), "guarded", 0)])
def test_forward_host_bytes_layout(L, shape, policy, forced):
    b, hq, hkv, lk = shape
    p = L.da_plan_make(b, hq, hkv, lk, 128, 1, 0, 148, policy, forced)
    for l_cap, seq, dt in ((lk, 0, L.DA_BF16), (lk + 77, 1, L.DA_F32)):
        kv = b * l_cap * hkv * 128 * 2
        want = (_align256(b * hq * 128 * 2) + 2 * _align256(kv) + _align256(4 * b if seq else 0)
                + _align256(b * hq * 128 * (4 if dt == L.DA_F32 else 2)) + _align256(4 * b * hq)
                + _align256(p.workspace_bytes if p.combine_mode == L.DA_COMBINE_KERNEL else 0))
        assert L.da_forward_host_bytes(p, l_cap, seq, dt) == want
    with pytest.raises(L.DecAttnError):
        L.da_forward_host_bytes(p, lk - 1, 0, L.DA_BF16)          # l_cap below the plan's length
    with pytest.raises(L.DecAttnError):
        L.da_forward_host_bytes(p, lk, 0, 7)                      # not a da_dtype


def test_forward_host_validation(L):
    p = L.da_plan_make(1, 8, 1, 512, 128, 1, 0, 148, "seq_aware", 0)
    need = L.da_forward_host_bytes(p, 512, 0, L.DA_BF16)

    def st(**kw):
        args = dict(q=A, k_cache=2 * A, v_cache=3 * A, l_cap=512, cache_seqlens=None, softmax_scale=0.0,
                    out_dtype=L.DA_BF16, out=4 * A, lse=5 * A, device_buffer=6 * A, device_buffer_bytes=need,
                    stream=0)
        args.update(kw)
        with pytest.raises(L.DecAttnError) as e:
            L.da_forward_host(p, **args)
        return e.value.status
    assert st(q=None) == L.DA_ERR_INVALID_ARG
    assert st(out=None) == L.DA_ERR_INVALID_ARG
    assert st(l_cap=100) == L.DA_ERR_INVALID_ARG
    assert st(device_buffer=None) == L.DA_ERR_WORKSPACE
    assert st(device_buffer_bytes=need - 1) == L.DA_ERR_WORKSPACE
    assert st(device_buffer=6 * A + 128) == L.DA_ERR_ALIGNMENT


def test_plan_make_varlen_matches_oracle(L):
    rng = random.Random(23)
    for _ in range(3000):
        B = rng.randint(1, 96)
        hkv = rng.choice([1, 2, 4, 8])
        G = rng.choice([1, 8, 16])
        l_cap = rng.choice([64, 512, 2048, 8192, 32768, 131072])
        sms = rng.choice([148, 132])
        kind = rng.random()
        if kind < 0.3:
            lens = [l_cap] * B
        elif kind < 0.6:
            lens = [rng.randint(0, l_cap) for _ in range(B)]
        else:
            lens = [rng.randint(0, max(1, l_cap // 32)) for _ in range(B)]
            lens[rng.randrange(B)] = l_cap
        p = L.da_plan_make_varlen(B, G * hkv, hkv, l_cap, 128, 1, 0, sms, lens)
        pol = OP.varlen_policy(B, G * hkv, hkv, l_cap, sms, 0, lens)
        assert p.policy == pol, (B, hkv, G, l_cap, lens[:4])
        ref = L.da_plan_make(B, G * hkv, hkv, l_cap, 128, 1, 0, sms, pol, 0)
        assert p.as_dict() == ref.as_dict()
    with pytest.raises(L.DecAttnError):
        L.da_plan_make_varlen(2, 8, 1, 512, 128, 1, 0, 148, [1])      # wrong length count


def test_peer_exchange_validation(L):
    A2 = 1 << 22
    slot, lo, fo = 4128, 4096, 2 * 4128                # B = 1, H_Q = 8: o 4096 B, lse 32 B
    def sig(**kw):
        a = dict(world=2, rank=0, peer_bases=A2, o_local=A2, lse_local=A2, batch=1, h_q=8, head_dim=128,
                 slot_bytes=slot, lse_offset=lo, flag_offset=fo, epoch=A2, stream=0)
        a.update(kw)
        with pytest.raises(L.DecAttnError) as e:
            L.da_peer_signal(**a)
        return e.value.status
    assert sig(world=0) == L.DA_ERR_INVALID_ARG
    assert sig(world=65) == L.DA_ERR_INVALID_ARG
    assert sig(rank=2) == L.DA_ERR_INVALID_ARG
    assert sig(peer_bases=None) == L.DA_ERR_INVALID_ARG
    assert sig(o_local=None) == L.DA_ERR_INVALID_ARG
    assert sig(head_dim=64) == L.DA_ERR_UNSUPPORTED
    assert sig(lse_offset=16) == L.DA_ERR_INVALID_ARG                 # o and lse overlap
    assert sig(slot_bytes=4112) == L.DA_ERR_INVALID_ARG               # lse past the slot
    assert sig(flag_offset=4128) == L.DA_ERR_INVALID_ARG              # flags inside slot 1
    assert sig(slot_bytes=4132, flag_offset=8272) == L.DA_ERR_ALIGNMENT
    assert sig(o_local=A2 + 4) == L.DA_ERR_ALIGNMENT

    def comb(**kw):
        a = dict(world=2, rank=1, peer_bases=A2, slot_bytes=slot, lse_offset=lo, flag_offset=fo, epoch=A2,
                 batch=1, h_q=8, head_dim=128, out_dtype=L.DA_BF16, out=A2, lse=A2, status=A2, timeout_ns=0,
                 stream=0)
        a.update(kw)
        with pytest.raises(L.DecAttnError) as e:
            L.da_combine_peers(**a)
        return e.value.status
    assert comb(status=None) == L.DA_ERR_INVALID_ARG              # the bounded wait needs its status word
    assert comb(status=A2 + 2) == L.DA_ERR_ALIGNMENT
    assert comb(out=None) == L.DA_ERR_INVALID_ARG
    assert comb(out_dtype=5) == L.DA_ERR_INVALID_ARG
    assert comb(epoch=None) == L.DA_ERR_INVALID_ARG
    assert comb(out=A2 + 8) == L.DA_ERR_ALIGNMENT


def test_forward_peer_validation(L):
    # da_forward_peer: the peer-layout and counter checks, then da_forward's, all before any CUDA call
    A2 = 1 << 22
    plan = L.da_plan_make(1, 8, 1, 512, 128, 1, 0, 148, "seq_aware", 0)
    slot, lo, fo = 4128, 4096, 2 * 4128

    def fwd(**kw):
        a = dict(plan=plan, q=A2, k_cache=A2, v_cache=A2, l_cap=512, cache_seqlens=None, strides=None,
                 softmax_scale=0.0, world=2, rank=0, peer_bases=A2, slot_bytes=slot, lse_offset=lo,
                 flag_offset=fo, epoch=A2, counter=A2, workspace=A2, workspace_bytes=1 << 20, stream=0)
        a.update(kw)
        with pytest.raises(L.DecAttnError) as e:
            L.da_forward_peer(**a)
        return e.value.status
    assert fwd(counter=None) == L.DA_ERR_INVALID_ARG
    assert fwd(counter=A2 + 2) == L.DA_ERR_ALIGNMENT
    assert fwd(epoch=None) == L.DA_ERR_INVALID_ARG
    assert fwd(rank=2) == L.DA_ERR_INVALID_ARG
    assert fwd(lse_offset=16) == L.DA_ERR_INVALID_ARG            # slot rows follow the plan's B x H_Q
    assert fwd(q=None) == L.DA_ERR_INVALID_ARG
    assert fwd(l_cap=100) == L.DA_ERR_INVALID_ARG
    assert fwd(k_cache=A2 + 8) == L.DA_ERR_ALIGNMENT
    wide = L.da_plan_make(1, 64, 8, 512, 128, 1, 0, 148, "seq_aware", 0)
    assert fwd(plan=wide) == L.DA_ERR_INVALID_ARG                # 64 rows do not fit the 8-row slot


def test_peer_layout():
    from paper_2604_00028_b200.dist import peer_layout
    for B, H, W in ((1, 64, 8), (3, 24, 2), (1, 8, 1), (128, 64, 64)):
        slot, lo, fo, llo, lls, tot = peer_layout(B, H, 128, W)
        assert lo >= B * H * 128 * 4 and lo % 16 == 0
        assert slot >= lo + 4 * B * H and slot % 16 == 0
        assert fo >= 2 * slot and fo % 16 == 0
        assert llo >= fo + 4 * W and llo % 16 == 0 and lls >= 8 * 129 * B * H and lls % 16 == 0
        assert tot >= llo + 2 * lls and tot % 16 == 0


def test_python_shape_checks_before_any_launch(L):
    # the binding refuses tensors that do not match the plan (the C ABI takes bare pointers)
    import torch
    from paper_2604_00028_b200 import api
    plan = L.da_plan_make(2, 16, 2, 300, 128, 1, 0, 148, "seq_aware", 0)
    bf = torch.bfloat16
    q, k, v = torch.zeros(2, 16, 128, dtype=bf), torch.zeros(2, 300, 2, 128, dtype=bf), torch.zeros(2, 300, 2, 128, dtype=bf)
    api._check_shapes(plan, q, k, v, torch.zeros(2, dtype=torch.int32))              # consistent: passes
    api._check_shapes(plan, q, torch.zeros(2, 512, 2, 128, dtype=bf), v)              # L_cap > L_K: fine
    bad = [dict(q=torch.zeros(2, 8, 128, dtype=bf)), dict(k_cache=torch.zeros(2, 299, 2, 128, dtype=bf)),
           dict(v_cache=torch.zeros(2, 300, 1, 128, dtype=bf)), dict(k_cache=torch.zeros(1, 300, 2, 128, dtype=bf)),
           dict(cache_seqlens=torch.zeros(3, dtype=torch.int32)), dict(out=torch.zeros(2, 16, 64, dtype=bf)),
           dict(lse=torch.zeros(16, dtype=torch.float32))]
    for kw in bad:
        a = dict(q=q, k_cache=k, v_cache=v, cache_seqlens=None, out=None, lse=None)
        a.update(kw)
        with pytest.raises(ValueError):
            api.forward_host(plan, a["q"], a["k_cache"], a["v_cache"], a["cache_seqlens"], out=a["out"], lse=a["lse"])


def test_forward_peer_combine_validation(L):
    # da_forward_peer_combine: one-wave NONE / CLUSTER plans only, checked before any CUDA call
    A2 = 1 << 22
    slot, lo, fo = 4128, 4096, 2 * 4128

    def fwd(plan, **kw):
        rows = plan.batch * plan.h_q
        a = dict(plan=plan, q=A2, k_cache=A2, v_cache=A2, l_cap=plan.l_k, cache_seqlens=None, strides=None,
                 softmax_scale=0.0, world=2, rank=0, peer_bases=A2, ll_offset=fo + 16, ll_slot_bytes=8 * 129 * rows + 16,
                 epoch=A2, counter=A2, out_dtype=L.DA_BF16, out=A2, lse=A2, status=A2, timeout_ns=0, workspace=None,
                 workspace_bytes=0, stream=0)
        a.update(kw)
        with pytest.raises(L.DecAttnError) as e:
            L.da_forward_peer_combine(**a)
        return e.value.status
    cluster = L.da_plan_make(1, 8, 1, 1500, 128, 1, 0, 148, "seq_aware", 0)
    assert cluster.combine_mode == L.DA_COMBINE_CLUSTER
    assert fwd(cluster, status=None) == L.DA_ERR_INVALID_ARG
    assert fwd(cluster, status=A2 + 2) == L.DA_ERR_ALIGNMENT
    assert fwd(cluster, out=None) == L.DA_ERR_INVALID_ARG
    assert fwd(cluster, out_dtype=7) == L.DA_ERR_INVALID_ARG
    assert fwd(cluster, counter=None) == L.DA_ERR_INVALID_ARG
    assert fwd(cluster, ll_slot_bytes=8 * 129 * 8 - 16) == L.DA_ERR_INVALID_ARG    # slot shorter than 8 rows
    assert fwd(cluster, ll_offset=fo + 8) == L.DA_ERR_ALIGNMENT
    assert fwd(cluster, world=0) == L.DA_ERR_INVALID_ARG
    assert fwd(cluster, out=A2 + 8) == L.DA_ERR_ALIGNMENT
    assert fwd(cluster, lse=A2 + 2) == L.DA_ERR_ALIGNMENT
    ws = L.da_plan_make(1, 8, 1, 4096, 128, 1, 0, 148, "guarded", 0)          # s = 28: workspace combine
    assert ws.combine_mode == L.DA_COMBINE_KERNEL and fwd(ws) == L.DA_ERR_WORKSPACE   # allowed, needs one
    dyn = L.da_plan_make(4, 16, 2, 3000, 128, 1, 0, 148, "dynamic", 0)
    assert dyn.combine_mode == L.DA_COMBINE_KERNEL and fwd(dyn) == L.DA_ERR_WORKSPACE     # allowed, needs one
    big = L.da_plan_make(64, 8, 1, 300, 128, 1, 0, 148, "guarded", 0)         # 64 CTAs... one wave: allowed
    wide = L.da_plan_make(256, 8, 1, 300, 128, 1, 0, 148, "guarded", 0)       # 256 CTAs > 148 SMs
    assert big.grid_x * big.grid_y * big.grid_z <= 148
    assert fwd(wide) == L.DA_ERR_UNSUPPORTED


def test_query_residency_validation(L):
    import ctypes
    plan = L.da_plan_make(1, 8, 1, 512, 128, 1, 0, 148, "seq_aware", 0)
    n = ctypes.c_int32(0)
    for kernel, exchange in ((2, 0), (-1, 0), (0, 3), (0, -1)):
        assert L.LIB.da_query_residency(ctypes.byref(plan), kernel, exchange, ctypes.byref(n)) == L.DA_ERR_INVALID_ARG
    assert L.LIB.da_query_residency(None, 0, 0, ctypes.byref(n)) == L.DA_ERR_INVALID_ARG
    assert L.LIB.da_query_residency(ctypes.byref(plan), 0, 0, None) == L.DA_ERR_INVALID_ARG
    bad = L.da_plan.from_buffer_copy(plan)
    bad.grid_x += 1                                              # an inconsistent (edited) plan
    assert L.LIB.da_query_residency(ctypes.byref(bad), 0, 0, ctypes.byref(n)) == L.DA_ERR_INVALID_ARG
