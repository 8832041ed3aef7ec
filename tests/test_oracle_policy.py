"""Pins for oracle/policy.py (C-pol) against what the paper (and SPEC's
paper-derived examples) fix.  CPU only."""

import csv
import os
import random
from fractions import Fraction

import pytest

from oracle import policy as P

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
H100_SMS = 132
B200_SMS = 148


def _rows(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return list(csv.DictReader(line for line in f if not line.startswith("#")))


def test_geometry_spec_examples():
    # S:L57-59 tile_geometry examples.
    g = P.geometry(1, 1, 1, 512, H100_SMS, 0)
    assert (g["nblk"], g["T"]) == (4, 1)
    g = P.geometry(1, 8, 8, 128, H100_SMS, 0)
    assert (g["nblk"], g["T"]) == (1, 8)
    g = P.geometry(8, 32, 32, 8192, H100_SMS, 0)
    assert (g["nblk"], g["T"]) == (64, 256)


def test_block_accounting_matches_paper_equivalences():
    # P:L91 "num_n_blocks <= 4 (L_K <= 512)"; "nblk <= 3 (e.g., L_K <= 384)".
    for lk in range(1, 2049):
        nblk = P.geometry(1, 8, 1, lk, H100_SMS, 0)["nblk"]
        assert (nblk <= 4) == (lk <= 512)
        assert (nblk <= 3) == (lk <= 384)
    # L_K >= 640 is where "the baseline efficiency loop already runs" (nblk >= 5).
    assert P.geometry(1, 8, 1, 640, H100_SMS, 0)["nblk"] == 5


def test_total_mblocks_is_batch_times_hkv_for_decode():
    # P:L73 / P:L99-100: "for decode (L_Q = 1), this reduces to batch_size * num_heads_kv".
    for b in (1, 2, 4, 8, 128):
        for hkv in (1, 2, 4, 8, 32):
            for G in (1, 8, 16, 64):
                assert P.geometry(b, hkv * G, hkv, 512, B200_SMS, 0)["T"] == b * hkv


def test_occupancy_eight_tiles_h100():
    # "8 tiles without sequence splitting translates to an occupancy ... of approximately 6%".
    num, den = P.occupancy_fraction(8, H100_SMS)
    assert Fraction(num, den) == Fraction(8, 132)
    assert round(100 * num / den) == 6
    # "leaving over 90% of the GPU SMs idle".
    assert Fraction(den - num, den) > Fraction(9, 10)
    assert P.occupancy_fraction(264, 132) == (132, 132)      # S:L69 saturation cap


def test_table1_decisions():
    # Table 1: speedup 1.00x rows ran identical split counts; the bold rows ran
    # s=1 (standard) vs s=3 (patched).  Batch = 1, H100.
    rows = _rows("table1.csv")
    assert len(rows) == 18
    for r in rows:
        lk, hkv = int(r["l_k"]), int(r["h_kv"])
        sg, _ = P.num_splits(1, 8 * hkv, hkv, lk, H100_SMS, 0, "guarded")
        ss, _ = P.num_splits(1, 8 * hkv, hkv, lk, H100_SMS, 0, "seq_aware")
        if r["speedup"] == "1.00":
            assert sg == ss, r
        else:
            assert (sg, ss) == (1, 3), r
        if lk <= 512:
            assert sg == 1, r          # the guard returns s=1 for L_K <= 512
        # speedup column is standard/patched rounded to 2 decimals ("21 to 24%")
        ratio = float(r["standard_us"]) / float(r["patched_us"])
        assert abs(ratio - float(r["speedup"])) < 0.006


def test_fig3_cascade_cases():
    for r in _rows("fig3_cases.csv"):
        nblk, T = int(r["nblk"]), int(r["T"])
        geo = {"nblk": nblk, "T": T, "U": H100_SMS}
        assert P.guarded_splits(geo)[0] == int(r["guarded"]), r
        assert P.seq_aware_splits(geo)[0] == int(r["seq_aware"]), r


def test_fig3_rules_named():
    geo = lambda nblk, T: {"nblk": nblk, "T": T, "U": B200_SMS}
    assert P.seq_aware_splits(geo(3, 1)) == (1, P.RULE_GUARD1)
    assert P.seq_aware_splits(geo(4, 4)) == (1, P.RULE_GUARD2)
    assert P.seq_aware_splits(geo(4, 3)) == (3, P.RULE_LOW_TILE)
    assert P.seq_aware_splits(geo(5, 1))[1] == P.RULE_EFF_LOOP
    assert P.guarded_splits(geo(4, 1)) == (1, P.RULE_GUARD_NBLK4)
    assert P.guarded_splits(geo(64, 1024)) == (1, P.RULE_SATURATED)


def test_boundary_sweep_section_4_1():
    # "unchanged behavior at L_K in {128, 256, 384}, a clear win at the representative
    # L_K=512 point ..., and unchanged behavior again ... (e.g., L_K >= 640)".  Low-tile shape.
    for sms in (H100_SMS, B200_SMS):
        for lk in list(range(1, 385)) + list(range(640, 9000, 7)):
            a = P.num_splits(1, 8, 1, lk, sms, 0, "guarded")[0]
            b = P.num_splits(1, 8, 1, lk, sms, 0, "seq_aware")[0]
            assert a == b, lk
        assert P.num_splits(1, 8, 1, 512, sms, 0, "seq_aware")[0] == 3


def test_regression_matrix_divergence_set():
    # P:L177-179 (§5.3): 160 configurations; "At L_K=512, wins appear only for H_KV in {1,2}";
    # "(e.g., Batch=8, H_KV=8), the sequence-aware guard defaults back to s=1".
    # divergence set is exactly {nblk = 4 and total_mblocks < 4}.
    for sms in (H100_SMS, B200_SMS):
        diverge = []
        for b in (1, 2, 4, 8):
            for lk in (128, 256, 384, 512, 1024, 2048, 4096, 8192):
                for hkv in (1, 2, 4, 8, 32):
                    a = P.num_splits(b, 8 * hkv, hkv, lk, sms, 0, "guarded")[0]
                    c = P.num_splits(b, 8 * hkv, hkv, lk, sms, 0, "seq_aware")[0]
                    if a != c:
                        diverge.append((b, lk, hkv, a, c))
        assert sorted(diverge) == [(1, 512, 1, 1, 3), (1, 512, 2, 1, 3), (2, 512, 1, 1, 3)]
        assert all(d[2] in (1, 2) for d in diverge if d[0] == 1)
        assert P.num_splits(8, 64, 8, 512, sms, 0, "seq_aware")[0] == 1


def test_unchanged_cases_theorem_random():
    # patched == baseline whenever not (nblk == 4 and T < 4); S:L152 1 <= s <= nblk.
    rng = random.Random(7)
    for _ in range(10000):
        b = rng.randint(1, 64)
        hkv = rng.choice([1, 2, 4, 8, 16, 32])
        G = rng.choice([1, 2, 4, 8, 16])
        lk = rng.randint(1, 40000)
        sms = rng.choice([H100_SMS, B200_SMS, 8, 3])
        margin = rng.randint(0, sms - 1)
        geo = P.geometry(b, hkv * G, hkv, lk, sms, margin)
        a, _ = P.num_splits(b, hkv * G, hkv, lk, sms, margin, "guarded")
        c, _ = P.num_splits(b, hkv * G, hkv, lk, sms, margin, "seq_aware")
        for s in (a, c):
            assert 1 <= s <= geo["nblk"]
        if not (geo["nblk"] == 4 and geo["T"] < 4):
            assert a == c
        elif not P.saturated(geo["T"], geo["U"]):
            assert (a, c) == (1, 3)


def _eff_loop_by_fractions(T, U, nblk):
    # Independent statement of the efficiency loop (C-amb-2) with exact rationals:
    # n_waves = T s / U, efficiency = n_waves / ceil(n_waves), pick the smallest s whose
    # efficiency >= 0.85 * max efficiency, over s = 1 .. min(128, U, nblk).
    smax = min(128, U, nblk)
    effs = []
    for s in range(1, smax + 1):
        n_waves = Fraction(T * s, U)
        ceil_w = -(-n_waves.numerator // n_waves.denominator)
        effs.append(n_waves / ceil_w)
    best = max(effs)
    for s, e in enumerate(effs, start=1):
        if e >= Fraction(85, 100) * best:
            return s
    raise AssertionError


def test_efficiency_loop_matches_rational_definition():
    for U in (1, 2, 3, 7, 100, 132, 148):
        for T in list(range(1, 40)) + [64, 100, 128, 200, 1024]:
            for nblk in list(range(1, 40)) + [64, 100, 128, 129, 1024]:
                assert P.efficiency_loop(T, U, nblk) == _eff_loop_by_fractions(T, U, nblk)


def test_efficiency_loop_single_wave_closed_form():
    # If T * m <= U with m = min(nblk, 128, U), every candidate is one wave, efficiency is
    # proportional to s and the rule gives s = ceil(17 m / 20).
    for U in (132, 148):
        for T in (1, 2, 3, 4, 8):
            for nblk in range(5, 300):
                m = min(nblk, 128, U)
                if T * m <= U:
                    assert P.efficiency_loop(T, U, nblk) == -(-17 * m // 20)


def test_appendix_a_regression_matrix():
    """Independent cross-check of the efficiency-loop reconstruction beyond one wave: SURVEY.md
    Appendix A's hand-computed guarded split counts over the paper's 160-configuration matrix
     at U = 148 and U = 132 (tests/golden/appendix_a_guarded.csv).  Multi-wave rows
    included, e.g. (B=8, H_KV=4, L_K=8192): T = 32 -> s = 4.  The paper never defines the loop
    (P:L85), so this pins the reconstruction against a second derivation, not
    against a printed value; the seq-aware column pins Fig. 3's divergence set."""
    rows = _rows("appendix_a_guarded.csv")
    assert len(rows) == 160
    multi_wave = 0
    for r in rows:
        b, hkv, lk = int(r["batch"]), int(r["h_kv"]), int(r["l_k"])
        for U, col in ((B200_SMS, "guarded_s_u148"), (H100_SMS, "guarded_s_u132")):
            assert P.num_splits(b, 8 * hkv, hkv, lk, U, 0, "guarded")[0] == int(r[col]), (b, hkv, lk, U)
            geo = P.geometry(b, 8 * hkv, hkv, lk, U, 0)
            m = min(geo["nblk"], 128, U)
            if geo["nblk"] >= 5 and not P.saturated(geo["T"], U) and geo["T"] * m > U:
                multi_wave += 1
        assert P.num_splits(b, 8 * hkv, hkv, lk, B200_SMS, 0, "seq_aware")[0] == int(r["seq_aware_s_u148"])
    assert multi_wave >= 40          # the table pins the loop well beyond its single-wave closed form


def test_spec_efficiency_examples():
    # S:L135 nblk=1 -> 1; S:L136 (nblk=64, T=256, 132 SMs) -> 1.
    assert P.efficiency_loop(5, 132, 1) == 1
    assert P.efficiency_loop(256, 132, 64) == 1
    # S:L137 claims 16 for (nblk=16, T=1, 132 SMs) but its own rule gives 14:
    # efficiency(s) = s/132 is linear, 0.85 * 16 = 13.6 -> smallest s is 14.
    assert P.efficiency_loop(1, 132, 16) == 14


def test_fixed_policy_and_validation():
    assert P.num_splits(1, 8, 1, 512, B200_SMS, 0, "fixed", 64) == (64, P.RULE_FORCED)
    with pytest.raises(ValueError):
        P.num_splits(1, 8, 1, 512, B200_SMS, 0, "fixed", 0)
    with pytest.raises(ValueError):
        P.num_splits(1, 8, 1, 512, B200_SMS, 0, "fixed", 257)
    with pytest.raises(ValueError):
        P.geometry(1, 6, 4, 512, B200_SMS, 0)          # h_q not a multiple of h_kv
    with pytest.raises(ValueError):
        P.geometry(1, 8, 1, 512, B200_SMS, B200_SMS)   # sm_margin >= num_sms


def test_sm_count_only_matters_in_efficiency_region():
    # The Fig. 3 region (nblk <= 4) decisions do not depend on the SM count (C-amb-18).
    for b in (1, 2, 4, 8):
        for hkv in (1, 2, 4, 8, 32):
            for lk in range(1, 513, 17):
                got = {P.num_splits(b, 8 * hkv, hkv, lk, sms, 0, "seq_aware")[0]
                       for sms in (132, 148, 1000)}
                assert len(got) == 1


def test_evolved_fragment():
    # Fig. 1.
    assert P.evolved_splits(1, 448) == (12, True, 0)
    assert P.evolved_splits(1, 128) == (16, True, 0)
    assert P.evolved_splits(2, 512) is None


# ---- policies beyond the paper's pair ---------------------------
def test_evolved_policy_literal_fig1():
    # batch == 1 -> 12, L_K < 256 -> 16; no clamp (s > nblk allowed).
    assert P.num_splits(1, 64, 8, 512, B200_SMS, 0, "evolved") == (12, P.RULE_EVOLVED)
    assert P.num_splits(1, 8, 1, 128, B200_SMS, 0, "evolved") == (16, P.RULE_EVOLVED)
    assert P.num_splits(1, 8, 1, 255, B200_SMS, 0, "evolved")[0] == 16
    assert P.num_splits(1, 8, 1, 256, B200_SMS, 0, "evolved")[0] == 12
    # batch != 1: the fragment is silent -> guarded default
    for lk in (128, 512, 4096):
        assert P.num_splits(2, 8, 1, lk, B200_SMS, 0, "evolved") == P.num_splits(2, 8, 1, lk, B200_SMS, 0, "guarded")


def test_cluster_fit_splits():
    # one wave never holds more CTAs than usable SMs (one CTA per SM in CLUSTER mode): T f <= U
    for U in (3, 16, 132, 148):
        prev = 16
        for T in range(1, 2 * U):
            f = P.cluster_fit_splits(T, U)
            assert 1 <= f <= prev                       # non-increasing in T
            assert f == 1 or T * f <= U
            prev = f
    # the B200 table (cudaOccupancyMaxActiveClusters): 7 clusters of 16, 8 of 10, 16 of 6, 33 of 4
    assert [P.cluster_fit_splits(T, 148) for T in (1, 7, 8, 11, 12, 16, 33, 34, 74, 75)] == \
        [16, 16, 10, 10, 9, 6, 4, 3, 2, 1]


def test_seq_aware_sm_structure():
    rng = random.Random(5)
    for _ in range(20000):
        b = rng.randint(1, 64)
        hkv = rng.choice([1, 2, 4, 8, 16, 32])
        lk = rng.randint(1, 140000)
        sms = rng.choice([132, 148, 16, 3])
        geo = P.geometry(b, 8 * hkv, hkv, lk, sms, 0)
        s, rule = P.num_splits(b, 8 * hkv, hkv, lk, sms, 0, "seq_aware_sm")
        g, grule = P.num_splits(b, 8 * hkv, hkv, lk, sms, 0, "guarded")
        n_u = -(-lk // 64)
        f = P.cluster_fit_splits(geo["T"], geo["U"])
        assert 1 <= s <= n_u                              # never an empty 64-token split
        if P.saturated(geo["T"], geo["U"]):
            assert (s, rule) == (g, grule)                # saturation guard unchanged
        elif geo["nblk"] <= 4:
            assert s == 1 or (s <= f and s <= 8)          # one wave of clusters
            if lk <= 256:
                assert s == 1                              # too few 64-token units to split
            assert s == 1 or s >= 3                        # a 2-way split does not pay
        else:
            e = P.efficiency_loop(geo["T"], geo["U"], geo["nblk"])
            assert (s == e) == (rule == P.RULE_EFF_LOOP)
            assert s == e or s <= f                       # deviates from the loop only to one wave
    # the calibrated points on B200
    assert P.num_splits(1, 8, 1, 512, B200_SMS, 0, "seq_aware_sm") == (8, P.RULE_SM_SPLIT)
    assert P.num_splits(1, 64, 8, 512, B200_SMS, 0, "seq_aware_sm") == (4, P.RULE_SM_SPLIT)
    assert P.num_splits(2, 128, 16, 512, B200_SMS, 0, "seq_aware_sm") == (4, P.RULE_SM_SPLIT)
    assert P.num_splits(1, 8, 1, 384, B200_SMS, 0, "seq_aware_sm")[0] == 6
    assert P.num_splits(1, 8, 1, 256, B200_SMS, 0, "seq_aware_sm") == (1, P.RULE_SM_SHORT)
    assert P.num_splits(1, 8, 1, 320, B200_SMS, 0, "seq_aware_sm") == (5, P.RULE_SM_SPLIT)
    assert P.num_splits(1, 8, 1, 192, B200_SMS, 0, "seq_aware_sm") == (1, P.RULE_SM_SHORT)
    assert P.num_splits(4, 64, 8, 256, B200_SMS, 0, "seq_aware_sm") == (1, P.RULE_SM_SHORT)
    # the SM count enters through f: T = 32 tiles on 148 SMs -> clusters of 4 fit; T = 64 -> only
    # clusters of 2 fit, which do not pay; T = 120 -> saturated
    assert P.num_splits(4, 64, 8, 512, B200_SMS, 0, "seq_aware_sm")[0] == 4
    assert P.num_splits(8, 64, 8, 512, B200_SMS, 0, "seq_aware_sm")[0] == 1
    assert P.num_splits(10, 64, 8, 512, B200_SMS, 0, "seq_aware_sm")[0] == 1
    assert P.num_splits(15, 64, 8, 512, B200_SMS, 0, "seq_aware_sm")[1] == P.RULE_SATURATED
    # efficiency region: the loop's workspace-combine split is moved to the one-wave cluster split
    assert P.num_splits(1, 64, 8, 2048, B200_SMS, 0, "seq_aware_sm") == (10, P.RULE_SM_FIT)
    assert P.num_splits(1, 64, 8, 131072, B200_SMS, 0, "seq_aware_sm") == (10, P.RULE_SM_FIT)
    assert P.num_splits(1, 8, 1, 4096, B200_SMS, 0, "seq_aware_sm") == (12, P.RULE_SM_FIT)   # cap 12
    # ... except for a long sequence with too few tiles to stream at HBM rate in one wave
    assert P.num_splits(1, 8, 1, 131072, B200_SMS, 0, "seq_aware_sm") == \
        P.num_splits(1, 8, 1, 131072, B200_SMS, 0, "guarded")
    # where the paper's rule splits (nblk = 4, T < 4) the generalisation splits too
    for hkv in (1, 2):
        assert P.num_splits(1, 8 * hkv, hkv, 512, B200_SMS, 0, "seq_aware_sm")[0] >= 3


def test_seq_aware_sm_wide_group_clause():
    # C-ext-1's wide-group clause (round 2): where the one-wave cluster fit leaves a <= 2-CTA split
    # for G >= 32, the efficiency loop's split runs on the tcgen05 kernel instead - the two
    # measured wins of profiles/r02zz4_wide_group_policy.log ...
    e = lambda b, hq, hkv, lk: P.efficiency_loop(P.geometry(b, hq, hkv, lk, B200_SMS, 0)["T"], B200_SMS,
                                                  P.geometry(b, hq, hkv, lk, B200_SMS, 0)["nblk"])
    assert P.num_splits(8, 64, 1, 4096, B200_SMS, 0, "seq_aware_sm") == (e(8, 64, 1, 4096), P.RULE_EFF_LOOP) == (16, 5)
    assert P.num_splits(16, 32, 1, 4096, B200_SMS, 0, "seq_aware_sm") == (8, P.RULE_EFF_LOOP)
    # ... and the shapes where the measured 2- / 4-split mma.sync plans stayed ahead keep them
    assert P.num_splits(16, 32, 1, 2048, B200_SMS, 0, "seq_aware_sm") == (2, P.RULE_SM_FIT)   # 32 units
    assert P.num_splits(8, 32, 1, 4096, B200_SMS, 0, "seq_aware_sm") == (4, P.RULE_SM_FIT)    # fit 4
    # the same loss for 16 < G < 32 (profiles/r02zz33_g17_31_policy.log: B16 L4096 s = 2 mma.sync
    # 13.6 us against the loop's s = 8 on tcgen05 11.0 us) ...
    assert P.num_splits(16, 24, 1, 4096, B200_SMS, 0, "seq_aware_sm") == (8, P.RULE_EFF_LOOP)
    assert P.num_splits(16, 20, 1, 4096, B200_SMS, 0, "seq_aware_sm") == (8, P.RULE_EFF_LOOP)
    # ... never for G <= 16 (one 16-row mma.sync CTA per KV head: the tcgen05 kernel is not used)
    assert P.num_splits(16, 16, 1, 4096, B200_SMS, 0, "seq_aware_sm") == (4, P.RULE_SM_FIT)
    # nor below 64 units (B8 G64 L2048 keeps s = 2), nor where the fit is > 2 (B4 G64 L4096: 4)
    assert P.num_splits(8, 64, 1, 2048, B200_SMS, 0, "seq_aware_sm") == (2, P.RULE_SM_FIT)
    assert P.num_splits(4, 64, 1, 4096, B200_SMS, 0, "seq_aware_sm") == (4, P.RULE_SM_FIT)


def _measured_grid(tag="r01h"):
    import csv
    import os
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
    grid = {}
    for name in (f"{tag}_ugrid.csv", f"{tag}_ugrid2.csv", f"{tag}_ugrid3.csv"):
        with open(os.path.join(root, name)) as fh:
            for r in csv.DictReader(fh):
                key = (int(r.get("batch", 1)), int(r["h_kv"]), int(r["l_k"]))
                grid.setdefault(key, {})[int(r["s"])] = float(r["latency_us"])
    return grid


@pytest.mark.parametrize("tag,bound", [("r01i", 1.02), ("r02a", 1.01)])
def test_seq_aware_sm_calibration_lowhead(tag, bound):
    """The 48 shapes of BASELINE configs[2] (profiles/<tag>_lowhead.csv: guarded, the paper's rule and
    the SM-count-aware pick, interleaved): every current pick was measured and is never more than
    1 % behind guarded - the paper's no-regression bar (>= 0.99x) - on the round-2 harness
    (r02a: identical plans share one graph, random arm order, host submission outside the timed
    region), 2 % on the round-1 harness (r01i, whose same-plan noise was ~2-4 %); at L_K = 512 it
    beats guarded by >= 1.2x for every T <= 32."""
    import csv
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        f"{tag}_lowhead.csv")
    meas = {}
    with open(path) as fh:
        for r in csv.DictReader(fh):
            meas.setdefault((int(r["batch"]), int(r["h_kv"]), int(r["l_k"])), {})[int(r["num_splits"])] = \
                float(r["latency_us"])
    assert len(meas) == 48
    for (b, hkv, lk), t in meas.items():
        s, _ = P.num_splits(b, 8 * hkv, hkv, lk, B200_SMS, 0, "seq_aware_sm")
        g, _ = P.num_splits(b, 8 * hkv, hkv, lk, B200_SMS, 0, "guarded")
        assert s in t and g in t, (b, hkv, lk, s)
        assert t[s] <= bound * t[g], (b, hkv, lk, s, g)
        if lk == 512 and b * hkv <= 32:
            assert t[g] / t[s] >= 1.2, (b, hkv, lk, s)


@pytest.mark.parametrize("tag,bound", [("r01h", 1.02), ("r01j", 1.02), ("r02a", 1.01)])
def test_seq_aware_sm_calibration(tag, bound):
    """C-ext-1's constants against the B200 measurements they were calibrated on
    (profiles/r01h_ugrid*.csv, forced-s latencies, G = 8), against the same grids re-measured
    on the final round-1 kernel (r01j) and on the round-2 harness (r02a): the pick is within 6 % of
    the best measured split (an unmeasured pick lies between two measured neighbours) and never
    slower than the guarded pick by more than the paper's no-regression bar, 1 % (>= 0.99x,
    P:L179), on the r02a grids; 2 % on the round-1 grids, whose harness noise was ~2-4 %."""
    grid = _measured_grid(tag)
    assert len(grid) >= 60
    for (b, hkv, lk), t in grid.items():
        s, _ = P.num_splits(b, 8 * hkv, hkv, lk, B200_SMS, 0, "seq_aware_sm")
        g, _ = P.num_splits(b, 8 * hkv, hkv, lk, B200_SMS, 0, "guarded")
        if s not in t:
            lo, hi = max(x for x in t if x < s), min(x for x in t if x > s)
            ts = max(t[lo], t[hi])
        else:
            ts = t[s]
        assert ts <= 1.06 * min(t.values()), (b, hkv, lk, s)
        if g in t:
            assert ts <= bound * t[g], (b, hkv, lk, s, g)


# ---- per-batch dynamic split counts (C-ext-2) -----------------------------------
def test_dynamic_schedule_examples():
    # hand-computed: one 32768-token sequence among fifteen 1024-token ones, 8 tiles per sequence:
    # units 512 + 15 x 16 = 752; W = ceil(752 * 8 / 148) = ceil(40.6) = 41; 512 // 41 = 12; 16 // 41 = 0 -> 1
    W, s, P_ = P.dynamic_schedule([32768] + [1024] * 15, 8, 148, 128)
    assert (W, s[0], s[1:]) == (41, 12, [1] * 15)
    assert P_[:3] == [0, 12, 13] and P_[-1] == 26
    # a single long sequence stays inside one wave: W = ceil(2048 * 8 / 148) = 111, 2048 // 111 = 18
    assert P.dynamic_schedule([131072], 8, 148, 128) == (111, [18], [0])          # 144 CTAs <= 148
    # T = 1: W = ceil(2048 / 148) = 14, 2048 // 14 = 146 -> the cap 128
    assert P.dynamic_schedule([131072], 1, 148, 128) == (14, [128], [0])
    # empty and one-token sequences still own one split (o = 0 / the single key)
    assert P.dynamic_schedule([0, 1, 64, 65], 1, 148, 2) == (1, [1, 1, 1, 2], [0, 1, 2, 3])
    assert P.num_splits(3, 24, 3, 700, B200_SMS, 0, "dynamic") == (11, P.RULE_DYNAMIC)   # cap ceil(700/64)


def test_dynamic_schedule_invariants():
    rng = random.Random(11)
    for _ in range(3000):
        B = rng.randint(1, 70)
        U = rng.choice([148, 132, 16, 3])
        tiles = rng.choice([1, 2, 8, 32])
        l_cap = rng.choice([64, 500, 4096, 131072])
        cap = P.dynamic_cap(l_cap)
        lens = [rng.choice([0, 1, rng.randint(0, l_cap), l_cap]) for _ in range(B)]
        W, s, P_ = P.dynamic_schedule(lens, tiles, U, cap)
        units = [-(-n // 64) for n in lens]
        assert W == max(1, -(-sum(units) * tiles // U))
        assert P_ == [sum(s[:b]) for b in range(B)]
        assert sum(s) <= P.dynamic_slots(B, tiles, U, cap)          # the launch always has the slots
        lifted = sum(1 for u in units if u < W)
        assert sum(s) * tiles <= U + lifted * tiles                   # one wave, except lifted short ones
        for u, v in zip(units, s):
            assert 1 <= v <= cap
            if v < cap and u >= W:
                assert u < (v + 1) * W                               # each split holds < 2 W units
                assert v * W <= u


# ---- the host-side plan for ragged batches (C-ext-3) --------------------------------------------
def test_varlen_policy_uniform_batches_stay_static():
    # uniform lengths: the static SM-count-aware plan is already balanced; never the dynamic path
    for B in (1, 2, 3, 4, 8, 16, 32, 64, 128):
        for hkv in (1, 2, 4, 8, 16, 32):
            for L in (1, 64, 65, 128, 300, 512, 513, 1000, 2048, 4096, 8192, 16384, 32768, 131072):
                for sms in (148, 132):
                    assert P.varlen_policy(B, 8 * hkv, hkv, L, sms, 0, [L] * B) == P.SEQ_AWARE_SM


def test_varlen_policy_cases():
    # hand-computed on B200 (U = 148):
    # one 32768-token sequence among fifteen of 1024, 8 tiles each: static s = 1 (T = 128 saturated),
    # c = 512 units; W = 41 (test_dynamic_schedule_examples) -> 512 > 82 and >= 32: dynamic
    assert P.varlen_policy(16, 64, 8, 32768, 148, 0, [32768] + [1024] * 15) == P.DYNAMIC
    # one 16384 among 63 of 512, 1 tile each: T = 64 -> static s = 2 (f = 2), c = 128; units
    # 256 + 63 x 8 = 760 -> W = ceil(760 / 148) = 6 -> 128 > 12: dynamic
    assert P.varlen_policy(64, 8, 1, 16384, 148, 0, [16384] + [512] * 63) == P.DYNAMIC
    # a long tail that is not long enough: 14794 among 127 of 1500 (T = 1024, static s = 1):
    # c = 232; units 232 + 127 x 24 = 3280 -> W = ceil(3280 * 8 / 148) = 178 -> 232 < 356: static
    assert P.varlen_policy(128, 64, 8, 16384, 148, 0, [14794] + [1500] * 127) == P.SEQ_AWARE_SM
    # skewed but short: the longest split would hold < 32 units (latency-bound): static
    assert P.varlen_policy(8, 8, 1, 1024, 148, 0, [1024] + [64] * 7) == P.SEQ_AWARE_SM
    # lengths are clamped to the capacity and empty batches are fine
    assert P.varlen_policy(4, 64, 8, 4096, 148, 0, [0, 0, 0, 0]) == P.SEQ_AWARE_SM


def test_rows_per_cta_and_wide_groups():
    # 8-row CTAs for G <= 8 and for short sequences; 16 for G > 8 beyond 64 units
    assert [P.rows_per_cta(G, L) for G, L in ((8, 10 ** 6), (16, 4096), (16, 4097), (64, 64), (32, 65536))] == \
        [8, 8, 16, 8, 16]
    # G = 16, short: the kernel launches 2 x 8 CTA groups per split -> T_k = 16 -> clusters of 6 fit,
    # and T_k > 8 caps the split at 4
    assert P.num_splits(1, 128, 8, 2048, B200_SMS, 0, "seq_aware_sm") == (4, P.RULE_SM_FIT)
    assert P.num_splits(1, 16, 1, 512, B200_SMS, 0, "seq_aware_sm") == (8, P.RULE_SM_SPLIT)
    # G = 16, long: 16-row CTAs stream better through the workspace split than a one-wave cluster
    # split, so the loop's choice stands (= guarded)
    assert P.num_splits(1, 128, 8, 65536, B200_SMS, 0, "seq_aware_sm") == \
        P.num_splits(1, 128, 8, 65536, B200_SMS, 0, "guarded")
    # launch: 8-row CTAs for G > 8 only while the whole grid is one wave
    assert P.launch_rows(1, 16, 8, 2048, 4, 148) == 8          # 8 x 2 x 4 = 64 CTAs
    assert P.launch_rows(1, 16, 8, 2048, 14, 148) == 16        # 224 CTAs: two waves
    assert P.launch_rows(64, 16, 8, 512, 1, 148) == 16
    assert P.launch_rows(1, 16, 8, 4097, 1, 148) == 16         # long: never 8
    assert all(P.launch_rows(b, 8, 8, 100, s, 148) == 8 for b in (1, 1000) for s in (1, 16))
    # the policy's own picks are one-wave grids: it launches the CTAs it planned for
    rng = random.Random(4)
    for _ in range(3000):
        b, hkv, G, lk = rng.randint(1, 16), rng.choice([1, 2, 4, 8]), rng.choice([12, 16, 32, 64]), rng.randint(1, 4096)
        s, rule = P.num_splits(b, G * hkv, hkv, lk, 148, 0, "seq_aware_sm")
        if rule in (P.RULE_SM_SPLIT, P.RULE_SM_FIT):
            assert P.launch_rows(b, G, hkv, lk, s, 148) == 8, (b, hkv, G, lk, s)
    # G <= 8: the CTA groups are the policy's tiles, the rule is unchanged
    rng = random.Random(3)
    for _ in range(2000):
        b, hkv, G, lk = rng.randint(1, 64), rng.choice([1, 2, 4, 8]), rng.choice([1, 2, 4, 8]), rng.randint(1, 9000)
        geo = P.geometry(b, G * hkv, hkv, lk, 148, 0)
        assert geo["T"] // geo["num_m_blocks"] * -(-G // P.rows_per_cta(G, lk)) == geo["T"]
