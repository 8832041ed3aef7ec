"""Pins for oracle/attention.py (C-att, C-part, C-comb) against closed forms,
invariants, library routines (scipy) and brute force.  CPU only."""

import math
import random

import numpy as np
import pytest
import scipy.special

from oracle import attention as A


def _rand(shape, rng, scale=1.0):
    return rng.standard_normal(shape) * scale


def _case(rng, B=2, HQ=4, HKV=2, L=9, d=8, seqlens=None):
    q = _rand((B, HQ, d), rng)
    k = _rand((B, L, HKV, d), rng)
    v = _rand((B, L, HKV, d), rng)
    if seqlens is None:
        seqlens = [L] * B
    return q, k, v, np.array(seqlens)


def test_single_key_returns_its_value():
    # n = 1: softmax over one key is 1, so out = v_0 and lse = scale * q . k_0.
    rng = np.random.default_rng(0)
    q, k, v, _ = _case(rng, L=5)
    out, lse = A.decode_attention(q, k, v, [1, 1], scale=0.3)
    G = 2
    for b in range(2):
        for h in range(4):
            assert np.array_equal(out[b, h], v[b, 0, h // G])
            assert lse[b, h] == pytest.approx(0.3 * float(np.dot(q[b, h], k[b, 0, h // G])), abs=1e-12)


def test_identical_keys_return_mean_of_values():
    # All keys equal: every score equals c, softmax is uniform: out = mean_j v_j, lse = c + ln n.
    rng = np.random.default_rng(1)
    q, k, v, _ = _case(rng, L=7)
    k[:] = k[:, :1]
    out, lse = A.decode_attention(q, k, v, [7, 4])
    sc = 1 / math.sqrt(8)
    for b, n in ((0, 7), (1, 4)):
        for h in range(4):
            g = h // 2
            np.testing.assert_allclose(out[b, h], v[b, :n, g].mean(axis=0), rtol=0, atol=1e-13)
            c = sc * float(np.dot(q[b, h], k[b, 0, g]))
            assert lse[b, h] == pytest.approx(c + math.log(n), abs=1e-12)


def test_matches_scipy_softmax_and_logsumexp():
    # Library routines: out = softmax(s) @ V and lse = logsumexp(s), row by row.
    rng = np.random.default_rng(2)
    q, k, v, seq = _case(rng, B=3, HQ=6, HKV=3, L=33, d=16, seqlens=[33, 20, 1])
    out, lse = A.decode_attention(q, k, v, seq, scale=0.7)
    for b in range(3):
        n = seq[b]
        for h in range(6):
            g = h // 2
            s = 0.7 * (k[b, :n, g] @ q[b, h])
            np.testing.assert_allclose(out[b, h], scipy.special.softmax(s) @ v[b, :n, g],
                                       rtol=1e-12, atol=1e-13)
            assert lse[b, h] == pytest.approx(scipy.special.logsumexp(s), abs=1e-12)


def test_brute_force_pure_python_tiny():
    # Pure-Python loops with math.exp / math.fsum on tiny inputs (B <= 2, L <= 8, d <= 8).
    rnd = random.Random(3)
    B, HQ, HKV, L, d = 2, 4, 2, 6, 5
    q = [[[rnd.uniform(-2, 2) for _ in range(d)] for _ in range(HQ)] for _ in range(B)]
    k = [[[[rnd.uniform(-2, 2) for _ in range(d)] for _ in range(HKV)] for _ in range(L)] for _ in range(B)]
    v = [[[[rnd.uniform(-2, 2) for _ in range(d)] for _ in range(HKV)] for _ in range(L)] for _ in range(B)]
    seq = [6, 3]
    out, lse = A.decode_attention(np.array(q), np.array(k), np.array(v), seq, scale=0.45)
    for b in range(B):
        for h in range(HQ):
            g = h * HKV // HQ
            w = [math.exp(0.45 * math.fsum(q[b][h][c] * k[b][j][g][c] for c in range(d)))
                 for j in range(seq[b])]
            z = math.fsum(w)
            for c in range(d):
                ref = math.fsum(w[j] * v[b][j][g][c] for j in range(seq[b])) / z
                assert out[b, h, c] == pytest.approx(ref, rel=1e-12, abs=1e-13)
            assert lse[b, h] == pytest.approx(math.log(z), abs=1e-12)


def test_permutation_invariance():
    rng = np.random.default_rng(4)
    q, k, v, seq = _case(rng, L=12)
    perm = rng.permutation(12)
    o1, l1 = A.decode_attention(q, k, v, seq)
    o2, l2 = A.decode_attention(q, k[:, perm], v[:, perm], seq)
    np.testing.assert_allclose(o1, o2, atol=1e-13)
    np.testing.assert_allclose(l1, l2, atol=1e-13)


def test_gqa_equals_mha_with_replicated_kv():
    # Pins the head mapping g = floor(h / G) (C-amb-11): H_Q=8, H_KV=2 (G=4) must equal
    # MHA over KV heads replicated as k_mha[..., h, :] = k[..., h // 4, :].
    rng = np.random.default_rng(5)
    q, k, v, seq = _case(rng, HQ=8, HKV=2, L=10)
    idx = np.arange(8) // 4
    o1, l1 = A.decode_attention(q, k, v, seq)
    o2, l2 = A.decode_attention(q, k[:, :, idx], v[:, :, idx], seq)
    np.testing.assert_allclose(o1, o2, atol=1e-13)
    np.testing.assert_allclose(l1, l2, atol=1e-13)
    # and a different grouping (h mod H_KV) gives a different answer on this input
    o3, _ = A.decode_attention(q, k[:, :, np.arange(8) % 2], v[:, :, np.arange(8) % 2], seq)
    assert not np.allclose(o1, o3)


def test_score_shift_moves_lse_only():
    # Appending a constant component c to q and 1 to every key shifts each score by scale*c:
    # out is unchanged and lse moves by exactly scale*c.
    rng = np.random.default_rng(6)
    q, k, v, seq = _case(rng, L=11, seqlens=[11, 5])
    c, sc = 3.25, 0.5
    q2 = np.concatenate([q, np.full(q.shape[:2] + (1,), c)], axis=-1)
    k2 = np.concatenate([k, np.ones(k.shape[:3] + (1,))], axis=-1)
    v2 = np.concatenate([v, np.zeros(v.shape[:3] + (1,))], axis=-1)
    o1, l1 = A.decode_attention(q, k, v, seq, scale=sc)
    o2, l2 = A.decode_attention(q2, k2, v2, seq, scale=sc)
    np.testing.assert_allclose(o2[..., :-1], o1, atol=1e-13)
    np.testing.assert_allclose(l2, l1 + sc * c, atol=1e-12)


def test_zero_query_is_uniform_average():
    rng = np.random.default_rng(7)
    q, k, v, seq = _case(rng, L=9, seqlens=[9, 2])
    q[:] = 0
    out, lse = A.decode_attention(q, k, v, seq)
    for b, n in ((0, 9), (1, 2)):
        for h in range(4):
            np.testing.assert_allclose(out[b, h], v[b, :n, h // 2].mean(0), atol=1e-13)
            assert lse[b, h] == pytest.approx(math.log(n), abs=1e-13)


def test_value_linearity():
    rng = np.random.default_rng(8)
    q, k, v, seq = _case(rng, L=9)
    o1, _ = A.decode_attention(q, k, v, seq)
    o2, _ = A.decode_attention(q, k, 3.0 * v + 1.0, seq)
    np.testing.assert_allclose(o2, 3.0 * o1 + 1.0, atol=1e-12)


def test_empty_sequence():
    rng = np.random.default_rng(9)
    q, k, v, _ = _case(rng, L=4)
    out, lse = A.decode_attention(q, k, v, [0, 4])
    assert (out[0] == 0).all() and np.isneginf(lse[0]).all()
    assert np.isfinite(lse[1]).all()


def test_default_scale_is_inverse_sqrt_d():
    rng = np.random.default_rng(10)
    q, k, v, seq = _case(rng, d=16)
    o1, l1 = A.decode_attention(q, k, v, seq)
    o2, l2 = A.decode_attention(q, k, v, seq, scale=0.25)
    np.testing.assert_array_equal(o1, o2)
    np.testing.assert_array_equal(l1, l2)


@pytest.mark.parametrize("num_splits", [1, 2, 3, 5, 16])
def test_any_partition_plus_combine_equals_unsplit(num_splits):
    rng = np.random.default_rng(11 + num_splits)
    q, k, v, seq = _case(rng, B=3, HQ=8, HKV=1, L=40, d=8, seqlens=[40, 17, 3])
    ref_o, ref_l = A.decode_attention(q, k, v, seq)
    # balanced partition with unit 4 and a random partition with empty pieces
    for ranges in ([A.partition(int(n), num_splits, 4) for n in seq],
                   [_random_ranges(int(n), num_splits, rng) for n in seq]):
        o, l = A.split_partials(q, k, v, seq, ranges)
        out, lse = A.lse_combine(o, l)
        np.testing.assert_allclose(out, ref_o, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(lse, ref_l, rtol=1e-12, atol=1e-13)
        # combine is invariant to the order of the splits
        perm = rng.permutation(num_splits)
        out2, lse2 = A.lse_combine(o[perm], l[perm])
        np.testing.assert_allclose(out2, out, atol=1e-13)
        np.testing.assert_allclose(lse2, lse, atol=1e-13)


def _random_ranges(n, s, rng):
    cuts = sorted(rng.integers(0, n + 1, size=s - 1).tolist())
    bounds = [0] + cuts + [n]
    return [(bounds[i], bounds[i + 1]) for i in range(s)]


def test_combine_closed_forms():
    # s = 1 is the identity; two splits follow logaddexp; empty splits are ignored.
    rng = np.random.default_rng(12)
    o = rng.standard_normal((1, 5, 4))
    l = rng.standard_normal((1, 5))
    out, lse = A.lse_combine(o, l)
    np.testing.assert_allclose(out, o[0], atol=1e-15)
    np.testing.assert_allclose(lse, l[0], atol=1e-15)
    o = rng.standard_normal((2, 5, 4))
    l = rng.standard_normal((2, 5)) * 4
    out, lse = A.lse_combine(o, l)
    np.testing.assert_allclose(lse, np.logaddexp(l[0], l[1]), atol=1e-13)
    w0 = 1 / (1 + np.exp(l[1] - l[0]))
    np.testing.assert_allclose(out, w0[:, None] * o[0] + (1 - w0)[:, None] * o[1], atol=1e-13)
    o3 = np.concatenate([o, np.zeros((1, 5, 4))])
    l3 = np.concatenate([l, np.full((1, 5), -np.inf)])
    out3, lse3 = A.lse_combine(o3, l3)
    np.testing.assert_allclose(out3, out, atol=1e-15)
    np.testing.assert_allclose(lse3, lse, atol=1e-15)
    out4, lse4 = A.lse_combine(np.zeros((3, 2, 4)), np.full((3, 2), -np.inf))
    assert (out4 == 0).all() and np.isneginf(lse4).all()


def test_partition_properties():
    for n in list(range(0, 300)) + [511, 512, 513, 131072]:
        for s in (1, 2, 3, 4, 5, 7, 16, 64, 256):
            r = A.partition(n, s, 64)
            assert len(r) == s and r[0][0] == 0 and r[-1][1] == n
            for (a0, a1), (b0, _) in zip(r, r[1:]):
                assert a1 == b0                        # contiguous cover of [0, n)
            sizes = [b - a for a, b in r]
            n_u = -(-n // 64)
            units = [-(-sz // 64) for sz in sizes]
            assert max(units) - min(units) <= 1        # balanced to one unit
            assert (min(sizes) == 0) == (s > n_u or n == 0)
            for a, _ in r:
                assert a % 64 == 0                     # splits start on unit boundaries
    # the paper's low-tile case: L_K = 512, s = 3 -> 2, 3, 3 units of 64 tokens
    assert A.partition(512, 3, 64) == [(0, 128), (128, 320), (320, 512)]


def test_bf16_round():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, -2.5, 0.0, 1e-40])
    r = A.bf16_round(x)
    assert r[0] == 1.0
    assert r[1] == 1.0                      # tie -> even
    assert r[2] == 1.0 + 2 ** -7            # above the tie -> up
    assert r[3] == -2.5 and r[4] == 0.0


def test_paged_identity_table_equals_dense():
    # pages laid out in sequence order (page j of sequence b = b * P + j) reproduce the dense cache
    rng = np.random.default_rng(20)
    B, HQ, HKV, d, ps, P = 2, 4, 2, 8, 4, 3
    q = rng.standard_normal((B, HQ, d))
    k = rng.standard_normal((B, P * ps, HKV, d))
    v = rng.standard_normal((B, P * ps, HKV, d))
    pages_k = k.reshape(B * P, ps, HKV, d)
    pages_v = v.reshape(B * P, ps, HKV, d)
    table = [[b * P + j for j in range(P)] for b in range(B)]
    seq = [P * ps, 7]
    o1, l1 = A.decode_attention(q, k, v, seq)
    o2, l2 = A.decode_attention_paged(q, pages_k, pages_v, table, seq, ps)
    np.testing.assert_array_equal(o1, o2)
    np.testing.assert_array_equal(l1, l2)


def test_paged_permuted_pool_is_invariant():
    # shuffling the physical pages (and the table with them) changes nothing; a wrong table does
    rng = np.random.default_rng(21)
    B, HQ, HKV, d, ps, P = 2, 4, 1, 8, 4, 3
    q = rng.standard_normal((B, HQ, d))
    pages_k = rng.standard_normal((B * P + 2, ps, HKV, d))
    pages_v = rng.standard_normal((B * P + 2, ps, HKV, d))
    table = [[b * P + j for j in range(P)] for b in range(B)]
    perm = rng.permutation(len(pages_k))
    inv = np.argsort(perm)
    table2 = [[int(inv[x]) for x in row] for row in table]
    seq = [12, 9]
    o1, l1 = A.decode_attention_paged(q, pages_k, pages_v, table, seq, ps)
    o2, l2 = A.decode_attention_paged(q, pages_k[perm], pages_v[perm], table2, seq, ps)
    np.testing.assert_allclose(o1, o2, atol=1e-13)
    np.testing.assert_allclose(l1, l2, atol=1e-13)
    o3, _ = A.decode_attention_paged(q, pages_k, pages_v, [row[::-1] for row in table], seq, ps)
    assert not np.allclose(o1, o3)


def test_gather_pages_token_mapping():
    pages = np.arange(5 * 2).reshape(5, 2, 1, 1).astype(float)   # page p, slot i -> value 2p + i
    g = A.gather_pages(pages, [[3, 0, 4]], [5], 2)
    assert g[0, :5, 0, 0].tolist() == [6, 7, 0, 1, 8]
