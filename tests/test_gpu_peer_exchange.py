"""The cross-GPU exchange over peer memory (da_peer_signal / da_combine_peers through
dist.PeerSeqShardedDecode) on the one GPU available: a one-rank NCCL group and torch symmetric
memory exercise the full path (symmetric buffer, device pointer table, epoch flags with system-scope
release / acquire, the pull-combine) against the oracle, eagerly and replayed from a CUDA graph.
Several ranks need several GPUs; the multi-rank host logic is covered on CPU (test_dist_gloo.py)."""

import os
import socket

import pytest
import torch

import synth
from oracle import attention as OA
from tests.helpers import assert_lse_close, assert_out_close

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def one_rank_group():
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("batch,h_q,h_kv,l_k", [(1, 64, 8, 4096), (2, 8, 1, 1500)])
def test_peer_exchange_matches_oracle(one_rank_group, batch, h_q, h_kv, l_k, fused):
    from paper_2604_00028_b200.dist import PeerSeqShardedDecode
    inp = synth.make_inputs(batch, h_q, h_kv, l_k, seed=1600, device="cuda")
    sd = PeerSeqShardedDecode(batch, h_q, h_kv, l_k, device="cuda", fused=fused)
    assert sd.world == 1 and sd.l_local == l_k
    ref_o, ref_l = OA.decode_attention(*(synth.to_f64(inp[n]) for n in ("q", "k", "v", "seqlens")))
    out = torch.empty((batch, h_q, 128), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((batch, h_q), dtype=torch.float32, device="cuda")
    for _ in range(3):                                    # eager steps: epochs 1, 2, 3
        out.zero_()
        sd.step(inp["q"], inp["k"], inp["v"], inp["seqlens"], out, lse)
        torch.cuda.synchronize()
        assert_out_close(synth.to_f64(out), ref_o)
        assert_lse_close(synth.to_f64(lse), ref_l)
    assert int(sd.epoch.item()) == 3
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(4):
            sd.step(inp["q"], inp["k"], inp["v"], inp["seqlens"], out, lse)
    for _ in range(2):                                    # replays keep advancing the epoch
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert_out_close(synth.to_f64(out), ref_o)
    assert int(sd.epoch.item()) == 3 + 2 * 4            # capture records, the two replays run
    assert int(sd.counter.item()) == 0                  # da_forward_peer leaves its counter at zero


@pytest.mark.parametrize("one_kernel", [True, False])
@pytest.mark.parametrize("batch,h_q,h_kv,l_k,policy,mode", [
    (1, 64, 8, 300, "seq_aware", 0),        # s = 1: the forward writes the slot rows, every CTA counts
    (2, 8, 1, 1500, "seq_aware", 1),        # cluster combine: the row owners write and count
    (3, 24, 3, 300, "seq_aware", 0),        # G = 8, several sequences: one wave of s = 1 CTAs
    (1, 64, 8, 4096, "seq_aware", 2),       # workspace combine: the combine kernel writes and counts
    (4, 16, 2, 3000, "dynamic", 2),         # dynamic: s_b = 1 rows from the forward, the rest combined
])
def test_forward_peer_every_combine_mode(one_rank_group, batch, h_q, h_kv, l_k, policy, mode, one_kernel):
    # da_forward_peer: the writer of the final rows publishes (slot e & 1, epoch flags), whichever
    # kernel that is; da_forward_peer_combine (static plans) exchanges LL words and merges the ranks'
    # partials inside that kernel (the forward for NONE / CLUSTER, the combine kernel for workspace
    # plans).  Checked against the oracle over several epochs (both slots).
    from paper_2604_00028_b200.dist import PeerSeqShardedDecode
    # ragged lengths everywhere: an empty sequence (lse = -inf partials) and a single-key one
    inp = synth.make_inputs(batch, h_q, h_kv, l_k, seed=1610, device="cuda",
                            variant="ragged" if (policy == "dynamic" or batch >= 2) else "normal")
    sd = PeerSeqShardedDecode(batch, h_q, h_kv, l_k, device="cuda", policy=policy, fused=True, one_kernel=one_kernel)
    assert sd.plan.combine_mode == mode
    assert sd.one_kernel == one_kernel       # the LL exchange in the kernel that finishes the rows
    ref_o, ref_l = OA.decode_attention(*(synth.to_f64(inp[n]) for n in ("q", "k", "v", "seqlens")))
    out = torch.empty((batch, h_q, 128), dtype=torch.float32, device="cuda")
    lse = torch.empty((batch, h_q), dtype=torch.float32, device="cuda")
    for e in range(1, 5):
        out.zero_()
        sd.step(inp["q"], inp["k"], inp["v"], inp["seqlens"], out, lse)
        torch.cuda.synchronize()
        assert_out_close(synth.to_f64(out), ref_o)
        assert_lse_close(synth.to_f64(lse), ref_l)
        assert int(sd.epoch.item()) == e and int(sd.counter.item()) == 0
    if sd.one_kernel:   # the LL words of the last step (slot 4 & 1 = 0) carry epoch 4
        words = sd.buf.view(torch.int64)[sd.ll_offset // 8: (sd.ll_offset + sd.ll_slot_bytes) // 8]
        rows = batch * h_q
        assert bool(((words[: rows * 129] >> 32) == 4).all())
    else:               # the partial of the last step sits in slot 0 of the exchange buffer, flag 0 holds 4
        flags = sd.buf.view(torch.int32)[sd.flag_offset // 4: sd.flag_offset // 4 + 1]
        assert int(flags.item()) == 4


@pytest.mark.parametrize("batch,h_q,h_kv,l_k,policy,mode", [
    (80, 64, 1, 300, "guarded", 0),          # tcgen05, s = 1: the forward does not publish -> forward + signal
    (4, 64, 1, 8192, "guarded", 2),          # tcgen05, s = 32: the combine kernel publishes / exchanges
])
def test_peer_exchange_tcgen05_plans(one_rank_group, batch, h_q, h_kv, l_k, policy, mode):
    from paper_2604_00028_b200.dist import PeerSeqShardedDecode
    inp = synth.make_inputs(batch, h_q, h_kv, l_k, seed=1650, device="cuda", variant="ragged")
    sd = PeerSeqShardedDecode(batch, h_q, h_kv, l_k, device="cuda", policy=policy)
    assert (sd.plan.path, sd.plan.combine_mode) == (2, mode)
    assert sd.one_kernel == (mode == 2) and sd.fused == (mode == 2)
    ref_o, ref_l = OA.decode_attention(*(synth.to_f64(inp[n]) for n in ("q", "k", "v", "seqlens")))
    out = torch.empty((batch, h_q, 128), dtype=torch.float32, device="cuda")
    lse = torch.empty((batch, h_q), dtype=torch.float32, device="cuda")
    for e in range(1, 4):
        out.zero_()
        sd.step(inp["q"], inp["k"], inp["v"], inp["seqlens"], out, lse)
        torch.cuda.synchronize()
        assert_out_close(synth.to_f64(out), ref_o)
        assert_lse_close(synth.to_f64(lse), ref_l)
        assert int(sd.epoch.item()) == e


# ---- bounded waits: a peer that never arrives fails the step instead of hanging the GPU ----------
def _fake_two_rank_buffers(batch, h_q, world=2):
    """Exchange buffers for `world` ranks on this GPU, where only rank 0 (this process) runs: the
    other ranks' buffers are plain zeroed allocations nobody writes, i.e. a peer that crashed or never
    reached the step.  Returns (bufs, bases tensor, layout)."""
    from paper_2604_00028_b200.dist import peer_layout
    lay = peer_layout(batch, h_q, 128, world)
    bufs = [torch.zeros(lay[-1] // 4, dtype=torch.float32, device="cuda") for _ in range(world)]
    bases = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    return bufs, bases, lay


@pytest.mark.parametrize("batch,h_q,h_kv,l_k,mode", [(1, 8, 1, 1500, 1), (1, 64, 8, 300, 0), (1, 64, 8, 4096, 2)])
def test_forward_peer_combine_times_out_on_a_missing_peer(batch, h_q, h_kv, l_k, mode):
    import time
    import paper_2604_00028_b200 as dec
    from paper_2604_00028_b200 import api
    inp = synth.make_inputs(batch, h_q, h_kv, l_k, seed=1620, device="cuda")
    plan = dec.make_plan(batch, h_q, h_kv, l_k, policy="seq_aware")
    assert plan.combine_mode == mode and api.one_kernel_exchange_ok(plan)
    bufs, bases, (slot, lo, fo, llo, lls, tot) = _fake_two_rank_buffers(batch, h_q)
    epoch = torch.zeros(1, dtype=torch.int32, device="cuda")
    counter = torch.zeros(1, dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    t0 = time.perf_counter()
    out, lse = api.forward_peer_combine(plan, inp["q"], inp["k"], inp["v"], None, 2, 0, bases, llo, lls, epoch,
                                        counter, status, timeout_ns=2_000_000)       # 2 ms bound
    torch.cuda.synchronize()
    elapsed = time.perf_counter() - t0
    assert int(status.item()) == dec.DA_ERR_TIMEOUT
    assert elapsed < 5.0                                 # bounded: no hang (every thread gives up)
    assert int(epoch.item()) == 1 and int(counter.item()) == 0   # the step still completes its bookkeeping
    # this rank's own LL words were published with epoch 1, in LL slot 1 & 1 = 1
    words = bufs[0].view(torch.int64)[(llo + lls) // 8: (llo + 2 * lls) // 8][: batch * h_q * 129]
    assert bool(((words >> 32) == 1).all())


def test_combine_peers_times_out_on_a_missing_flag():
    import time
    import paper_2604_00028_b200 as dec
    from paper_2604_00028_b200 import _lib as L
    batch, h_q = 2, 16
    bufs, bases, (slot, lo, fo, llo, lls, tot) = _fake_two_rank_buffers(batch, h_q)
    o = torch.randn(batch, h_q, 128, device="cuda")
    lse_local = torch.randn(batch, h_q, device="cuda")
    epoch = torch.zeros(1, dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = torch.empty(batch, h_q, 128, dtype=torch.float32, device="cuda")
    lse = torch.empty(batch, h_q, dtype=torch.float32, device="cuda")
    L.da_peer_signal(2, 0, bases, o, lse_local, batch, h_q, 128, slot, lo, fo, epoch)   # rank 0 signals epoch 1
    t0 = time.perf_counter()
    L.da_combine_peers(2, 0, bases, slot, lo, fo, epoch, batch, h_q, 128, L.DA_F32, out, lse, status, 2_000_000)
    torch.cuda.synchronize()
    assert time.perf_counter() - t0 < 5.0
    assert int(status.item()) == dec.DA_ERR_TIMEOUT       # rank 1's flag never reached epoch 1
    # with both flags present the same call completes without touching status
    status.zero_()
    flags = bufs[0].view(torch.int32)[fo // 4: fo // 4 + 2]
    flags[1] = 1
    L.da_combine_peers(2, 0, bases, slot, lo, fo, epoch, batch, h_q, 128, L.DA_F32, out, lse, status, 2_000_000)
    torch.cuda.synchronize()
    assert int(status.item()) == 0


def test_peer_step_check_reports_timeout(one_rank_group):
    # PeerSeqShardedDecode.check(): a clean run reads status 0
    from paper_2604_00028_b200.dist import PeerSeqShardedDecode
    inp = synth.make_inputs(1, 8, 1, 1500, seed=1621, device="cuda")
    sd = PeerSeqShardedDecode(1, 8, 1, 1500, device="cuda", timeout_ns=50_000_000)
    sd.step(inp["q"], inp["k"], inp["v"])
    sd.check()
    sd.status.fill_(6)
    with pytest.raises(Exception):
        sd.check()


# ---- the north_star's NCCL path: all-gather of the packed [o | lse] partials + da_combine ----------
@pytest.mark.parametrize("batch,h_q,h_kv,l_k,policy", [(1, 64, 8, 4096, "seq_aware"), (3, 24, 3, 1500, "seq_aware_sm"),
                                                       (2, 8, 1, 700, "seq_aware")])
def test_nccl_seq_sharded_matches_oracle(one_rank_group, batch, h_q, h_kv, l_k, policy):
    from paper_2604_00028_b200.dist import SeqShardedDecode
    inp = synth.make_inputs(batch, h_q, h_kv, l_k, seed=1630, device="cuda",
                            variant="ragged" if batch >= 2 else "normal")
    sd = SeqShardedDecode(batch, h_q, h_kv, l_k, device="cuda", policy=policy)
    # the packed chunk is padded to 16 bytes: da_combine reads the partials with that split stride
    assert sd.chunk % 4 == 0 and sd.chunk >= batch * h_q * 129
    ref_o, ref_l = OA.decode_attention(*(synth.to_f64(inp[n]) for n in ("q", "k", "v", "seqlens")))
    for dt in (torch.bfloat16, torch.float32):
        out = torch.zeros((batch, h_q, 128), dtype=dt, device="cuda")
        lse = torch.empty((batch, h_q), dtype=torch.float32, device="cuda")
        sd.step(inp["q"], inp["k"], inp["v"], inp["seqlens"], out, lse)
        torch.cuda.synchronize()
        assert_out_close(synth.to_f64(out), ref_o)
        assert_lse_close(synth.to_f64(lse), ref_l)
    # graph-captured steps (the bench's launch configuration)
    out = torch.zeros((batch, h_q, 128), dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        sd.step(inp["q"], inp["k"], inp["v"], inp["seqlens"], out, lse)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(3):
            sd.step(inp["q"], inp["k"], inp["v"], inp["seqlens"], out, lse)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert_out_close(synth.to_f64(out), ref_o)
    assert_lse_close(synth.to_f64(lse), ref_l)


# ---- the multi-rank LL protocol with world > 1, emulated in ONE launch on one GPU --------------------
# (separate launches that spin on each other's words are not guaranteed to be co-scheduled on one GPU:
#  da_forward_peer_combine with rank = -1 runs every rank's grid in a single launch instead)
@pytest.mark.parametrize("world,batch,h_q,h_kv,l_total,policy", [
    (2, 2, 64, 8, 1024, "guarded"),        # s = 1 NONE plans, ragged lengths (an empty and a 1-token sequence)
    (4, 1, 8, 1, 4096, "seq_aware_sm"),    # cluster plans: the owner CTAs of each rank exchange
    (8, 1, 64, 8, 4095, "seq_aware"),      # world 8, shards of 511 / 512 tokens (lengths per rank)
    (3, 3, 24, 3, 1500, "seq_aware_sm"),
])
def test_emulated_ranks_one_kernel_exchange(world, batch, h_q, h_kv, l_total, policy):
    import paper_2604_00028_b200 as dec
    from paper_2604_00028_b200 import _lib as L
    from paper_2604_00028_b200.dist import peer_layout, shard_range
    inp = synth.make_inputs(batch, h_q, h_kv, l_total, seed=1640, device="cuda",
                            variant="ragged" if batch >= 2 else "normal")
    ref_o, ref_l = OA.decode_attention(*(synth.to_f64(inp[n]) for n in ("q", "k", "v", "seqlens")))
    shards = [shard_range(l_total, r, world) for r in range(world)]
    l_cap = max(t1 - t0 for t0, t1 in shards)
    k = torch.full((world * batch, l_cap, h_kv, 128), float("nan"), dtype=torch.bfloat16, device="cuda")
    v = torch.full_like(k, float("nan"))
    lens = torch.zeros(world * batch, dtype=torch.int32)
    for r, (t0, t1) in enumerate(shards):
        k[r * batch:(r + 1) * batch, : t1 - t0] = inp["k"][:, t0:t1]
        v[r * batch:(r + 1) * batch, : t1 - t0] = inp["v"][:, t0:t1]
        for b in range(batch):
            lens[r * batch + b] = min(max(int(inp["seqlens"][b]) - t0, 0), t1 - t0)
    lens = lens.to("cuda")
    plan = dec.make_plan(batch, h_q, h_kv, l_cap, policy=policy)
    assert plan.combine_mode in (0, 1)
    lay = peer_layout(batch, h_q, 128, world)
    slot, lo, fo, llo, lls, tot = lay
    bufs = [torch.zeros(tot // 4, dtype=torch.float32, device="cuda") for _ in range(world)]
    bases = torch.tensor([x.data_ptr() for x in bufs], dtype=torch.int64, device="cuda")
    epoch = torch.zeros(world, dtype=torch.int32, device="cuda")
    counter = torch.zeros(world, dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = torch.empty((world, batch, h_q, 128), dtype=torch.float32, device="cuda")
    lse = torch.empty((world, batch, h_q), dtype=torch.float32, device="cuda")
    strides = (inp["q"].stride(0), inp["q"].stride(1), k.stride(0), k.stride(1), k.stride(2),
               v.stride(0), v.stride(1), v.stride(2))
    for e in range(1, 6):                                 # both LL slots, several epochs
        out.zero_()
        L.da_forward_peer_combine(plan, inp["q"], k, v, l_cap, lens, strides, 0.0, world, -1, bases, llo, lls,
                                  epoch, counter, L.DA_F32, out, lse, status, 2_000_000_000)
        torch.cuda.synchronize()
        assert int(status.item()) == 0
        for r in range(world):                            # every emulated rank holds the full result
            assert_out_close(synth.to_f64(out[r]), ref_o, f"rank {r} out")
            assert_lse_close(synth.to_f64(lse[r]), ref_l, f"rank {r} lse")
        assert epoch.tolist() == [e] * world and counter.tolist() == [0] * world


def test_emulation_validation():
    import paper_2604_00028_b200 as dec
    from paper_2604_00028_b200 import _lib as L
    plan = dec.make_plan(1, 64, 8, 131072, policy="seq_aware")           # s = 16: workspace combine
    x = torch.zeros(4, dtype=torch.int64, device="cuda")
    with pytest.raises(L.DecAttnError) as e:
        L.da_forward_peer_combine(plan, x, x, x, 131072, None, None, 0.0, 2, -1, x, 0, 8 * 129 * 64, x, x, L.DA_F32,
                                  x, x, x, 0, x, 1 << 30)
    assert e.value.status == L.DA_ERR_UNSUPPORTED
    big = dec.make_plan(1, 64, 8, 1024, policy="guarded")                 # s = 7 clusters: 8 per rank
    with pytest.raises(L.DecAttnError) as e:
        L.da_forward_peer_combine(big, x, x, x, 1024, None, None, 0.0, 8, -1, x, 0, 8 * 129 * 64, x, x, L.DA_F32,
                                  x, x, x, 0)
    assert e.value.status == L.DA_ERR_UNSUPPORTED                        # 8 ranks x 8 clusters do not fit
