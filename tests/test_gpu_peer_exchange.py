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
