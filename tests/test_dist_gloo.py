"""Multi-GPU layer host logic with world_size 2 on CPU (gloo): sharding ranges and the
long-context exchange (all-gather of packed [o | lse] partials + combine) against the
unsharded oracle.  The local attention / combine are injected with oracle functions
(test infrastructure); the CUDA versions are exercised by the GPU tests."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_ranges_cover_exactly():
    from paper_2604_00028_b200.dist import head_shard, shard_range
    for n in (0, 1, 7, 8, 128, 131072):
        for world in (1, 2, 3, 4, 8):
            rs = [shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
    (k0, k1), (q0, q1) = head_shard(64, 8, 7, 8)
    assert (k0, k1, q0, q1) == (7, 8, 56, 64)     # TP-8: one KV head per device
    with pytest.raises(ValueError):
        head_shard(64, 8, 0, 3)


def _worker(rank, world, port, B, HQ, HKV, L, seqlens, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from oracle import attention as OA
        from paper_2604_00028_b200.dist import SeqShardedDecode, local_seqlens

        inp = synth.make_inputs(B, HQ, HKV, L, seed=77)     # every rank draws the same global cache
        q, k, v = (synth.to_f64(inp[n]) for n in ("q", "k", "v"))

        def local(qt, kt, vt, sl, o_out, lse_out):
            # sl: whole-sequence lengths (the CUDA path takes the shard's part via the plan's
            # seq_offset; this injected oracle does it on the host)
            sl = local_seqlens(sl, sd.t0, sd.l_local)
            o, l = OA.decode_attention(q, synth.to_f64(kt), synth.to_f64(vt), sl.numpy())
            o_out.copy_(torch.from_numpy(o).float())
            lse_out.copy_(torch.from_numpy(l).float())

        def comb(o_parts, lse_parts, out, lse):
            o, l = OA.lse_combine(o_parts.double().numpy(), lse_parts.double().numpy())
            out.copy_(torch.from_numpy(o))
            lse.copy_(torch.from_numpy(l))

        sd = SeqShardedDecode(B, HQ, HKV, L, 128, device="cpu", local_attention=local, combine=comb)
        kl, vl = inp["k"][:, sd.t0:sd.t0 + sd.l_local], inp["v"][:, sd.t0:sd.t0 + sd.l_local]
        sl = torch.tensor(seqlens, dtype=torch.int32)
        out = torch.empty(B, HQ, 128, dtype=torch.float32)
        lse = torch.empty(B, HQ, dtype=torch.float32)
        sd.step(inp["q"], kl, vl, sl, out, lse)
        ref_o, ref_l = OA.decode_attention(q, k, v, np.array(seqlens))
        ok_o = np.allclose(out.numpy(), ref_o, atol=1e-5, rtol=1e-5)
        fin = np.isfinite(ref_l)
        ok_l = (np.isneginf(lse.numpy()) == ~fin).all() and np.allclose(lse.numpy()[fin], ref_l[fin], atol=1e-5)
        ret[rank] = bool(ok_o and ok_l)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seqlens", [[300, 300], [300, 100], [0, 151]])
def test_seq_sharded_exchange_matches_unsharded(seqlens):
    world, B, HQ, HKV, L = 2, 2, 16, 2, 300
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), B, HQ, HKV, L, seqlens, ret), nprocs=world, join=True)
    assert dict(ret) == {0: True, 1: True}
