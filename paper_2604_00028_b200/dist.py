"""Multi-GPU layer: one process per GPU, torch.distributed (NCCL over NVLink 5 /
NVSwitch) for the plumbing.  SURVEY §8(e).

Two ways the decode-attention path shards across one 8xB200 box:

* Throughput configs (batch x KV-head units are independent, "work
  tiles = Batch x H_KV"): each rank owns a contiguous range of batches (or of
  KV heads with their G query heads - the tensor-parallel mapping of P:L123)
  and runs the single-GPU path on it.  No collective: every rank owns its
  outputs (``shard_range``, ``BatchShard``).
* Long-context configs: rank r holds tokens [r L/P, (r+1) L/P) of every
  sequence (contiguous sequence shard).  Each rank runs the split-KV forward
  with fp32 output to get its (o_r, lse_r) partial - the same partial the
  in-GPU splits produce - then ONE exchange step: an all-gather of the packed
  [o_r | lse_r] fp32 buffer, followed by the same LSE-combine kernel with
  s = P (``SeqShardedDecode``).  Merging per-GPU partials is the identity
  behind sequence splitting (C-comb), so the result equals single-GPU
  attention over the whole sequence.

``PeerSeqShardedDecode`` replaces the all-gather + combine pair with an exchange over peer
memory: every rank's partial is written into its own buffer of a symmetric allocation mapped
on all GPUs (torch symmetric memory), a one-thread kernel releases a step epoch into every
peer's flag slot, and the combine kernel acquires the flags and reads the partials straight
from the peers' buffers over NVLink (``da_peer_signal`` / ``da_combine_peers``).

Host-side only: the arithmetic runs in libdecattn.so's kernels.  The local
attention and the combine are injectable so that the exchange logic can be
tested with world_size 2 on CPU (gloo) against the oracle.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int):
    """Contiguous, balanced [start, end) of n units for ``rank`` of ``world``."""
    if world < 1 or not (0 <= rank < world) or n < 0:
        raise ValueError("bad shard arguments")
    return (n * rank) // world, (n * (rank + 1)) // world


def head_shard(h_q: int, h_kv: int, rank: int, world: int):
    """KV heads [k0, k1) and their query heads [k0 G, k1 G) owned by ``rank``
    (tensor-parallel head mapping).  Requires world | h_kv."""
    if h_kv % world:
        raise ValueError("h_kv must be divisible by the world size for head sharding")
    G = h_q // h_kv
    k0, k1 = shard_range(h_kv, rank, world)
    return (k0, k1), (k0 * G, k1 * G)


def local_seqlens(seqlens_global: torch.Tensor, t0: int, l_local: int) -> torch.Tensor:
    """Tokens of each sequence that fall in this rank's shard [t0, t0 + l_local) (host reference of
    what the kernel derives from the plan's seq_offset; injected local attentions use it)."""
    return (seqlens_global.to(torch.int64) - t0).clamp_(0, l_local).to(torch.int32)


def _all_gather_flat(recv: torch.Tensor, send: torch.Tensor, group=None):
    backend = dist.get_backend(group)
    if backend == "nccl":
        dist.all_gather_into_tensor(recv, send, group=group)
    else:  # gloo (CPU tests): list form
        world = dist.get_world_size(group)
        dist.all_gather(list(recv.view(world, -1).unbind(0)), send, group=group)


class BatchShard:
    """Throughput mode: rank r owns batches [b0, b1) of a global batch; no collective."""

    def __init__(self, global_batch: int, rank: int, world: int):
        self.b0, self.b1 = shard_range(global_batch, rank, world)
        self.local_batch = self.b1 - self.b0


class SeqShardedDecode:
    """Long-context mode: sequence-sharded KV cache + all-gather + LSE combine.

    ``local_attention(q, k, v, seqlens, o_out, lse_out)`` must write this rank's
    fp32 partial into the given views (``seqlens``: whole-sequence lengths or None; the shard
    holds tokens [t0, t0 + l_local)); ``combine(o_parts, lse_parts, out, lse)``
    merges P partials ([P, B, H_Q, d] / [P, B, H_Q] views of the gather
    buffer).  Both default to the CUDA path.
    """

    def __init__(self, batch: int, h_q: int, h_kv: int, l_k_total: int, head_dim: int = 128, *,
                 group=None, policy="seq_aware", device=None, local_attention=None, combine=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.batch, self.h_q, self.h_kv, self.d = batch, h_q, h_kv, head_dim
        self.t0, t1 = shard_range(l_k_total, self.rank, self.world)
        self.l_local = t1 - self.t0
        if self.l_local < 1:
            raise ValueError("every rank needs at least one token of the sequence")
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
        # floats per rank: [o | lse], padded to 16 bytes so every rank's o is 16-byte aligned
        self.chunk = -(-(batch * h_q * (head_dim + 1)) // 4) * 4
        self.send = torch.empty(self.chunk, dtype=torch.float32, device=self.device)
        self.recv = torch.empty(self.world * self.chunk, dtype=torch.float32, device=self.device)
        self.plan = None
        if local_attention is None or combine is None:
            from . import api
            # seq_offset = t0: cache_seqlens stay whole-sequence lengths, the kernel takes this shard's
            # part of each (no per-step length arithmetic on the host or in extra launches)
            self.plan = api.make_plan(batch, h_q, h_kv, self.l_local, head_dim, True, 0, None, policy,
                                      seq_offset=self.t0)
            self._ws = api.workspace_for(self.plan, self.device)
        self._local = local_attention or self._cuda_local
        self._combine = combine or self._cuda_combine

    # -- views of the packed buffers ---------------------------------------
    def _o_view(self, flat):
        return flat[: self.batch * self.h_q * self.d].view(self.batch, self.h_q, self.d)

    def _lse_view(self, flat):
        n_o = self.batch * self.h_q * self.d
        return flat[n_o:n_o + self.batch * self.h_q].view(self.batch, self.h_q)

    def gathered(self):
        r = self.recv.view(self.world, self.chunk)
        o = r[:, : self.batch * self.h_q * self.d].view(self.world, self.batch, self.h_q, self.d)
        n_o = self.batch * self.h_q * self.d
        lse = r[:, n_o:n_o + self.batch * self.h_q].view(self.world, self.batch, self.h_q)
        return o, lse

    # -- default CUDA implementations --------------------------------------
    def _cuda_local(self, q, k, v, seqlens, o_out, lse_out):
        from . import api
        api.forward(self.plan, q, k, v, seqlens, out=o_out, lse=lse_out, workspace=self._ws,
                    out_dtype=torch.float32)

    def _cuda_combine(self, o_parts, lse_parts, out, lse):
        from . import _lib as L
        L.da_combine(self.world, self.batch, self.h_q, self.d, o_parts, self.chunk, lse_parts,
                     self.chunk, L.DA_F32 if out.dtype == torch.float32 else L.DA_BF16, out, lse)

    def step(self, q, k_local, v_local, cache_seqlens=None, out=None, lse=None):
        """One decode step: local partial -> all-gather -> combine.  ``cache_seqlens``: whole-sequence
        lengths (device int32 [B]) or None (every sequence l_k_total long).  Returns (out, lse)."""
        self._local(q, k_local, v_local, cache_seqlens, self._o_view(self.send), self._lse_view(self.send))
        _all_gather_flat(self.recv, self.send, self.group)
        if out is None:
            out = torch.empty((self.batch, self.h_q, self.d), dtype=torch.bfloat16, device=self.device)
        if lse is None:
            lse = torch.empty((self.batch, self.h_q), dtype=torch.float32, device=self.device)
        o_parts, lse_parts = self.gathered()
        self._combine(o_parts, lse_parts, out, lse)
        return out, lse


def _align16(n: int) -> int:
    return (n + 15) // 16 * 16


def peer_layout(batch: int, h_q: int, head_dim: int, world: int):
    """Byte layout of one rank's exchange buffer (include/decattn.h): two slots of slot_bytes, each
    [0, lse_offset) o fp32 [B, H_Q, d] and [lse_offset, ...) lse fp32 [B, H_Q]; one uint32 flag per
    rank at flag_offset (da_forward_peer / da_peer_signal / da_combine_peers); two LL slots of
    ll_slot_bytes, uint64 [B H_Q][d + 1], at ll_offset (da_forward_peer_combine).  Returns
    (slot_bytes, lse_offset, flag_offset, ll_offset, ll_slot_bytes, total_bytes), 16-byte aligned."""
    if min(batch, h_q, head_dim, world) < 1:
        raise ValueError("bad peer layout arguments")
    lse_offset = _align16(batch * h_q * head_dim * 4)
    slot_bytes = _align16(lse_offset + batch * h_q * 4)
    flag_offset = 2 * slot_bytes
    ll_offset = flag_offset + _align16(4 * world)
    ll_slot_bytes = _align16(8 * (head_dim + 1) * batch * h_q)
    return slot_bytes, lse_offset, flag_offset, ll_offset, ll_slot_bytes, ll_offset + 2 * ll_slot_bytes


class PeerSeqShardedDecode:
    """Long-context mode with the exchange over peer memory.  fused (default): when the plan's grid
    is one wave (NONE / CLUSTER combine), da_forward_peer_combine runs the whole step in ONE kernel
    (publish the partial into slot epoch & 1 of this rank's symmetric buffer, release the epoch to
    every rank from the last CTA, wait for every rank's flag, LSE-merge the ranks' partials of the
    rows each CTA wrote); otherwise da_forward_peer (publish) -> da_combine_peers (acquire every
    flag, read the partials from the peers' buffers, LSE-merge).  one_kernel=False forces the
    latter.  fused=False: forward into a local fp32 partial -> da_peer_signal (copy + release) ->
    da_combine_peers.  No NCCL call on the step; every call can be captured in a CUDA graph
    (monotonic epochs)."""

    def __init__(self, batch: int, h_q: int, h_kv: int, l_k_total: int, head_dim: int = 128, *,
                 group=None, policy="seq_aware", device=None, fused: bool = True, one_kernel: bool = True,
                 timeout_ns: int = 0):
        import torch.distributed._symmetric_memory as symm

        from . import api
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.batch, self.h_q, self.h_kv, self.d = batch, h_q, h_kv, head_dim
        self.t0, t1 = shard_range(l_k_total, self.rank, self.world)
        self.l_local = t1 - self.t0
        if self.l_local < 1:
            raise ValueError("every rank needs at least one token of the sequence")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.slot_bytes, self.lse_offset, self.flag_offset, self.ll_offset, self.ll_slot_bytes, total = \
            peer_layout(batch, h_q, head_dim, self.world)
        self.buf = symm.empty((total // 4,), dtype=torch.float32, device=self.device)
        pg = group if group is not None else dist.group.WORLD
        self.hdl = symm.rendezvous(self.buf, pg.group_name)
        self.buf.zero_()                                   # flags start at 0 (epochs start at 1)
        torch.cuda.synchronize(self.device)
        dist.barrier(group)                                # every buffer zeroed before any signal
        self.bases = torch.tensor([int(x) for x in self.hdl.buffer_ptrs], dtype=torch.int64, device=self.device)
        self.epoch = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.counter = torch.zeros(1, dtype=torch.int32, device=self.device)   # da_forward_peer: writer CTAs
        self.plan = api.make_plan(batch, h_q, h_kv, self.l_local, head_dim, True, 0, None, policy,
                                  seq_offset=self.t0)      # cache_seqlens: whole-sequence lengths
        from . import _lib as L
        if self.plan.path == L.DA_PATH_TC and self.plan.combine_mode != L.DA_COMBINE_KERNEL:
            fused = False        # the tcgen05 forward (s = 1) does not publish: forward + da_peer_signal
        self.fused = fused
        # every rank must take the same protocol (LL words vs slot + flags): the shards' lengths can
        # differ by one token, so their plans - and whether the one-kernel grid is resident - can
        # differ; the decision is the minimum over the group
        ok = torch.tensor([1 if (fused and one_kernel and api.one_kernel_exchange_ok(self.plan)) else 0],
                          dtype=torch.int32, device=self.device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        self.one_kernel = bool(ok.item())
        # bounded exchange waits: a peer's words / flags that do not arrive within timeout_ns
        # (0: the library's default, 10 s) set status = DA_ERR_TIMEOUT instead of hanging the GPU
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.timeout_ns = int(timeout_ns)
        self._ws = api.workspace_for(self.plan, self.device)
        self.o_local = torch.empty((batch, h_q, head_dim), dtype=torch.float32, device=self.device)
        self.lse_local = torch.empty((batch, h_q), dtype=torch.float32, device=self.device)

    def step(self, q, k_local, v_local, cache_seqlens=None, out=None, lse=None):
        """One decode step: local partial (published to the peers) -> pull-combine.  ``cache_seqlens``:
        whole-sequence lengths (device int32 [B]) or None.  Returns (out, lse)."""
        from . import _lib as L
        from . import api
        if self.one_kernel:
            return api.forward_peer_combine(self.plan, q, k_local, v_local, cache_seqlens, self.world, self.rank,
                                            self.bases, self.ll_offset, self.ll_slot_bytes, self.epoch, self.counter,
                                            self.status, timeout_ns=self.timeout_ns, out=out, lse=lse,
                                            workspace=self._ws)
        if self.fused:
            api.forward_peer(self.plan, q, k_local, v_local, cache_seqlens, self.world, self.rank, self.bases,
                             self.slot_bytes, self.lse_offset, self.flag_offset, self.epoch, self.counter,
                             workspace=self._ws)
        else:
            api.forward(self.plan, q, k_local, v_local, cache_seqlens, out=self.o_local, lse=self.lse_local,
                        workspace=self._ws, out_dtype=torch.float32)
            L.da_peer_signal(self.world, self.rank, self.bases, self.o_local, self.lse_local, self.batch,
                             self.h_q, self.d, self.slot_bytes, self.lse_offset, self.flag_offset, self.epoch)
        if out is None:
            out = torch.empty((self.batch, self.h_q, self.d), dtype=torch.bfloat16, device=self.device)
        if lse is None:
            lse = torch.empty((self.batch, self.h_q), dtype=torch.float32, device=self.device)
        L.da_combine_peers(self.world, self.rank, self.bases, self.slot_bytes, self.lse_offset, self.flag_offset,
                           self.epoch, self.batch, self.h_q, self.d,
                           L.DA_F32 if out.dtype == torch.float32 else L.DA_BF16, out, lse, self.status,
                           self.timeout_ns)
        return out, lse

    def check(self):
        """Raise DecAttnError(DA_ERR_TIMEOUT) if an exchange wait of any step so far ran past its bound
        (reads the device status word: synchronises with the steps enqueued before it)."""
        from . import _lib as L
        st = int(self.status.item())
        if st != 0:
            raise L.DecAttnError(st, "PeerSeqShardedDecode exchange")
