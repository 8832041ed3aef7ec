// Cross-GPU exchange from inside the producing kernel.
//   da_forward_peer: the kernel that produces a rank's final (o, lse) rows writes them straight
//     into its exchange slot and the last CTA releases the step's epoch to every rank (one
//     system fence), so no separate signal kernel or copy sits before da_combine_peers.
//   da_forward_peer_combine: every CTA writes its rows as LL words (value and epoch in one 8-byte
//     store), polls the same words of every rank and LSE-merges them: the whole step in one
//     kernel, with no fence and no flag on its critical path.
#pragma once

#include <cstdint>

#include "internal.h"
#include "ptx.cuh"

namespace decattn {

// Base of this step's slot (e = *epoch + 1 uses slot e & 1).  The epoch advances only after
// every writer CTA has counted, i.e. after each of them read it here.
static __device__ __forceinline__ uint64_t pub_slot(const PubParams& pb) {
  const uint32_t e = static_cast<uint32_t>(*reinterpret_cast<const volatile int32_t*>(pb.epoch)) + 1u;
  return pb.bases[pb.rank] + static_cast<uint64_t>(pb.slot_bytes) * (e & 1u);
}

// One thread per writer CTA, after the CTA's row stores are ordered before it (a CTA or warp
// barrier): count the CTA (its rows ordered before the count at GPU scope: every writer runs on
// this GPU); the last one, after a system-scope acquire-release fence (cumulative: it covers the
// rows of every writer it observed through the count), releases e = *epoch + 1 into flag `rank`
// of every rank's buffer, resets the count and sets *epoch = e.  One system-scope fence per step.
static __device__ __noinline__ void pub_arrive(const uint64_t* bases, int32_t* epoch, uint32_t* count,
                                        int64_t flag_offset, int32_t world, int32_t rank, int32_t writers) {
  ptx::fence_acq_rel_gpu();                         // this CTA's rows before its count
  const uint32_t prev = atomicAdd(count, 1u);
  if (prev + 1u != static_cast<uint32_t>(writers)) return;
  ptx::fence_acq_rel_sys();                         // every writer's rows before the flags
  const uint32_t e = static_cast<uint32_t>(*reinterpret_cast<volatile int32_t*>(epoch)) + 1u;
  *reinterpret_cast<volatile uint32_t*>(count) = 0u;
  for (int q = 0; q < world; ++q) {   // fence above + strong stores = one release pattern per flag
    uint32_t* flags = reinterpret_cast<uint32_t*>(bases[q] + static_cast<uint64_t>(flag_offset));
    ptx::st_relaxed_sys_u32(flags + rank, e);
  }
  *reinterpret_cast<volatile int32_t*>(epoch) = static_cast<int32_t>(e);
}

static __device__ __forceinline__ void pub_arrive(const PubParams& pb) {
  pub_arrive(pb.bases, pb.epoch, pb.count, pb.flag_offset, pb.world, pb.rank, pb.writers);
}

// ---- da_forward_peer_combine: LL (low-latency) words, data and epoch in one 8-byte store ----
constexpr int kLLRowWords = 129;                  // 128 o floats + lse per row

static __device__ __forceinline__ uint64_t* pub_ll_row(const PubParams& pb, int q, uint32_t e, size_t row) {
  return reinterpret_cast<uint64_t*>(pb.bases[q] + static_cast<uint64_t>(pb.ll_offset) +
                                     static_cast<uint64_t>(pb.ll_slot_bytes) * (e & 1u)) + row * kLLRowWords;
}
static __device__ __forceinline__ void st_ll(uint64_t* p, uint32_t e, float v) {
  const uint64_t w = (static_cast<uint64_t>(e) << 32) | __float_as_uint(v);
  asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
static __device__ __forceinline__ uint64_t ld_ll(const uint64_t* p) {
  uint64_t w;
  asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}
// Row `row`, float4 column d4 (and the lse when d4 == 0) of this rank's partial, as LL words.
static __device__ __forceinline__ void pub_ll_store(const PubParams& pb, uint32_t e, size_t row, int d4, float4 v,
                                                    float lse) {
  uint64_t* w = pub_ll_row(pb, pb.rank, e, row) + 4 * d4;
  st_ll(w, e, v.x);
  st_ll(w + 1, e, v.y);
  st_ll(w + 2, e, v.z);
  st_ll(w + 3, e, v.w);
  if (d4 == 0) st_ll(pub_ll_row(pb, pb.rank, e, row) + 128, e, lse);
}
// Bounded wait: poll `p` until its epoch is e, at most pb.timeout_ns after the first
// failed poll; past that (or once another thread has timed out) record DA_ERR_TIMEOUT in
// *pb.status and return what the word holds, so the kernel completes and the host sees the failure.
static __device__ __noinline__ uint64_t ld_ll_wait(const PubParams& pb, const uint64_t* p, uint64_t w, uint32_t e) {
  const uint64_t t0 = ptx::globaltimer();
  while (static_cast<uint32_t>(w >> 32) != e) {
    if (*reinterpret_cast<const volatile int32_t*>(pb.status) != 0) break;
    if (ptx::globaltimer() - t0 > pb.timeout_ns) {
      atomicExch(pb.status, static_cast<int32_t>(DA_ERR_TIMEOUT));
      break;
    }
    w = ld_ll(p);
  }
  return w;
}
// Every rank's (o, lse) words of row / d4, polled until they carry epoch e (each word validates
// itself: no flag, no fence), LSE-merged (C-comb) into the final out / lse.
static __device__ __forceinline__ void pub_ll_merge_row(const PubParams& pb, uint32_t e, size_t row, int d4) {
  constexpr float kLog2e = 1.4426950408889634f;
  float m = -__builtin_huge_valf(), L = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int q = 0; q < pb.world; ++q) {
    const uint64_t* rw = pub_ll_row(pb, q, e, row);
    uint64_t w[5];
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = ld_ll(rw + 4 * d4 + i);
    w[4] = ld_ll(rw + 128);
#pragma unroll
    for (int i = 0; i < 5; ++i)
      if (static_cast<uint32_t>(w[i] >> 32) != e) w[i] = ld_ll_wait(pb, i < 4 ? rw + 4 * d4 + i : rw + 128, w[i], e);
    const float li = __uint_as_float(static_cast<uint32_t>(w[4])) * kLog2e;
    const float4 oi = make_float4(__uint_as_float(static_cast<uint32_t>(w[0])), __uint_as_float(static_cast<uint32_t>(w[1])),
                                  __uint_as_float(static_cast<uint32_t>(w[2])), __uint_as_float(static_cast<uint32_t>(w[3])));
    const float mb = fmaxf(m, li);
    if (mb == -__builtin_huge_valf()) continue;           // every partial so far empty
    const float r = ptx::ex2(m - mb), wt = ptx::ex2(li - mb);
    L = fmaf(L, r, wt);
    acc = make_float4(fmaf(acc.x, r, wt * oi.x), fmaf(acc.y, r, wt * oi.y), fmaf(acc.z, r, wt * oi.z),
                      fmaf(acc.w, r, wt * oi.w));
    m = mb;
  }
  const float inv = L > 0.f ? ptx::rcp(L) : 0.f;
  const float4 v = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  if (pb.out_f32) {
    reinterpret_cast<float4*>(pb.out)[row * 32 + d4] = v;
  } else {
    uint2 w2;
    w2.x = ptx::pack_bf16(v.x, v.y);
    w2.y = ptx::pack_bf16(v.z, v.w);
    reinterpret_cast<uint2*>(pb.out)[row * 32 + d4] = w2;
  }
  if (d4 == 0 && pb.lse != nullptr) pb.lse[row] = L > 0.f ? (m + ptx::lg2(L)) * (1.f / kLog2e) : -__builtin_huge_valf();
}
// One thread per CTA, after the CTA read the epoch: the last of the grid's CTAs advances it (the
// next step's kernel reads it after griddepcontrol.wait) and resets the count.
static __device__ __forceinline__ void pub_count_advance(const PubParams& pb, uint32_t e) {
  const uint32_t prev = atomicAdd(pb.count, 1u);
  if (prev + 1u != static_cast<uint32_t>(pb.writers)) return;
  *reinterpret_cast<volatile uint32_t*>(pb.count) = 0u;
  *reinterpret_cast<volatile int32_t*>(pb.epoch) = static_cast<int32_t>(e);
}

// The exchange parameters of the rank this CTA acts for: the caller's rank, or under multi-rank
// emulation (PubParams::emulate) rank `erank` with its own epoch, count, output and lse
// (`rows` = B H_Q rows per rank).
static __device__ __forceinline__ PubParams pub_rank_view(const PubParams& pb, int erank, size_t rows) {
  PubParams v = pb;
  if (pb.emulate) {
    v.rank = erank;
    v.epoch = pb.epoch + erank;
    v.count = pb.count + erank;
    v.out = static_cast<char*>(pb.out) + rows * static_cast<size_t>(erank) * 128 * (pb.out_f32 ? 4 : 2);
    if (pb.lse != nullptr) v.lse = pb.lse + rows * static_cast<size_t>(erank);
  }
  return v;
}

// The epoch this step publishes (e = *epoch + 1), read before the CTA counts itself.
static __device__ __forceinline__ uint32_t pub_epoch(const PubParams& pb) {
  return static_cast<uint32_t>(*reinterpret_cast<const volatile int32_t*>(pb.epoch)) + 1u;
}

}  // namespace decattn
