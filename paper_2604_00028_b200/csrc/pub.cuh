// Fused peer publish (da_forward_peer): the kernel that produces a rank's final
// (o, lse) rows writes them straight into its exchange slot and the last CTA releases the step's
// epoch to every rank, so no separate signal kernel or copy sits between the forward and the
// cross-GPU combine.
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

// The epoch this step publishes (e = *epoch + 1), read before the CTA counts itself.
static __device__ __forceinline__ uint32_t pub_epoch(const PubParams& pb) {
  return static_cast<uint32_t>(*reinterpret_cast<const volatile int32_t*>(pb.epoch)) + 1u;
}

// Warp 0 of the CTA (lane q polls rank q's flag) waits until every rank has published epoch e.
// Spinning is safe only when every CTA of this grid is resident (the host checks one wave).
static __device__ __forceinline__ void pub_wait_all(const PubParams& pb, uint32_t e, int lane) {
  const uint32_t* flags = reinterpret_cast<const uint32_t*>(pb.bases[pb.rank] + static_cast<uint64_t>(pb.flag_offset));
  for (int q = lane; q < pb.world; q += 32)
    while (ptx::ld_acquire_sys_u32(flags + q) < e) {
    }
}

// LSE merge (C-comb) of row `row`, float4 column d4, across the world partials of slot e & 1
// (o fp32 at slot + row * 512, lse at slot + lse_offset + row * 4), read from the ranks' buffers
// (NVLink loads for peers); writes the final out / lse.
static __device__ __forceinline__ void pub_merge_row(const PubParams& pb, uint32_t e, size_t row, int d4) {
  const uint64_t slot_off = static_cast<uint64_t>(pb.slot_bytes) * (e & 1u);
  constexpr float kLog2e = 1.4426950408889634f;
  float m = -__builtin_huge_valf(), L = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int q = 0; q < pb.world; ++q) {
    const uint64_t base = pb.bases[q] + slot_off;
    const float li = reinterpret_cast<const float*>(base + static_cast<uint64_t>(pb.lse_offset))[row] * kLog2e;
    const float4 oi = reinterpret_cast<const float4*>(base)[row * 32 + d4];
    const float mb = fmaxf(m, li);
    if (mb == -__builtin_huge_valf()) continue;           // every partial so far empty
    const float r = ptx::ex2(m - mb), w = ptx::ex2(li - mb);
    L = fmaf(L, r, w);
    acc = make_float4(fmaf(acc.x, r, w * oi.x), fmaf(acc.y, r, w * oi.y), fmaf(acc.z, r, w * oi.z),
                      fmaf(acc.w, r, w * oi.w));
    m = mb;
  }
  const float inv = L > 0.f ? __frcp_rn(L) : 0.f;
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

}  // namespace decattn
