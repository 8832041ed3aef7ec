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

}  // namespace decattn
