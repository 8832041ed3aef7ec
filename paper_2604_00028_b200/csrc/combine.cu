// LSE combine of split partials (C-comb):
//   M = max_i lse_i,  lse = M + ln sum_i exp(lse_i - M),
//   out = sum_i exp(lse_i - lse) o_i;  every split empty -> out = 0, lse = -inf.
// The paper counts this merge as the cost that grows with s ("final
// reductions"; the right arm of the U-curve; "atomic
// combination overhead").
//
// One warp per (b, h) row: lanes read the s lse values (warp-shuffle max and
// sum), then each lane streams its 4 of the 128 head dims of every partial
// (128-bit loads, 512 B per warp per split).  Launched with programmatic
// dependent launch so its launch latency hides under the forward kernel's
// tail; griddepcontrol.wait orders its reads after the forward's writes.
#include <cuda_runtime.h>

#include <cstdint>

#include "config.h"
#include "internal.h"
#include "ptx.cuh"

namespace decattn {

using namespace ptx;

namespace {

constexpr float kNegInf = -__builtin_huge_valf();
constexpr float kLog2e = 1.4426950408889634f;

__global__ void __launch_bounds__(kCombineRowsPerCta * 32)
    lse_combine_kernel(const CombineParams p) {
  pdl_launch_dependents();   // the next step's forward may start its prologue
  pdl_wait();                // partials are written by the preceding forward kernel
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * kCombineRowsPerCta + warp;
  if (row >= p.rows) return;
  const int s = p.num_splits;
  const float* lse_in = p.lse_in + row;

  float M = kNegInf;
  for (int i = lane; i < s; i += 32) M = fmaxf(M, __ldg(lse_in + i * p.lse_stride));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
  const bool empty = M == kNegInf;
  float L = 0.f;
  if (!empty)
    for (int i = lane; i < s; i += 32) L += ex2((__ldg(lse_in + i * p.lse_stride) - M) * kLog2e);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) L += __shfl_xor_sync(0xffffffffu, L, off);
  const float lse = empty ? kNegInf : M + lg2(L) * (1.f / kLog2e);

  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (!empty) {
    const float4* o = reinterpret_cast<const float4*>(p.o + static_cast<int64_t>(row) * kHeadDim) + lane;
    const int64_t ostride4 = p.o_stride / 4;
#pragma unroll 4
    for (int i = 0; i < s; ++i) {
      const float li = __ldg(lse_in + i * p.lse_stride);
      const float w = ex2((li - lse) * kLog2e);          // empty split: exp(-inf) = 0
      const float4 oi = __ldg(o + i * ostride4);
      acc.x = fmaf(w, oi.x, acc.x);
      acc.y = fmaf(w, oi.y, acc.y);
      acc.z = fmaf(w, oi.z, acc.z);
      acc.w = fmaf(w, oi.w, acc.w);
    }
  }
  if (p.out_f32) {
    reinterpret_cast<float4*>(p.out)[static_cast<int64_t>(row) * (kHeadDim / 4) + lane] = acc;
  } else {
    uint2 w;
    w.x = pack_bf16(acc.x, acc.y);
    w.y = pack_bf16(acc.z, acc.w);
    reinterpret_cast<uint2*>(p.out)[static_cast<int64_t>(row) * (kHeadDim / 4) + lane] = w;
  }
  if (lane == 0 && p.lse != nullptr) p.lse[row] = lse;
}

}  // namespace

cudaError_t launch_lse_combine(const CombineParams& p, bool pdl, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((p.rows + kCombineRowsPerCta - 1) / kCombineRowsPerCta, 1, 1);
  cfg.blockDim = dim3(kCombineRowsPerCta * 32, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, lse_combine_kernel, p);
}

}  // namespace decattn
