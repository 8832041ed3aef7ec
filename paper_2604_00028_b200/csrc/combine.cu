// LSE combine of split partials (C-comb):
//   M = max_i lse_i,  lse = M + ln sum_i exp(lse_i - M),
//   out = sum_i exp(lse_i - lse) o_i;  every split empty -> out = 0, lse = -inf.
// The paper counts this merge as the cost that grows with s ("final
// reductions"; the right arm of the U-curve; "atomic
// combination overhead").
//
// One CTA (4 warps) per (b, h) row: every warp reduces the s lse values to
// M with warp shuffles; warp w then accumulates splits w, w+4, ... with every
// lane owning 4 of the 128 head dims (128-bit loads; the loads of 8 splits
// are issued before their FMAs), and warp 0 adds the four partial sums.  Two
// L2 round trips whatever s is.  Launched with programmatic dependent launch
// so its launch latency hides under the forward kernel's tail;
// griddepcontrol.wait orders its reads after the forward's writes.
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

__global__ void __launch_bounds__(kCombineThreads)
    lse_combine_kernel(const CombineParams p) {
  pdl_launch_dependents();   // the next step's forward may start its prologue
  pdl_wait();                // partials are written by the preceding forward kernel
  constexpr int kWarps = kCombineThreads / 32;
  __shared__ float4 s_acc[kWarps][32];
  __shared__ float s_l[kWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x;
  const int s = p.num_splits;
  DA_DASSERT(row < p.rows && s >= 1);
  const float* lse_in = p.lse_in + row;

  // (1) M = max_i lse_i: every warp reduces all s values (one L2 round trip)
  float M = kNegInf;
  for (int i = lane; i < s; i += 32) M = fmaxf(M, __ldg(lse_in + i * p.lse_stride));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
  const bool empty = M == kNegInf;

  // (2) warp w accumulates splits w, w + kWarps, ...: lane owns dims 4 lane .. 4 lane + 3.
  //     The loads of 8 splits are issued before their FMAs (second L2 round trip).
  float Lw = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (!empty) {
    const float4* o = reinterpret_cast<const float4*>(p.o + static_cast<int64_t>(row) * kHeadDim) + lane;
    const int64_t ostride4 = p.o_stride / 4;
    for (int i0 = warp; i0 < s; i0 += 8 * kWarps) {
      float li[8];
      float4 oi[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = i0 + j * kWarps;
        li[j] = kNegInf;
        oi[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < s) {
          li[j] = __ldg(lse_in + i * p.lse_stride);
          oi[j] = __ldg(o + i * ostride4);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float wgt = ex2((li[j] - M) * kLog2e);     // empty split or past s: exp(-inf) = 0
        Lw += wgt;
        acc.x = fmaf(wgt, oi[j].x, acc.x);
        acc.y = fmaf(wgt, oi[j].y, acc.y);
        acc.z = fmaf(wgt, oi[j].z, acc.z);
        acc.w = fmaf(wgt, oi[j].w, acc.w);
      }
    }
  }
  s_acc[warp][lane] = acc;
  if (lane == 0) s_l[warp] = Lw;
  __syncthreads();
  if (warp != 0) return;

  // (3) warp 0 sums the warps' partial sums and writes the row
  float L = 0.f;
  float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    L += s_l[w];
    const float4 a = s_acc[w][lane];
    sum.x += a.x;
    sum.y += a.y;
    sum.z += a.z;
    sum.w += a.w;
  }
  const float inv = L > 0.f ? __frcp_rn(L) : 0.f;
  sum = make_float4(sum.x * inv, sum.y * inv, sum.z * inv, sum.w * inv);
  const float lse = empty ? kNegInf : M + lg2(L) * (1.f / kLog2e);
  if (p.out_f32) {
    reinterpret_cast<float4*>(p.out)[static_cast<int64_t>(row) * (kHeadDim / 4) + lane] = sum;
  } else {
    uint2 w2;
    w2.x = pack_bf16(sum.x, sum.y);
    w2.y = pack_bf16(sum.z, sum.w);
    reinterpret_cast<uint2*>(p.out)[static_cast<int64_t>(row) * (kHeadDim / 4) + lane] = w2;
  }
  if (lane == 0 && p.lse != nullptr) p.lse[row] = lse;
}

}  // namespace

cudaError_t launch_lse_combine(const CombineParams& p, bool pdl, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.rows, 1, 1);
  cfg.blockDim = dim3(kCombineThreads, 1, 1);
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
