// Device helpers shared by the split-KV forward kernels (fwd.cu: mma.sync / scalar paths;
// fwd_tc.cu: the tcgen05 path for wide query groups).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "config.h"
#include "internal.h"
#include "ptx.cuh"

namespace decattn {
namespace {

constexpr float kNegInf = -__builtin_huge_valf();
constexpr float kLn2 = 0.6931471805599453f;
constexpr int kHalfBytes = kTileN * 128;     // one 64-token x 64-dim box: 8 KB

__device__ __forceinline__ void store_out(const FwdParams& p, void* out, size_t row, int d4, float4 v) {
  DA_DASSERT(row < static_cast<size_t>(p.batch) * p.h_q && d4 >= 0 && d4 < kHeadDim / 4);
  if (p.out_f32) {
    reinterpret_cast<float4*>(out)[row * (kHeadDim / 4) + d4] = v;
  } else {
    uint2 w;
    w.x = ptx::pack_bf16(v.x, v.y);
    w.y = ptx::pack_bf16(v.z, v.w);
    reinterpret_cast<uint2*>(out)[row * (kHeadDim / 4) + d4] = w;
  }
}

// floor(x / d) for a launch-invariant d given m = ceil(2^38 / d) (internal.h div_magic; exact
// while x d < 2^38): a 32 x 64-bit multiply and a shift instead of an integer divide.
__device__ __forceinline__ uint32_t udiv_magic(uint32_t x, uint64_t m) {
  return static_cast<uint32_t>((static_cast<uint64_t>(x) * m) >> 38);
}

// Tokens [t0, t_end) of split `split` of s for a sequence of n tokens: units of kTileN
// tokens, split i covering units [floor(i n_u / s), floor((i+1) n_u / s)) (C-pol item 6),
// evaluated as i q + floor(i r / s) with n_u = q s + r so every quotient is exact (n_u < 2^25,
// i r < 2^16, s <= 256).
__device__ __forceinline__ void split_range(int n, int split, int s, uint64_t s_magic, int& t0, int& t_end,
                                            int& n_tiles) {
  const uint32_t nu = (static_cast<uint32_t>(n) + (kTileN - 1)) / kTileN;
  const uint32_t q = udiv_magic(nu, s_magic);
  const uint32_t r = nu - q * static_cast<uint32_t>(s);
  const uint32_t i0 = static_cast<uint32_t>(split), i1 = i0 + 1;
  const uint32_t u0 = i0 * q + udiv_magic(i0 * r, s_magic);
  const uint32_t u1 = i1 * q + udiv_magic(i1 * r, s_magic);
  t0 = static_cast<int>(u0) * kTileN;
  t_end = min(static_cast<int>(u1) * kTileN, n);
  n_tiles = static_cast<int>(u1 - u0);
}

}  // namespace
}  // namespace decattn
