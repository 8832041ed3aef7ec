// LSE combine of split partials (C-comb):
//   M = max_i lse_i,  lse = M + ln sum_i exp(lse_i - M),
//   out = sum_i exp(lse_i - lse) o_i;  every split empty -> out = 0, lse = -inf.
// The paper counts this merge as the cost that grows with s ("final
// reductions"; the right arm of the U-curve; "atomic
// combination overhead").
//
// One CTA (4 warps) per (b, h) row: warp w merges splits w, w+4, ... online
// against its own running maximum, every lane owning 4 of the 128 head dims
// (128-bit loads; the lse and o loads of 8 splits are issued together, so
// s <= 32 costs one L2 round trip), and warp 0 merges the four warps'
// (max, sum, accumulator) triples with the same identity.  Launched with programmatic dependent launch
// so its launch latency hides under the forward kernel's tail;
// griddepcontrol.wait orders its reads after the forward's writes.
#include <cuda_runtime.h>

#include <cstdint>

#include "config.h"
#include "internal.h"
#include "ptx.cuh"
#include "pub.cuh"

namespace decattn {

using namespace ptx;

namespace {

constexpr float kNegInf = -__builtin_huge_valf();
constexpr float kLog2e = 1.4426950408889634f;

// development timeline tracing (-DDECATTN_TRACE builds only): per row < 64, globaltimer ns at
// entry (0), after griddepcontrol.wait (1), after the output store (2)
#ifdef DECATTN_TRACE
__device__ unsigned long long g_trace_comb[64 * 4];
__device__ __forceinline__ void ctrace(int slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (blockIdx.x < 64) g_trace_comb[blockIdx.x * 4 + slot] = t;
}
#define CTRACE(slot) do { if (threadIdx.x == 0) ctrace(slot); } while (0)
#else
#define CTRACE(slot) do { } while (0)
#endif

__global__ void __launch_bounds__(kCombineThreads)
    lse_combine_kernel(const CombineParams p) {
  CTRACE(0);
  pdl_launch_dependents();   // the next step's forward may start its prologue
  pdl_wait();                // partials are written by the preceding forward kernel
  CTRACE(1);
  constexpr int kWarps = kCombineThreads / 32;
  constexpr int kBatch = 8;
  __shared__ float4 s_acc[kWarps][32];
  __shared__ float s_m[kWarps], s_l[kWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x;
  int s = p.num_splits;
  int64_t prow = row;                  // partial row of split 0
  if (p.meta != nullptr) {             // DA_POLICY_DYNAMIC: row (b, h) merges slots P_b .. P_b + s_b - 1
    const int b = row / p.h_q, h = row - b * p.h_q;
    prow = static_cast<int64_t>(__ldg(p.meta + b)) * p.h_q + h;
    s = __ldg(p.meta + p.batch + b);
    if (s == 1 && p.pub.out == nullptr) {   // one split: the forward wrote this row's out / lse itself
      if (p.pub.bases != nullptr && threadIdx.x == 0) pub_arrive(p.pub);
      return;
    }                                  // (LL exchange: the forward left it in the workspace, merged below)
  }
  DA_DASSERT(row < p.rows && s >= 1);
  const float* lse_in = p.lse_in + prow;
  const float4* o = reinterpret_cast<const float4*>(p.o + prow * kHeadDim) + lane;
  const int64_t ostride4 = p.o_stride / 4;

  // (1) warp w merges splits w, w + 4, ...: the lse and o loads of 8 splits are issued together
  //     (one L2 round trip for s <= 32), merged online against the warp's running maximum m
  //     (in log2 units); lane owns dims 4 lane .. 4 lane + 3.
  float m = kNegInf, Lw = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i0 = warp; i0 < s; i0 += kBatch * kWarps) {
    float li[kBatch];
    float4 oi[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int i = i0 + j * kWarps;
      li[j] = kNegInf;
      oi[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < s) {
        li[j] = __ldg(lse_in + i * p.lse_stride) * kLog2e;
        oi[j] = __ldg(o + i * ostride4);
      }
    }
    float mb = m;
#pragma unroll
    for (int j = 0; j < kBatch; ++j) mb = fmaxf(mb, li[j]);
    if (mb == kNegInf) continue;                           // every split so far empty
    const float r = ex2(m - mb);                           // m = -inf -> 0 (acc, Lw are 0)
    Lw *= r;
    acc = make_float4(acc.x * r, acc.y * r, acc.z * r, acc.w * r);
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const float wgt = ex2(li[j] - mb);                   // empty split or past s: 0
      Lw += wgt;
      acc.x = fmaf(wgt, oi[j].x, acc.x);
      acc.y = fmaf(wgt, oi[j].y, acc.y);
      acc.z = fmaf(wgt, oi[j].z, acc.z);
      acc.w = fmaf(wgt, oi[j].w, acc.w);
    }
    m = mb;
  }
  s_acc[warp][lane] = acc;
  if (lane == 0) { s_m[warp] = m; s_l[warp] = Lw; }
  __syncthreads();
  if (warp != 0) return;

  // (2) warp 0 merges the warps' (m, L, acc): M = max m_w, weights 2^(m_w - M)
  float M = kNegInf;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) M = fmaxf(M, s_m[w]);
  const bool empty = M == kNegInf;
  float L = 0.f;
  float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
  if (!empty) {
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float c = ex2(s_m[w] - M);                     // empty warp: 2^-inf = 0
      L = fmaf(c, s_l[w], L);
      const float4 a = s_acc[w][lane];
      sum.x = fmaf(c, a.x, sum.x);
      sum.y = fmaf(c, a.y, sum.y);
      sum.z = fmaf(c, a.z, sum.z);
      sum.w = fmaf(c, a.w, sum.w);
    }
  }
  const float inv = L > 0.f ? ptx::rcp(L) : 0.f;
  sum = make_float4(sum.x * inv, sum.y * inv, sum.z * inv, sum.w * inv);
  const float lse = empty ? kNegInf : (M + lg2(L)) * (1.f / kLog2e);
  if (p.pub.out != nullptr) {
    // da_forward_peer_combine: this row of this rank's partial goes out as LL words, the same words
    // of every rank are polled back and LSE-merged into the final row (the cross-rank combine in
    // the kernel that produces the row; the grid is co-resident, so the spinning is safe)
    const uint32_t e = pub_epoch(p.pub);
    pub_ll_store(p.pub, e, static_cast<size_t>(row), lane, sum, lse);
    __syncwarp();
    if (lane == 0) pub_count_advance(p.pub, e);
    pub_ll_merge_row(p.pub, e, static_cast<size_t>(row), lane);
    CTRACE(2);
    return;
  }
  // final rows: out / lse, or this step's slot of the exchange buffer (da_forward_peer)
  void* o_dst = p.out;
  float* l_dst = p.lse;
  if (p.pub.bases != nullptr) {
    const uint64_t sb = pub_slot(p.pub);
    o_dst = reinterpret_cast<void*>(sb);
    l_dst = reinterpret_cast<float*>(sb + static_cast<uint64_t>(p.pub.lse_offset));
  }
  if (p.out_f32) {
    reinterpret_cast<float4*>(o_dst)[static_cast<int64_t>(row) * (kHeadDim / 4) + lane] = sum;
  } else {
    uint2 w2;
    w2.x = pack_bf16(sum.x, sum.y);
    w2.y = pack_bf16(sum.z, sum.w);
    reinterpret_cast<uint2*>(o_dst)[static_cast<int64_t>(row) * (kHeadDim / 4) + lane] = w2;
  }
  if (lane == 0 && l_dst != nullptr) l_dst[row] = lse;
  if (p.pub.bases != nullptr) {
    __syncwarp();
    if (lane == 0) pub_arrive(p.pub);
  }
  CTRACE(2);
}

// ---- cross-GPU exchange over peer memory --------------------------------------
// Every rank owns a buffer mapped on every GPU (torch symmetric memory) with two partial slots
// (o fp32 [B, H_Q, d] at 0, lse fp32 [B, H_Q] at lse_offset within a slot of slot_bytes) and one
// uint32 flag per source rank at flag_offset.  The flags carry a step epoch (monotonic: no reset,
// CUDA-graph replayable); step e uses slot e & 1, so a rank that runs ahead overwrites the slot of
// step e - 1 only: every peer has finished reading it (it signalled step e after combining e - 1).

// One CTA: e = *epoch + 1; copy this rank's partial (written by the forward into local memory)
// into slot e & 1 of its own exchange buffer; fence (system scope); release e into slot `rank`
// of every peer's flags; *epoch = e.
__global__ void __launch_bounds__(256)
    peer_signal_kernel(const uint64_t* peer_bases, int32_t world, int32_t rank, const float* o_local,
                       const float* lse_local, int32_t rows, int64_t slot_bytes, int64_t lse_offset,
                       int64_t flag_offset, int32_t* epoch) {
  const uint32_t e = static_cast<uint32_t>(*epoch) + 1u;
  const uint64_t slot = peer_bases[rank] + static_cast<uint64_t>(slot_bytes) * (e & 1u);
  float4* dst = reinterpret_cast<float4*>(slot);
  const float4* src = reinterpret_cast<const float4*>(o_local);
  for (int i = threadIdx.x; i < rows * (kHeadDim / 4); i += blockDim.x) dst[i] = src[i];
  float* dl = reinterpret_cast<float*>(slot + static_cast<uint64_t>(lse_offset));
  for (int i = threadIdx.x; i < rows; i += blockDim.x) dl[i] = lse_local != nullptr ? lse_local[i] : kNegInf;
  __syncthreads();
  if (threadIdx.x != 0) return;
  fence_acq_rel_sys();                // + the strong stores below: one release pattern per flag
  for (int q = 0; q < world; ++q) {
    uint32_t* flags = reinterpret_cast<uint32_t*>(peer_bases[q] + static_cast<uint64_t>(flag_offset));
    st_relaxed_sys_u32(flags + rank, e);
  }
  *epoch = static_cast<int32_t>(e);
}

// One CTA (4 warps) per (b, h) row: warp 0 acquires every rank's flag at this step's epoch, then
// the row's P partials are read from the peers' buffers (NVLink loads, coherent: no __ldg) and
// merged exactly like lse_combine_kernel (per-warp online max, warp-level rescale merge).
__global__ void __launch_bounds__(kCombineThreads)
    peer_combine_kernel(const uint64_t* peer_bases, int64_t slot_bytes, int64_t lse_offset, int64_t flag_offset,
                        const int32_t* epoch, int32_t world, int32_t rank, int32_t rows, int32_t out_f32,
                        void* out, float* lse_out, int32_t* status, uint64_t timeout_ns) {
  constexpr int kWarps = kCombineThreads / 32;
  __shared__ float4 s_acc[kWarps][32];
  __shared__ float s_m[kWarps], s_l[kWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x;
  // the pointer table is set up once, before any step: read it while the producer drains, so the
  // step's dependent chain is epoch -> flags -> partials
  const uint64_t own = peer_bases[rank];
  const uint64_t first = warp < world ? peer_bases[warp] : 0;
  pdl_launch_dependents();
  pdl_wait();
  const uint32_t e = static_cast<uint32_t>(*epoch);
  if (warp == 0) {   // lane q polls rank q's flag (q, q + 32): the P acquires overlap
    const uint32_t* flags = reinterpret_cast<const uint32_t*>(own + static_cast<uint64_t>(flag_offset));
    for (int q = lane; q < world; q += 32) {
      if (ld_acquire_sys_u32(flags + q) >= e) continue;
      // bounded wait: a flag still behind timeout_ns after the first failed poll
      // records DA_ERR_TIMEOUT and ends the wait (the merge below then reads stale slots)
      const uint64_t t0 = globaltimer();
      while (ld_acquire_sys_u32(flags + q) < e) {
        if (*reinterpret_cast<const volatile int32_t*>(status) != 0) break;
        if (globaltimer() - t0 > timeout_ns) {
          atomicExch(status, static_cast<int32_t>(DA_ERR_TIMEOUT));
          break;
        }
      }
    }
  }
  __syncthreads();
  const uint64_t slot_off = static_cast<uint64_t>(slot_bytes) * (e & 1u);
  float m = kNegInf, Lw = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = warp; i < world; i += kWarps) {
    const uint64_t base = (i == warp ? first : peer_bases[i]) + slot_off;
    const float li = reinterpret_cast<const float*>(base + static_cast<uint64_t>(lse_offset))[row] * kLog2e;
    const float4 oi = reinterpret_cast<const float4*>(base)[static_cast<int64_t>(row) * (kHeadDim / 4) + lane];
    const float mb = fmaxf(m, li);
    if (mb == kNegInf) continue;                           // every partial so far empty
    const float r = ex2(m - mb), wgt = ex2(li - mb);
    Lw = fmaf(Lw, r, wgt);
    acc = make_float4(fmaf(acc.x, r, wgt * oi.x), fmaf(acc.y, r, wgt * oi.y), fmaf(acc.z, r, wgt * oi.z),
                      fmaf(acc.w, r, wgt * oi.w));
    m = mb;
  }
  s_acc[warp][lane] = acc;
  if (lane == 0) { s_m[warp] = m; s_l[warp] = Lw; }
  __syncthreads();
  if (warp != 0) return;
  float M = kNegInf;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) M = fmaxf(M, s_m[w]);
  const bool empty = M == kNegInf;
  float L = 0.f;
  float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
  if (!empty) {
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float c = ex2(s_m[w] - M);
      L = fmaf(c, s_l[w], L);
      const float4 a = s_acc[w][lane];
      sum = make_float4(fmaf(c, a.x, sum.x), fmaf(c, a.y, sum.y), fmaf(c, a.z, sum.z), fmaf(c, a.w, sum.w));
    }
  }
  const float inv = L > 0.f ? ptx::rcp(L) : 0.f;
  sum = make_float4(sum.x * inv, sum.y * inv, sum.z * inv, sum.w * inv);
  DA_DASSERT(row < rows);
  if (out_f32) {
    reinterpret_cast<float4*>(out)[static_cast<int64_t>(row) * (kHeadDim / 4) + lane] = sum;
  } else {
    uint2 w2;
    w2.x = pack_bf16(sum.x, sum.y);
    w2.y = pack_bf16(sum.z, sum.w);
    reinterpret_cast<uint2*>(out)[static_cast<int64_t>(row) * (kHeadDim / 4) + lane] = w2;
  }
  if (lane == 0 && lse_out != nullptr) lse_out[row] = empty ? kNegInf : (M + lg2(L)) * (1.f / kLog2e);
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

#ifdef DECATTN_TRACE
extern "C" __attribute__((visibility("default"))) int da_trace_fetch_combine(unsigned long long* host, int n) {
  if (n > 64 * 4) n = 64 * 4;
  return cudaMemcpyFromSymbol(host, g_trace_comb, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 1;
}
#endif

cudaError_t launch_peer_signal(const uint64_t* peer_bases, int32_t world, int32_t rank, const float* o_local,
                               const float* lse_local, int32_t rows, int64_t slot_bytes, int64_t lse_offset,
                               int64_t flag_offset, int32_t* epoch, cudaStream_t stream) {
  peer_signal_kernel<<<1, 256, 0, stream>>>(peer_bases, world, rank, o_local, lse_local, rows, slot_bytes,
                                            lse_offset, flag_offset, epoch);
  return cudaGetLastError();
}

cudaError_t launch_peer_combine(const uint64_t* peer_bases, int64_t slot_bytes, int64_t lse_offset,
                                int64_t flag_offset, const int32_t* epoch, int32_t world, int32_t rank, int32_t rows,
                                int32_t out_f32, void* out, float* lse, int32_t* status, uint64_t timeout_ns,
                                cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(rows, 1, 1);
  cfg.blockDim = dim3(kCombineThreads, 1, 1);
  cfg.stream = stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, peer_combine_kernel, peer_bases, slot_bytes, lse_offset, flag_offset, epoch,
                            world, rank, rows, out_f32, out, lse, status, timeout_ns);
}

cudaError_t combine_residency(int* out) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  if ((err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return err;
  if ((err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lse_combine_kernel, kCombineThreads, 0)) !=
      cudaSuccess)
    return err;
  *out = per_sm * sms;
  return cudaSuccess;
}

}  // namespace decattn
