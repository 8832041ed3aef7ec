// Split-KV decode-attention forward for sm_100a.
//
// One CTA = one (split, head-group, batch) work unit; grid = (s, Y, B) with
// Y = H_KV * ceil(G / rows) on the pack_gqa tensor-core path or Y = H_Q on
// the scalar path.  The s CTAs of a head-group partition its sequence
// ("num_splits ... sequence-level parallelization across SMs", §3.1),
// so s is exactly the paper's knob: s = 1 launches B*H_KV CTAs ("as few as 8
// Thread Blocks"), s = 3 triples them.
// DA_POLICY_DYNAMIC (kDyn, C-ext-2): grid = (Y, slots, 1); the (sequence, split)
// of a slot is derived on the device from cache_seqlens (dyn_schedule).
//
// Inside a CTA, NS ring stages and NW consumer warps per combine
// mode (config.h: NONE 7 / 7, CLUSTER 6 / 3 + 4 helper warps, KERNEL 4 / 4):
//   warp NW     TMA producer: one lane streams 64-token tiles, one 5-D box for K
//               and one for V (64 tokens x 2 x 64 dims, 128B-swizzled, 32 KB per
//               stage) through the mbarrier ring (step a3, KV streaming).
//   warps 0..NW-1  consumers: warp w owns ring stages w, w+NW, ... (tiles w,
//               w+NW, ...) and keeps its own online-softmax state (a4-a6):
//               MMA path  S^T = K Q^T and O^T += V^T P^T with
//                         mma.sync.m16n8k16 (bf16 -> fp32): tokens and head
//                         dims fill the M = 16 side, the G query rows the
//                         N = 8 side, so no MMA lane is padding for G = 8;
//                         P^T is re-laid out register-to-register with
//                         movmatrix.trans and enters the PV product as the
//                         bf16 pair P_hi + P_lo (two MMAs).
//               scalar    lane-per-token fp32 dot products, warp-shuffle
//                         max / sum, lane-per-4-dims PV.
//   helpers     (CLUSTER) idle through the main loop, then join the merges.
//   epilogue    the consumer warps' (m, l, O) merge in shared memory; then
//               NONE     : bf16/fp32 out + lse written directly (a7);
//               CLUSTER  : the s CTAs form one thread-block cluster; row g is
//                          owned by rank g mod s, every rank st.async-pushes
//                          its (m, l, O) of g into the owner's shared memory
//                          (bytes counted on the owner's mbarrier) and the
//                          owner does the LSE combine (a8): no workspace, no
//                          second launch, no cluster-wide barrier on exit;
//               KERNEL   : normalised fp32 partials + lse go to the
//                          workspace for lse_combine_kernel (combine.cu).
//   kPub (sequence-sharded steps, pub.cuh): 1 = the final rows go to this
//               rank's exchange slot and the last CTA releases the epoch
//               (da_forward_peer); 2 = the rows go out as LL words, every CTA
//               polls the same words of every rank and LSE-merges them into
//               the final out / lse (da_forward_peer_combine: one kernel).
// Programmatic dependent launch: the prologue overlaps the previous kernel's
// tail; griddepcontrol.wait precedes the first global read.  Scores are kept in
// the log2 domain; lse is returned in natural log (C-amb-10).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "config.h"
#include "internal.h"
#include "ptx.cuh"
#include "pub.cuh"
#include "tile_common.cuh"

namespace decattn {

using namespace ptx;

namespace {


// ---- development timeline tracing (only in -DDECATTN_TRACE builds; no-op otherwise) ----
#ifdef DECATTN_TRACE
__device__ unsigned long long g_trace[64 * 64];
__device__ unsigned long long g_prev_end;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int trace_cta() { return (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x; }
#define TRACE(slot) do { const int c_ = trace_cta(); if (c_ < 64) g_trace[c_ * 64 + (slot)] = gtime(); } while (0)
// timestamp once the value v has been produced (the compare waits for it)
#define TRACE_DEP(slot, v, on) do { if ((on) && __float_as_uint(v) != 0x7fc0beefu) TRACE(slot); } while (0)
#else
#define TRACE(slot) do { } while (0)
#define TRACE_DEP(slot, v, on) do { } while (0)
#endif
constexpr int kEpiStride = kHeadDim + 4;     // fp32 row stride of epilogue buffers (bank spread)

// ---------------------------------------------------------------------------
// MMA path: one 64-token tile for one warp.  sK / sV: smem addresses of the
// K / V half-0 boxes (half 1 follows at +8 KB).  Box layout: row r (token)
// at r*128 B, 16-byte chunk c at ((c ^ (r & 7)) * 16)  (TMA SWIZZLE_128B).
// ---------------------------------------------------------------------------
template <int NB>
__device__ __forceinline__ void mma_tile(uint32_t sK, uint32_t sV, int valid,
                                         const uint32_t (&qf)[8][NB][2], float (&o)[8][NB][4],
                                         float (&m)[NB][2], float (&l)[NB][2], float scale_log2,
                                         int lane, uint32_t vbar, uint32_t vparity, bool tr = false) {
  const uint32_t sw = static_cast<uint32_t>(lane & 7);
  tr = tr && lane == 0;                                    // trace builds: time the steps of this tile
  // ---- S^T[token, g] = sum_d K[token, d] Q[g, d]  (4 token blocks x NB g-blocks)
  float s[4][NB][4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int c = 0; c < 4; ++c) s[j][nb][c] = 0.f;

  {
    // A operand = K rows: lane provides row (lane & 7) + 8*((lane >> 3) & 1), k-chunk lane >> 4.
    const uint32_t row_off = static_cast<uint32_t>(((lane & 7) + ((lane >> 3) & 1) * 8) * 128);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t chunk = static_cast<uint32_t>(((kk & 3) << 1) + (lane >> 4));
      const uint32_t base = sK + (kk >> 2) * kHalfBytes + row_off + ((chunk ^ sw) << 4);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t a0, a1, a2, a3;
        ldmatrix_x4(base + j * 16 * 128, a0, a1, a2, a3);
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) mma_bf16_16816(s[j][nb], a0, a1, a2, a3, qf[kk][nb][0], qf[kk][nb][1]);
      }
    }
  }

  TRACE_DEP(32, s[0][0][0] + s[3][NB - 1][3], tr);       // QK^T done
  // ---- online softmax over the tile's tokens, per query row g (a5)
  // C layout: s[j][nb][c] holds token 16j + (lane >> 2) + 8*(c >> 1), g = 8nb + 2(lane & 3) + (c & 1).
  float mx[NB][2];
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) mx[nb][0] = mx[nb][1] = kNegInf;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int tok = 16 * j + (lane >> 2);
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int t = tok + 8 * (c >> 1);
        s[j][nb][c] = t < valid ? s[j][nb][c] * scale_log2 : kNegInf;
        mx[nb][c & 1] = fmaxf(mx[nb][c & 1], s[j][nb][c]);
      }
    }
  }
#pragma unroll
  for (int nb = 0; nb < NB; ++nb)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float v = mx[nb][c];
      v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 4));
      v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 8));
      v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 16));
      const float m_new = fmaxf(m[nb][c], v);           // finite: the tile has >= 1 valid token
      const float alpha = ex2(m[nb][c] - m_new);        // m_old = -inf -> 0
      m[nb][c] = m_new;
      l[nb][c] *= alpha;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        o[i][nb][c] *= alpha;
        o[i][nb][c + 2] *= alpha;
      }
    }

  // P = exp2(S - m) as an unevaluated sum of two bf16 terms, P = P_hi + P_lo with
  // P_hi = bf16(P) and P_lo = bf16(P - P_hi): the PV product then carries ~16 mantissa bits
  // of P instead of 8 (a single bf16 P is off by up to 2^-9 relative per weight, which short
  // sequences with cancelling V rows turn into > 2e-3 absolute error).  Each 8x8 block is
  // transposed so P^T's C layout becomes the B-operand layout of the PV product.
  uint32_t pb[4][NB][2], pl[4][NB][2];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      float p[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        p[c] = ex2(s[j][nb][c] - m[nb][c & 1]);         // masked: exp2(-inf) = 0
        l[nb][c & 1] += p[c];
      }
      const uint32_t h01 = pack_bf16(p[0], p[1]), h23 = pack_bf16(p[2], p[3]);
      pb[j][nb][0] = movmatrix_trans(h01);
      pb[j][nb][1] = movmatrix_trans(h23);
      pl[j][nb][0] = movmatrix_trans(pack_bf16(p[0] - bf16lo(h01), p[1] - bf16hi(h01)));
      pl[j][nb][1] = movmatrix_trans(pack_bf16(p[2] - bf16lo(h23), p[3] - bf16hi(h23)));
    }

  TRACE_DEP(33, __uint_as_float(pl[3][NB - 1][1] ^ pb[0][0][0]), tr);   // softmax + P done
  // ---- V: wait for its half of the stage (it lands while QK^T and the softmax run); rows past
  // the range may hold anything (even NaN): zero them so the P = 0 rows stay 0
  mbar_wait(vbar, vparity);
  if (tr) TRACE(34);                                       // V landed
  if (valid < kTileN) {
    for (int idx = lane; idx < (kTileN - valid) * 16; idx += 32) {
      const int r = valid + (idx >> 4);
      const int c = idx & 15;
      sts128(sV + (c >> 3) * kHalfBytes + r * 128 + (c & 7) * 16, make_uint4(0, 0, 0, 0));
    }
    __syncwarp();
  }

  // ---- O^T[d, g] += sum_token V^T[d, token] P^T[token, g]   (8 d-blocks x 4 token blocks)
  {
    // A operand = V^T via ldmatrix.trans: lane provides token row (lane & 7) + 8*(lane >> 4),
    // d-chunk 2i + ((lane >> 3) & 1).
    const uint32_t row_off = static_cast<uint32_t>(((lane & 7) + (lane >> 4) * 8) * 128);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t chunk = static_cast<uint32_t>(((2 * i) & 7) + ((lane >> 3) & 1));
      const uint32_t base = sV + (i >> 2) * kHalfBytes + row_off + ((chunk ^ sw) << 4);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t a0, a1, a2, a3;
        ldmatrix_x4_trans(base + j * 16 * 128, a0, a1, a2, a3);
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
          mma_bf16_16816(o[i][nb], a0, a1, a2, a3, pb[j][nb][0], pb[j][nb][1]);
          mma_bf16_16816(o[i][nb], a0, a1, a2, a3, pl[j][nb][0], pl[j][nb][1]);
        }
      }
    }
  }
  TRACE_DEP(35, o[0][0][0] + o[7][NB - 1][3], tr);        // PV done
}

// ---------------------------------------------------------------------------
// Scalar path: one 64-token tile for one warp, one query row.  Lane t scores
// tokens t and t + 32; lane owns head dims 4*lane .. 4*lane + 3 of O.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void scalar_tile(uint32_t sK, uint32_t sV, int valid, const uint4 (&qv)[16],
                                            float (&o)[4], float& m, float& l, float scale_log2,
                                            int lane) {
  float sc[2];
#pragma unroll
  for (int tt = 0; tt < 2; ++tt) {
    const int r = lane + 32 * tt;
    const uint32_t row = sK + static_cast<uint32_t>(r * 128);
    const uint32_t sw = static_cast<uint32_t>(r & 7);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 kv = lds128(row + h * kHalfBytes + ((static_cast<uint32_t>(c) ^ sw) << 4));
        const uint4 qq = qv[h * 8 + c];
        acc[0] = fmaf(bf16lo(kv.x), bf16lo(qq.x), acc[0]);
        acc[1] = fmaf(bf16hi(kv.x), bf16hi(qq.x), acc[1]);
        acc[2] = fmaf(bf16lo(kv.y), bf16lo(qq.y), acc[2]);
        acc[3] = fmaf(bf16hi(kv.y), bf16hi(qq.y), acc[3]);
        acc[0] = fmaf(bf16lo(kv.z), bf16lo(qq.z), acc[0]);
        acc[1] = fmaf(bf16hi(kv.z), bf16hi(qq.z), acc[1]);
        acc[2] = fmaf(bf16lo(kv.w), bf16lo(qq.w), acc[2]);
        acc[3] = fmaf(bf16hi(kv.w), bf16hi(qq.w), acc[3]);
      }
    const float dot = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    sc[tt] = r < valid ? dot * scale_log2 : kNegInf;
  }
  float mx = fmaxf(sc[0], sc[1]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  const float m_new = fmaxf(m, mx);
  const float alpha = ex2(m - m_new);
  m = m_new;
  const float p0 = ex2(sc[0] - m_new), p1 = ex2(sc[1] - m_new);
  l = l * alpha + (p0 + p1);
#pragma unroll
  for (int e = 0; e < 4; ++e) o[e] *= alpha;

  // PV over the valid tokens: row t, 8 bytes at dims 4*lane.
  const uint32_t half = static_cast<uint32_t>(lane >> 4);
  const uint32_t chunk = static_cast<uint32_t>((lane & 15) >> 1);
  const uint32_t vcol = sV + half * kHalfBytes + static_cast<uint32_t>((lane & 1) * 8);
#pragma unroll 4
  for (int t = 0; t < valid; ++t) {
    const float pt = __shfl_sync(0xffffffffu, t < 32 ? p0 : p1, t & 31);
    const uint2 vv = lds64(vcol + static_cast<uint32_t>(t * 128) + ((chunk ^ static_cast<uint32_t>(t & 7)) << 4));
    o[0] = fmaf(pt, bf16lo(vv.x), o[0]);
    o[1] = fmaf(pt, bf16hi(vv.x), o[1]);
    o[2] = fmaf(pt, bf16lo(vv.y), o[2]);
    o[3] = fmaf(pt, bf16hi(vv.y), o[3]);
  }
}

// DA_POLICY_DYNAMIC (C-ext-2, oracle/policy.py dynamic_schedule): one warp derives the per-batch
// split counts from the lengths - W = max(1, ceil(sum_b n_u_b * T_b / U)), s_b = min(cap,
// max(1, floor(n_u_b / W))), first slot P_b = s_0 + ... + s_{b-1} - and returns the (sequence,
// split, s_b, length) that split slot `slot` serves, or x = -1 for an unused slot.  Every CTA
// runs the same integer arithmetic; the CTA of slot 0, head group 0 records (P_b, s_b) for the
// combine kernel.
constexpr int kDynScratch = kStageBytes / 4;   // sequences whose unit count is cached in shared memory

__device__ __forceinline__ int dyn_len(const FwdParams& p, int b) {
  return min(max(p.seqlens != nullptr ? (max(__ldg(p.seqlens + b), 0) - p.seq_offset) : p.l_default, 0), p.l_cap);
}

__device__ __noinline__ int4 dyn_schedule(const FwdParams& p, uint32_t slot, bool record, int lane,
                                          int* lens) {
  // lens: shared-memory scratch (the ring, idle until the first TMA) holding n_b for b < kDynScratch
  const int B = p.batch;
  uint32_t tot = 0;
#pragma unroll 4
  for (int b0 = 0; b0 < B; b0 += 32) {
    const int bb = b0 + lane;
    if (bb < B) {
      const int n = dyn_len(p, bb);
      if (bb < kDynScratch) lens[bb] = n;
      tot += (static_cast<uint32_t>(n) + (kTileN - 1)) / kTileN;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
  const uint32_t T = static_cast<uint32_t>(p.dyn_tiles), U = static_cast<uint32_t>(p.dyn_u);
  uint32_t W;
  if (tot <= 0xffffffffu / T) {                        // the common case: a 32-bit quotient
    W = (tot * T + U - 1) / U;
  } else {
    W = static_cast<uint32_t>((static_cast<uint64_t>(tot) * T + U - 1) / U);
  }
  W = max(W, 1u);
  const uint32_t cap = static_cast<uint32_t>(p.num_splits);
  int4 mine = make_int4(-1, 0, 0, 0);
  uint32_t base = 0;
  for (int b0 = 0; b0 < B; b0 += 32) {
    const int bb = b0 + lane;
    uint32_t sb = 0;
    int n = 0;
    if (bb < B) {
      n = bb < kDynScratch ? lens[bb] : dyn_len(p, bb);
      sb = min(max(((static_cast<uint32_t>(n) + (kTileN - 1)) / kTileN) / W, 1u), cap);
    }
    uint32_t inc = sb;                                  // inclusive warp scan of s_b
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, inc, off);
      if (lane >= off) inc += v;
    }
    const uint32_t first = base + inc - sb;
    if (bb < B) {
      if (record) {
        p.ws_meta[bb] = static_cast<int32_t>(first);
        p.ws_meta[B + bb] = static_cast<int32_t>(sb);
      }
      if (slot >= first && slot < first + sb) mine = make_int4(bb, static_cast<int>(slot - first), static_cast<int>(sb), n);
    }
    base += __shfl_sync(0xffffffffu, inc, 31);
  }
  const unsigned hit = __ballot_sync(0xffffffffu, mine.x >= 0);   // at most one lane matches
  const int src = hit ? __ffs(hit) - 1 : 0;
  int4 r;
  r.x = hit ? __shfl_sync(0xffffffffu, mine.x, src) : -1;
  r.y = __shfl_sync(0xffffffffu, mine.y, src);
  r.z = __shfl_sync(0xffffffffu, mine.z, src);
  r.w = __shfl_sync(0xffffffffu, mine.w, src);
  return r;
}

// ---------------------------------------------------------------------------
// The kernel.  kPath: DA_PATH_SCALAR / DA_PATH_MMA; kNB: g-blocks of 8 query
// rows (MMA path); kCombine: da_combine_mode; NS: ring stages; NW: consumer warps
// (NS a multiple of NW: warp w owns stages w, w + NW, ... and consumes them in order).
// ---------------------------------------------------------------------------
template <int kPath, int kNB, int kCombine, int NS, int NW, bool kDyn, int kPub, bool kBal, bool kPaged>
__global__ void __launch_bounds__(threads_for(NW, helpers_for(kCombine)), 1)
    split_kv_fwd_kernel(const __grid_constant__ CUtensorMap tmap_k,
                        const __grid_constant__ CUtensorMap tmap_v, const FwdParams p) {
  static_assert(NS % NW == 0, "each consumer warp must own whole ring stages");
  static_assert(!kDyn || kCombine == DA_COMBINE_KERNEL, "dynamic split counts use the workspace combine");
  constexpr int kT = threads_for(NW, helpers_for(kCombine));   // consumers + producer + helpers
  constexpr int R = kPath == DA_PATH_MMA ? 8 * kNB : 1;    // query rows of this CTA
  constexpr int kIters = (R * 32 + kT - 1) / kT;           // merge passes: element = (row, float4)
  constexpr bool kCluster = kCombine == DA_COMBINE_CLUSTER;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[NS];    // K of the stage has landed
  __shared__ __align__(8) uint64_t fullv_bar[NS];   // V of the stage has landed (QK^T need not wait)
  __shared__ __align__(8) uint64_t empty_bar[NS];
  __shared__ __align__(8) uint64_t push_bar;              // CLUSTER: pushes of the rows this CTA owns
  // tail balancing (cluster plans with long splits): the tile each ring stage holds, written by the
  // producer before it arms the stage (-1: no more tiles for the warp that owns the stage), and the
  // cluster's ticket counter for the pooled tail chunks (rank 0's copy is the one used)
  // (a separate instantiation, kBal: launched only when some sequence can be long enough, so the
  // latency-regime cluster plans run without the balancing code - it cost them 5 %)
  constexpr bool kBalCapable = kCluster && !kDyn && kPub == 0 && kBal;
  __shared__ int stage_tile[kBalCapable ? NS : 1];
  __shared__ uint32_t bal_next;

  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  float* const epi = reinterpret_cast<float*>(smem_raw + (sbase - raw));
  // epilogue carve-up (aliases the ring once every tile is consumed)
  float* const epi_o = epi;                                          // [NW][16][kEpiStride]
  float2* const epi_ml = reinterpret_cast<float2*>(epi_o + NW * 16 * kEpiStride);  // [NW][16] (m, l)
  // CLUSTER push slots, past the ring (peers write them while this CTA may still stream):
  // [source slot 0..s-2][owned row 0..ceil(R/s)-1][kSlotRowFloats]
  float* const slots = epi + NS * kStageBytes / 4;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // kDyn: blockIdx.x is the head group and blockIdx.y the split slot, so that consecutive CTAs
  // read the heads of one sequence (shared DRAM rows, like the static (split, group, batch) order)
  const int grp = kDyn ? blockIdx.x : blockIdx.y;
  const uint32_t dslot = kDyn ? blockIdx.y : 0u;
  int split = blockIdx.x, b = blockIdx.z;       // kDyn: assigned from the schedule below
  // batch index of the K / V cache and cache_seqlens: b, except under multi-rank emulation
  // (kPub == 2, tests on one GPU), where z spans every rank's batch and the rank's shard sits at
  // cache batch z while q / out use b = z mod B
  int bkv = blockIdx.z, erank = 0;
  if constexpr (kPub == 2) {
    if (p.pub.emulate) {
      erank = blockIdx.z / p.batch;
      b = blockIdx.z - erank * p.batch;
    }
  }
  bool dyn_single = false;                       // kDyn: this sequence has one split (s_b = 1)
  int kvh, hq0, rows_valid;
  if constexpr (kPath == DA_PATH_MMA) {
    kvh = static_cast<int>(udiv_magic(static_cast<uint32_t>(grp), p.mb_magic));
    const int rg = grp - kvh * p.mblocks_per_head;
    hq0 = kvh * p.G + rg * R;
    rows_valid = min(R, p.G - rg * R);
  } else {
    hq0 = grp;
    kvh = hq0 / p.G;
    rows_valid = 1;
  }
  DA_DASSERT(rows_valid >= 1 && hq0 + rows_valid <= p.h_q && kvh * p.G <= hq0);
  DA_DASSERT(!kCluster || (p.num_splits >= 2 && p.num_splits <= kMaxClusterSplits));
  // CLUSTER: rank r owns rows g = r, r + s, r + 2s, ... and emits them
  const int s_cl = kCluster ? p.num_splits : 1;
  const uint32_t rank = kCluster ? cluster_ctarank() : 0u;
  const int rows_per_owner = kCluster ? static_cast<int>(udiv_magic(R + s_cl - 1, p.s_magic)) : R;

  if (threadIdx.x == 0) TRACE(0);
#ifdef DECATTN_TRACE
  if (threadIdx.x == 0 && trace_cta() < 64) g_trace[trace_cta() * 64 + 60] = clock64();
#endif
  if (threadIdx.x == 0) {
#pragma unroll 1
    for (int i = 0; i < NS; ++i) {
      mbar_init(smem_u32(&full_bar[i]), 1);
      mbar_init(smem_u32(&fullv_bar[i]), 1);
      mbar_init(smem_u32(&empty_bar[i]), 1);
    }
    if constexpr (kBalCapable) bal_next = 0u;
    if constexpr (kCluster) {
      // expect s pushes (every rank, this one included) of (O row, m, l) for every valid row
      // this rank owns, counted in st.async bytes
      const int owned = rows_valid > static_cast<int>(rank)
          ? static_cast<int>(udiv_magic(rows_valid - 1 - static_cast<int>(rank), p.s_magic)) + 1 : 0;
      mbar_init(smem_u32(&push_bar), 1);
      mbar_arrive_expect_tx(smem_u32(&push_bar), static_cast<uint32_t>(s_cl * owned * (kHeadDim * 4 + 8)));
    }
    fence_mbarrier_init();
  }
  if (warp == NW && lane == 0) {
    prefetch_tmap(&tmap_k);
    prefetch_tmap(&tmap_v);
    // the lengths are read right after griddepcontrol.wait: pull their line into L2 now (a
    // prefetch never returns data, so it cannot observe a stale value)
    if (!kDyn && p.seqlens != nullptr) prefetch_l2(p.seqlens + bkv);
  }
  if (kDyn && warp == NW && p.seqlens != nullptr && lane * 32 < p.batch)
    prefetch_l2(p.seqlens + lane * 32);          // the first 1024 lengths, one 128-byte line per lane
  __syncthreads();
  if constexpr (kCluster) cluster_arrive_relaxed();   // "my push barrier is initialised"

  // ---- this split's token range (C-pol item 6), in units of kTileN tokens.  With uniform
  // lengths (cache_seqlens == NULL) it depends on no global value, so it is computed before
  // griddepcontrol.wait and the producer issues the first TMA the moment the wait returns.
  int t0 = 0, t_end = 0, n_tiles = 0;
  if constexpr (!kDyn) {
    // the range at the plan's length: exact when cache_seqlens == NULL; with cache_seqlens it is
    // only a guess for the prefetch below (the lengths may still be written by the preceding
    // kernel, so they are read after the wait and the range recomputed there)
    split_range(min(max(p.l_default, 0), p.l_cap), split, p.num_splits, p.s_magic, t0, t_end, n_tiles);
    // paged cache: the block table may still be written by the preceding kernel, so the values
    // read here only steer L2 prefetches of the pages the ring loads first (a stale or torn entry
    // costs a useless prefetch; out-of-range pages are clipped by the tensor map); the producer
    // re-reads the table after the wait for the loads themselves
    if (kPaged && warp == NW && lane == 0 && n_tiles >= 1 && n_tiles <= 2 * NS) {
      const int32_t* bt = p.block_table + static_cast<int64_t>(b) * p.bt_stride;
      const uint32_t tpp = static_cast<uint32_t>(p.page_size / kTileN);
      const uint32_t tile0 = static_cast<uint32_t>(t0 / kTileN);
      uint32_t j = udiv_magic(tile0, p.page_magic), k = tile0 - j * tpp;
      const int np = min(n_tiles, NS);
      for (int i = 0; i < np; ++i) {
        const int page = *reinterpret_cast<const volatile int32_t*>(bt + j);
        tma_prefetch_5d(&tmap_k, 0, static_cast<int>(k) * kTileN, 0, kvh, page);
        tma_prefetch_5d(&tmap_v, 0, static_cast<int>(k) * kTileN, 0, kvh, page);
        if (++k == tpp) { k = 0; ++j; }
      }
    }
    // pull the tiles the ring loads first into L2 while the previous kernel drains; L2 is the point
    // of coherence, so the loads after griddepcontrol.wait still see the preceding kernel's writes
    // (latency regime: Llama 3.57 -> 3.12 us; streaming splits: the DRAM idles less between
    // kernels).  A wrong guess only costs DRAM reads.
    if (DECATTN_SPECULATE || p.seqlens == nullptr) {
      if (warp == NW && lane == 0 && n_tiles >= 1 && (DECATTN_PREFETCH_LONG || n_tiles <= 2 * NS) &&
          !kPaged) {
        const int np = min(n_tiles, NS);
        // (single-thread issue loops stay rolled here and below: the latency-bound launches pay
        // for every instruction they fetch)
#pragma unroll 1
        for (int i = 0; i < np; ++i) tma_prefetch_5d(&tmap_k, 0, t0 + i * kTileN, 0, kvh, bkv);
#pragma unroll 1
        for (int i = 0; i < np; ++i) tma_prefetch_5d(&tmap_v, 0, t0 + i * kTileN, 0, kvh, bkv);
      }
    }
  }

  // Let the next kernel in the stream start its prologue now (it waits in its own
  // griddepcontrol.wait for this grid to finish), then wait for our inputs, which
  // the preceding kernel may still be writing.
  pdl_launch_dependents();
  pdl_wait();
#ifdef DECATTN_TRACE
  if (threadIdx.x == 0) {
    TRACE(1);
    const int c_ = trace_cta();
    if (c_ < 64) g_trace[c_ * 64 + 63] = *(volatile unsigned long long*)&g_prev_end;
  }
#endif
  if constexpr (kDyn) {
    __shared__ int4 sched;
    if (warp == 0) {
      const int4 r = dyn_schedule(p, dslot, dslot == 0 && grp == 0 && p.ws_meta != nullptr,
                                  lane, reinterpret_cast<int*>(epi));
      if (lane == 0) sched = r;
    }
    __syncthreads();
    const int4 r = sched;
    if (r.x < 0) return;                          // unused slot (the launch provides an upper bound)
    b = r.x;
    bkv = b;                                      // the sequence's cache batch and length index
    split = r.y;
    dyn_single = r.z == 1;
    // split r.y of r.z over n = r.w tokens; (split + 1) n_u < 2^32 since r.z <= 128, n_u < 2^25
    const uint32_t nu = (static_cast<uint32_t>(r.w) + (kTileN - 1)) / kTileN;
    const uint32_t u0 = static_cast<uint32_t>(r.y) * nu / static_cast<uint32_t>(r.z);
    const uint32_t u1 = static_cast<uint32_t>(r.y + 1) * nu / static_cast<uint32_t>(r.z);
    t0 = static_cast<int>(u0) * kTileN;
    t_end = min(static_cast<int>(u1) * kTileN, r.w);
    n_tiles = static_cast<int>(u1 - u0);
  } else if (p.seqlens != nullptr) {
    split_range(min(max((max(__ldg(p.seqlens + bkv), 0) - p.seq_offset), 0), p.l_cap), split, p.num_splits, p.s_magic, t0, t_end, n_tiles);
  }
  // tail balancing (kBalCapable): every split of this sequence holds >= kBalMinTiles tiles (uniform
  // over the cluster: one sequence, one length); n_seq = the sequence's length
  bool bal = false;
  int n_seq = 0, tail_chunks = 0;
  if constexpr (kBalCapable) {
    n_seq = min(max(p.seqlens != nullptr ? (max(__ldg(p.seqlens + bkv), 0) - p.seq_offset) : p.l_default, 0), p.l_cap);
    const int nu = (n_seq + kTileN - 1) / kTileN;
    bal = !kPaged && nu >= kBalMinTiles * p.num_splits;
    tail_chunks = nu / p.num_splits / kBalTailDiv / kBalChunk;   // pooled chunks per split (>= 2)
  }

  if (warp == NW) {
    // ================= TMA producer =================
    if constexpr (kBalCapable) {
      if (bal) cluster_wait();       // rank 0's ticket counter is initialised (the epilogue skips it)
    }
    if (lane == 0) {
      if (kBalCapable && bal) {
        // the head of this split's range, [t0, t_end - pooled tail), then pooled tail chunks: ticket j
        // is chunk k = j mod tc of split i = j / tc's tail, the tickets fetched one chunk ahead; a
        // ticket past the pool ends the CTA's share
        const int tc = tail_chunks, s_ = p.num_splits, nu = (n_seq + kTileN - 1) / kTileN;
        const int q = nu / s_, r = nu - q * s_;
        const int head_end = n_tiles - tc * kBalChunk;      // tiles of the head
        const uint32_t tkt = mapa(smem_u32(&bal_next), 0);
        int i = 0;
        auto issue = [&](int tile) {
          const int st = i % NS;
          if (i >= NS) mbar_wait(smem_u32(&empty_bar[st]), ((i / NS) - 1) & 1);
          stage_tile[st] = tile;
          const uint32_t fb = smem_u32(&full_bar[st]), fvb = smem_u32(&fullv_bar[st]);
          mbar_arrive_expect_tx(fb, kStageBytes / 2);
          mbar_arrive_expect_tx(fvb, kStageBytes / 2);
          const uint32_t dst = sbase + st * kStageBytes;
          tma_load_5d(dst, &tmap_k, fb, 0, tile * kTileN, 0, kvh, bkv);
          tma_load_5d(dst + 2 * kHalfBytes, &tmap_v, fvb, 0, tile * kTileN, 0, kvh, bkv);
          if (i < 8) TRACE(2 + i);
          ++i;
        };
        const int tile0 = t0 / kTileN;
        for (int t = 0; t < head_end; ++t) issue(tile0 + t);
        const uint32_t pool = static_cast<uint32_t>(s_ * tc);
        uint32_t jn = atom_add_cluster(tkt, 1u);
        while (jn < pool) {
          const int j = static_cast<int>(jn);
          jn = atom_add_cluster(tkt, 1u);                    // the next ticket, in flight
          const int si = j / tc, k = j - si * tc;
          const int u1 = (si + 1) * q + ((si + 1) * r) / s_;  // end of split si's range (split_range)
          const int c0 = u1 - (tc - k) * kBalChunk;
          for (int c = 0; c < kBalChunk; ++c) issue(c0 + c);
        }
        // every consumer warp's next stage says "no more tiles"
        for (int w = 0; w < NW; ++w) {
          const int st = i % NS;
          if (i >= NS) mbar_wait(smem_u32(&empty_bar[st]), ((i / NS) - 1) & 1);
          stage_tile[st] = -1;
          mbar_arrive(smem_u32(&full_bar[st]));
          ++i;
        }
      } else if (!kPaged && n_tiles <= NS) {
        // latency regime (every tile has its own stage): all K boxes first, then all V boxes, so
        // every consumer starts QK^T one V box earlier than in tile order
#pragma unroll 1
        for (int i = 0; i < n_tiles; ++i) {
          const uint32_t fb = smem_u32(&full_bar[i]);
          mbar_arrive_expect_tx(fb, kStageBytes / 2);
          tma_load_5d(sbase + i * kStageBytes, &tmap_k, fb, 0, t0 + i * kTileN, 0, kvh, bkv);
          if (i < 8) TRACE(2 + i);
        }
#pragma unroll 1
        for (int i = 0; i < n_tiles; ++i) {
          const uint32_t fvb = smem_u32(&fullv_bar[i]);
          mbar_arrive_expect_tx(fvb, kStageBytes / 2);
          tma_load_5d(sbase + i * kStageBytes + 2 * kHalfBytes, &tmap_v, fvb, 0, t0 + i * kTileN, 0, kvh, bkv);
        }
      } else if (!kPaged) {
#pragma unroll 1
        for (int i = 0; i < n_tiles; ++i) {
          const int st = i % NS;
          if (i >= NS) mbar_wait(smem_u32(&empty_bar[st]), ((i / NS) - 1) & 1);
          DA_DASSERT(t0 + i * kTileN < max(t_end, 1) + kTileN);
          const uint32_t fb = smem_u32(&full_bar[st]), fvb = smem_u32(&fullv_bar[st]);
          mbar_arrive_expect_tx(fb, kStageBytes / 2);
          mbar_arrive_expect_tx(fvb, kStageBytes / 2);
          const uint32_t dst = sbase + st * kStageBytes;
          const int t = t0 + i * kTileN;
          tma_load_5d(dst, &tmap_k, fb, 0, t, 0, kvh, bkv);                   // K: both 64-dim halves
          tma_load_5d(dst + 2 * kHalfBytes, &tmap_v, fvb, 0, t, 0, kvh, bkv);  // V
          if (i < 8) TRACE(2 + i);
        }
      } else {
        // paged cache: tile i of the split lives in page block_table[b][t / page_size] at token
        // t % page_size (a tile never spans pages).  The page indices of the next NS tiles are
        // loaded ahead so the lookups do not throttle the ring; both the current tile and the
        // look-ahead walk the pages with a (page, tile-in-page) cursor, one division in all.
        // Out-of-range indices fall outside the tensor map and read as zeros.
        const int32_t* bt = p.block_table + static_cast<int64_t>(b) * p.bt_stride;
        const uint32_t tpp = static_cast<uint32_t>(p.page_size / kTileN);   // tiles per page
        const uint32_t tile0 = static_cast<uint32_t>(t0 / kTileN);
        uint32_t cj = udiv_magic(tile0, p.page_magic), ck = tile0 - cj * tpp;   // current tile
        uint32_t lj = cj, lk = ck;                                              // look-ahead
        int pg[NS];
#pragma unroll
        for (int j = 0; j < NS; ++j) {
          pg[j] = j < n_tiles ? __ldg(bt + lj) : 0;
          if (++lk == tpp) { lk = 0; ++lj; }
        }
        for (int i = 0; i < n_tiles; ++i) {
          const int st = i % NS;
          if (i >= NS) mbar_wait(smem_u32(&empty_bar[st]), ((i / NS) - 1) & 1);
          const uint32_t fb = smem_u32(&full_bar[st]), fvb = smem_u32(&fullv_bar[st]);
          mbar_arrive_expect_tx(fb, kStageBytes / 2);
          mbar_arrive_expect_tx(fvb, kStageBytes / 2);
          const uint32_t dst = sbase + st * kStageBytes;
          const int page = pg[0];
          const int slot = static_cast<int>(ck) * kTileN;
          if (++ck == tpp) { ck = 0; ++cj; }
#pragma unroll
          for (int j = 0; j + 1 < NS; ++j) pg[j] = pg[j + 1];
          pg[NS - 1] = i + NS < n_tiles ? __ldg(bt + lj) : 0;
          if (++lk == tpp) { lk = 0; ++lj; }
          tma_load_5d(dst, &tmap_k, fb, 0, slot, 0, kvh, page);
          tma_load_5d(dst + 2 * kHalfBytes, &tmap_v, fvb, 0, slot, 0, kvh, page);
        }
      }
    }
    __syncwarp();
    asm volatile("bar.sync 0;" ::: "memory");   // (A) pairs with the consumers' barrier
  } else if (warp > NW) {
    // ================= helpers: idle until the epilogue merges =================
    asm volatile("bar.sync 0;" ::: "memory");   // (A)
  } else {
    // ================= consumers: warp w handles tiles w, w + NW, ... (stages it owns) =======
    const uint16_t* qrow = p.q + static_cast<int64_t>(b) * p.q_sb;
    if constexpr (kPath == DA_PATH_MMA) {
      uint32_t qf[8][kNB][2];
#pragma unroll
      for (int nb = 0; nb < kNB; ++nb) {
        const int g = nb * 8 + (lane >> 2);
        const bool ok = g < rows_valid;
        const uint16_t* qg = qrow + static_cast<int64_t>(hq0 + (ok ? g : 0)) * p.q_sh + 2 * (lane & 3);
        DA_DASSERT(hq0 + (ok ? g : 0) < p.h_q && b < p.batch);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          qf[kk][nb][0] = ok ? __ldg(reinterpret_cast<const uint32_t*>(qg + kk * 16)) : 0u;
          qf[kk][nb][1] = ok ? __ldg(reinterpret_cast<const uint32_t*>(qg + kk * 16 + 8)) : 0u;
        }
      }
      float o[8][kNB][4];
      float m[kNB][2], l[kNB][2];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int nb = 0; nb < kNB; ++nb)
#pragma unroll
          for (int c = 0; c < 4; ++c) o[i][nb][c] = 0.f;
#pragma unroll
      for (int nb = 0; nb < kNB; ++nb) m[nb][0] = m[nb][1] = kNegInf, l[nb][0] = l[nb][1] = 0.f;

      for (int i = warp; bal || i < n_tiles; i += NW) {
        const int st = i % NS;
        const uint32_t sK = sbase + st * kStageBytes;
        const uint32_t sV = sK + 2 * kHalfBytes;
        mbar_wait(smem_u32(&full_bar[st]), (i / NS) & 1);      // K: QK^T and the softmax start now
        if (lane == 0 && i < 8) TRACE(10 + i);
        int valid;
        if (kBalCapable && bal) {
          const int tile = *reinterpret_cast<volatile int*>(&stage_tile[st]);
          if (tile < 0) break;                                  // no more tiles for this warp
          valid = min(kTileN, n_seq - tile * kTileN);
        } else {
          valid = min(kTileN, t_end - (t0 + i * kTileN));
        }
        mma_tile<kNB>(sK, sV, valid, qf, o, m, l, p.scale_log2, lane, smem_u32(&fullv_bar[st]), (i / NS) & 1, i == 0);
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&empty_bar[st]));
        if (lane == 0 && i < 8) TRACE(18 + i);
      }
      // finish l: sum the partial sums of the 8 lanes that share a g column
#pragma unroll
      for (int nb = 0; nb < kNB; ++nb)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float v = l[nb][c];
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          v += __shfl_xor_sync(0xffffffffu, v, 8);
          v += __shfl_xor_sync(0xffffffffu, v, 16);
          l[nb][c] = v;
        }
      asm volatile("bar.sync 0;" ::: "memory");   // (A) every tile consumed: the ring is free
      // (tail balancing: every warp writes; one that took no tile holds m = -inf, l = 0, O = 0)
      if ((bal || warp < n_tiles) && lane < 4) {
#pragma unroll
        for (int nb = 0; nb < kNB; ++nb)
#pragma unroll
          for (int c = 0; c < 2; ++c) epi_ml[warp * 16 + nb * 8 + 2 * lane + c] = make_float2(m[nb][c], l[nb][c]);
      }
      if (bal || warp < n_tiles) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int nb = 0; nb < kNB; ++nb)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int g = nb * 8 + 2 * (lane & 3) + (c & 1);
              const int d = 16 * i + (lane >> 2) + 8 * (c >> 1);
              epi_o[(warp * 16 + g) * kEpiStride + d] = o[i][nb][c];
            }
      }
    } else {
      uint4 qv[16];
      const uint4* q4 = reinterpret_cast<const uint4*>(qrow + static_cast<int64_t>(hq0) * p.q_sh);
#pragma unroll
      for (int c = 0; c < 16; ++c) qv[c] = __ldg(q4 + c);
      float o[4] = {0.f, 0.f, 0.f, 0.f};
      float m = kNegInf, l = 0.f;
      for (int i = warp; bal || i < n_tiles; i += NW) {
        const int st = i % NS;
        const uint32_t sK = sbase + st * kStageBytes;
        mbar_wait(smem_u32(&full_bar[st]), (i / NS) & 1);
        int valid;
        if (kBalCapable && bal) {
          const int tile = *reinterpret_cast<volatile int*>(&stage_tile[st]);
          if (tile < 0) break;
          valid = min(kTileN, n_seq - tile * kTileN);
        } else {
          valid = min(kTileN, t_end - (t0 + i * kTileN));
        }
        mbar_wait(smem_u32(&fullv_bar[st]), (i / NS) & 1);
        scalar_tile(sK, sK + 2 * kHalfBytes, valid, qv, o, m, l, p.scale_log2, lane);
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&empty_bar[st]));
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
      asm volatile("bar.sync 0;" ::: "memory");   // (A)
      if (bal || warp < n_tiles) {
        if (lane == 0) epi_ml[warp * 16] = make_float2(m, l);
        *reinterpret_cast<float4*>(&epi_o[(warp * 16) * kEpiStride + 4 * lane]) =
            make_float4(o[0], o[1], o[2], o[3]);
      }
    }
  }
  __syncthreads();                                // (B) every warp's (m, l, O) is in shared memory
  if (threadIdx.x == 0) TRACE(26);

  // ================= merge the consumer warps (every thread of the CTA) =================
  // Element e = (row g = e / 32, float4 column d4 = e % 32) of the CTA's [R x 128] result.
  // Only the n_active = min(NW, n_tiles) warps that received tiles wrote a partial; the
  // passes are branch-free (predicated loads), so the loads of all passes issue back to back.
  const int n_active = bal ? NW : min(NW, n_tiles);
  float eM[kIters], eL[kIters];
  float4 eO[kIters];
#pragma unroll
  for (int it = 0; it < kIters; ++it) {
    const int e = threadIdx.x + it * kT;
    const int g = (e >> 5) & 15, d4 = e & 31;
    float2 ml[NW];
    float4 ow[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      ml[w] = make_float2(kNegInf, 0.f);
      ow[w] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (w < n_active) {
        ml[w] = epi_ml[w * 16 + g];
        ow[w] = *reinterpret_cast<const float4*>(&epi_o[(w * 16 + g) * kEpiStride + 4 * d4]);
      }
    }
    float M = kNegInf;
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, ml[w].x);
    float Lsum = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float f = ml[w].x == kNegInf ? 0.f : ex2(ml[w].x - M);
      Lsum = fmaf(f, ml[w].y, Lsum);
      acc.x = fmaf(f, ow[w].x, acc.x);
      acc.y = fmaf(f, ow[w].y, acc.y);
      acc.z = fmaf(f, ow[w].z, acc.z);
      acc.w = fmaf(f, ow[w].w, acc.w);
    }
    eM[it] = M;
    eL[it] = Lsum;
    eO[it] = acc;
  }
  if (threadIdx.x == 0) TRACE(27);

  // final rows: out / lse, or (kPub, da_forward_peer) this step's slot of the exchange buffer
  void* o_dst = p.out;
  float* l_dst = p.lse;
  uint32_t e_pub = 0;
  if constexpr (kPub == 1) e_pub = pub_epoch(p.pub);
  if constexpr (kPub == 2) e_pub = pub_epoch(pub_rank_view(p.pub, erank, static_cast<size_t>(p.batch) * p.h_q));
  if constexpr (kPub == 1) {
    const uint64_t sb = pub_slot(p.pub);
    o_dst = reinterpret_cast<void*>(sb);
    l_dst = reinterpret_cast<float*>(sb + static_cast<uint64_t>(p.pub.lse_offset));
  }
  if constexpr (!kCluster) {
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
      const int e = threadIdx.x + it * kT;
      const int g = e >> 5, d4 = e & 31;
      if (e >= R * 32 || g >= rows_valid) continue;
      const float inv = eL[it] > 0.f ? rcp(eL[it]) : 0.f;
      const float4 v = make_float4(eO[it].x * inv, eO[it].y * inv, eO[it].z * inv, eO[it].w * inv);
      const float lse_v = eL[it] > 0.f ? (eM[it] + lg2(eL[it])) * kLn2 : kNegInf;
      const size_t row = static_cast<size_t>(b) * p.h_q + hq0 + g;
      if (kCombine == DA_COMBINE_NONE || (kDyn && dyn_single && !p.dyn_via_combine)) {   // kDyn, s_b = 1: the final row
        if constexpr (kPub == 2) {
          pub_ll_store(pub_rank_view(p.pub, erank, static_cast<size_t>(p.batch) * p.h_q), e_pub, row, d4, v, lse_v);
        } else {
          store_out(p, o_dst, row, d4, v);
          if (d4 == 0 && l_dst != nullptr) l_dst[row] = lse_v;
        }
      } else {  // DA_COMBINE_KERNEL: normalised partial o_i, lse_i (C-part); kDyn: slot-major rows
        const size_t prow = kDyn ? static_cast<size_t>(dslot) * p.h_q + hq0 + g
                                 : static_cast<size_t>(split) * p.batch * p.h_q + row;
        DA_DASSERT(prow < (kDyn ? static_cast<size_t>(gridDim.y) * p.h_q
                                : static_cast<size_t>(p.num_splits) * p.batch * p.h_q));
        reinterpret_cast<float4*>(p.ws_o)[prow * (kHeadDim / 4) + d4] = v;
        if (d4 == 0) p.ws_lse[prow] = lse_v;
      }
    }
  } else {
    // ================= LSE combine across the s CTAs of the cluster (a8) =================
    // Row g belongs to rank g mod s.  Non-owned rows are pushed into the owner's slot with
    // st.async (bytes counted on the owner's push barrier; no fence, no cluster barrier on the
    // exit path); owned rows wait for the s - 1 pushes, merge, and are written out.
    if (!(bal && warp == NW)) cluster_wait();       // every peer's push barrier is initialised
                                                    // (a balancing producer warp waited already)
    const int s = s_cl;
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
      const int e = threadIdx.x + it * kT;
      const int g = e >> 5, d4 = e & 31;
      if (e >= R * 32 || g >= rows_valid) continue;
      const int gq = static_cast<int>(udiv_magic(g, p.s_magic));   // g / s
      const int owner = g - gq * s;
      // slot [source rank][row g / s of the owner]
      float* const dst = slots + (static_cast<int>(rank) * rows_per_owner + gq) * kSlotRowFloats;
      DA_DASSERT(static_cast<int>(rank) * rows_per_owner + gq < kMaxSlotRows && g < R && owner == g % s);
      const uint32_t rbar = mapa(smem_u32(&push_bar), owner);
      st_async_v4(mapa(smem_u32(dst + 4 * d4), owner), eO[it], rbar);
      if (d4 == 0) st_async_v2(mapa(smem_u32(dst + kHeadDim), owner), eM[it], eL[it], rbar);
    }
    {
      const uint32_t pb = smem_u32(&push_bar);
      while (!mbar_try_wait_cluster(pb, 0)) {
      }
    }
    if (threadIdx.x == 0) TRACE(29);
    // this rank's rows: element t = (owned row t / 32, float4 column t % 32)
    for (int t = threadIdx.x; t < rows_per_owner * 32; t += kT) {
      const int rl = t >> 5, d4 = t & 31;
      const int g = static_cast<int>(rank) + rl * s;
      if (g >= rows_valid) break;   // rows of a rank ascend with t: the rest are invalid too
      // two passes without a loop-carried max: (1) M = max over the s pushed lse's,
      // (2) independent weighted sums, so the slot loads of consecutive ranks overlap
      const float* const row0 = slots + rl * kSlotRowFloats;
      DA_DASSERT((s - 1) * rows_per_owner + rl < kMaxSlotRows);
      const int rstride = rows_per_owner * kSlotRowFloats;
      float M = kNegInf;
#pragma unroll 4
      for (int r = 0; r < s; ++r) M = fmaxf(M, row0[r * rstride + kHeadDim]);
      if (t == 0) TRACE(44);
      float Lsum = 0.f;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      if (M != kNegInf) {
#pragma unroll 4
        for (int r = 0; r < s; ++r) {
          const float2 ml = *reinterpret_cast<const float2*>(row0 + r * rstride + kHeadDim);
          const float4 ow = *reinterpret_cast<const float4*>(row0 + r * rstride + 4 * d4);
          const float f = ex2(ml.x - M);                 // empty rank: exp2(-inf) = 0
          Lsum = fmaf(f, ml.y, Lsum);
          acc.x = fmaf(f, ow.x, acc.x);
          acc.y = fmaf(f, ow.y, acc.y);
          acc.z = fmaf(f, ow.z, acc.z);
          acc.w = fmaf(f, ow.w, acc.w);
        }
      }
      if (t == 0) TRACE(45);
      const float inv = Lsum > 0.f ? rcp(Lsum) : 0.f;
      const size_t row = static_cast<size_t>(b) * p.h_q + hq0 + g;
      if constexpr (kPub == 2) {
        pub_ll_store(pub_rank_view(p.pub, erank, static_cast<size_t>(p.batch) * p.h_q), e_pub, row, d4,
                     make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv),
                     Lsum > 0.f ? (M + lg2(Lsum)) * kLn2 : kNegInf);
      } else {
        store_out(p, o_dst, row, d4, make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv));
        if (d4 == 0 && l_dst != nullptr) l_dst[row] = Lsum > 0.f ? (M + lg2(Lsum)) * kLn2 : kNegInf;
      }
      if (t == 0) TRACE(46);
    }
  }
  if (threadIdx.x == 0) TRACE(47);
  if constexpr (kPub == 1 && kCombine != DA_COMBINE_KERNEL) {   // this kernel wrote the final rows
    __syncthreads();
    if (threadIdx.x == 0) pub_arrive(p.pub);
  }
  if constexpr (kPub == 2) {
    // da_forward_peer_combine: the rows this CTA wrote as LL words, polled back from every rank and
    // LSE-merged here (the cross-GPU combine fused into the forward; the grid is one wave, so the
    // spinning is safe); the epoch advances once every CTA has read it
    __syncthreads();
    const PubParams pbr = pub_rank_view(p.pub, erank, static_cast<size_t>(p.batch) * p.h_q);
    if (threadIdx.x == 0) pub_count_advance(pbr, e_pub);
    const int s = kCluster ? s_cl : 1;
    for (int t = threadIdx.x; t < rows_per_owner * 32; t += kT) {
      const int rl = t >> 5, d4 = t & 31;
      const int g = static_cast<int>(rank) + rl * s;
      if (g >= rows_valid) break;
      pub_ll_merge_row(pbr, e_pub, static_cast<size_t>(b) * p.h_q + hq0 + g, d4);
    }
  }
#ifdef DECATTN_TRACE
  __syncthreads();
  if (threadIdx.x == 0) {
    TRACE(30);
    if (trace_cta() < 64) g_trace[trace_cta() * 64 + 61] = clock64();
    if (rank == 0 && blockIdx.x == 0) g_prev_end = gtime();
  }
#endif
}

// The kernel instantiation a plan launches, its shared memory and block size, with the one-time
// (per device) opt-in to > 48 KB of dynamic shared memory and to non-portable cluster sizes.
template <int kPath, int kNB, int kCombine, bool kDyn = false, int kPub = 0, bool kBal = false, bool kPaged = false>
struct FwdKernel {
  static constexpr bool kCluster = kCombine == DA_COMBINE_CLUSTER;
  // dynamic split counts: mostly one split per sequence, so the streaming (s = 1) configuration
  static constexpr int NS = kDyn ? kStagesNone : stages_for(kCombine);
  static constexpr int NW = kDyn ? kWarpsNone : warps_for(kCombine);
  static constexpr int kSmem = smem_for(NS, kCluster);
  static constexpr int kThreads = threads_for(NW, helpers_for(kCombine));
  static constexpr auto kern = split_kv_fwd_kernel<kPath, kNB, kCombine, NS, NW, kDyn, kPub, kBal, kPaged>;

  static cudaError_t prepare() {
    static std::atomic<uint64_t> attr_done{0};
    int dev = 0;
    cudaError_t err = cudaGetDevice(&dev);
    if (err != cudaSuccess) return err;
    const uint64_t bit = 1ull << (dev & 63);
    if ((attr_done.load(std::memory_order_acquire) & bit) == 0) {
      err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
      if (err != cudaSuccess) return err;
      if (kCluster) {   // clusters of 9..16 CTAs are a non-portable size
        err = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (err != cudaSuccess) return err;
      }
      attr_done.fetch_or(bit, std::memory_order_acq_rel);
    }
    return cudaSuccess;
  }

  static void config(const da_plan& plan, cudaStream_t stream, cudaLaunchConfig_t& cfg, cudaLaunchAttribute* attrs) {
    cfg = {};
    cfg.gridDim = dim3(plan.grid_x, plan.grid_y, plan.grid_z);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = stream;
    int na = 0;
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
    if (kCluster) {
      attrs[na].id = cudaLaunchAttributeClusterDimension;
      attrs[na].val.clusterDim.x = static_cast<unsigned>(plan.num_splits);
      attrs[na].val.clusterDim.y = 1;
      attrs[na].val.clusterDim.z = 1;
      ++na;
    }
    cfg.attrs = attrs;
    cfg.numAttrs = na;
  }

  static cudaError_t launch(const da_plan& plan, const CUtensorMap& tk, const CUtensorMap& tv, const FwdParams& p,
                            cudaStream_t stream) {
    cudaError_t err = prepare();
    if (err != cudaSuccess) return err;
    if (kThreads != plan.block_threads || kSmem != plan.smem_bytes) return cudaErrorInvalidConfiguration;
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute attrs[2];
    config(plan, stream, cfg, attrs);
    return cudaLaunchKernelEx(&cfg, kern, tk, tv, p);
  }

  // Launch units of this instantiation that can be co-resident on the current device: clusters of
  // plan.num_splits CTAs (cudaOccupancyMaxActiveClusters) for a cluster kernel, CTAs otherwise.
  static cudaError_t residency(const da_plan& plan, int* out) {
    cudaError_t err = prepare();
    if (err != cudaSuccess) return err;
    if (kCluster) {
      cudaLaunchConfig_t cfg;
      cudaLaunchAttribute attrs[2];
      config(plan, nullptr, cfg, attrs);
      return cudaOccupancyMaxActiveClusters(out, kern, &cfg);
    }
    int dev = 0, sms = 0, per_sm = 0;
    if ((err = cudaGetDevice(&dev)) != cudaSuccess) return err;
    if ((err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return err;
    if ((err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, kSmem)) != cudaSuccess)
      return err;
    *out = per_sm * sms;
    return cudaSuccess;
  }
};

template <int kPath, int kNB, int kCombine, bool kDyn = false, int kPub = 0, bool kBal = false>
cudaError_t launch_impl(const da_plan& plan, const CUtensorMap& tk, const CUtensorMap& tv,
                        const FwdParams& p, cudaStream_t stream) {
  // paged and dense caches run separate instantiations (kPaged): the page walk's code stays out of
  // the dense kernels, whose latency-bound launches pay for every instruction they fetch
  if (p.block_table != nullptr)
    return FwdKernel<kPath, kNB, kCombine, kDyn, kPub, false, true>::launch(plan, tk, tv, p, stream);
  return FwdKernel<kPath, kNB, kCombine, kDyn, kPub, kBal, false>::launch(plan, tk, tv, p, stream);
}

// The balancing instantiation is launched when the plan's length gives every split >=
// kBalMinTiles tiles (dense cache).  Either instantiation is exact for any length: the other one
// only never balances, so a serving plan made for short sequences in a large cache keeps the lean
// latency kernel even though its cache capacity would allow long ones
inline bool balancing_possible(const da_plan& plan, const FwdParams& p) {
  return p.block_table == nullptr &&
         (static_cast<int64_t>(plan.l_k) + kTileN - 1) / kTileN >= static_cast<int64_t>(kBalMinTiles) * plan.num_splits;
}

template <int kPath, int kNB>
cudaError_t residency_combine(const da_plan& plan, int pub, int* out) {
  switch (plan.combine_mode) {
    case DA_COMBINE_NONE:
      if (pub == 2) return FwdKernel<kPath, kNB, DA_COMBINE_NONE, false, 2>::residency(plan, out);
      if (pub == 1) return FwdKernel<kPath, kNB, DA_COMBINE_NONE, false, 1>::residency(plan, out);
      return FwdKernel<kPath, kNB, DA_COMBINE_NONE>::residency(plan, out);
    case DA_COMBINE_CLUSTER:
      if (pub == 2) return FwdKernel<kPath, kNB, DA_COMBINE_CLUSTER, false, 2>::residency(plan, out);
      if (pub == 1) return FwdKernel<kPath, kNB, DA_COMBINE_CLUSTER, false, 1>::residency(plan, out);
      return FwdKernel<kPath, kNB, DA_COMBINE_CLUSTER>::residency(plan, out);
    default:
      if (is_dynamic(plan)) {
        if (pub) return FwdKernel<kPath, kNB, DA_COMBINE_KERNEL, true, 1>::residency(plan, out);
        return FwdKernel<kPath, kNB, DA_COMBINE_KERNEL, true>::residency(plan, out);
      }
      return FwdKernel<kPath, kNB, DA_COMBINE_KERNEL>::residency(plan, out);
  }
}

template <int kPath, int kNB>
cudaError_t dispatch_combine(const da_plan& plan, const CUtensorMap& tk, const CUtensorMap& tv,
                             const FwdParams& p, cudaStream_t stream) {
  // kPub (da_forward_peer) instantiations only where the forward writes final rows; with the
  // workspace combine the combine kernel publishes and the forward is the plain one
  // (kPub = 2: publish + the in-kernel cross-rank combine, one-wave NONE / CLUSTER plans)
  const int pub = p.pub.bases == nullptr ? 0 : (p.pub.out != nullptr ? 2 : 1);
  switch (plan.combine_mode) {
    case DA_COMBINE_NONE:
      if (pub == 2) return launch_impl<kPath, kNB, DA_COMBINE_NONE, false, 2>(plan, tk, tv, p, stream);
      if (pub == 1) return launch_impl<kPath, kNB, DA_COMBINE_NONE, false, 1>(plan, tk, tv, p, stream);
      return launch_impl<kPath, kNB, DA_COMBINE_NONE>(plan, tk, tv, p, stream);
    case DA_COMBINE_CLUSTER:
      if (pub == 2) return launch_impl<kPath, kNB, DA_COMBINE_CLUSTER, false, 2>(plan, tk, tv, p, stream);
      if (pub == 1) return launch_impl<kPath, kNB, DA_COMBINE_CLUSTER, false, 1>(plan, tk, tv, p, stream);
      if (balancing_possible(plan, p)) return launch_impl<kPath, kNB, DA_COMBINE_CLUSTER, false, 0, true>(plan, tk, tv, p, stream);
      return launch_impl<kPath, kNB, DA_COMBINE_CLUSTER>(plan, tk, tv, p, stream);
    default:
      if (is_dynamic(plan)) {   // s_b = 1 rows are final rows written by the forward
        if (pub) return launch_impl<kPath, kNB, DA_COMBINE_KERNEL, true, 1>(plan, tk, tv, p, stream);
        return launch_impl<kPath, kNB, DA_COMBINE_KERNEL, true>(plan, tk, tv, p, stream);
      }
      return launch_impl<kPath, kNB, DA_COMBINE_KERNEL>(plan, tk, tv, p, stream);
  }
}

}  // namespace

cudaError_t launch_split_kv_fwd(const da_plan& plan, const CUtensorMap& tmap_k,
                                const CUtensorMap& tmap_v, const FwdParams& p,
                                cudaStream_t stream) {
  if (plan.path == DA_PATH_TC) return launch_split_kv_fwd_tc(plan, tmap_k, tmap_v, p, stream);
  if (plan.path == DA_PATH_SCALAR) return dispatch_combine<DA_PATH_SCALAR, 1>(plan, tmap_k, tmap_v, p, stream);
  if (plan.rows_per_cta == 8) return dispatch_combine<DA_PATH_MMA, 1>(plan, tmap_k, tmap_v, p, stream);
  return dispatch_combine<DA_PATH_MMA, 2>(plan, tmap_k, tmap_v, p, stream);
}

cudaError_t forward_residency(const da_plan& plan, int pub, int* out) {
  if (plan.path == DA_PATH_TC) return forward_tc_residency(out);
  if (plan.path == DA_PATH_SCALAR) return residency_combine<DA_PATH_SCALAR, 1>(plan, pub, out);
  if (plan.rows_per_cta == 8) return residency_combine<DA_PATH_MMA, 1>(plan, pub, out);
  return residency_combine<DA_PATH_MMA, 2>(plan, pub, out);
}

#ifdef DECATTN_TRACE
extern "C" __attribute__((visibility("default"))) int da_trace_fetch(unsigned long long* host, int n) {
  if (n > 64 * 64) n = 64 * 64;
  return cudaMemcpyFromSymbol(host, g_trace, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 1;
}
#endif
}  // namespace decattn
