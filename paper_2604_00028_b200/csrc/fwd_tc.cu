// Split-KV decode-attention forward on the 5th-generation tensor cores (tcgen05 + TMEM) for wide
// query groups: DA_PATH_TC, pack_gqa with G = H_Q / H_KV > 16 (MQA / wide GQA) on splits of >= 4
// tiles of 64 tokens with >= U / 2 CTAs (plan.cpp tc_path), SURVEY §8(a) steps a2-a7.  There the G
// query rows of a KV head make a real dense contraction per KV tile, which the mma.sync path could
// only run as 16-row CTAs that read every K / V tile ceil(G / 16) times and issue 96+ HMMAs per warp
// per tile (MQA G = 64 measured 2.6 TB/s there, 6.6-6.8 TB/s here).
//
// One CTA = 64 query rows of one KV head (rows hq0 .. hq0 + 63; G < 64 padded with zero rows) x one
// split x one batch entry; grid = (s, H_KV * ceil(G / 64), B) as on the other paths.  Stages of 128
// tokens (two 64-token tiles); K and V of a stage each [half][128 tokens][64 dims], 128B-swizzled,
// 32 KB, in separate rings (2 K slots, freed when S(s) is computed; 5 V slots, freed when PV(s) is).
//   warp 8       TMA producer: one 5-D box per 64-token tile and 64-dim half (dense or paged cache),
//                issued K(0), K(1), then V(s), K(s + 2); a split's last stage may hold one tile.
//   warp 9       TMEM allocator and MMA issuer (one lane), tcgen05.mma kind::f16 with A from TMEM:
//                S(s) = Q K(s)^T at M = 64 rows, N = 128 tokens, K = 128 dims into TMEM buffer s & 1,
//                then O += P(s) V(s) at M = 128, N = 128 dims, K = 128 tokens with the pair
//                P = P_hi + P_lo stacked along M (B = the V box, MN-major): two S stages ahead, so the
//                tensor pipe runs PV(s) and S(s + 2) while the softmax warps work on stage s + 1.
//                The pipe executes in issue order, so S(s + 2) overwrites the buffer only after PV(s)
//                read P(s) from it; tcgen05.commit releases ring stages, S and O to their waiters.
//   warps 0-7    softmax and epilogue: row r lives on TMEM lane 32 (r / 16) + r mod 16 (M = 64,
//                scripts/microbench_tcgen05_rows.cu); the 16-lane TMEM shapes give thread t rows
//                16 q + t / 4 and + 8 (q = w mod 4), the 4 threads of a row reduce with shuffles,
//                and warps q, q + 4 take the two 64-token halves of a stage (row maxima exchanged
//                through shared memory; DECATTN_TC_SMX_WARPS = 4: warps 0-3 take both halves).
//                Online softmax in fp32 / log2 units; P = exp2(S - m) as the bf16
//                pair P_hi + P_lo (the precision of fwd.cu's PV) written over S.  The
//                running maximum m is a reference that moves only when a stage's maximum exceeds it
//                by more than 8 (log2 units); then the O rows are rescaled in TMEM (tcgen05.ld /
//                st) and l with them.  P <= 2^8 otherwise, and out = O / l and lse = m + log2 l hold
//                for any reference, so the result is the exact softmax (C-att).
//   epilogue     O = the hi lanes' part + the lo lanes' part, / l: out + lse (s = 1, NONE) or the
//                normalised fp32 partial + lse (s > 1, KERNEL; merged by lse_combine_kernel).
// Programmatic dependent launch as in fwd.cu: the prologue (barriers, TMEM allocation, tensor-map
// prefetch, L2 prefetch of the CTA's Q rows and of the first ring tiles) overlaps the previous kernel.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "config.h"
#include "internal.h"
#include "ptx.cuh"
#include "tile_common.cuh"

namespace decattn {

using namespace ptx;

namespace {

constexpr int kTcM = kTcRows;                    // query rows of a CTA (the S MMA's M)
constexpr int kTcT = 2 * kTileN;                 // tokens per stage (the S MMA's N): two 64-token tiles
constexpr int kTcSlotBytes = kStageBytes;        // K or V of a stage: [half][128 tokens][64 dims], 32 KB
constexpr int kTcHalfStride = kTcSlotBytes / 2;  // the 64-dim halves of a slot
constexpr int kTcKSlots = DECATTN_TC_KSLOTS;     // K ring (released when S(s) is computed)
constexpr int kTcVSlots = DECATTN_TC_VSLOTS;     // V ring (released when PV(s) is done)
constexpr int kTcSoftmaxWarps = DECATTN_TC_SMX_WARPS;
constexpr int kTcHalvesPerWarp = 8 / kTcSoftmaxWarps;   // 64-token halves of a stage per softmax warp
static_assert(kTcSoftmaxWarps == 4 || kTcSoftmaxWarps == 8, "one or two softmax warps per lane quadrant");
constexpr int kTcThreads = (kTcSoftmaxWarps + 2) * 32;   // + TMA producer warp + MMA warp
constexpr int kTcProducerWarp = kTcSoftmaxWarps, kTcMmaWarp = kTcSoftmaxWarps + 1;
// TMEM columns (512 allocated): two S buffers (P is written over S once the softmax warps read it),
// the O accumulator and Q (the S MMA's A operand, two bf16 per 32-bit column, row r on the
// accumulator's lane).  The PV product runs at M = 128 with the P pair stacked along M: in warp
// quadrant q, TMEM lanes 32 q + i hold P_hi and lanes 32 q + 16 + i hold P_lo of row 16 q + i
// (i < 16), so the O rows on those lanes are the hi and lo parts of the row's output (summed in
// the epilogue) and every lane a thread touches stays in its warp's quadrant: one pass over V at
// M = 128, N = 128 instead of two passes at M = 64 (each at half the tensor rate).
constexpr int kTcTmemCols = 512;
constexpr uint32_t kTcColSP = 0, kTcColO = 2 * kTcT, kTcColQ = kTcColO + 128;
constexpr int kTcSmem = (kTcKSlots + kTcVSlots) * kTcSlotBytes + 1024;
static_assert(kTcSmem <= 227 * 1024, "tcgen05 path shared memory");
static_assert(kTcSmem == kTcSmemCfg && kTcThreads == kTcThreadsCfg, "the planner's launch fields (config.h)");
static_assert(kTcColQ + 64 <= kTcTmemCols, "TMEM columns");
constexpr float kTcRescaleLog2 = 8.f;            // rescale O only when the maximum grows by > 2^8


// development timeline tracing (-DDECATTN_TRACE builds): globaltimer ns of tiles 16..23 of the
// first 64 CTAs: 0+k K TMA issued, 8+k S issued, 16+k S seen by softmax warp 0, 24+k P written,
// 32+k PV issued, 40+k P(s) seen complete by the MMA thread, 48+k S start, 56+k PV start
#ifdef DECATTN_TRACE
__device__ unsigned long long g_trace_tc[64 * 64];
__device__ unsigned long long g_clock_tc[4];   // globaltimer / clock64 at S(16), S(23) of CTA 0
__device__ unsigned long long g_cta_tc[8 * 1024];   // per CTA (first 1024): after the PDL wait, end, SM id,
// entry, Q in TMEM (MMA thread), first S seen, last PV seen (softmax thread 0)
__device__ __forceinline__ void tc_trace_cta(int slot) {
  const int c = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  if (c >= 1024) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_cta_tc[slot * 1024 + c] = t;
  if (slot == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_cta_tc[2 * 1024 + c] = smid;
  }
}
#define TC_TRACE_CTA(slot) tc_trace_cta(slot)
__device__ __forceinline__ void tc_trace(int slot_base, int i) {
  const int k = i - 16;
  if (k < 0 || k >= 8) return;
  const int c = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  if (c >= 64) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_trace_tc[c * 64 + slot_base + k] = t;
}
#define TC_TRACE(base, i) tc_trace(base, i)
// softmax-internal stamps of warp 0 / lane 0 in CTA 0, stages 16..23 (slot j: 0 S loaded, 1 maximum
// exchanged, 2 P computed, 3 P stored)
__device__ unsigned long long g_trace_smx[4 * 8];
__device__ unsigned long long g_trace_pw[16 * 8];   // P stored, per softmax warp (lane 0), CTA 0, stages 16..23
#define TC_TRACE_PW(s)                                                                              \
  do {                                                                                              \
    if (lane == 0 && blockIdx.x + blockIdx.y + blockIdx.z == 0 && (s) >= 16 && (s) < 24) {          \
      unsigned long long t_;                                                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                        \
      g_trace_pw[warp * 8 + (s) - 16] = t_;                                                         \
    }                                                                                               \
  } while (0)
#define TC_TRACE_SMX(j, s)                                                                        \
  do {                                                                                            \
    if (threadIdx.x == 0 && blockIdx.x + blockIdx.y + blockIdx.z == 0 && (s) >= 16 && (s) < 24) { \
      unsigned long long t_;                                                                      \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                      \
      g_trace_smx[(j) * 8 + (s) - 16] = t_;                                                       \
    }                                                                                             \
  } while (0)
#else
#define TC_TRACE(base, i) do { } while (0)
#define TC_TRACE_CTA(slot) do { } while (0)
#define TC_TRACE_SMX(j, s) do { } while (0)
#define TC_TRACE_PW(s) do { } while (0)
#endif

// development watchdog (-DDECATTN_TC_WATCHDOG builds): a wait that has not completed after 2 s
// prints its barrier tag, stage and thread, then traps
#ifdef DECATTN_TC_WATCHDOG
}  // namespace
}  // namespace decattn
#include <cstdio>
namespace decattn {
namespace {
__device__ __forceinline__ void tc_wait(uint32_t bar, uint32_t parity, int tag, int s) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (!mbar_try_wait(bar, parity)) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 2000000000ull) {
      printf("tc watchdog: tag %d stage %d parity %u thread %d block %d %d %d\n", tag, s, parity, (int)threadIdx.x,
             (int)blockIdx.x, (int)blockIdx.y, (int)blockIdx.z);
      asm volatile("trap;");
    }
  }
}
#else
__device__ __forceinline__ void tc_wait(uint32_t bar, uint32_t parity, int, int) { mbar_wait(bar, parity); }
#endif

// ---- tcgen05 helpers --------------------------------------------------------------------------
// shared-memory matrix descriptor: start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46),
// version 1 [46,48), layout SWIZZLE_128B (2) [61,64)
__device__ __forceinline__ uint64_t tc_sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3fffu) | (static_cast<uint64_t>((lbo >> 4) & 0x3fffu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor, kind::f16: D fp32 (bit 4), A / B bf16 (bits 7, 10), A / B MN-major
// (bits 15, 16), N >> 3 at bit 17, M >> 4 at bit 24
__host__ __device__ constexpr uint32_t tc_idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
         (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
               "l"(a), "l"(b), "r"(id), "r"(acc)
               : "memory");
}
// A operand from TMEM ("TS"): a_tmem = the first column of the K16 step
__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
               "r"(a_tmem), "l"(b), "r"(id), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 32 consecutive TMEM columns of this warp's lane quadrant: v[i] = column col + i of lane (lane)
__device__ __forceinline__ void tc_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tc_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])),
      "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])),
      "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])),
      "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}
__device__ __forceinline__ void tc_st32u(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
// 16x256b: of the warp's 16 lanes L0..L0+15, thread t holds lanes L0 + t / 4 and L0 + t / 4 + 8,
// columns 2 (t % 4) and 2 (t % 4) + 1 of every 8-column group: v[4 g + 0..1] = lane t / 4,
// v[4 g + 2..3] = lane t / 4 + 8 (CUTLASS SM100_TMEM_LOAD_16dp256b layout)
template <int NG>
__device__ __forceinline__ void tc_ld16x256(uint32_t taddr, uint32_t (&v)[4 * NG]) {
  static_assert(NG == 8, "x8 only");
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tc_st16x256_x8(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
// 16x128b: thread t writes lanes L0 + t / 4 (v[2 g]) and L0 + t / 4 + 8 (v[2 g + 1]), column
// 4 g + t % 4 of every 4-column group g
__device__ __forceinline__ void tc_st16x128_x8(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x128b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// P = P_hi + P_lo for two values (x0 in the low half of each word), both rounded to nearest.
// (Exact truncation by byte permutes instead of cvt measured no faster.)
__device__ __forceinline__ void tc_pair(float x0, float x1, uint32_t& hw, uint32_t& lw) {
  hw = pack_bf16(x0, x1);
  lw = pack_bf16(x0 - bf16lo(hw), x1 - bf16hi(hw));
}

// byte offset of 16-byte chunk c (8 bf16) of row r in a 128B-swizzled box of 128-byte rows
__device__ __forceinline__ uint32_t sw128_chunk(int r, int c) {
  return static_cast<uint32_t>(r * 128 + (((c ^ r) & 7) << 4));
}

__global__ void __launch_bounds__(kTcThreads, 1)
    split_kv_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmap_k, const __grid_constant__ CUtensorMap tmap_v,
                           const FwdParams p, int kernel_combine) {
  constexpr int NK = kTcKSlots, NV = kTcVSlots;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t fullk_bar[NK];   // K(s) has landed in slot s % NK
  __shared__ __align__(8) uint64_t emptyk_bar[NK];  // S(s) done: slot free (tcgen05.commit)
  __shared__ __align__(8) uint64_t fullv_bar[NV];   // V(s) has landed in slot s % NV
  __shared__ __align__(8) uint64_t emptyv_bar[NV];  // PV(s) done: slot free (tcgen05.commit)
  __shared__ __align__(8) uint64_t q_bar;           // Q is in TMEM (every softmax thread)
  __shared__ __align__(8) uint64_t s_full[2];       // S(s) in TMEM buffer s & 1 (commit)
  __shared__ __align__(8) uint64_t p_full[2];       // P(s) written over S(s) (every softmax warp)
  __shared__ __align__(8) uint64_t pv_done[2];      // O += P(s) V(s) done for s & 1 == b (commit)
  __shared__ uint32_t tmem_base;
  __shared__ float red_x[2][2][kTcM];               // [stage parity][token half] row maxima (8 warps)
  __shared__ float red_l[2][kTcM];                  // [token half] row sums (8 warps)

  const uint32_t raw = smem_u32(smem_raw);
  if (threadIdx.x == 0) TC_TRACE_CTA(3);
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int grp = blockIdx.y, split = blockIdx.x, b = blockIdx.z;
  const int kvh = static_cast<int>(udiv_magic(static_cast<uint32_t>(grp), p.mb_magic));
  const int rg = grp - kvh * p.mblocks_per_head;
  const int hq0 = kvh * p.G + rg * kTcM;
  const int rows_valid = min(kTcM, p.G - rg * kTcM);
  // pull this CTA's Q rows (two 128-byte lines each) into L2 before anything else: the softmax
  // warps read them right after griddepcontrol.wait, when the ring's first K / V loads of every
  // CTA already queue at the DRAM (a prefetch returns no data, so it cannot observe a stale Q)
  if (DECATTN_TC_QPREFETCH && threadIdx.x < 2 * kTcM && (threadIdx.x >> 1) < rows_valid)
    prefetch_l2(p.q + static_cast<int64_t>(b) * p.q_sb + static_cast<int64_t>(hq0 + (threadIdx.x >> 1)) * p.q_sh +
                (threadIdx.x & 1) * 64);

  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NK; ++i) {
      mbar_init(smem_u32(&fullk_bar[i]), 1);
      mbar_init(smem_u32(&emptyk_bar[i]), 1);
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      mbar_init(smem_u32(&fullv_bar[i]), 1);
      mbar_init(smem_u32(&emptyv_bar[i]), 1);
    }
    mbar_init(smem_u32(&q_bar), kTcSoftmaxWarps * 32);
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&s_full[i]), 1);
      mbar_init(smem_u32(&p_full[i]), kTcSoftmaxWarps);
      mbar_init(smem_u32(&pv_done[i]), 1);
    }
    fence_mbarrier_init();
  }
  if (warp == kTcMmaWarp) {   // TMEM: S / P double buffer, O accumulator, Q
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(kTcTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == kTcProducerWarp && lane == 0) {
    prefetch_tmap(&tmap_k);
    prefetch_tmap(&tmap_v);
    if (p.seqlens != nullptr) prefetch_l2(p.seqlens + b);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  // this split's range at the plan's length (exact without cache_seqlens; a guess for the L2
  // prefetch otherwise, recomputed after the wait as in fwd.cu); tiles of 64 tokens, stages of two
  int t0 = 0, t_end = 0, n_tiles = 0;
  split_range(min(max(p.l_default, 0), p.l_cap), split, p.num_splits, p.s_magic, t0, t_end, n_tiles);
  if (p.block_table == nullptr && warp == kTcProducerWarp && lane == 0 && n_tiles >= 1) {
    const int np = min(n_tiles, 2 * NK);
    for (int i = 0; i < np; ++i)
      for (int h = 0; h < 2; ++h) {
        tma_prefetch_5d(&tmap_k, 0, t0 + i * kTileN, h, kvh, b);
        tma_prefetch_5d(&tmap_v, 0, t0 + i * kTileN, h, kvh, b);
      }
  }
  pdl_launch_dependents();
  pdl_wait();
  if (p.seqlens != nullptr)
    split_range(min(max(max(__ldg(p.seqlens + b), 0) - p.seq_offset, 0), p.l_cap), split, p.num_splits, p.s_magic,
                t0, t_end, n_tiles);
  const int n_st = (n_tiles + 1) >> 1;                 // 128-token stages
  if (threadIdx.x == 0) TC_TRACE_CTA(0);

  if (warp == kTcProducerWarp) {
    // ================= TMA producer (dense or paged cache) =================
    // a stage holds K then V of two 64-token tiles as [half][128 tokens][64 dims] (one 8 KB box per
    // tile and half); the second tile of a split's last stage may be missing (not loaded: its
    // tokens are masked and its V rows zeroed by the softmax warps)
    if (lane == 0) {
      const int32_t* bt = p.block_table != nullptr ? p.block_table + static_cast<int64_t>(b) * p.bt_stride : nullptr;
      const uint32_t tpp = p.page_size > 0 ? static_cast<uint32_t>(p.page_size / kTileN) : 1u;
      const uint32_t tile0 = static_cast<uint32_t>(t0 / kTileN);
      // K and V of a stage go to their own rings in the order the tensor pipe needs them:
      // K(0), K(1), then V(s), K(s + 2) (S runs two stages ahead of PV).  Each ring walks the
      // split's tiles (and, paged, the block table) on its own
      struct Walk {
        uint32_t cj, ck;
      };
      Walk wk{bt != nullptr ? udiv_magic(tile0, p.page_magic) : 0u, 0u}, wv{0u, 0u};
      wk.ck = tile0 - wk.cj * tpp;
      wv = wk;
      auto load = [&](const CUtensorMap* tm, Walk& w, uint32_t slot, uint32_t bar, int s) {
        const int nsub = min(2, n_tiles - 2 * s);
        mbar_arrive_expect_tx(bar, nsub * 2 * kHalfBytes);
        for (int sub = 0; sub < nsub; ++sub) {
          int major = b, tok = t0 + (2 * s + sub) * kTileN;
          if (bt != nullptr) {   // paged: tile in page block_table[b][t / page_size] at t % page_size
            major = __ldg(bt + w.cj);
            tok = static_cast<int>(w.ck) * kTileN;
            if (++w.ck == tpp) { w.ck = 0; ++w.cj; }
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) tma_load_5d(slot + h * kTcHalfStride + sub * kHalfBytes, tm, bar, 0, tok, h, kvh, major);
        }
      };
      auto load_k = [&](int s) {
        const int st = s % NK;
        if (s >= NK) tc_wait(smem_u32(&emptyk_bar[st]), ((s / NK) - 1) & 1, 1, s);
        load(&tmap_k, wk, sbase + st * kTcSlotBytes, smem_u32(&fullk_bar[st]), s);
        TC_TRACE(0, s);
      };
      auto load_v = [&](int s) {
        const int st = s % NV;
        if (s >= NV) tc_wait(smem_u32(&emptyv_bar[st]), ((s / NV) - 1) & 1, 2, s);
        load(&tmap_v, wv, sbase + (NK + st) * kTcSlotBytes, smem_u32(&fullv_bar[st]), s);
      };
      if (n_st > 0) load_k(0);
      if (n_st > 1) load_k(1);
      for (int s = 0; s < n_st; ++s) {
        load_v(s);
        if (s + 2 < n_st) load_k(s + 2);
      }
    }
  } else if (warp == kTcMmaWarp) {
    // ================= MMA issuer (one lane) =================
    if (lane == 0 && n_st > 0) {
      constexpr uint32_t id_s = tc_idesc(kTcM, kTcT, 0, 0);             // S: M = 64, N = 128 tokens
      constexpr uint32_t id_o = tc_idesc(2 * kTcM, kHeadDim, 0, 1);     // O: [P_hi; P_lo] stacked along M
      tc_wait(smem_u32(&q_bar), 0, 3, 0);
      TC_TRACE_CTA(4);
      // S(s) = Q K(s)^T into TMEM buffer s & 1.  The buffer held P(s - 2), read by PV(s - 2), which
      // was issued before: the tensor pipe executes in issue order
      auto issue_s = [&](int s) {
        const int st = s % NK, sb = s & 1;
        tc_wait(smem_u32(&fullk_bar[st]), (s / NK) & 1, 4, s);
        tc_fence_after();
#ifndef DECATTN_TRACE_VWAIT
        TC_TRACE(48, s);
#endif
        const uint32_t sK = sbase + st * kTcSlotBytes;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {   // 16 dims per step: K half kk / 4, +32 B per step in the row
          const uint64_t bk = tc_sdesc(sK + (kk >> 2) * kTcHalfStride + (kk & 3) * 32, 16, 1024);
          tc_mma_ts(tmem + kTcColSP + sb * kTcT, tmem + kTcColQ + kk * 8, bk, id_s, kk > 0 ? 1u : 0u);
        }
        tc_commit(smem_u32(&s_full[sb]));
        tc_commit(smem_u32(&emptyk_bar[st]));
        TC_TRACE(8, s);
#ifdef DECATTN_TRACE
        if ((s == 16 || s == 23) && blockIdx.x + blockIdx.y + blockIdx.z == 0) {
          g_clock_tc[s == 16 ? 2 : 3] = clock64();
          unsigned long long t_;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
          g_clock_tc[s == 16 ? 0 : 1] = t_;
        }
#endif
      };
      // O += P(s) V(s), once the softmax warps wrote P(s) (over S(s)) and V(s) landed
      auto issue_pv = [&](int s) {
        const int st = s % NV, pb = s & 1;
        tc_wait(smem_u32(&p_full[pb]), (s >> 1) & 1, 5, s);
        TC_TRACE(40, s);
        tc_wait(smem_u32(&fullv_bar[st]), (s / NV) & 1, 6, s);
#ifdef DECATTN_TRACE_VWAIT
        TC_TRACE(48, s);   // development: V(s) seen, before the fence (slot of "S start")
#endif
        tc_fence_after();
        TC_TRACE(56, s);
        const uint32_t sV = sbase + (NK + st) * kTcSlotBytes;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {   // 16 tokens (8 packed columns, 16 V rows) per step
          const uint64_t bv = tc_sdesc(sV + kk * 2048, kTcHalfStride, 1024);
          tc_mma_ts(tmem + kTcColO, tmem + kTcColSP + pb * kTcT + kk * 8, bv, id_o, (s > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(smem_u32(&pv_done[pb]));
        tc_commit(smem_u32(&emptyv_bar[st]));
        TC_TRACE(32, s);
      };
      // two S stages ahead, then PV(s) and S(s + 2): the tensor pipe runs PV(s) and S(s + 2) while
      // the softmax warps work on stage s + 1, whose S is already there
      issue_s(0);
      if (n_st > 1) issue_s(1);
      for (int s = 0; s < n_st; ++s) {
        issue_pv(s);
        if (s + 2 < n_st) issue_s(s + 2);
      }
    }
  } else {
    // ================= softmax + epilogue =================
    // warp w reads TMEM lanes 32 q .. 32 q + 15 (q = w mod 4) = rows 16 q .. 16 q + 15 (M = 64) with
    // the 16-lane shapes: thread t holds rows rA = 16 q + t / 4 and rB = rA + 8, and of each 8-token
    // group the tokens 2 a, 2 a + 1 (a = t % 4); the 4 threads of a row reduce with xor shuffles
    // 1, 2.  With 8 softmax warps, warps q and q + 4 share the quadrant and split every stage's 128
    // tokens (and O's 128 columns) into halves hh = w / 4: two warps per SM sub-partition hide each
    // other's MUFU / conversion latency; the row maximum is exchanged through shared memory
    // (named barrier 1 + q, 64 threads) and the row sums are added in the epilogue
    const int q4 = warp & 3, hh = warp >> 2;
    const int a4 = lane & 3;
    const int rA = 16 * q4 + (lane >> 2), rB = rA + 8;
    const uint32_t lane_addr = static_cast<uint32_t>(q4 * 32) << 16;
    auto pair_sync = [&]() {
      if (kTcSoftmaxWarps == 8) asm volatile("bar.sync %0, 64;" ::"r"(1 + q4) : "memory");
    };
    // Q -> TMEM (the S MMA's A operand: u32 column j = dims 2 j, 2 j + 1), 16x128b layout: column
    // 4 g + a of rows rA, rB; zero past G.  Warp half hh writes dims [64 h, + 64) for its halves h
    {
      const uint32_t* qA = reinterpret_cast<const uint32_t*>(p.q + static_cast<int64_t>(b) * p.q_sb +
                                                              static_cast<int64_t>(hq0 + min(rA, rows_valid - 1)) * p.q_sh);
      const uint32_t* qB = reinterpret_cast<const uint32_t*>(p.q + static_cast<int64_t>(b) * p.q_sb +
                                                              static_cast<int64_t>(hq0 + min(rB, rows_valid - 1)) * p.q_sh);
#pragma unroll
      for (int hi = 0; hi < kTcHalvesPerWarp; ++hi) {
        const int h = hh * kTcHalvesPerWarp + hi;
        uint32_t qv[16];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          qv[2 * g] = rA < rows_valid ? __ldg(qA + 32 * h + 4 * g + a4) : 0u;
          qv[2 * g + 1] = rB < rows_valid ? __ldg(qB + 32 * h + 4 * g + a4) : 0u;
        }
        tc_st16x128_x8(tmem + lane_addr + kTcColQ + 32 * h, qv);
      }
      tc_wait_st();
      tc_fence_before();
      mbar_arrive(smem_u32(&q_bar));
    }
    constexpr int NSV = 32 * kTcHalvesPerWarp;            // S values per thread and stage
    float mA = kNegInf, mB = kNegInf, lA = 0.f, lB = 0.f;   // reference maxima (log2 units), partial sums
    for (int s = 0; s < n_st; ++s) {
      const int sb = s & 1;
      const uint32_t sp = tmem + lane_addr + kTcColSP + sb * kTcT;   // the S / P buffer of this stage
      const int valid = min(kTcT, t_end - (t0 + s * kTcT));
      tc_wait(smem_u32(&s_full[sb]), (s >> 1) & 1, 7, s);
      tc_fence_after();
      if (threadIdx.x == 0) TC_TRACE(16, s);
      if (threadIdx.x == 0 && s == 0) TC_TRACE_CTA(5);
      float sv[NSV];   // [half hi][group g][4]: tokens 64 h + 8 g + 2 a (+1) of rows rA, rB
#pragma unroll
      for (int hi = 0; hi < kTcHalvesPerWarp; ++hi) {
        uint32_t r0[32];
        tc_ld16x256<8>(sp + 64 * (hh * kTcHalvesPerWarp + hi), r0);
        tc_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; ++c) sv[32 * hi + c] = __uint_as_float(r0[c]);
      }
      TC_TRACE_SMX(0, s);
      const int tok0 = 64 * hh * kTcHalvesPerWarp;       // first token of this warp's values
      if (valid < tok0 + NSV * 2) {                       // tokens past the range
#pragma unroll
        for (int g = 0; g < NSV / 4; ++g)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const bool ok = tok0 + 8 * g + 2 * a4 + c < valid;
            sv[4 * g + c] = ok ? sv[4 * g + c] : kNegInf;
            sv[4 * g + 2 + c] = ok ? sv[4 * g + 2 + c] : kNegInf;
          }
      }
      float xA = fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[4], sv[5]));
      float xB = fmaxf(fmaxf(sv[2], sv[3]), fmaxf(sv[6], sv[7]));
      float yA = fmaxf(fmaxf(sv[8], sv[9]), fmaxf(sv[12], sv[13]));
      float yB = fmaxf(fmaxf(sv[10], sv[11]), fmaxf(sv[14], sv[15]));
#pragma unroll
      for (int g = 4; g < NSV / 4; g += 2) {
        xA = fmaxf(xA, fmaxf(sv[4 * g], sv[4 * g + 1]));
        xB = fmaxf(xB, fmaxf(sv[4 * g + 2], sv[4 * g + 3]));
        yA = fmaxf(yA, fmaxf(sv[4 * g + 4], sv[4 * g + 5]));
        yB = fmaxf(yB, fmaxf(sv[4 * g + 6], sv[4 * g + 7]));
      }
      xA = fmaxf(xA, yA);
      xB = fmaxf(xB, yB);
      xA = fmaxf(xA, __shfl_xor_sync(0xffffffffu, xA, 1));
      xB = fmaxf(xB, __shfl_xor_sync(0xffffffffu, xB, 1));
      xA = fmaxf(xA, __shfl_xor_sync(0xffffffffu, xA, 2));
      xB = fmaxf(xB, __shfl_xor_sync(0xffffffffu, xB, 2));
      if (kTcSoftmaxWarps == 8) {   // the other token half's maximum (parity-double-buffered slots)
        if (a4 == 0) red_x[sb][hh][rA] = xA, red_x[sb][hh][rB] = xB;
        pair_sync();
        xA = fmaxf(xA, red_x[sb][hh ^ 1][rA]);
        xB = fmaxf(xB, red_x[sb][hh ^ 1][rB]);
      }
      TC_TRACE_SMX(1, s);
      const float mxA = xA * p.scale_log2, mxB = xB * p.scale_log2;   // >= 1 valid token: finite
      if (s == 0) mA = mxA, mB = mxB;                    // PV(0) starts O (accumulate = 0)
      // the reference moves only when this stage's maximum exceeds it by more than 2^8: then the
      // row's O (PV(0 .. s-1): wait for PV(s - 1)) and l are rescaled by exp2(m_old - m_new).  The
      // TMEM load / store is warp-collective: every lane takes part, factor 1 for unchanged rows.
      // Both warps of a quadrant see the same maxima, so they take the same decision, each for its
      // O columns
      const bool resA = s > 0 && mxA > mA + kTcRescaleLog2, resB = s > 0 && mxB > mB + kTcRescaleLog2;
      if (__any_sync(0xffffffffu, resA || resB)) {
        const float alA = resA ? ex2(mA - mxA) : 1.f, alB = resB ? ex2(mB - mxB) : 1.f;
        mbar_wait(smem_u32(&pv_done[(s - 1) & 1]), ((s - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int i = 0; i < 2 * kTcHalvesPerWarp; ++i) {   // hi / lo lanes x this warp's O column halves
          const int h = hh * kTcHalvesPerWarp + (i >> 1);
          uint32_t ov[32];
          const uint32_t ta = tmem + lane_addr + (static_cast<uint32_t>(16 * (i & 1)) << 16) + kTcColO + 64 * h;
          tc_ld16x256<8>(ta, ov);
          tc_wait_ld();
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            ov[4 * g] = __float_as_uint(__uint_as_float(ov[4 * g]) * alA);
            ov[4 * g + 1] = __float_as_uint(__uint_as_float(ov[4 * g + 1]) * alA);
            ov[4 * g + 2] = __float_as_uint(__uint_as_float(ov[4 * g + 2]) * alB);
            ov[4 * g + 3] = __float_as_uint(__uint_as_float(ov[4 * g + 3]) * alB);
          }
          tc_st16x256_x8(ta, ov);
        }
        tc_wait_st();
        if (resA) lA *= alA, mA = mxA;
        if (resB) lB *= alB, mB = mxB;
      }
      // P = exp2(scale S - m) <= 2^8 as the pair P_hi + P_lo, written over S(s): u32 column
      // j = tokens 2 j, 2 j + 1 = 4 g + a (16x128b layout: the S layout's token pair of group g);
      // P_hi on lanes 32 q + i, P_lo on lanes 32 q + 16 + i
      const float nA = -mA, nB = -mB;
      float sA0 = 0.f, sA1 = 0.f, sB0 = 0.f, sB1 = 0.f;
#pragma unroll
      for (int hi = 0; hi < kTcHalvesPerWarp; ++hi) {
        const int h = hh * kTcHalvesPerWarp + hi;
        uint32_t hw[16], lw[16];
#pragma unroll
        for (int g8 = 0; g8 < 8; ++g8) {
          const int g = 8 * hi + g8;
          const float pa0 = ex2(fmaf(sv[4 * g], p.scale_log2, nA)), pa1 = ex2(fmaf(sv[4 * g + 1], p.scale_log2, nA));
          const float pb0 = ex2(fmaf(sv[4 * g + 2], p.scale_log2, nB)), pb1 = ex2(fmaf(sv[4 * g + 3], p.scale_log2, nB));
          if (g8 & 1) sA1 += pa0 + pa1, sB1 += pb0 + pb1;
          else sA0 += pa0 + pa1, sB0 += pb0 + pb1;
          tc_pair(pa0, pa1, hw[2 * g8], lw[2 * g8]);
          tc_pair(pb0, pb1, hw[2 * g8 + 1], lw[2 * g8 + 1]);
        }
        tc_st16x128_x8(sp + 32 * h, hw);
        tc_st16x128_x8(sp + (16u << 16) + 32 * h, lw);
      }
      lA += sA0 + sA1;
      lB += sB0 + sB1;
      TC_TRACE_SMX(2, s);
      if (valid < kTcT) {
        // V rows past the range may hold anything (stale or NaN): zero them (P = 0 there)
        const int st = s % NV;
        tc_wait(smem_u32(&fullv_bar[st]), (s / NV) & 1, 8, s);
        const uint32_t sV = sbase + (NK + st) * kTcSlotBytes;
        for (int e = threadIdx.x; e < (kTcT - valid) * 16; e += kTcSoftmaxWarps * 32) {
          const int row = valid + (e >> 4), c = e & 15;
          sts128(sV + (c >> 3) * kTcHalfStride + sw128_chunk(row, c & 7), make_uint4(0, 0, 0, 0));
        }
        fence_proxy_async_smem();
      }
      tc_wait_st();
      TC_TRACE_SMX(3, s);
      TC_TRACE_PW(s);
      tc_fence_before();
      __syncwarp();
      if (threadIdx.x == 0) TC_TRACE(24, s);
      if (lane == 0) mbar_arrive(smem_u32(&p_full[sb]));
    }
    // ================= epilogue =================
    lA += __shfl_xor_sync(0xffffffffu, lA, 1);
    lB += __shfl_xor_sync(0xffffffffu, lB, 1);
    lA += __shfl_xor_sync(0xffffffffu, lA, 2);
    lB += __shfl_xor_sync(0xffffffffu, lB, 2);
    if (kTcSoftmaxWarps == 8) {   // both token halves' sums (same reference maxima in both warps)
      if (a4 == 0) red_l[hh][rA] = lA, red_l[hh][rB] = lB;
      pair_sync();
      lA += red_l[hh ^ 1][rA];
      lB += red_l[hh ^ 1][rB];
    }
    float invA = 0.f, invB = 0.f, lseA = kNegInf, lseB = kNegInf;
    if (n_st > 0) {
      mbar_wait(smem_u32(&pv_done[(n_st - 1) & 1]), ((n_st - 1) >> 1) & 1);
      if (threadIdx.x == 0) TC_TRACE_CTA(6);
      tc_fence_after();
      invA = lA > 0.f ? rcp(lA) : 0.f;
      invB = lB > 0.f ? rcp(lB) : 0.f;
      lseA = lA > 0.f ? (mA + lg2(lA)) * kLn2 : kNegInf;
      lseB = lB > 0.f ? (mB + lg2(lB)) * kLn2 : kNegInf;
    }
    const size_t rowA = static_cast<size_t>(b) * p.h_q + hq0 + rA, rowB = rowA + 8;
    const size_t prowA = static_cast<size_t>(split) * p.batch * p.h_q + rowA, prowB = prowA + 8;
    const bool wA = rA < rows_valid, wB = rB < rows_valid;
#pragma unroll
    for (int hi = 0; hi < kTcHalvesPerWarp; ++hi) {
      const int h = hh * kTcHalvesPerWarp + hi;
      uint32_t ov[32];
      if (n_st > 0) {   // O = the hi lanes' part + the lo lanes' part
        uint32_t ol[32];
        tc_ld16x256<8>(tmem + lane_addr + kTcColO + 64 * h, ov);
        tc_ld16x256<8>(tmem + lane_addr + (16u << 16) + kTcColO + 64 * h, ol);
        tc_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; ++c) ov[c] = __float_as_uint(__uint_as_float(ov[c]) + __uint_as_float(ol[c]));
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) ov[c] = 0u;
      }
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const int col = 64 * h + 8 * g + 2 * a4;            // dims col, col + 1
        const float2 vA = make_float2(__uint_as_float(ov[4 * g]) * invA, __uint_as_float(ov[4 * g + 1]) * invA);
        const float2 vB = make_float2(__uint_as_float(ov[4 * g + 2]) * invB, __uint_as_float(ov[4 * g + 3]) * invB);
        if (kernel_combine) {
          if (wA) *reinterpret_cast<float2*>(p.ws_o + prowA * kHeadDim + col) = vA;
          if (wB) *reinterpret_cast<float2*>(p.ws_o + prowB * kHeadDim + col) = vB;
        } else if (p.out_f32) {
          if (wA) *reinterpret_cast<float2*>(static_cast<float*>(p.out) + rowA * kHeadDim + col) = vA;
          if (wB) *reinterpret_cast<float2*>(static_cast<float*>(p.out) + rowB * kHeadDim + col) = vB;
        } else {
          if (wA) *reinterpret_cast<uint32_t*>(static_cast<uint16_t*>(p.out) + rowA * kHeadDim + col) = pack_bf16(vA.x, vA.y);
          if (wB) *reinterpret_cast<uint32_t*>(static_cast<uint16_t*>(p.out) + rowB * kHeadDim + col) = pack_bf16(vB.x, vB.y);
        }
      }
    }
    if (a4 == 0 && hh == 0) {
      if (kernel_combine) {
        if (wA) p.ws_lse[prowA] = lseA;
        if (wB) p.ws_lse[prowB] = lseB;
      } else if (p.lse != nullptr) {
        if (wA) p.lse[rowA] = lseA;
        if (wB) p.lse[rowB] = lseB;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) TC_TRACE_CTA(1);
  if (warp == kTcMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcTmemCols));
  }
}

cudaError_t tc_prepare() {
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  const uint64_t bit = 1ull << (dev & 63);
  if ((attr_done.load(std::memory_order_acquire) & bit) == 0) {
    err = cudaFuncSetAttribute(split_kv_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem);
    if (err != cudaSuccess) return err;
    attr_done.fetch_or(bit, std::memory_order_acq_rel);
  }
  return cudaSuccess;
}

}  // namespace

cudaError_t launch_split_kv_fwd_tc(const da_plan& plan, const CUtensorMap& tmap_k, const CUtensorMap& tmap_v,
                                   const FwdParams& p, cudaStream_t stream) {
  cudaError_t err = tc_prepare();
  if (err != cudaSuccess) return err;
  if (plan.block_threads != kTcThreads || plan.smem_bytes != kTcSmem || plan.rows_per_cta != kTcM)
    return cudaErrorInvalidConfiguration;
  if (plan.combine_mode != DA_COMBINE_NONE && plan.combine_mode != DA_COMBINE_KERNEL) return cudaErrorInvalidValue;
  if (p.pub.bases != nullptr) return cudaErrorNotSupported;   // the C ABI rejects these calls first
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(plan.grid_x, plan.grid_y, plan.grid_z);
  cfg.blockDim = dim3(kTcThreads, 1, 1);
  cfg.dynamicSmemBytes = kTcSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int kernel_combine = plan.combine_mode == DA_COMBINE_KERNEL ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, split_kv_fwd_tc_kernel, tmap_k, tmap_v, p, kernel_combine);
}

cudaError_t forward_tc_residency(int* out) {
  cudaError_t err = tc_prepare();
  if (err != cudaSuccess) return err;
  int dev = 0, sms = 0, per_sm = 0;
  if ((err = cudaGetDevice(&dev)) != cudaSuccess) return err;
  if ((err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return err;
  if ((err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, split_kv_fwd_tc_kernel, kTcThreads, kTcSmem)) !=
      cudaSuccess)
    return err;
  *out = per_sm * sms;
  return cudaSuccess;
}

#ifdef DECATTN_TRACE
extern "C" __attribute__((visibility("default"))) int da_trace_fetch_tc(unsigned long long* host, int n) {
  if (n > 64 * 64) n = 64 * 64;
  return cudaMemcpyFromSymbol(host, g_trace_tc, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 1;
}
extern "C" __attribute__((visibility("default"))) int da_trace_fetch_tc_smx(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_trace_smx, sizeof(unsigned long long) * 4 * 8) == cudaSuccess ? 0 : 1;
}
extern "C" __attribute__((visibility("default"))) int da_trace_fetch_tc_pw(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_trace_pw, sizeof(unsigned long long) * 16 * 8) == cudaSuccess ? 0 : 1;
}
extern "C" __attribute__((visibility("default"))) int da_trace_fetch_tc_cta(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_cta_tc, sizeof(unsigned long long) * 8 * 1024) == cudaSuccess ? 0 : 1;
}
extern "C" __attribute__((visibility("default"))) int da_trace_fetch_tc_clock(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_clock_tc, sizeof(unsigned long long) * 4) == cudaSuccess ? 0 : 1;
}
#endif

int tc_block_threads() { return kTcThreads; }
int tc_smem_bytes() { return kTcSmem; }

}  // namespace decattn
