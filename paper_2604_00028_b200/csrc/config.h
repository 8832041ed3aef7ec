// Compile-time configuration shared by the planner (plan.cpp), the C ABI
// (capi.cpp) and the kernels (fwd.cu, combine.cu).  DESIGN.md §5 explains
// every number.
#pragma once

#ifdef __CUDACC__
#define DA_HD __host__ __device__
#else
#define DA_HD
#endif

namespace decattn {

// ---- policy accounting (paper side) -------------------------
constexpr int kPolicyBlockN = 128;     // nblk = ceil(L_K / 128)  (C-amb-1)
constexpr int kPolicyBlockM = 64;      // num_m_blocks = ceil(G / 64)
constexpr int kLowTileSplits = 3;      // Fig. 3 "return 3" (C-amb-5)
constexpr int kEffMaxSplits = 128;     // efficiency-loop candidate cap (C-amb-2)
constexpr int kMaxForcedSplits = 256;

// ---- kernel geometry (B200 side) -----------------------------
constexpr int kHeadDim = 128;          // v1 supports d = 128 only
constexpr int kTileN = 64;             // tokens per pipeline stage (= split unit)
constexpr int kSplitUnit = kTileN;     // partition unit (C-pol item 6)
constexpr int kStageBytes = 4 * kTileN * 128;   // K|V x two 64-dim halves, 128 B rows = 32 KB
// Each consumer warp owns exactly one ring stage (stages == consumer warps), so
// a warp never waits on a stage another warp consumes: no mbarrier phase aliasing.
constexpr int kStagesDefault = 7;      // s == 1 and workspace-combine kernels: 224 KB ring, 8 warps
constexpr int kStagesCluster = 6;      // cluster-combine kernels: 192 KB ring + DSMEM push slots
constexpr int kMaxClusterSplits = 8;   // portable cluster size
// One pushed row: O[128] fp32, (m, l), padding to 16 bytes.  A rank owns ceil(R/s) rows and
// receives them from all s ranks (itself included): at most max_s s ceil(16/s) = 21 rows (s = 7).
constexpr int kSlotRowFloats = kHeadDim + 4;
constexpr int kMaxSlotRows = 21;
DA_HD constexpr int threads_for(int stages) { return (stages + 1) * 32; }   // + 1 TMA producer warp
DA_HD constexpr int smem_for(int stages, bool cluster) {
  return stages * kStageBytes + (cluster ? kMaxSlotRows * kSlotRowFloats * 4 : 0) + 1024;
}
constexpr int kCombineRowsPerCta = 4;  // combine kernel: one warp per (b, h) row

}  // namespace decattn
