// Compile-time configuration shared by the planner (plan.cpp), the C ABI
// (capi.cpp) and the kernels (fwd.cu, combine.cu).  DESIGN.md §5 explains
// every number.
#pragma once

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
constexpr int kStages = 6;             // TMA ring depth
constexpr int kConsumerWarps = 4;      // warp w consumes stages w, w+4, ...
constexpr int kThreads = (kConsumerWarps + 1) * 32;   // + 1 TMA producer warp
constexpr int kStageBytes = 4 * kTileN * 128;         // K|V x two 64-column halves, 128 B rows
constexpr int kSmemBytes = kStages * kStageBytes + 1024;  // + 1024 B alignment slack (SWIZZLE_128B)
constexpr int kMaxClusterSplits = 8;   // portable cluster size
constexpr int kCombineRowsPerCta = 4;  // combine kernel: one warp per (b, h) row

}  // namespace decattn
