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
constexpr int kEvolvedSplits = 12, kEvolvedShortSplits = 16, kEvolvedShortLk = 256;  // Fig. 1
// SM-count-aware generalisation (DESIGN.md C-ext-1): B200-calibrated, frozen constants
constexpr int kSmUnit = 64, kSmMinUnits = 5, kSmMinUnitsWide = 8, kSmWideT = 16, kSmMinSplits = 3;
constexpr int kSmNarrowT = 4, kSmNarrowSplits = 8, kSmMaxSplits = 4;
constexpr int kSmStreamUnits = 16, kSmMidT = 8, kSmMidUnits = 64, kSmClusterCap = 12;
// wide groups: a <= 2-CTA cluster split gives way to the efficiency loop's split on the tcgen05
// kernel (oracle/policy.py SM_TC_*; the kernel's own constants kTcMinG / kTcMinTiles / kTcRows)
constexpr int kSmTcMaxFit = 2, kSmTcUnits = 64;
constexpr int kDynMaxSplits = 128;   // DA_POLICY_DYNAMIC per-sequence cap (C-ext-2)
constexpr int kVarlenMinUnits = 32;  // da_plan_make_varlen: dynamic only for splits >= 2048 tokens (C-ext-3)

// ---- kernel geometry (B200 side) -----------------------------
constexpr int kHeadDim = 128;          // v1 supports d = 128 only
constexpr int kTileN = 64;             // tokens per pipeline stage (= split unit)
constexpr int kSplitUnit = kTileN;     // partition unit (C-pol item 6)
constexpr int kStageBytes = 4 * kTileN * 128;   // K|V x two 64-dim halves, 128 B rows = 32 KB
// Ring stages and consumer warps: stages are a multiple of warps and warp w owns stages
// w, w + NW, ... (consuming them in tile order), so no warp can observe a stale mbarrier
// phase.  Few consumer warps keep the cross-warp merge small (it reads one partial per
// warp); a deep ring keeps a single CTA's TMA ingest busy.  DESIGN.md §5.
// Per combine mode (A/B-measured on B200, scripts/ab_variants.py):
//   NONE (s == 1)        7 stages / 7 warps: a single CTA is TMA-ingest bound, keep 224 KB in flight
//   CLUSTER (2..8)       6 stages / 3 warps: few tiles per CTA, small cross-warp merge, + push slots
//   KERNEL (s > 8)       4 stages / 4 warps: HBM-streaming splits (long context)
// (each value can be overridden with -DDECATTN_<MODE>_<STAGES|WARPS>=n for A/B builds)
#ifndef DECATTN_NONE_STAGES
#define DECATTN_NONE_STAGES 7
#endif
#ifndef DECATTN_NONE_WARPS
#define DECATTN_NONE_WARPS 7
#endif
#ifndef DECATTN_CLUSTER_STAGES
#define DECATTN_CLUSTER_STAGES 6
#endif
#ifndef DECATTN_CLUSTER_WARPS
#define DECATTN_CLUSTER_WARPS 3
#endif
#ifndef DECATTN_KERNEL_STAGES
#define DECATTN_KERNEL_STAGES 4
#endif
#ifndef DECATTN_KERNEL_WARPS
#define DECATTN_KERNEL_WARPS 4
#endif
constexpr int kStagesNone = DECATTN_NONE_STAGES, kWarpsNone = DECATTN_NONE_WARPS;
constexpr int kStagesCluster = DECATTN_CLUSTER_STAGES, kWarpsCluster = DECATTN_CLUSTER_WARPS;
constexpr int kStagesKernel = DECATTN_KERNEL_STAGES, kWarpsKernel = DECATTN_KERNEL_WARPS;
DA_HD constexpr int stages_for(int combine_mode) {
  return combine_mode == 0 ? kStagesNone : (combine_mode == 1 ? kStagesCluster : kStagesKernel);
}
DA_HD constexpr int warps_for(int combine_mode) {
  return combine_mode == 0 ? kWarpsNone : (combine_mode == 1 ? kWarpsCluster : kWarpsKernel);
}
// Helper warps idle through the main loop and join the epilogue merges so that every merge
// is a single pass (cluster kernels: 3 consumers + producer + 4 helpers = 256 threads).
#ifndef DECATTN_CLUSTER_HELPERS
#define DECATTN_CLUSTER_HELPERS 4
#endif
DA_HD constexpr int helpers_for(int combine_mode) { return combine_mode == 1 ? DECATTN_CLUSTER_HELPERS : 0; }
#ifndef DECATTN_SPECULATE
#define DECATTN_SPECULATE 1   // prefetch the plan-length range also when cache_seqlens is given
#endif
// Tail balancing of cluster plans: when every split holds >= kBalMinTiles tiles, each
// CTA streams the first (1 - 1/kBalTailDiv) of its range and the last 1/kBalTailDiv of every range is
// pooled in chunks of kBalChunk tiles, handed out by a ticket counter in rank 0's shared memory, so
// CTAs on faster SMs take more of the pool and the cluster's CTAs end together.
#ifndef DECATTN_BAL_MIN_TILES
#define DECATTN_BAL_MIN_TILES 32
#endif
#ifndef DECATTN_BAL_TAIL_DIV
#define DECATTN_BAL_TAIL_DIV 4
#endif
#ifndef DECATTN_BAL_CHUNK
#define DECATTN_BAL_CHUNK 4
#endif
constexpr int kBalMinTiles = DECATTN_BAL_MIN_TILES, kBalTailDiv = DECATTN_BAL_TAIL_DIV, kBalChunk = DECATTN_BAL_CHUNK;
// tcgen05 path (fwd_tc.cu, DA_PATH_TC): pack_gqa with G >= kTcMinG; 64 query rows per CTA (the
// MMA's M), 8 softmax warps + a TMA producer warp + an MMA warp, separate K and V rings of
// 128-token slots (Q, S, P and O live in TMEM).  Never a cluster combine.
#ifndef DECATTN_TC_KSLOTS
#define DECATTN_TC_KSLOTS 2       // tcgen05 path: K ring slots of 128 tokens (32 KB)
#endif
#ifndef DECATTN_TC_VSLOTS
#define DECATTN_TC_VSLOTS 5       // tcgen05 path: V ring slots of 128 tokens (32 KB)
#endif
#ifndef DECATTN_TC_MIN_G
#define DECATTN_TC_MIN_G 17       // G > 16: the mma.sync kernel's 16-row CTAs would read K / V twice or more
#endif
#ifndef DECATTN_TC_MIN_TILES
#define DECATTN_TC_MIN_TILES 4    // 64-token tiles per split at the plan's length (and >= U / 2 CTAs)
#endif
constexpr int kTcMinG = DECATTN_TC_MIN_G, kTcMinTiles = DECATTN_TC_MIN_TILES;
constexpr int kTcRows = 64;
#ifndef DECATTN_TC_QPREFETCH
#define DECATTN_TC_QPREFETCH 1    // L2 prefetch of the CTA's Q rows at kernel entry
#endif
#ifndef DECATTN_TC_SMX_WARPS
#define DECATTN_TC_SMX_WARPS 8    // softmax warps: 4 (one per TMEM lane quadrant) or 8 (two, token halves)
#endif
constexpr int kTcThreadsCfg = (DECATTN_TC_SMX_WARPS + 2) * 32;
constexpr int kTcSmemCfg = (DECATTN_TC_KSLOTS + DECATTN_TC_VSLOTS) * kStageBytes + 1024;   // 128-token stages; Q, S, P, O in TMEM
#ifndef DECATTN_L2_PROMOTION
#define DECATTN_L2_PROMOTION 3    // CU_TENSOR_MAP_L2_PROMOTION_L2_256B for the K / V tensor maps
#endif
#ifndef DECATTN_PREFETCH_LONG
#define DECATTN_PREFETCH_LONG 1   // the pre-wait L2 prefetch of the first ring tiles also for long splits
#endif
constexpr int kMaxPageSize = 1 << 18;     // da_forward_paged: tiles per page < 2^13 (exact magic division)
constexpr int kMaxClusterSplits = 16;
constexpr int kMaxPeers = 64;          // da_peer_signal / da_combine_peers: ranks of one exchange  // cluster combine up to 16 CTAs (non-portable size, B200)
// One pushed row: O[128] fp32, (m, l), padding to 16 bytes.  A rank owns ceil(R/s) rows and
// receives them from all s ranks (itself included): at most max_{s<=16} s ceil(16/s) = 30 rows (s = 15).
constexpr int kSlotRowFloats = kHeadDim + 4;
constexpr int kMaxSlotRows = 30;
// Co-resident clusters of s CTAs (one CTA per SM, the cluster kernel's ~221 KB of shared memory)
// measured on B200 (148 SMs): the CUDA occupancy API's answer for these exact kernels
// (da_query_residency), recorded by scripts/measure_residency.py in profiles/cluster_fit_b200.json;
// tests/test_abi_cpu.py checks this copy against that record and tests/test_gpu_residency.py both
// against the device.  Cluster placement is GPC-bound, hence not simply 148 / s.  Index: s.
constexpr int kMaxActiveClustersB200[17] = {0, 148, 74, 45, 33, 26, 22, 15, 15, 15, 11, 7, 7, 7, 7, 7, 7};
DA_HD constexpr int threads_for(int warps, int helpers = 0) { return (warps + 1 + helpers) * 32; }   // + TMA producer
DA_HD constexpr int smem_for(int stages, bool cluster) {
  return stages * kStageBytes + (cluster ? kMaxSlotRows * kSlotRowFloats * 4 : 0) + 1024;
}
constexpr int kCombineThreads = 128;   // combine kernel: one CTA of 4 warps per (b, h) row

}  // namespace decattn
