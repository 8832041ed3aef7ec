// Split planner: da_plan_make / da_plan_make_varlen / da_plan_set_combine (host-only,
// integer-only).
//
// Implements the decision the paper is about: how many sequence splits a
// decode-attention launch uses.  The paper's two policies, plus FIXED, the
// evolved Fig. 1 fragment, the SM-count-aware generalisation (C-ext-1), the
// per-batch dynamic counts (C-ext-2) and the host-side choice between them (C-ext-3):
//   * guarded   - FA3's default (§2.2 "returns s=1 if the sequence
//                 length L_K <= 512"; §4.2 "strictly enforced s=1 when
//                 num_n_blocks <= 4"), behind the saturation guard and ahead
//                 of the efficiency loop (DESIGN.md C-amb-2..4);
//   * seq-aware - the paper's Fig. 3 cascade: Guard 1, Guard 2,
//                 the low-tile override s = 3, else the unchanged loop.
// Every comparison is an exact integer cross-multiplication (C-amb-3), so the
// result is bit-identical to the CPU oracle's (tests/test_abi_cpu.py).
// This file shares no code with oracle/: it is the product-side statement.
#include <cstdint>

#include "../../include/decattn.h"
#include "config.h"

namespace decattn {
namespace {

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// FA3-style first guard: total_mblocks >= 0.8 * usable SMs  <=>  5T >= 4U.
inline bool saturated(int64_t T, int64_t U) { return 5 * T >= 4 * U; }

// Efficiency loop (referenced by P:L85; reconstruction in
// DESIGN.md C-amb-2).  Candidates s = 1..min(128, U, nblk); waves
// w_s = ceil(T s / U); efficiency(s) = T s / (U w_s).  Smallest s with
// efficiency(s) >= 0.85 * best, i.e. 20 s w* >= 17 s* w_s.
int efficiency_loop(int64_t T, int64_t U, int64_t nblk) {
  int64_t smax = kEffMaxSplits;
  if (U < smax) smax = U;
  if (nblk < smax) smax = nblk;
  int64_t best_s = 1, best_w = ceil_div(T, U);
  for (int64_t s = 2; s <= smax; ++s) {
    const int64_t w = ceil_div(T * s, U);
    if (s * best_w > best_s * w) { best_s = s; best_w = w; }
  }
  for (int64_t s = 1; s <= smax; ++s) {
    const int64_t w = ceil_div(T * s, U);
    if (20 * s * best_w >= 17 * best_s * w) return static_cast<int>(s);
  }
  return 1;
}

// Query rows per CTA on the tensor-core path: 8, or 16 for G > 8 beyond kSmMidUnits units (two
// 8-row CTAs halve the per-warp MMA work and keep the kernel inside the instruction cache on
// short sequences; on long ones they would read every KV tile twice).
int64_t mma_rows(int64_t G, int64_t l_k) { return G <= 8 || ceil_div(l_k, kSmUnit) <= kSmMidUnits ? 8 : 16; }

// Largest s in 1..16 whose T clusters of s CTAs are all co-resident in one wave of U SMs
// (the B200 table in config.h scaled by U / 148); s = 1 always qualifies.
int64_t cluster_fit_splits(int64_t T, int64_t U) {
  int64_t best = 1;
  for (int s = 2; s <= kMaxClusterSplits; ++s)
    if (T <= static_cast<int64_t>(kMaxActiveClustersB200[s]) * U / 148) best = s;
  return best;
}

void decide(int64_t batch, int64_t l_k, int64_t T, int64_t U, int64_t nblk, int64_t G, int64_t mblocks,
            int policy, int forced, int* s, int* rule) {
  if (policy == DA_POLICY_FIXED) { *s = forced; *rule = DA_RULE_FORCED; return; }
  if (policy == DA_POLICY_DYNAMIC) {          // C-ext-2: the cap; counts are decided per batch on the device
    int64_t cap = ceil_div(l_k, kSplitUnit);
    if (cap > kDynMaxSplits) cap = kDynMaxSplits;
    *s = static_cast<int>(cap < 1 ? 1 : cap);
    *rule = DA_RULE_DYNAMIC;
    return;
  }
  if (policy == DA_POLICY_EVOLVED) {
    if (batch == 1) {                                                    // Fig. 1
      *s = l_k < kEvolvedShortLk ? kEvolvedShortSplits : kEvolvedSplits;
      *rule = DA_RULE_EVOLVED;
      return;
    }
    policy = DA_POLICY_GUARDED;      // the fragment shows no batch != 1 branch: FA3 default
  }
  if (saturated(T, U)) { *s = 1; *rule = DA_RULE_SATURATED; return; }
  if (policy == DA_POLICY_SEQ_AWARE_SM) {                                 // C-ext-1
    const int64_t n_u = ceil_div(l_k, kSmUnit);
    // the CTA groups the kernel launches per split (= T for G <= 8)
    const int64_t rows = mma_rows(G, l_k);
    const int64_t Tk = T / mblocks * ceil_div(G, rows);
    const int64_t f = cluster_fit_splits(Tk, U);
    if (nblk <= 4) {
      if (n_u < kSmMinUnits || (n_u < kSmMinUnitsWide && Tk > kSmWideT)) {
        *s = 1; *rule = DA_RULE_SM_SHORT; return;
      }
      int64_t v = Tk <= kSmNarrowT ? kSmNarrowSplits : kSmMaxSplits;
      if (n_u < v) v = n_u;
      if (f < v) v = f;
      if (v < kSmMinSplits) { *s = 1; *rule = DA_RULE_SM_SHORT; return; }
      *s = static_cast<int>(v);
      *rule = DA_RULE_SM_SPLIT;
      return;
    }
    const int64_t e = efficiency_loop(T, U, nblk);
    const int64_t c = Tk <= kSmNarrowT ? kSmNarrowSplits : kSmMaxSplits;
    int64_t v;
    if (e <= f) {
      int64_t floor_s = c;
      if (n_u < floor_s) floor_s = n_u;
      if (f < floor_s) floor_s = f;
      v = e > floor_s ? e : floor_s;
    } else if (f >= 2 && rows == 8 && (n_u <= kSmStreamUnits * f || 2 * Tk * f >= U)) {
      v = f;
    } else {
      *s = static_cast<int>(e);            // streaming: the loop's split as is
      *rule = DA_RULE_EFF_LOOP;
      return;
    }
    if (n_u <= kSmMidUnits) {               // short sequences: at most 4 (T > 8) or 12 splits
      const int64_t cap = Tk > kSmMidT ? kSmMaxSplits : kSmClusterCap;
      if (v > cap) v = cap;
    }
    // wide groups: a <= 2-CTA cluster split gives way to the loop's split on the tcgen05 kernel
    // when that kernel's rule (tc_path) accepts it and the sequence has >= kSmTcUnits units
    if (G >= kTcMinG && v <= kSmTcMaxFit && n_u >= kSmTcUnits && n_u >= static_cast<int64_t>(kTcMinTiles) * e &&
        2 * (T / mblocks) * ceil_div(G, static_cast<int64_t>(kTcRows)) * e >= U) {
      *s = static_cast<int>(e);
      *rule = DA_RULE_EFF_LOOP;
      return;
    }
    *s = static_cast<int>(v);
    *rule = v == e ? DA_RULE_EFF_LOOP : DA_RULE_SM_FIT;
    return;
  } else if (policy == DA_POLICY_GUARDED) {
    if (nblk <= 4) { *s = 1; *rule = DA_RULE_GUARD_NBLK4; return; }
  } else {  // DA_POLICY_SEQ_AWARE, Fig. 3 in order
    if (nblk <= 3) { *s = 1; *rule = DA_RULE_GUARD1; return; }
    if (nblk <= 4 && T >= 4) { *s = 1; *rule = DA_RULE_GUARD2; return; }
    if (nblk == 4 && T < 4) { *s = kLowTileSplits; *rule = DA_RULE_LOW_TILE; return; }
  }
  *s = efficiency_loop(T, U, nblk);
  *rule = DA_RULE_EFF_LOOP;
}

}  // namespace

// DA_POLICY_DYNAMIC with a cap above one: the split CTAs are slots assigned on the device.
bool is_dynamic(const da_plan& p) { return p.policy == DA_POLICY_DYNAMIC && p.num_splits > 1; }

// Rows per CTA on the tensor-core path: mma_rows, except that 8-row CTAs for G > 8 need the
// whole grid (B x H_KV x ceil(G / 8) x s CTAs) in one wave; past it 16-row CTAs stand.
static int64_t launch_rows(const da_plan& p) {
  const int64_t G = p.h_q / p.h_kv;
  int64_t rows = mma_rows(G, p.l_k);
  if (rows == 8 && G > 8 &&
      static_cast<int64_t>(p.batch) * p.h_kv * ceil_div(G, 8) * p.num_splits > p.usable_sms)
    rows = 16;
  return rows;
}

// pack_gqa plans with G >= kTcMinG and a static split count run the tcgen05 kernel (fwd_tc.cu: 64
// query rows per CTA, no cluster combine) when every split holds >= kTcMinTiles tiles and its grid
// has >= U / 2 CTAs; otherwise the mma.sync kernel (8 / 16-row CTAs: 4x the CTAs at G = 64, few-tile
// CTAs spread over 3-7 warps and merged through clusters), which wins on short or few splits
// (profiles/r02ze_mid.log).  da_plan_set_path overrides the choice.
bool tc_path(const da_plan& p) {
  const int64_t G = p.h_q / p.h_kv;
  if (p.pack_gqa == 0 || G < 2 || is_dynamic(p)) return false;
  if (p.path_override == DA_PATH_TC) return true;
  if (p.path_override == DA_PATH_MMA) return false;
  const int64_t ctas = static_cast<int64_t>(p.batch) * p.h_kv * ceil_div(G, kTcRows) * p.num_splits;
  return G >= kTcMinG &&
         ceil_div(static_cast<int64_t>(p.l_k), kSplitUnit) >= static_cast<int64_t>(kTcMinTiles) * p.num_splits &&
         2 * ctas >= p.usable_sms;
}

// Launch geometry for a plan whose decision fields are set.  Shared by
// da_plan_make, da_plan_set_combine and da_forward's consistency check.
void derive_launch(da_plan* p) {
  const int G = p->h_q / p->h_kv;
  const bool mma = p->pack_gqa != 0 && G >= 2;
  p->path = mma ? DA_PATH_MMA : DA_PATH_SCALAR;
  p->rows_per_cta = mma ? static_cast<int32_t>(launch_rows(*p)) : 1;
  p->grid_x = p->num_splits;
  p->grid_y = mma ? p->h_kv * static_cast<int32_t>(ceil_div(G, p->rows_per_cta)) : p->h_q;
  p->grid_z = p->batch;
  if (is_dynamic(*p)) {
    // split slots: sum_b s_b <= sum_b n_u_b / W + B <= U / T_b + B for any lengths (C-ext-2)
    const int64_t tiles = static_cast<int64_t>(p->h_kv) * p->num_m_blocks;
    int64_t slots = ceil_div(p->usable_sms, tiles) + p->batch;
    const int64_t most = static_cast<int64_t>(p->batch) * p->num_splits;
    p->grid_x = p->grid_y;                                 // head groups innermost (DRAM row sharing)
    p->grid_y = static_cast<int32_t>(slots < most ? slots : most);
    p->grid_z = 1;
  }
  const bool cluster = p->combine_mode == DA_COMBINE_CLUSTER;
  p->block_threads = threads_for(warps_for(p->combine_mode), helpers_for(p->combine_mode));
  p->cluster_x = cluster ? p->num_splits : 1;
  p->smem_bytes = smem_for(stages_for(p->combine_mode), cluster);
  if (is_dynamic(*p)) {   // mostly one split per sequence: the streaming (s = 1) configuration
    p->block_threads = threads_for(kWarpsNone, 0);
    p->smem_bytes = smem_for(kStagesNone, false);
  }
  if (tc_path(*p)) {      // tcgen05 kernel: the G query rows of a KV head in ceil(G / 64) CTAs
    p->path = DA_PATH_TC;
    p->rows_per_cta = kTcRows;
    p->grid_y = p->h_kv * static_cast<int32_t>(ceil_div(G, kTcRows));
    p->block_threads = kTcThreadsCfg;
    p->smem_bytes = kTcSmemCfg;
    p->cluster_x = 1;
  }
  p->workspace_bytes = p->num_splits > 1
      ? static_cast<int64_t>(p->num_splits) * p->batch * p->h_q * (p->head_dim + 1) * 4
      : 0;
  if (is_dynamic(*p))   // partials per slot, then the schedule (first slot, split count) per b
    p->workspace_bytes = static_cast<int64_t>(p->grid_y) * p->h_q * (p->head_dim + 1) * 4 + 8LL * p->batch;
}

// s == 1: NONE.  2 <= s <= 16: CLUSTER when every cluster of the launch is co-resident in one
// wave (the B200 table in config.h, scaled by the usable SM count), else the workspace +
// combine-kernel path, which has no placement constraint.
int default_combine_mode(const da_plan& p) {
  const int s = p.num_splits;
  if (s == 1) return DA_COMBINE_NONE;
  if (is_dynamic(p)) return DA_COMBINE_KERNEL;   // per-batch split counts: no uniform cluster shape
  if (tc_path(p)) return DA_COMBINE_KERNEL;       // the tcgen05 kernel has no cluster combine
  if (s > kMaxClusterSplits) return DA_COMBINE_KERNEL;
  const int G = p.h_q / p.h_kv;
  const bool mma = p.pack_gqa != 0 && G >= 2;
  const int64_t rows = mma ? launch_rows(p) : 1;
  const int64_t clusters = static_cast<int64_t>(p.batch) * (mma ? p.h_kv * ceil_div(G, rows) : p.h_q);
  const int64_t fit = static_cast<int64_t>(kMaxActiveClustersB200[s]) * p.num_sms / 148;
  return clusters <= fit ? DA_COMBINE_CLUSTER : DA_COMBINE_KERNEL;
}

bool combine_mode_valid(int mode, int s) {
  switch (mode) {
    case DA_COMBINE_NONE: return s == 1;
    case DA_COMBINE_CLUSTER: return s >= 2 && s <= kMaxClusterSplits;
    case DA_COMBINE_KERNEL: return s >= 2;
    default: return false;
  }
}

}  // namespace decattn

using namespace decattn;

extern "C" da_status da_plan_make(int32_t batch, int32_t h_q, int32_t h_kv, int32_t l_k,
                                  int32_t head_dim, int32_t pack_gqa, int32_t sm_margin,
                                  int32_t num_sms, int32_t policy, int32_t forced_splits,
                                  da_plan* out) {
  if (out == nullptr) return DA_ERR_INVALID_ARG;
  if (batch < 1 || h_q < 1 || h_kv < 1 || l_k < 1 || head_dim < 1 || num_sms < 1)
    return DA_ERR_INVALID_ARG;
  if (h_q % h_kv != 0) return DA_ERR_INVALID_ARG;
  if (sm_margin < 0 || sm_margin >= num_sms) return DA_ERR_INVALID_ARG;
  if (pack_gqa != 0 && pack_gqa != 1) return DA_ERR_INVALID_ARG;
  if (policy < DA_POLICY_GUARDED || policy > DA_POLICY_DYNAMIC) return DA_ERR_INVALID_ARG;
  if (policy == DA_POLICY_FIXED && (forced_splits < 1 || forced_splits > kMaxForcedSplits))
    return DA_ERR_INVALID_ARG;
  if (head_dim != kHeadDim) return DA_ERR_UNSUPPORTED;

  da_plan p{};
  p.batch = batch; p.h_q = h_q; p.h_kv = h_kv; p.l_k = l_k; p.head_dim = head_dim;
  p.pack_gqa = pack_gqa; p.sm_margin = sm_margin; p.num_sms = num_sms;
  p.policy = policy; p.forced_splits = policy == DA_POLICY_FIXED ? forced_splits : 0;

  const int64_t G = h_q / h_kv;
  p.usable_sms = num_sms - sm_margin;                                // C-amb-8
  p.block_n = kPolicyBlockN;
  p.num_n_blocks = static_cast<int32_t>(ceil_div(l_k, kPolicyBlockN));
  p.num_m_blocks = static_cast<int32_t>(ceil_div(G, kPolicyBlockM));
  const int64_t T = static_cast<int64_t>(batch) * h_kv * p.num_m_blocks;
  if (T > INT32_MAX) return DA_ERR_INVALID_ARG;
  p.total_mblocks = static_cast<int32_t>(T);

  int s = 1, rule = 0;
  decide(batch, l_k, T, p.usable_sms, p.num_n_blocks, G, p.num_m_blocks, policy, forced_splits, &s, &rule);
  p.num_splits = s;
  p.rule = rule;
  p.split_unit = kSplitUnit;
  const int64_t units = ceil_div(l_k, kSplitUnit);
  p.nonempty_splits = static_cast<int32_t>(units < s ? units : s);
  p.combine_mode = default_combine_mode(p);
  derive_launch(&p);
  *out = p;
  return DA_OK;
}

// C-ext-3: the plan for a ragged batch whose lengths are on the host.  The static SM-count-aware
// plan for the capacity, unless its longest split would hold more than 2 W units (W the dynamic
// schedule's per-CTA work) and at least kVarlenMinUnits; then DA_POLICY_DYNAMIC.
extern "C" da_status da_plan_make_varlen(int32_t batch, int32_t h_q, int32_t h_kv, int32_t l_cap,
                                         int32_t head_dim, int32_t pack_gqa, int32_t sm_margin,
                                         int32_t num_sms, const int32_t* host_seqlens, da_plan* out) {
  if (host_seqlens == nullptr || out == nullptr) return DA_ERR_INVALID_ARG;
  da_plan st{};
  da_status r = da_plan_make(batch, h_q, h_kv, l_cap, head_dim, pack_gqa, sm_margin, num_sms,
                             DA_POLICY_SEQ_AWARE_SM, 0, &st);
  if (r != DA_OK) return r;
  int64_t total = 0, u_max = 0;
  for (int32_t b = 0; b < batch; ++b) {
    int64_t n = host_seqlens[b];
    n = n < 0 ? 0 : (n > l_cap ? l_cap : n);
    const int64_t u = ceil_div(n, kSplitUnit);
    total += u;
    if (u > u_max) u_max = u;
  }
  const int64_t tiles = static_cast<int64_t>(h_kv) * st.num_m_blocks;
  int64_t W = ceil_div(total * tiles, st.usable_sms);
  if (W < 1) W = 1;
  const int64_t c = ceil_div(u_max, st.num_splits);
  if (c > 2 * W && c >= kVarlenMinUnits)
    return da_plan_make(batch, h_q, h_kv, l_cap, head_dim, pack_gqa, sm_margin, num_sms,
                        DA_POLICY_DYNAMIC, 0, out);
  *out = st;
  return DA_OK;
}

extern "C" da_status da_plan_set_seq_offset(da_plan* plan, int32_t seq_offset) {
  if (plan == nullptr || seq_offset < 0) return DA_ERR_INVALID_ARG;
  plan->seq_offset = seq_offset;
  return DA_OK;
}

extern "C" da_status da_plan_set_path(da_plan* plan, int32_t path) {
  if (plan == nullptr) return DA_ERR_INVALID_ARG;
  const int32_t G = plan->h_kv > 0 ? plan->h_q / plan->h_kv : 0;
  if (plan->pack_gqa == 0 || G < 2) return DA_ERR_INVALID_ARG;          // the scalar kernel only
  if (path != -1 && path != DA_PATH_MMA && path != DA_PATH_TC) return DA_ERR_INVALID_ARG;
  if (path == DA_PATH_TC && is_dynamic(*plan)) return DA_ERR_INVALID_ARG;
  plan->path_override = path == -1 ? 0 : path;
  if (tc_path(*plan) && plan->combine_mode == DA_COMBINE_CLUSTER) plan->combine_mode = DA_COMBINE_KERNEL;
  if (!tc_path(*plan) && plan->combine_mode == DA_COMBINE_KERNEL && plan->num_splits <= kMaxClusterSplits)
    plan->combine_mode = default_combine_mode(*plan);                 // the mma.sync kernel's own choice
  derive_launch(plan);
  return DA_OK;
}

extern "C" da_status da_plan_set_combine(da_plan* plan, int32_t combine_mode) {
  if (plan == nullptr) return DA_ERR_INVALID_ARG;
  if (!combine_mode_valid(combine_mode, plan->num_splits)) return DA_ERR_INVALID_ARG;
  if (is_dynamic(*plan) && combine_mode != DA_COMBINE_KERNEL) return DA_ERR_INVALID_ARG;
  if (tc_path(*plan) && combine_mode == DA_COMBINE_CLUSTER) return DA_ERR_INVALID_ARG;
  plan->combine_mode = combine_mode;
  derive_launch(plan);
  return DA_OK;
}
