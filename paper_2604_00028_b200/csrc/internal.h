// Internal (non-ABI) declarations shared by capi.cpp and the .cu files.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/decattn.h"

namespace decattn {

// Arguments of the split-KV forward kernel (everything except the two
// tensor maps, which are passed as __grid_constant__ parameters).
// da_forward_peer: the kernel that writes the final rows writes them into slot e & 1 (e = *epoch
// + 1) of this rank's exchange buffer, and the last of its `writers` CTAs releases e into flag
// `rank` of every rank's buffer (the da_peer_signal step fused into the producer of the rows).
// bases == nullptr: off.
struct PubParams {
  const uint64_t* bases;    // device [world]: every rank's exchange buffer as mapped on this GPU
  int32_t* epoch;           // device: this rank's step epoch
  uint32_t* count;          // device: CTAs of this step that wrote their rows (0 between steps)
  int64_t slot_bytes, lse_offset, flag_offset;
  int32_t world, rank;
  int32_t writers;          // CTAs of the writing launch
  // da_forward_peer_combine (one-wave NONE / CLUSTER forwards): every CTA writes its rows as
  // self-validating 8-byte words (epoch << 32 | fp32 bits; no fence, no flag) into LL slot e & 1,
  // polls the same words of every rank and LSE-merges them into out / lse
  int64_t ll_offset, ll_slot_bytes;   // two LL slots [B H_Q][129] uint64 at ll_offset
  void* out;                // final [B, H_Q, d] bf16 or fp32
  float* lse;               // final [B, H_Q] or nullptr
  int32_t out_f32;
  // bounded spin: a peer word still not at this step's epoch timeout_ns after the
  // first failed poll ends the wait and sets *status = DA_EXCHANGE_TIMEOUT (the kernel completes)
  int32_t* status;
  uint64_t timeout_ns;
  // multi-rank emulation (da_forward_peer_combine with rank = -1; tests on one GPU): the launch
  // holds all `world` ranks' grids along z (rank r's CTAs at z in [r B, (r + 1) B), its K / V shard
  // at cache batches r B ..), and rank r has its own epoch[r], count[r], out[r] and lse[r]
  int32_t emulate;
};

struct FwdParams {
  const uint16_t* q;        // bf16 [B, H_Q, d]
  int64_t q_sb, q_sh;       // strides in elements
  const int32_t* seqlens;   // device int32 [B] or nullptr: whole-sequence lengths
  int32_t seq_offset;       // tokens before this cache (sequence shard): n_b = seqlens[b] - seq_offset
  int32_t l_default;        // length used when seqlens == nullptr (plan->l_k)
  int32_t l_cap;            // cache capacity (clamp bound)
  int32_t num_splits;       // s
  uint64_t s_magic;         // ceil(2^38 / s): floor(x / s) = (x * s_magic) >> 38 for x s < 2^38
  int32_t G;                // H_Q / H_KV
  int32_t h_q;
  int32_t batch;
  int32_t mblocks_per_head; // MMA path: ceil(G / rows_per_cta); SCALAR: 1
  uint64_t mb_magic;        // ceil(2^38 / mblocks_per_head) (udiv_magic: no integer divide on the device)
  float scale_log2;         // softmax_scale * log2(e)
  void* out;                // [B, H_Q, d] bf16 or f32
  int32_t out_f32;
  float* lse;               // [B, H_Q] or nullptr
  float* ws_o;              // KERNEL combine: [s, B, H_Q, d]
  float* ws_lse;            // KERNEL combine: [s, B, H_Q]
  // paged KV cache (da_forward_paged); block_table == nullptr for a dense cache
  const int32_t* block_table;   // [B, bt_stride] page indices
  int64_t bt_stride;
  int32_t page_size;            // tokens per page, a multiple of kTileN, <= kMaxPageSize
  uint64_t page_magic;          // ceil(2^38 / (page_size / kTileN))
  // DA_POLICY_DYNAMIC (C-ext-2): blockIdx.x is a split slot; the (sequence, split) it serves is
  // decided on the device from the lengths.  ws_meta[b] / ws_meta[B + b] receive the schedule.
  int32_t dyn_tiles;            // T_b = H_KV * num_m_blocks
  int32_t dyn_u;                // usable SMs U
  int32_t* ws_meta;             // [2, B] int32 (first slot, split count) or nullptr
  int32_t dyn_via_combine;      // kDyn: s_b = 1 rows also go through the combine kernel (LL exchange)
  PubParams pub;                // fused peer publish (NONE / CLUSTER: this kernel writes the rows)
};

// Division by a launch-invariant divisor d without an integer divide: with m = ceil(2^38 / d),
// floor(x / d) = (x m) >> 38 exactly whenever x d < 2^38 (m d = 2^38 + delta, delta < d, so the
// product overshoots x / d by less than x / 2^38 < 1 / d, which cannot cross the next integer).
inline uint64_t div_magic(uint32_t d) { return ((uint64_t(1) << 38) + d - 1) / d; }

struct CombineParams {
  const float* o;           // split i at o + i * o_stride, [rows, d]
  int64_t o_stride;
  const float* lse_in;      // split i at lse_in + i * lse_stride, [rows]
  int64_t lse_stride;
  int32_t num_splits;
  int32_t rows;             // B * H_Q
  void* out;
  int32_t out_f32;
  float* lse;               // [rows] or nullptr
  // DA_POLICY_DYNAMIC: row r = (b, h) merges meta[B + b] splits starting at slot meta[b]; the
  // partial of slot j sits at o + (j * h_q + h) * d (o_stride / lse_stride give the slot stride)
  const int32_t* meta;      // [2, B] or nullptr (uniform: num_splits at o + i * o_stride)
  int32_t h_q;
  int32_t batch;
  PubParams pub;            // fused peer publish (KERNEL combine: this kernel writes the rows)
};

// plan.cpp
void derive_launch(da_plan* p);
bool is_dynamic(const da_plan& p);
bool tc_path(const da_plan& p);
bool combine_mode_valid(int mode, int s);

// fwd.cu
cudaError_t launch_split_kv_fwd(const da_plan& plan, const CUtensorMap& tmap_k,
                                const CUtensorMap& tmap_v, const FwdParams& p,
                                cudaStream_t stream);
// combine.cu
cudaError_t launch_lse_combine(const CombineParams& p, bool pdl, cudaStream_t stream);
cudaError_t launch_peer_signal(const uint64_t* peer_bases, int32_t world, int32_t rank, const float* o_local,
                               const float* lse_local, int32_t rows, int64_t slot_bytes, int64_t lse_offset,
                               int64_t flag_offset, int32_t* epoch, cudaStream_t stream);
cudaError_t launch_peer_combine(const uint64_t* peer_bases, int64_t slot_bytes, int64_t lse_offset,
                                int64_t flag_offset, const int32_t* epoch, int32_t world, int32_t rank, int32_t rows,
                                int32_t out_f32, void* out, float* lse, int32_t* status, uint64_t timeout_ns,
                                cudaStream_t stream);
// co-residency queries (da_query_residency): launch units of the instantiation a plan launches
// that fit the current device at once (fwd.cu: clusters for CLUSTER plans, else CTAs; pub = the
// exchange variant 0 / 1 / 2), and CTAs of the combine kernel (combine.cu)
cudaError_t forward_residency(const da_plan& plan, int pub, int* out);
// fwd_tc.cu (DA_PATH_TC)
cudaError_t launch_split_kv_fwd_tc(const da_plan& plan, const CUtensorMap& tmap_k, const CUtensorMap& tmap_v,
                                   const FwdParams& p, cudaStream_t stream);
cudaError_t forward_tc_residency(int* out);
cudaError_t combine_residency(int* out);

}  // namespace decattn
