// C ABI: da_forward / da_forward_paged / da_forward_host / da_combine / da_peer_signal / da_combine_peers /
// da_status_string / da_abi_version
// (da_plan_make, da_plan_set_combine live in plan.cpp).  See
// include/decattn.h for the contract of every entry point.
//
// This layer validates arguments (every host-checkable error returns before
// any launch, with no side effects), builds the two TMA tensor maps that
// describe the caller's K / V cache, and launches the kernels on the
// caller's stream.  It never allocates, synchronises or prints.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "../../include/decattn.h"
#include "config.h"
#include "internal.h"

using namespace decattn;

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  // Resolved once through the runtime (no -lcuda link dependency).
  static PFN_cuTensorMapEncodeTiled_v12000 fn = []() -> PFN_cuTensorMapEncodeTiled_v12000 {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }();
  return fn;
}

// True when [a, a + bytes) lies inside one CUDA-registered allocation (pinned host or device
// memory; the driver reports the allocation range), so one DMA may span it.  Pageable memory,
// or a driver without the attribute, answers false.
bool one_allocation(const void* a, size_t bytes) {
  using Fn = CUresult (*)(void*, CUpointer_attribute, CUdeviceptr);
  static Fn fn = []() -> Fn {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    if (cudaGetDriverEntryPoint("cuPointerGetAttribute", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<Fn>(ptr);
  }();
  if (fn == nullptr) return false;
  CUdeviceptr start = 0;
  size_t size = 0;
  const CUdeviceptr p = reinterpret_cast<CUdeviceptr>(a);
  if (fn(&start, CU_POINTER_ATTRIBUTE_RANGE_START_ADDR, p) != CUDA_SUCCESS ||
      fn(&size, CU_POINTER_ATTRIBUTE_RANGE_SIZE, p) != CUDA_SUCCESS)
    return false;
  return p >= start && p + bytes <= start + size;
}

// K or V cache [B, l_cap, H_KV, d] as a 5-D TMA tensor (d_lo = 64, t, d_hi = 2, H_KV, B):
// the head dim is split into two 64-element halves (d_hi stride 128 B) so one box of
// 64 x 64 x 2 x 1 x 1 brings a whole 64-token tile of K (or V) in a single TMA op, laid out
// in shared memory as [half][token][64 dims] with 128-byte rows and the 128-byte swizzle
// the consumers' ldmatrix addressing expects.  Tokens past l_cap read as zero.
// For a paged pool [num_pages, page_size, H_KV, d] the same map is built with (num_pages,
// page_size, page stride) in place of (B, l_cap, batch stride).
// box_halves: 2 = one box per 64-token tile (both 64-dim halves, the mma.sync kernels); 1 = one
// box per tile and half (the tcgen05 kernel's [half][128 tokens][64 dims] stages)
bool make_kv_tmap(CUtensorMap* map, const void* base, int32_t batch, int32_t l_cap, int32_t h_kv,
                  int64_t sb, int64_t st, int64_t sh, uint32_t box_halves = 2) {
  auto fn = encode_fn();
  if (fn == nullptr) return false;
  cuuint64_t dims[5] = {64, static_cast<cuuint64_t>(l_cap), 2, static_cast<cuuint64_t>(h_kv),
                        static_cast<cuuint64_t>(batch)};
  cuuint64_t strides[4] = {static_cast<cuuint64_t>(st) * 2, 128, static_cast<cuuint64_t>(sh) * 2,
                           static_cast<cuuint64_t>(sb) * 2};
  cuuint32_t box[5] = {64, static_cast<cuuint32_t>(kTileN), box_halves, 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  static_cast<CUtensorMapL2promotion>(DECATTN_L2_PROMOTION), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

constexpr uint64_t kDefaultTimeoutNs = 10ull * 1000 * 1000 * 1000;   // bounded exchange wait: 10 s

// Co-resident launch units of a kernel variant on the current device (da_query_residency),
// memoised per (device, kernel, exchange, path, rows, combine, cluster size): the answer depends on
// the compiled kernel and the device only.
cudaError_t residency(const da_plan& plan, int kernel, int exchange, int* out) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int, int, int, int>, int> memo;
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  const auto key = kernel == 1 ? std::make_tuple(dev, 1, 0, 0, 0, 0, 0)
                               : std::make_tuple(dev, 0, exchange, plan.path, plan.rows_per_cta, plan.combine_mode,
                                                 plan.combine_mode == DA_COMBINE_CLUSTER ? plan.num_splits : 0);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = memo.find(key);
    if (it != memo.end()) { *out = it->second; return cudaSuccess; }
  }
  int n = 0;
  err = kernel == 1 ? combine_residency(&n) : forward_residency(plan, exchange, &n);
  if (err != cudaSuccess) return err;
  std::lock_guard<std::mutex> g(mu);
  memo[key] = n;
  *out = n;
  return cudaSuccess;
}

// A plan may be edited by its owner; re-derive what the launch depends on.
da_status check_plan(const da_plan* plan) {
  if (plan->batch < 1 || plan->h_q < 1 || plan->h_kv < 1 || plan->l_k < 1) return DA_ERR_INVALID_ARG;
  if (plan->h_q % plan->h_kv != 0) return DA_ERR_INVALID_ARG;
  if (plan->head_dim != kHeadDim) return DA_ERR_UNSUPPORTED;
  if (plan->num_splits < 1 || plan->num_splits > kMaxForcedSplits) return DA_ERR_INVALID_ARG;
  if (plan->pack_gqa != 0 && plan->pack_gqa != 1) return DA_ERR_INVALID_ARG;
  if (!combine_mode_valid(plan->combine_mode, plan->num_splits)) return DA_ERR_INVALID_ARG;
  if (plan->seq_offset < 0) return DA_ERR_INVALID_ARG;
  if (plan->path_override != 0 && plan->path_override != DA_PATH_MMA && plan->path_override != DA_PATH_TC)
    return DA_ERR_INVALID_ARG;
  da_plan chk = *plan;
  derive_launch(&chk);
  if (chk.path != plan->path || chk.rows_per_cta != plan->rows_per_cta ||
      chk.grid_x != plan->grid_x || chk.grid_y != plan->grid_y || chk.grid_z != plan->grid_z ||
      chk.block_threads != plan->block_threads || chk.cluster_x != plan->cluster_x ||
      chk.smem_bytes != plan->smem_bytes || chk.workspace_bytes != plan->workspace_bytes)
    return DA_ERR_INVALID_ARG;
  if (plan->grid_y > 65535 || plan->grid_z > 65535) return DA_ERR_UNSUPPORTED;
  return DA_OK;
}

struct PagedArgs {
  const int32_t* block_table = nullptr;
  int64_t bt_stride = 0;
  int32_t page_size = 0;
  int32_t num_pages = 0;
};

// Shared body of da_forward / da_forward_paged.  For a paged cache, k_cache / v_cache are the
// page pools [num_pages, page_size, H_KV, d], strides[2..7] are (page, token, head) strides,
// and l_cap = max_pages_per_seq * page_size bounds the per-sequence length.
da_status forward_impl(const da_plan* plan, const void* q, const void* k_cache, const void* v_cache,
                       int32_t l_cap, const int32_t* cache_seqlens, const int64_t* strides,
                       float softmax_scale, int32_t out_dtype, void* out, float* lse, void* workspace,
                       int64_t workspace_bytes, void* cuda_stream, const PagedArgs& pg,
                       const PubParams* pub = nullptr) {
  // pub (da_forward_peer): the final rows go to the exchange slot, out / lse are unused
  if (plan == nullptr || q == nullptr || k_cache == nullptr || v_cache == nullptr || (out == nullptr && !pub))
    return DA_ERR_INVALID_ARG;
  da_status st = check_plan(plan);
  if (st != DA_OK) return st;
  if (l_cap < plan->l_k) return DA_ERR_INVALID_ARG;
  if (out_dtype != DA_BF16 && out_dtype != DA_F32) return DA_ERR_INVALID_ARG;
  if (!(softmax_scale <= 0.f) && !std::isfinite(softmax_scale)) return DA_ERR_INVALID_ARG;
  const bool paged = pg.block_table != nullptr;
  // the tcgen05 kernel does not publish into a peer exchange itself: with s == 1 the peer paths take
  // da_forward + da_peer_signal instead (with s > 1 the combine kernel publishes, as for any plan)
  if (pub != nullptr && plan->path == DA_PATH_TC && plan->combine_mode != DA_COMBINE_KERNEL) return DA_ERR_UNSUPPORTED;

  const int64_t B = plan->batch, HQ = plan->h_q, HKV = plan->h_kv, D = kHeadDim;
  const int64_t rows_per_major = paged ? pg.page_size : l_cap;   // tokens per batch entry / page
  int64_t sd[8];
  if (strides != nullptr) {
    std::memcpy(sd, strides, sizeof(sd));
  } else {
    sd[0] = HQ * D; sd[1] = D;                                   // q (b, h)
    sd[2] = rows_per_major * HKV * D; sd[3] = HKV * D; sd[4] = D; // k (b | page, t, h)
    sd[5] = sd[2]; sd[6] = sd[3]; sd[7] = sd[4];                  // v
  }
  for (int i = 0; i < 8; ++i) {
    if (sd[i] < 0) return DA_ERR_INVALID_ARG;
    if (sd[i] % 8 != 0) return DA_ERR_ALIGNMENT;
  }
  if (!aligned16(q) || !aligned16(k_cache) || !aligned16(v_cache) || (!pub && !aligned16(out)) ||
      (lse != nullptr && (reinterpret_cast<uintptr_t>(lse) & 3u) != 0))
    return DA_ERR_ALIGNMENT;
  if (cache_seqlens != nullptr && (reinterpret_cast<uintptr_t>(cache_seqlens) & 3u) != 0)
    return DA_ERR_ALIGNMENT;
  if (paged && (reinterpret_cast<uintptr_t>(pg.block_table) & 3u) != 0) return DA_ERR_ALIGNMENT;

  float* ws_o = nullptr;
  float* ws_lse = nullptr;
  int32_t* ws_meta = nullptr;
  const bool dyn = is_dynamic(*plan);
  // partial rows: static [s][B][H_Q]; dynamic [slot][H_Q] then the schedule [2][B] int32
  const int64_t prows = dyn ? int64_t(plan->grid_y) * HQ : int64_t(plan->num_splits) * B * HQ;
  if (plan->combine_mode == DA_COMBINE_KERNEL) {
    if (workspace == nullptr || workspace_bytes < plan->workspace_bytes) return DA_ERR_WORKSPACE;
    if (!aligned16(workspace)) return DA_ERR_ALIGNMENT;
    ws_o = static_cast<float*>(workspace);
    ws_lse = ws_o + prows * D;
    if (dyn) ws_meta = reinterpret_cast<int32_t*>(ws_lse + prows);
  }

  CUtensorMap tk, tv;
  // multi-rank emulation (da_forward_peer_combine, rank = -1): the cache holds every rank's shard
  const int32_t emul = (pub != nullptr && pub->emulate) ? pub->world : 1;
  const int32_t major = paged ? pg.num_pages : plan->batch * emul;
  const int32_t rows = paged ? pg.page_size : l_cap;
  const uint32_t halves = plan->path == DA_PATH_TC ? 1u : 2u;
  if (!make_kv_tmap(&tk, k_cache, major, rows, plan->h_kv, sd[2], sd[3], sd[4], halves) ||
      !make_kv_tmap(&tv, v_cache, major, rows, plan->h_kv, sd[5], sd[6], sd[7], halves))
    return DA_ERR_CUDA;

  FwdParams p{};
  p.q = static_cast<const uint16_t*>(q);
  p.q_sb = sd[0];
  p.q_sh = sd[1];
  p.seqlens = cache_seqlens;
  p.seq_offset = plan->seq_offset;
  p.l_default = plan->l_k;
  p.l_cap = l_cap;
  p.num_splits = plan->num_splits;
  p.s_magic = div_magic(static_cast<uint32_t>(plan->num_splits));
  p.G = plan->h_q / plan->h_kv;
  p.h_q = plan->h_q;
  p.batch = plan->batch;
  p.mblocks_per_head = plan->path != DA_PATH_SCALAR ? (p.G + plan->rows_per_cta - 1) / plan->rows_per_cta : 1;
  p.mb_magic = div_magic(static_cast<uint32_t>(p.mblocks_per_head));
  const float scale = softmax_scale > 0.f ? softmax_scale : 1.0f / std::sqrt(float(D));
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = out;
  p.out_f32 = out_dtype == DA_F32;
  p.lse = lse;
  p.ws_o = ws_o;
  p.ws_lse = ws_lse;
  p.block_table = pg.block_table;
  p.bt_stride = pg.bt_stride;
  p.page_size = pg.page_size;
  p.page_magic = pg.page_size > 0 ? div_magic(static_cast<uint32_t>(pg.page_size / kTileN)) : 0;
  p.dyn_tiles = plan->h_kv * plan->num_m_blocks;
  p.dyn_u = plan->usable_sms;
  p.ws_meta = ws_meta;
  // LL exchange of a dynamic plan: every row, s_b = 1 included, is finished by the combine kernel
  p.dyn_via_combine = (pub != nullptr && pub->out != nullptr && dyn) ? 1 : 0;
  if (pub != nullptr && !(pub->out != nullptr && plan->combine_mode == DA_COMBINE_KERNEL)) {
    p.pub = *pub;     // NONE / CLUSTER: every CTA of the forward writes final rows and counts
    p.pub.writers = plan->grid_x * plan->grid_y * plan->grid_z;
  }

  cudaStream_t stream = static_cast<cudaStream_t>(cuda_stream);
  da_plan lp = *plan;
  lp.grid_z *= emul;                            // every emulated rank's grid in one launch
  if (lp.grid_z > 65535) return DA_ERR_UNSUPPORTED;
  if (launch_split_kv_fwd(lp, tk, tv, p, stream) != cudaSuccess) return DA_ERR_CUDA;
  if (plan->combine_mode == DA_COMBINE_KERNEL) {
    CombineParams c{};
    c.o = ws_o;
    c.o_stride = dyn ? HQ * D : B * HQ * D;   // dynamic: consecutive slots of one sequence
    c.lse_in = ws_lse;
    c.lse_stride = dyn ? HQ : B * HQ;
    c.meta = ws_meta;
    c.h_q = static_cast<int32_t>(HQ);
    c.batch = static_cast<int32_t>(B);
    c.num_splits = plan->num_splits;
    c.rows = static_cast<int32_t>(B * HQ);
    c.out = out;
    c.out_f32 = p.out_f32;
    c.lse = lse;
    if (pub != nullptr) {
      c.pub = *pub;   // KERNEL: one combine CTA per row writes it and counts
      c.pub.writers = c.rows;
    }
    if (launch_lse_combine(c, /*pdl=*/true, stream) != cudaSuccess) return DA_ERR_CUDA;
  }
  return DA_OK;
}

}  // namespace

extern "C" da_status da_forward(const da_plan* plan, const void* q, const void* k_cache,
                                const void* v_cache, int32_t l_cap, const int32_t* cache_seqlens,
                                const int64_t* strides, float softmax_scale, int32_t out_dtype,
                                void* out, float* lse, void* workspace, int64_t workspace_bytes,
                                void* cuda_stream) {
  return forward_impl(plan, q, k_cache, v_cache, l_cap, cache_seqlens, strides, softmax_scale,
                      out_dtype, out, lse, workspace, workspace_bytes, cuda_stream, PagedArgs{});
}

extern "C" da_status da_forward_paged(const da_plan* plan, const void* q, const void* k_pages,
                                      const void* v_pages, int32_t num_pages, int32_t page_size,
                                      const int32_t* block_table, int64_t block_table_stride,
                                      int32_t max_pages_per_seq, const int32_t* cache_seqlens,
                                      const int64_t* strides, float softmax_scale, int32_t out_dtype,
                                      void* out, float* lse, void* workspace, int64_t workspace_bytes,
                                      void* cuda_stream) {
  if (block_table == nullptr || num_pages < 1 || max_pages_per_seq < 1) return DA_ERR_INVALID_ARG;
  if (page_size < kTileN || page_size % kTileN != 0 || page_size > kMaxPageSize) return DA_ERR_UNSUPPORTED;
  if (block_table_stride < max_pages_per_seq) return DA_ERR_INVALID_ARG;
  const int64_t cap = int64_t(max_pages_per_seq) * page_size;
  if (cap > INT32_MAX) return DA_ERR_INVALID_ARG;
  PagedArgs pg;
  pg.block_table = block_table;
  pg.bt_stride = block_table_stride;
  pg.page_size = page_size;
  pg.num_pages = num_pages;
  return forward_impl(plan, q, k_pages, v_pages, static_cast<int32_t>(cap), cache_seqlens, strides,
                      softmax_scale, out_dtype, out, lse, workspace, workspace_bytes, cuda_stream, pg);
}

namespace {

// da_forward_host's staging layout in the device buffer (256-byte aligned regions).
struct HostStaging {
  int64_t q, k, v, seq, out, lse, ws, total;
};

inline int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

bool host_staging(const da_plan* plan, int32_t l_cap, bool with_seqlens, int32_t out_dtype,
                  HostStaging* h) {
  if (plan == nullptr || check_plan(plan) != DA_OK || l_cap < plan->l_k) return false;
  if (out_dtype != DA_BF16 && out_dtype != DA_F32) return false;
  const int64_t B = plan->batch, HQ = plan->h_q, HKV = plan->h_kv, D = kHeadDim;
  int64_t off = 0;
  h->q = off;   off = align256(off + B * HQ * D * 2);
  h->k = off;   off = align256(off + B * int64_t(l_cap) * HKV * D * 2);
  h->v = off;   off = align256(off + B * int64_t(l_cap) * HKV * D * 2);
  h->seq = off; off = align256(off + (with_seqlens ? B * 4 : 0));
  h->out = off; off = align256(off + B * HQ * D * (out_dtype == DA_F32 ? 4 : 2));
  h->lse = off; off = align256(off + B * HQ * 4);
  h->ws = off;  off = align256(off + (plan->combine_mode == DA_COMBINE_KERNEL ? plan->workspace_bytes : 0));
  h->total = off;
  return true;
}

}  // namespace

extern "C" int64_t da_forward_host_bytes(const da_plan* plan, int32_t l_cap, int32_t with_seqlens,
                                         int32_t out_dtype) {
  HostStaging h;
  return host_staging(plan, l_cap, with_seqlens != 0, out_dtype, &h) ? h.total : -1;
}

extern "C" da_status da_forward_host(const da_plan* plan, const void* q, const void* k_cache,
                                     const void* v_cache, int32_t l_cap, const int32_t* cache_seqlens,
                                     float softmax_scale, int32_t out_dtype, void* out, float* lse,
                                     void* device_buffer, int64_t device_buffer_bytes, void* cuda_stream) {
  if (plan == nullptr || q == nullptr || k_cache == nullptr || v_cache == nullptr || out == nullptr)
    return DA_ERR_INVALID_ARG;
  da_status st = check_plan(plan);
  if (st != DA_OK) return st;
  HostStaging h;
  if (!host_staging(plan, l_cap, cache_seqlens != nullptr, out_dtype, &h)) return DA_ERR_INVALID_ARG;
  if (device_buffer == nullptr || device_buffer_bytes < h.total) return DA_ERR_WORKSPACE;
  if ((reinterpret_cast<uintptr_t>(device_buffer) & 255u) != 0) return DA_ERR_ALIGNMENT;
  char* base = static_cast<char*>(device_buffer);
  cudaStream_t stream = static_cast<cudaStream_t>(cuda_stream);
  const int64_t B = plan->batch, HQ = plan->h_q, HKV = plan->h_kv, D = kHeadDim;
  const size_t kv_bytes = size_t(B) * size_t(l_cap) * size_t(HKV * D * 2);
  // K and V of one [2, B, l_cap, H_KV, d] host allocation land adjacent in the staging buffer too:
  // one DMA instead of two (at 1-2 MB the per-copy cost dominates the PCIe time)
  const bool kv_joint = static_cast<const char*>(v_cache) == static_cast<const char*>(k_cache) + kv_bytes &&
                        h.v == h.k + static_cast<int64_t>(kv_bytes) && one_allocation(k_cache, 2 * kv_bytes);
  if (cudaMemcpyAsync(base + h.q, q, size_t(B * HQ * D * 2), cudaMemcpyHostToDevice, stream) != cudaSuccess)
    return DA_ERR_CUDA;
  if (kv_joint) {
    if (cudaMemcpyAsync(base + h.k, k_cache, 2 * kv_bytes, cudaMemcpyHostToDevice, stream) != cudaSuccess)
      return DA_ERR_CUDA;
  } else if (cudaMemcpyAsync(base + h.k, k_cache, kv_bytes, cudaMemcpyHostToDevice, stream) != cudaSuccess ||
             cudaMemcpyAsync(base + h.v, v_cache, kv_bytes, cudaMemcpyHostToDevice, stream) != cudaSuccess) {
    return DA_ERR_CUDA;
  }
  const int32_t* dseq = nullptr;
  if (cache_seqlens != nullptr) {
    if (cudaMemcpyAsync(base + h.seq, cache_seqlens, size_t(B * 4), cudaMemcpyHostToDevice, stream) != cudaSuccess)
      return DA_ERR_CUDA;
    dseq = reinterpret_cast<const int32_t*>(base + h.seq);
  }
  float* dlse = reinterpret_cast<float*>(base + h.lse);
  const bool kernel_ws = plan->combine_mode == DA_COMBINE_KERNEL;
  st = forward_impl(plan, base + h.q, base + h.k, base + h.v, l_cap, dseq, nullptr, softmax_scale,
                    out_dtype, base + h.out, dlse, kernel_ws ? base + h.ws : nullptr,
                    kernel_ws ? plan->workspace_bytes : 0, cuda_stream, PagedArgs{});
  if (st != DA_OK) return st;
  const size_t out_bytes = size_t(B * HQ * D) * (out_dtype == DA_F32 ? 4 : 2);
  const size_t lse_bytes = size_t(B * HQ * 4);
  const bool ol_joint = lse != nullptr && reinterpret_cast<char*>(lse) == static_cast<char*>(out) + out_bytes &&
                        h.lse == h.out + static_cast<int64_t>(out_bytes) && one_allocation(out, out_bytes + lse_bytes);
  if (ol_joint) {
    if (cudaMemcpyAsync(out, base + h.out, out_bytes + lse_bytes, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
      return DA_ERR_CUDA;
  } else {
    if (cudaMemcpyAsync(out, base + h.out, out_bytes, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
      return DA_ERR_CUDA;
    if (lse != nullptr && cudaMemcpyAsync(lse, dlse, lse_bytes, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
      return DA_ERR_CUDA;
  }
  return DA_OK;
}

namespace {
// da_peer_signal / da_combine_peers: the exchange-buffer layout of include/decattn.h.
da_status check_peer_layout(int32_t world, int32_t rank, const uint64_t* peer_bases, const void* epoch,
                            int32_t batch, int32_t h_q, int32_t head_dim, int64_t slot_bytes, int64_t lse_offset,
                            int64_t flag_offset, int64_t* rows_out) {
  if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world || peer_bases == nullptr || epoch == nullptr ||
      batch < 1 || h_q < 1)
    return DA_ERR_INVALID_ARG;
  if (head_dim != kHeadDim) return DA_ERR_UNSUPPORTED;
  const int64_t rows = int64_t(batch) * h_q;
  if (rows > INT32_MAX) return DA_ERR_INVALID_ARG;
  if (lse_offset < rows * kHeadDim * 4 || slot_bytes < lse_offset + rows * 4 || flag_offset < 2 * slot_bytes)
    return DA_ERR_INVALID_ARG;
  if ((slot_bytes & 15) != 0 || (lse_offset & 15) != 0 || (flag_offset & 3) != 0 ||
      (reinterpret_cast<uintptr_t>(epoch) & 3u) != 0)
    return DA_ERR_ALIGNMENT;
  *rows_out = rows;
  return DA_OK;
}
}  // namespace

extern "C" da_status da_peer_signal(int32_t world, int32_t rank, const uint64_t* peer_bases, const float* o_local,
                                    const float* lse_local, int32_t batch, int32_t h_q, int32_t head_dim,
                                    int64_t slot_bytes, int64_t lse_offset, int64_t flag_offset, int32_t* epoch,
                                    void* cuda_stream) {
  int64_t rows = 0;
  da_status st = check_peer_layout(world, rank, peer_bases, epoch, batch, h_q, head_dim, slot_bytes, lse_offset,
                                   flag_offset, &rows);
  if (st != DA_OK) return st;
  if (o_local == nullptr) return DA_ERR_INVALID_ARG;
  if (!aligned16(o_local) || (lse_local != nullptr && (reinterpret_cast<uintptr_t>(lse_local) & 3u) != 0))
    return DA_ERR_ALIGNMENT;
  return launch_peer_signal(peer_bases, world, rank, o_local, lse_local, static_cast<int32_t>(rows), slot_bytes,
                            lse_offset, flag_offset, epoch, static_cast<cudaStream_t>(cuda_stream)) == cudaSuccess
             ? DA_OK
             : DA_ERR_CUDA;
}

extern "C" da_status da_forward_peer(const da_plan* plan, const void* q, const void* k_cache,
                                     const void* v_cache, int32_t l_cap, const int32_t* cache_seqlens,
                                     const int64_t* strides, float softmax_scale, int32_t world, int32_t rank,
                                     const uint64_t* peer_bases, int64_t slot_bytes, int64_t lse_offset,
                                     int64_t flag_offset, int32_t* epoch, uint32_t* counter, void* workspace,
                                     int64_t workspace_bytes, void* cuda_stream) {
  if (plan == nullptr) return DA_ERR_INVALID_ARG;
  int64_t rows = 0;
  da_status st = check_peer_layout(world, rank, peer_bases, epoch, plan->batch, plan->h_q, plan->head_dim,
                                   slot_bytes, lse_offset, flag_offset, &rows);
  if (st != DA_OK) return st;
  if (counter == nullptr) return DA_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(counter) & 3u) != 0) return DA_ERR_ALIGNMENT;
  PubParams pub{};
  pub.bases = peer_bases;
  pub.epoch = epoch;
  pub.count = counter;
  pub.slot_bytes = slot_bytes;
  pub.lse_offset = lse_offset;
  pub.flag_offset = flag_offset;
  pub.world = world;
  pub.rank = rank;
  return forward_impl(plan, q, k_cache, v_cache, l_cap, cache_seqlens, strides, softmax_scale, DA_F32, nullptr,
                      nullptr, workspace, workspace_bytes, cuda_stream, PagedArgs{}, &pub);
}

extern "C" da_status da_forward_peer_combine(const da_plan* plan, const void* q, const void* k_cache,
                                             const void* v_cache, int32_t l_cap, const int32_t* cache_seqlens,
                                             const int64_t* strides, float softmax_scale, int32_t world,
                                             int32_t rank, const uint64_t* peer_bases, int64_t ll_offset,
                                             int64_t ll_slot_bytes, int32_t* epoch, uint32_t* counter,
                                             int32_t out_dtype, void* out, float* lse, int32_t* status,
                                             int64_t timeout_ns, void* workspace, int64_t workspace_bytes,
                                             void* cuda_stream) {
  // rank = -1: emulate all `world` ranks in this one launch (tests on one GPU; include/decattn.h)
  if (plan == nullptr || world < 1 || world > kMaxPeers || rank < -1 || rank >= world || peer_bases == nullptr ||
      epoch == nullptr || counter == nullptr || out == nullptr || status == nullptr ||
      (out_dtype != DA_BF16 && out_dtype != DA_F32))
    return DA_ERR_INVALID_ARG;
  const bool emulate = rank < 0;
  if ((reinterpret_cast<uintptr_t>(status) & 3u) != 0) return DA_ERR_ALIGNMENT;
  if (plan->head_dim != kHeadDim) return DA_ERR_UNSUPPORTED;
  const int64_t rows = int64_t(plan->batch) * plan->h_q;
  if (ll_offset < 0 || ll_slot_bytes < rows * 129 * 8) return DA_ERR_INVALID_ARG;
  if ((ll_offset & 15) != 0 || (ll_slot_bytes & 15) != 0 || (reinterpret_cast<uintptr_t>(epoch) & 3u) != 0 ||
      (reinterpret_cast<uintptr_t>(counter) & 3u) != 0 || !aligned16(out) ||
      (lse != nullptr && (reinterpret_cast<uintptr_t>(lse) & 3u) != 0))
    return DA_ERR_ALIGNMENT;
  {
    da_status cs = check_plan(plan);
    if (cs != DA_OK) return cs;
  }
  // the CTAs that write the final rows spin on the ranks' words: their whole grid must be
  // resident at once - the forward for NONE plans (CTAs) and CLUSTER plans (clusters of s CTAs,
  // GPC-bound placement), the combine kernel (one CTA per row) for workspace plans - as the
  // occupancy API answers for the exact kernel, scaled to the usable SMs.  Host-only checks first:
  // a bound no device can beat (one forward CTA per SM: its shared memory; 32 CTAs per SM) and the
  // workspace, then the query.
  const bool kernel_ws = plan->combine_mode == DA_COMBINE_KERNEL;
  if (emulate && kernel_ws) return DA_ERR_UNSUPPORTED;   // emulation: one-kernel (NONE / CLUSTER) plans only
  const int64_t ranks_here = emulate ? world : 1;
  const int64_t need = ranks_here * (kernel_ws ? rows
                       : plan->combine_mode == DA_COMBINE_CLUSTER ? int64_t(plan->grid_y) * plan->grid_z
                                                                  : int64_t(plan->grid_x) * plan->grid_y * plan->grid_z);
  const int64_t ctas = ranks_here * (kernel_ws ? rows : int64_t(plan->grid_x) * plan->grid_y * plan->grid_z);
  if (ctas > int64_t(plan->usable_sms) * (kernel_ws ? 32 : 1)) return DA_ERR_UNSUPPORTED;
  if (kernel_ws && (workspace == nullptr || workspace_bytes < plan->workspace_bytes)) return DA_ERR_WORKSPACE;
  int units = 0;
  if (residency(*plan, kernel_ws ? 1 : 0, 2, &units) != cudaSuccess) return DA_ERR_CUDA;
  if (need > int64_t(units) * plan->usable_sms / (plan->num_sms > 0 ? plan->num_sms : 1)) return DA_ERR_UNSUPPORTED;
  PubParams pub{};
  pub.bases = peer_bases;
  pub.epoch = epoch;
  pub.count = counter;
  pub.ll_offset = ll_offset;
  pub.ll_slot_bytes = ll_slot_bytes;
  pub.world = world;
  pub.rank = emulate ? 0 : rank;
  pub.emulate = emulate ? 1 : 0;
  pub.out = out;
  pub.lse = lse;
  pub.out_f32 = out_dtype == DA_F32;
  pub.status = status;
  pub.timeout_ns = timeout_ns > 0 ? static_cast<uint64_t>(timeout_ns) : kDefaultTimeoutNs;
  return forward_impl(plan, q, k_cache, v_cache, l_cap, cache_seqlens, strides, softmax_scale, DA_F32, nullptr,
                      nullptr, workspace, workspace_bytes, cuda_stream, PagedArgs{}, &pub);
}

extern "C" da_status da_combine_peers(int32_t world, int32_t rank, const uint64_t* peer_bases, int64_t slot_bytes,
                                      int64_t lse_offset, int64_t flag_offset, const int32_t* epoch, int32_t batch,
                                      int32_t h_q, int32_t head_dim, int32_t out_dtype, void* out, float* lse,
                                      int32_t* status, int64_t timeout_ns, void* cuda_stream) {
  int64_t rows = 0;
  da_status st = check_peer_layout(world, rank, peer_bases, epoch, batch, h_q, head_dim, slot_bytes, lse_offset,
                                   flag_offset, &rows);
  if (st != DA_OK) return st;
  if (out == nullptr || status == nullptr || (out_dtype != DA_BF16 && out_dtype != DA_F32)) return DA_ERR_INVALID_ARG;
  if (!aligned16(out) || (lse != nullptr && (reinterpret_cast<uintptr_t>(lse) & 3u) != 0) ||
      (reinterpret_cast<uintptr_t>(status) & 3u) != 0)
    return DA_ERR_ALIGNMENT;
  return launch_peer_combine(peer_bases, slot_bytes, lse_offset, flag_offset, epoch, world, rank,
                             static_cast<int32_t>(rows), out_dtype == DA_F32, out, lse, status,
                             timeout_ns > 0 ? static_cast<uint64_t>(timeout_ns) : kDefaultTimeoutNs,
                             static_cast<cudaStream_t>(cuda_stream)) == cudaSuccess
             ? DA_OK
             : DA_ERR_CUDA;
}

extern "C" da_status da_combine(int32_t num_splits, int32_t batch, int32_t h_q, int32_t head_dim,
                                const float* o_partial, int64_t o_split_stride,
                                const float* lse_partial, int64_t lse_split_stride,
                                int32_t out_dtype, void* out, float* lse, void* cuda_stream) {
  if (o_partial == nullptr || lse_partial == nullptr || out == nullptr) return DA_ERR_INVALID_ARG;
  if (num_splits < 1 || num_splits > 4096 || batch < 1 || h_q < 1 || head_dim < 1)
    return DA_ERR_INVALID_ARG;
  if (head_dim != kHeadDim) return DA_ERR_UNSUPPORTED;
  if (out_dtype != DA_BF16 && out_dtype != DA_F32) return DA_ERR_INVALID_ARG;
  const int64_t rows = int64_t(batch) * h_q;
  if (rows > INT32_MAX / 2) return DA_ERR_UNSUPPORTED;   // one CTA per row (grid.x)
  if (num_splits > 1 && (o_split_stride < rows * kHeadDim || lse_split_stride < rows))
    return DA_ERR_INVALID_ARG;
  if (o_split_stride % 4 != 0 || !aligned16(o_partial) || !aligned16(out) ||
      (reinterpret_cast<uintptr_t>(lse_partial) & 3u) != 0 ||
      (lse != nullptr && (reinterpret_cast<uintptr_t>(lse) & 3u) != 0))
    return DA_ERR_ALIGNMENT;
  CombineParams c{};
  c.o = o_partial;
  c.o_stride = o_split_stride;
  c.lse_in = lse_partial;
  c.lse_stride = lse_split_stride;
  c.num_splits = num_splits;
  c.rows = static_cast<int32_t>(rows);
  c.out = out;
  c.out_f32 = out_dtype == DA_F32;
  c.lse = lse;
  if (launch_lse_combine(c, /*pdl=*/true, static_cast<cudaStream_t>(cuda_stream)) != cudaSuccess)
    return DA_ERR_CUDA;
  return DA_OK;
}

extern "C" const char* da_status_string(int32_t status) {
  switch (status) {
    case DA_OK: return "DA_OK";
    case DA_ERR_INVALID_ARG: return "DA_ERR_INVALID_ARG: invalid argument or inconsistent plan";
    case DA_ERR_UNSUPPORTED: return "DA_ERR_UNSUPPORTED: configuration not supported (head_dim must be 128)";
    case DA_ERR_ALIGNMENT: return "DA_ERR_ALIGNMENT: pointer not 16-byte aligned or stride not a multiple of 8 elements";
    case DA_ERR_WORKSPACE: return "DA_ERR_WORKSPACE: workspace missing or smaller than plan->workspace_bytes";
    case DA_ERR_CUDA: return "DA_ERR_CUDA: a CUDA runtime/driver call failed";
    case DA_ERR_TIMEOUT: return "DA_ERR_TIMEOUT: a cross-GPU exchange wait ran past its bound (a peer is late, crashed or out of step)";
    default: return "unknown da_status";
  }
}

extern "C" da_status da_query_residency(const da_plan* plan, int32_t kernel, int32_t exchange, int32_t* out) {
  if (plan == nullptr || out == nullptr || kernel < 0 || kernel > 1 || exchange < 0 || exchange > 2)
    return DA_ERR_INVALID_ARG;
  da_status st = check_plan(plan);
  if (st != DA_OK) return st;
  int n = 0;
  if (residency(*plan, kernel, exchange, &n) != cudaSuccess) return DA_ERR_CUDA;
  *out = n;
  return DA_OK;
}

extern "C" int32_t da_abi_version(void) { return DA_ABI_VERSION; }
