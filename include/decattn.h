/*
 * decattn.h - C ABI of the B200 (sm_100a) split-KV decode-attention library
 * (libdecattn.so) built for arxiv/paper_2604_00028, "sequence-aware split
 * policy for low-head-count decode attention".
 *
 * Citations: P:Lnn = PAPER.md line nn (section / figure / table beside it),
 * S:Lnn = SPEC.md line nn.  DESIGN.md §2 restates every entry point.
 *
 * The three calls follow the paper's statement of the problem:
 *   - da_plan_make: the split decision.  Inputs are the shape tuple
 *     (Batch, L_Q=1, L_K, H_Q, H_KV, D) (§5.1) and the three knobs the
 *     paper exposes - num_splits, pack_gqa, sm_margin (§3.1) - plus
 *     the SM count (132 on H100 P:L12; 148 on B200).  The policy is the FA3
 *     guarded default (§2.2, §4.2), the paper's sequence-aware
 *     cascade (Fig. 3) or a forced split.  Host-only integer code,
 *     computed once per shape like the precomputed scheduler metadata the
 *     paper's measurements use (§5.1).
 *   - da_forward: split-KV decode attention (L_Q = 1) over a bf16 KV cache:
 *     each of num_splits sequence chunks ("sequence-level parallelization
 *     across SMs") is reduced by its own CTA(s), then the partials are
 *     merged by the log-sum-exp combine (the "final reductions").
 *   - da_combine: the log-sum-exp combine of s (out, lse) partials on its
 *     own; also used to merge per-GPU partials of a sequence-sharded cache.
 *
 * Conventions for every call:
 *   - All device buffers are caller-owned (PyTorch allocates them); the
 *     library never allocates or frees device memory, never synchronises,
 *     never prints and never throws across the ABI.  It keeps no mutable
 *     global state except one-time kernel-attribute / driver-entry-point
 *     setup (thread-safe), so all calls are reentrant.
 *   - Every host-checkable error is returned BEFORE any launch, with no side
 *     effects.  Device-side values (cache_seqlens) cannot be checked without
 *     a sync: the kernels clamp them to [0, l_cap].  Asynchronous faults
 *     surface at the caller's next synchronisation of cuda_stream.
 *   - Layouts are row-major with the innermost dimension contiguous.  bf16 is
 *     IEEE bfloat16 (2 bytes); "lse" is the natural-log log-sum-exp in fp32
 *     (the FA softmax_lse convention; reading C-amb-10).
 */
#ifndef DECATTN_H
#define DECATTN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DA_ABI_VERSION 7

#if defined(__GNUC__)
#define DA_API __attribute__((visibility("default")))
#else
#define DA_API
#endif

/* Return codes. */
typedef enum da_status {
  DA_OK = 0,
  DA_ERR_INVALID_ARG = 1,  /* a dim < 1, h_q % h_kv != 0, sm_margin
                              outside [0, num_sms), forced split outside
                              [1, 256], a null pointer, l_cap < l_k,
                              an inconsistent plan */
  DA_ERR_UNSUPPORTED = 2,  /* head_dim != 128, or a configuration this build
                              has no kernel for */
  DA_ERR_ALIGNMENT = 3,    /* a base pointer not 16-byte aligned, or a stride
                              that is not a multiple of 8 elements */
  DA_ERR_WORKSPACE = 4,    /* combine_mode == DA_COMBINE_KERNEL and the
                              workspace is missing or too small */
  DA_ERR_CUDA = 5,         /* a CUDA runtime / driver call failed */
  DA_ERR_TIMEOUT = 6       /* a cross-GPU exchange wait ran past its bound (the device status
                              word of da_combine_peers / da_forward_peer_combine; never returned
                              by a call itself) */
} da_status;

/* Split policies (P:L34-39 knobs; decision functions SURVEY §8(c) C-pol). */
typedef enum da_policy {
  DA_POLICY_GUARDED = 0,    /* FA3 default: saturation guard, then s = 1 when
                               L_K <= 512, else efficiency loop */
  DA_POLICY_SEQ_AWARE = 1,  /* Fig. 3: Guard 1, Guard 2, low-tile
                               override s = 3, else efficiency loop */
  DA_POLICY_FIXED = 2,      /* s = forced_splits (the U-curve sweep) */
  DA_POLICY_EVOLVED = 3,    /* Fig. 1: batch == 1 -> 12 (16 when
                               L_K < 256); batch != 1 -> guarded            */
  DA_POLICY_SEQ_AWARE_SM = 4, /* SM-count-aware generalisation (DESIGN.md
                               C-ext-1), n_u = ceil(L_K/64),
                               T_k = B H_KV ceil(G / r) the CTA groups (r = 8
                               when G <= 8 or n_u <= 64, else 16),
                               f = largest s <= 16 whose T_k clusters fit
                               one wave, c = T_k <= 4 ? 8 : 4: nblk <= 4 ->
                               min(n_u, c, f) (1 when below 3, n_u < 5, or
                               n_u < 8 and T_k > 16);
                               else the efficiency loop's e, raised to
                               min(c, n_u, f) when e <= f, or moved to f when
                               e > f >= 2, r = 8 and (n_u <= 16 f or
                               2 T_k f >= U), then for n_u <= 64 at most 4
                               (T_k > 8) or 12; B200-calibrated             */
  DA_POLICY_DYNAMIC = 5     /* per-batch split counts from cache_seqlens on the
                               device (DESIGN.md C-ext-2):
                               W = max(1, ceil(sum_b ceil(n_b/64) * T_b / U)),
                               s_b = min(cap, max(1, floor(ceil(n_b/64) / W)))
                               with T_b = H_KV * num_m_blocks and cap =
                               min(128, ceil(L_K/64)) (= plan->num_splits);
                               always the workspace combine              */
} da_policy;

/* Which step of the cascade decided num_splits (SPEC's "source"). */
typedef enum da_rule {
  DA_RULE_SATURATED = 0,    /* 5 T >= 4 U (T >= 0.8 usable SMs)             */
  DA_RULE_GUARD_NBLK4 = 1,  /* guarded: num_n_blocks <= 4           */
  DA_RULE_GUARD1 = 2,       /* seq-aware: nblk <= 3           */
  DA_RULE_GUARD2 = 3,       /* seq-aware: nblk <= 4, T >= 4         */
  DA_RULE_LOW_TILE = 4,     /* seq-aware: nblk == 4, T < 4 -> 3     */
  DA_RULE_EFF_LOOP = 5,     /* efficiency loop (DESIGN.md C-amb-2)   */
  DA_RULE_FORCED = 6,       /* DA_POLICY_FIXED                               */
  DA_RULE_EVOLVED = 7,      /* DA_POLICY_EVOLVED, batch == 1      */
  DA_RULE_SM_SHORT = 8,     /* DA_POLICY_SEQ_AWARE_SM: too few units or splits */
  DA_RULE_SM_SPLIT = 9,     /* DA_POLICY_SEQ_AWARE_SM: nblk <= 4 split        */
  DA_RULE_SM_FIT = 10,      /* DA_POLICY_SEQ_AWARE_SM: nblk >= 5, the loop's
                               split moved to a one-wave cluster split      */
  DA_RULE_DYNAMIC = 11      /* DA_POLICY_DYNAMIC: num_splits is the cap, the
                               counts are decided per batch on the device   */
} da_rule;

/* Element types of outputs. */
typedef enum da_dtype { DA_BF16 = 0, DA_F32 = 1 } da_dtype;

/* How the s > 1 split partials are merged. */
typedef enum da_combine_mode {
  DA_COMBINE_NONE = 0,     /* s == 1: the split CTA writes out/lse directly   */
  DA_COMBINE_CLUSTER = 1,  /* 2 <= s <= 16: the s split CTAs of one tile form a
                              thread-block cluster and merge through
                              distributed shared memory inside the forward
                              kernel (no workspace, no second launch)          */
  DA_COMBINE_KERNEL = 2    /* s >= 2: fp32 partials go to the workspace and the
                              LSE-combine kernel (da_combine's kernel) merges
                              them, launched with programmatic dependent launch */
} da_combine_mode;

/* Kernel family selected by the plan. */
typedef enum da_path {
  DA_PATH_SCALAR = 0,  /* one query row per CTA (pack_gqa = 0, or G = 1):
                          fp32 FMA dot products + warp-shuffle softmax          */
  DA_PATH_MMA = 1,     /* pack_gqa with G >= 2: the G query rows of a KV head
                          share each K/V tile; QK^T and PV on tensor cores
                          (mma.sync, 8 or 16 rows per CTA)                     */
  DA_PATH_TC = 2       /* pack_gqa with G > 16 (MQA / wide GQA) and a static
                          split count: 64 query rows per CTA on tcgen05 (TMEM
                          accumulators); combine NONE (s == 1) or KERNEL     */
} da_path;

/*
 * da_plan - a plain value (copyable, no handles).  Fields marked (in) echo
 * the da_plan_make arguments; the rest are derived.
 */
typedef struct da_plan {
  int32_t batch, h_q, h_kv, l_k, head_dim, pack_gqa, sm_margin, num_sms; /* (in) */
  int32_t policy, forced_splits;                                          /* (in) */
  int32_t usable_sms;      /* U = num_sms - sm_margin (DESIGN.md C-amb-8)      */
  int32_t block_n;         /* 128: the policy's token accounting (C-amb-1)     */
  int32_t num_n_blocks;    /* nblk = ceil(l_k / 128)                           */
  int32_t num_m_blocks;    /* ceil(G / 64) (= 1 for G <= 64)                   */
  int32_t total_mblocks;   /* T = batch * h_kv * num_m_blocks      */
  int32_t num_splits;      /* s                                                */
  int32_t nonempty_splits; /* min(s, ceil(l_k / split_unit))                   */
  int32_t rule;            /* da_rule                                          */
  int32_t split_unit;      /* 64 tokens: the partition unit                    */
  int32_t path;            /* da_path                                          */
  int32_t rows_per_cta;    /* query rows one CTA computes: SCALAR 1; MMA 8,
                              or 16 when G > 8 and (n_u > 64 or the 8-row
                              grid B H_KV ceil(G/8) s exceeds U); TC 64   */
  int32_t combine_mode;    /* da_combine_mode                                  */
  int32_t grid_x;          /* = num_splits; DA_POLICY_DYNAMIC: the head groups
                              (grid_y's static value)                        */
  int32_t grid_y;          /* MMA / TC: h_kv * ceil(G / rows_per_cta); SCALAR: h_q;
                              DA_POLICY_DYNAMIC: split slots,
                              min(B * cap, ceil(U / T_b) + B)                */
  int32_t grid_z;          /* = batch; DA_POLICY_DYNAMIC: 1                    */
  int32_t block_threads;   /* threads per CTA                                  */
  int32_t cluster_x;       /* CTAs per cluster along x (s in CLUSTER mode)     */
  int32_t smem_bytes;      /* dynamic shared memory per CTA                    */
  int64_t workspace_bytes; /* s * batch * h_q * (head_dim + 1) * 4 when s > 1,
                              else 0.  Only DA_COMBINE_KERNEL reads/writes it.
                              DA_POLICY_DYNAMIC: grid_y * h_q * (head_dim + 1)
                              * 4 + 8 * batch (partials per slot, then the
                              schedule: first slot and split count per b)  */
  int32_t seq_offset;      /* (in, da_plan_set_seq_offset; 0 from da_plan_make)
                              tokens of every sequence that precede this cache:
                              cache_seqlens hold whole-sequence lengths and
                              batch b attends to tokens [0, seqlens[b] -
                              seq_offset) of this cache (clamped to
                              [0, l_cap]) - the shard of a sequence-sharded
                              KV cache that starts at token seq_offset
                              (DESIGN.md §6).  Not applied when cache_seqlens
                              is NULL (then every sequence has plan->l_k).  */
  int32_t path_override;   /* (in, da_plan_set_path; 0 from da_plan_make) 0 =
                              the planner's kernel choice, else the da_path
                              forced: DA_PATH_MMA or DA_PATH_TC (A/B, tests) */
} da_plan;

/*
 * da_plan_make - decide num_splits and the launch geometry for one shape.
 *   batch, h_q, h_kv, l_k, head_dim : the shape; all >= 1,
 *                                     h_q % h_kv == 0.
 *   pack_gqa   : 0/1.  Does not change the decision (C-amb-17), only
 *                the kernel path (MMA when pack_gqa && G >= 2).
 *   sm_margin  : SMs excluded from the policy's count, 0 <= sm_margin < num_sms
 *                (S:L37-41).
 *   num_sms    : SM count of the device (148 on B200).
 *   policy     : da_policy; forced_splits is read only for DA_POLICY_FIXED and
 *                must be in [1, 256] (forced_splits > nblk is allowed: empty
 *                splits produce o = 0, lse = -inf partials; C-amb-6).
 *   out        : written on DA_OK only.
 * Pure host code: no CUDA call, no allocation.  Errors: DA_ERR_INVALID_ARG,
 * DA_ERR_UNSUPPORTED (head_dim != 128).
 * Default combine mode: NONE for s == 1; CLUSTER for 2 <= s <= 16 when all
 * clusters of the launch fit one wave on the device (measured B200 co-residency
 * table, scaled by num_sms / 148); else KERNEL.
 */
DA_API da_status da_plan_make(int32_t batch, int32_t h_q, int32_t h_kv, int32_t l_k,
                       int32_t head_dim, int32_t pack_gqa, int32_t sm_margin,
                       int32_t num_sms, int32_t policy, int32_t forced_splits,
                       da_plan* out);

/*
 * da_plan_make_varlen - the plan for a ragged batch whose lengths are known on the host (the
 * metadata-then-launch path of P:L125; DESIGN.md C-ext-3).  Arguments as da_plan_make with
 * l_cap = the cache capacity, plus host_seqlens (host int32 [batch], clamped to [0, l_cap]).
 * Returns the DA_POLICY_SEQ_AWARE_SM plan for l_cap, unless its longest split would hold more
 * than twice the per-CTA work W of the dynamic schedule (and at least 32 units of 64 tokens);
 * then the DA_POLICY_DYNAMIC plan.  plan->policy tells which.  Pure host code.
 * Errors: as da_plan_make; DA_ERR_INVALID_ARG for a NULL host_seqlens.
 */
DA_API da_status da_plan_make_varlen(int32_t batch, int32_t h_q, int32_t h_kv, int32_t l_cap,
                                     int32_t head_dim, int32_t pack_gqa, int32_t sm_margin,
                                     int32_t num_sms, const int32_t* host_seqlens, da_plan* out);

/*
 * da_plan_set_combine - switch an existing plan to another combine mode and
 * re-derive its launch fields.  NONE requires s == 1, CLUSTER 2 <= s <= 16,
 * KERNEL s >= 2.  Errors: DA_ERR_INVALID_ARG.
 */
DA_API da_status da_plan_set_combine(da_plan* plan, int32_t combine_mode);

/*
 * da_plan_set_seq_offset - make the plan one sequence shard's: cache_seqlens passed to the
 * forwards are then whole-sequence lengths and the cache holds tokens [seq_offset, seq_offset +
 * l_cap) of each sequence (the kernel attends to min(max(seqlens[b] - seq_offset, 0), l_cap)
 * of them).  Sequence sharding across GPUs (north_star: "only long-context configs
 * shard the sequence") without a per-step length kernel.  seq_offset >= 0, else
 * DA_ERR_INVALID_ARG.  Pure host code.
 */
DA_API da_status da_plan_set_seq_offset(da_plan* plan, int32_t seq_offset);

/*
 * da_plan_set_path - force the kernel of a pack_gqa plan with G >= 2 and re-derive its launch
 * fields: DA_PATH_MMA (mma.sync, 8 / 16 rows per CTA) or DA_PATH_TC (tcgen05, 64 rows per CTA; static
 * split counts only, never a cluster combine: a CLUSTER plan becomes KERNEL); -1 restores the
 * planner's choice.  The planner's own rule: DA_PATH_TC when G > 16, every split
 * holds >= 4 tiles of 64 tokens and the tcgen05 grid has >= U / 2 CTAs.  Errors: DA_ERR_INVALID_ARG
 * (scalar plans, dynamic plans asked for DA_PATH_TC, unknown paths).  Pure host code.
 */
DA_API da_status da_plan_set_path(da_plan* plan, int32_t path);

/*
 * da_forward - decode attention for one step (L_Q = 1), asynchronously on
 * cuda_stream (a cudaStream_t; NULL = legacy default stream).
 *   q        bf16 [B, H_Q, d]             device; strides (q_b, q_h) elements
 *   k_cache  bf16 [B, l_cap, H_KV, d]     device; strides (k_b, k_t, k_h)
 *   v_cache  bf16 [B, l_cap, H_KV, d]     device; strides (v_b, v_t, v_h)
 *   l_cap    cache capacity in tokens, >= plan->l_k
 *   cache_seqlens  device int32 [B], tokens of batch b that attend (clamped
 *            to [0, l_cap] on the device); NULL means plan->l_k for every b.
 *   strides  host int64[8] = {q_b, q_h, k_b, k_t, k_h, v_b, v_t, v_h} in
 *            elements (innermost dim contiguous); NULL = contiguous.  Each must
 *            be a multiple of 8 elements (16 bytes, for TMA / 128-bit loads).
 *   softmax_scale  <= 0 selects 1/sqrt(d) (C-amb-9).
 *   out_dtype      DA_BF16 (round-to-nearest-even once at the end, C-amb-13)
 *            or DA_F32 (unrounded: the per-GPU partial of a sequence shard).
 *   out      [B, H_Q, d] contiguous, out_dtype.  Query head h uses KV head
 *            floor(h / G) (C-amb-11).  An empty sequence gives out = 0.
 *   lse      fp32 [B, H_Q] contiguous natural-log LSE, -inf for an empty
 *            sequence (C-amb-12); may be NULL (not written).
 *   workspace, workspace_bytes  fp32 partials [s, B, H_Q, d] followed by
 *            [s, B, H_Q]; required (>= plan->workspace_bytes, 16-byte
 *            aligned) only for DA_COMBINE_KERNEL, ignored otherwise.
 * The result equals exact softmax attention over tokens [0, n_b) for every
 * split count (SURVEY §8(c) C-att / C-comb).
 */
DA_API da_status da_forward(const da_plan* plan, const void* q, const void* k_cache,
                     const void* v_cache, int32_t l_cap,
                     const int32_t* cache_seqlens, const int64_t* strides,
                     float softmax_scale, int32_t out_dtype, void* out, float* lse,
                     void* workspace, int64_t workspace_bytes, void* cuda_stream);

/*
 * da_forward_paged - da_forward over a paged KV cache (vLLM-style block tables; SURVEY
 * §8(f4)).  Same plan, q, cache_seqlens, softmax_scale, out, lse, workspace and stream
 * semantics as da_forward, with the cache given as page pools:
 *   k_pages, v_pages  bf16 [num_pages, page_size, H_KV, d]; strides (as in da_forward)
 *                     are {q_b, q_h, k_page, k_t, k_h, v_page, v_t, v_h} in elements,
 *                     NULL = contiguous pools
 *   page_size         tokens per page: a multiple of 64 (one kernel tile never spans pages)
 *                     and at most 262144, else DA_ERR_UNSUPPORTED
 *   block_table       device int32 [B, block_table_stride]: entry j of row b is the page
 *                     holding tokens [j page_size, (j+1) page_size) of sequence b.  Entries
 *                     past a sequence's length are never read; an index outside
 *                     [0, num_pages) reads zeros (no out-of-bounds access)
 *   max_pages_per_seq pages per sequence: max_pages_per_seq * page_size >= plan->l_k and
 *                     bounds every cache_seqlens value (clamped on the device)
 * The result is decode attention over the gathered sequence (oracle.gather_pages).
 */
DA_API da_status da_forward_paged(const da_plan* plan, const void* q, const void* k_pages,
                                  const void* v_pages, int32_t num_pages, int32_t page_size,
                                  const int32_t* block_table, int64_t block_table_stride,
                                  int32_t max_pages_per_seq, const int32_t* cache_seqlens,
                                  const int64_t* strides, float softmax_scale, int32_t out_dtype,
                                  void* out, float* lse, void* workspace, int64_t workspace_bytes,
                                  void* cuda_stream);

/*
 * da_forward_host_bytes - device staging bytes da_forward_host needs for `plan` and a cache of
 * l_cap tokens: q, K, V, cache_seqlens (with_seqlens != 0), out (out_dtype), lse and the
 * workspace (DA_COMBINE_KERNEL), each 256-byte aligned, in that order.  Returns -1 when the plan
 * is invalid, l_cap < plan->l_k or out_dtype is not a da_dtype.  Pure host code.
 */
DA_API int64_t da_forward_host_bytes(const da_plan* plan, int32_t l_cap, int32_t with_seqlens,
                                     int32_t out_dtype);

/*
 * da_forward_host - da_forward with HOST inputs and outputs, for callers whose KV cache lives
 * in host memory (the end-to-end path the benchmark's e2e figure times).  All work is
 * enqueued on cuda_stream in this order: host->device copies of q [B, H_Q, d], k_cache and
 * v_cache [B, l_cap, H_KV, d] (bf16, contiguous host memory) and cache_seqlens int32 [B]
 * (NULL = plan->l_k for every b) into device_buffer; the forward (as da_forward with
 * contiguous strides); device->host copies of out [B, H_Q, d] (out_dtype) and lse fp32
 * [B, H_Q] (NULL = not copied).  The host outputs are valid once the stream has
 * synchronised.  Page-locked host memory makes every copy asynchronous; pageable memory
 * works but then copies synchronously.  When v_cache starts where k_cache ends inside one
 * CUDA-registered allocation (a [2, B, l_cap, H_KV, d] host cache), K and V travel in one DMA;
 * so do out and lse when lse starts where out ends inside one allocation.
 *   device_buffer, device_buffer_bytes: device scratch of at least
 *   da_forward_host_bytes(plan, l_cap, cache_seqlens != NULL, out_dtype) bytes, 256-byte
 *   aligned, owned by the caller and reusable once the stream has passed this call.
 * Errors: as da_forward; DA_ERR_WORKSPACE when device_buffer is NULL or too small,
 * DA_ERR_CUDA when a copy cannot be enqueued.
 */
DA_API da_status da_forward_host(const da_plan* plan, const void* q, const void* k_cache,
                                 const void* v_cache, int32_t l_cap, const int32_t* cache_seqlens,
                                 float softmax_scale, int32_t out_dtype, void* out, float* lse,
                                 void* device_buffer, int64_t device_buffer_bytes,
                                 void* cuda_stream);

/*
 * da_combine - LSE-combine of s partials (C-comb):
 *   M = max_i lse_i, lse = M + ln sum_i exp(lse_i - M),
 *   out = sum_i exp(lse_i - lse) o_i; all splits empty -> out = 0, lse = -inf.
 *   o_partial   fp32, split i at o_partial + i * o_split_stride, each
 *               [B, H_Q, d] contiguous (16-byte aligned; stride multiple of 4)
 *   lse_partial fp32, split i at lse_partial + i * lse_split_stride, [B, H_Q]
 *   (the strides let one NCCL all-gather buffer of [P][o | lse] be passed as is)
 *   out         [B, H_Q, d] out_dtype;  lse fp32 [B, H_Q] or NULL.
 * 1 <= num_splits <= 4096; head_dim must be 128.
 */
DA_API da_status da_combine(int32_t num_splits, int32_t batch, int32_t h_q, int32_t head_dim,
                     const float* o_partial, int64_t o_split_stride,
                     const float* lse_partial, int64_t lse_split_stride,
                     int32_t out_dtype, void* out, float* lse, void* cuda_stream);

/*
 * Cross-GPU exchange of sequence-shard partials over peer memory (the long-context
 * configs shard the sequence across GPUs and merge the per-GPU (out, lse) partials).
 * Every rank owns an exchange buffer mapped on all ranks (e.g. torch symmetric memory), all with
 * one layout: two partial slots of slot_bytes at 0 and slot_bytes, each
 *   [0, lse_offset)            o fp32 [batch, h_q, head_dim]
 *   [lse_offset, ...)          lse fp32 [batch, h_q]
 * then, at flag_offset >= 2 slot_bytes, one uint32 flag per source rank, zero before the first
 * step.  slot_bytes and lse_offset are multiples of 16.
 * peer_bases: DEVICE array of `world` base addresses (uint64), entry q = rank q's buffer as mapped
 * on this GPU.  epoch: device int32 owned by this rank, zero before the first step.
 *
 * da_peer_signal - e = *epoch + 1: copy this rank's partial (o_local fp32 [batch, h_q, head_dim],
 * lse_local fp32 [batch, h_q] - da_forward with out_dtype = DA_F32 writes them; lse_local NULL
 * means empty rows) into slot e & 1 of its own buffer, fence (system scope), release e into flag
 * slot `rank` of every rank's buffer, *epoch = e.  Enqueue after the forward.
 * da_combine_peers - every CTA waits (acquire, system scope) until all `world` flags of this
 * rank's buffer reach *epoch, then merges the world partials of slot *epoch & 1, read from the
 * peers' buffers, with the LSE identity of da_combine (C-comb) into out (out_dtype) and lse (fp32,
 * may be NULL).
 * A rank overwrites slot e & 1 again only at step e + 2, after every peer has signalled step e + 1,
 * i.e. finished combining step e.  The flags carry monotonic epochs, so both calls can be captured
 * in a CUDA graph and replayed.
 * Bounded wait: a flag still below *epoch timeout_ns after the first failed poll (<= 0: 10 s) ends
 * the wait; the CTA stores DA_ERR_TIMEOUT into *status (device int32 owned by the caller, zero
 * before the step; it is never cleared by the library) and merges what the slots hold, so the
 * kernel completes and the caller reads the failure from *status instead of hanging on a peer that
 * is late, crashed or out of step.
 * Errors: DA_ERR_INVALID_ARG (world not in [1, 64], rank, NULL pointers incl. status, overlapping
 * regions), DA_ERR_UNSUPPORTED (head_dim != 128), DA_ERR_ALIGNMENT, DA_ERR_CUDA.
 */
DA_API da_status da_peer_signal(int32_t world, int32_t rank, const uint64_t* peer_bases, const float* o_local,
                                const float* lse_local, int32_t batch, int32_t h_q, int32_t head_dim,
                                int64_t slot_bytes, int64_t lse_offset, int64_t flag_offset, int32_t* epoch,
                                void* cuda_stream);
DA_API da_status da_combine_peers(int32_t world, int32_t rank, const uint64_t* peer_bases, int64_t slot_bytes,
                                  int64_t lse_offset, int64_t flag_offset, const int32_t* epoch, int32_t batch,
                                  int32_t h_q, int32_t head_dim, int32_t out_dtype, void* out, float* lse,
                                  int32_t* status, int64_t timeout_ns, void* cuda_stream);

/*
 * da_forward_peer - da_forward (out_dtype = DA_F32) and da_peer_signal in one: the kernel that
 * produces this rank's final rows (the forward for DA_COMBINE_NONE / CLUSTER plans, the combine
 * kernel for DA_COMBINE_KERNEL) writes them straight into slot e & 1 (e = *epoch + 1) of this
 * rank's exchange buffer (layout above), and the last of its CTAs to finish (device counter)
 * fences at system scope, releases e into flag `rank` of every rank's buffer, resets *counter to
 * 0 and sets *epoch = e.  No copy and no signal launch between the forward and da_combine_peers
 * (DESIGN.md §6).  Dense caches only.
 *   plan, q, k_cache, v_cache, l_cap, cache_seqlens, strides, softmax_scale, workspace,
 *   workspace_bytes: as da_forward (plan->batch, h_q, head_dim define the slot rows);
 *   world, rank, peer_bases, slot_bytes, lse_offset, flag_offset, epoch: as da_peer_signal;
 *   counter: device uint32 owned by this rank, zero before the first step (left zero after each).
 * Errors: those of da_forward and da_peer_signal; DA_ERR_INVALID_ARG for a NULL counter,
 * DA_ERR_ALIGNMENT for a counter not 4-byte aligned.
 */
DA_API da_status da_forward_peer(const da_plan* plan, const void* q, const void* k_cache,
                                 const void* v_cache, int32_t l_cap, const int32_t* cache_seqlens,
                                 const int64_t* strides, float softmax_scale, int32_t world, int32_t rank,
                                 const uint64_t* peer_bases, int64_t slot_bytes, int64_t lse_offset,
                                 int64_t flag_offset, int32_t* epoch, uint32_t* counter, void* workspace,
                                 int64_t workspace_bytes, void* cuda_stream);

/*
 * da_forward_peer_combine - the whole sequence-sharded step with the exchange inside the kernel
 * that produces the final rows (the forward for NONE / CLUSTER plans: ONE kernel per step; the
 * combine kernel for workspace plans).  e = *epoch + 1.  Every CTA of that kernel writes its
 * final fp32 rows (o, then lse) into LL slot e & 1 of this rank's exchange buffer as
 * self-validating 8-byte words ((e << 32) | fp32 bits, one system-scope relaxed
 * store each: no fence, no flag), then polls the same words of every rank's slot (NVLink loads for
 * peers) until they carry e and LSE-merges (C-comb) the world partials of its rows into out
 * (out_dtype [B, H_Q, d]) and lse (fp32 [B, H_Q], or NULL); the last CTA to have read the epoch
 * (device counter) advances *epoch.  The exchange and the combine fused into the kernel that
 * finishes the rows.
 *   ll_offset, ll_slot_bytes: the two LL slots (uint64 [B * H_Q][129] each, ll_slot_bytes >=
 *     8 * 129 * B * H_Q, both multiples of 16) inside every rank's exchange buffer (same layout on
 *     every rank, zero before the first step); a rank reuses slot e & 1 at step e + 2 only (the
 *     stream order then guarantees every peer has read it).
 *   counter: device uint32 owned by this rank, zero before the first step (left zero after each).
 * The CTAs spin, so the writing grid must be resident at once on an otherwise idle GPU, which the
 * call checks against the device's own occupancy answer for the exact kernel (da_query_residency,
 * scaled by usable_sms / SM count): NONE plans with grid_x * grid_y * grid_z CTAs, CLUSTER plans
 * with grid_y * grid_z clusters of num_splits CTAs (cluster placement is GPC-bound: not SMs / s),
 * or DA_COMBINE_KERNEL plans (static or DA_POLICY_DYNAMIC, whose single-split rows then also pass
 * through the combine kernel) with B * H_Q combine CTAs (workspace, workspace_bytes as
 * da_forward); DA_ERR_UNSUPPORTED otherwise (use da_forward_peer + da_combine_peers).
 * status, timeout_ns: the bounded wait of da_combine_peers, for the LL words.
 * rank = -1 (testing the multi-rank protocol on ONE GPU, where separate launches cannot be made to
 *   wait on one another): one launch runs every rank's grid along z (NONE / CLUSTER plans only,
 *   DA_ERR_UNSUPPORTED otherwise; the residency check covers all world grids).  Then k_cache /
 *   v_cache hold the world shards stacked along the batch dimension ([world * B, l_cap, H_KV, d],
 *   rank r's sequence b at cache batch r * B + b), cache_seqlens is [world * B] (or NULL), epoch
 *   and counter are arrays [world], out is [world, B, H_Q, d] and lse [world, B, H_Q] (or NULL):
 *   emulated rank r publishes into peer_bases[r], polls every rank's words and writes out[r].
 * Errors: as da_forward; DA_ERR_INVALID_ARG for world / rank / NULL pointers / a short LL slot,
 * DA_ERR_ALIGNMENT for misaligned offsets, counter, epoch, status, out or lse; DA_ERR_CUDA when the
 * occupancy query fails.
 */
DA_API da_status da_forward_peer_combine(const da_plan* plan, const void* q, const void* k_cache,
                                         const void* v_cache, int32_t l_cap, const int32_t* cache_seqlens,
                                         const int64_t* strides, float softmax_scale, int32_t world,
                                         int32_t rank, const uint64_t* peer_bases, int64_t ll_offset,
                                         int64_t ll_slot_bytes, int32_t* epoch, uint32_t* counter,
                                         int32_t out_dtype, void* out, float* lse, int32_t* status,
                                         int64_t timeout_ns, void* workspace, int64_t workspace_bytes,
                                         void* cuda_stream);

/*
 * da_query_residency - how many launch units of the kernel a plan launches can be resident on the
 * CURRENT device at once, as the CUDA occupancy API answers for the exact instantiation (its
 * threads, registers and shared memory): the measurement behind the planner's cluster-fit table
 * (config.h kMaxActiveClustersB200) and the residency guard of
 * da_forward_peer_combine.
 *   kernel 0: the split-KV forward of the plan (exchange 0 = da_forward, 1 = da_forward_peer,
 *             2 = da_forward_peer_combine): clusters of num_splits CTAs for a DA_COMBINE_CLUSTER
 *             plan (cudaOccupancyMaxActiveClusters), CTAs otherwise;
 *   kernel 1: the LSE combine kernel: CTAs (the plan is only validated).
 * *out: the count for the whole device (all SMs, sm_margin not applied).
 * Errors: DA_ERR_INVALID_ARG (NULL, inconsistent plan, kernel / exchange out of range),
 * DA_ERR_CUDA (no device, or the query failed).
 */
DA_API da_status da_query_residency(const da_plan* plan, int32_t kernel, int32_t exchange, int32_t* out);

/* Static, NUL-terminated description of a status code (never NULL). */
DA_API const char* da_status_string(int32_t status);

/* DA_ABI_VERSION of the loaded library. */
DA_API int32_t da_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DECATTN_H */
