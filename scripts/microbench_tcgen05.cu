// tcgen05 feasibility microbenchmark for the decode tile (development tool, not part of the product).
//
// One CTA, 4 warps.  The smem operands use exactly the product's layouts (csrc/fwd.cu): a 64-token
// K tile and V tile as two 128B-swizzled boxes of 64 tokens x 64 dims each (what the TMA ring
// holds), the 8 query rows as K-major 128B-swizzled atoms, P as one K-major atom [8 rows][64 tokens].
//   S^T[tok, g] = sum_d K[tok, d] Q[g, d]   tcgen05.mma kind::f16 M=64  N=8 K=128 (8 x K16), A = K (K-major)
//   O^T[d, g]   = sum_t V[t, d] P[g, t]     tcgen05.mma kind::f16 M=128 N=8 K=64  (4 x K16), A = V^T (MN-major)
// Checks both against a host fp32 reference, reports where the M = 64 accumulator rows land in TMEM,
// and times (clock64) the MMA issue -> commit -> mbarrier round trips and the tcgen05.ld.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/mb_tc scripts/microbench_tcgen05.cu && /tmp/mb_tc
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// byte offset of element (row r, column c) in a 128B-swizzled box of 128-byte rows (64 bf16)
__host__ __device__ inline uint32_t sw128(int r, int c) { return r * 128 + ((((c >> 3) ^ (r & 7)) & 7) << 4) + (c & 7) * 2; }

// SM100 shared-memory matrix descriptor (cute::UMMA::SmemDescriptor): start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version 1 [46,48), base offset 0, lbo mode 0, layout type [61,64) (2 = SWIZZLE_128B)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor kind::f16: c_format F32 (bit 4), a/b BF16 (bits 7, 10), a/b major, N>>3 at 17, M>>4 at 24
__host__ __device__ constexpr uint32_t idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t id, int acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(bar), "r"(ph) : "memory");
}
__device__ __forceinline__ void ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// out_s: [128 lanes][8] (raw TMEM dump of the S accumulator), out_o: [128 d][8 g], cyc: timings
__global__ void __launch_bounds__(128) tile_kernel(const __nv_bfloat16* K, const __nv_bfloat16* V,
                                                    const __nv_bfloat16* Q, const __nv_bfloat16* P,
                                                    float* out_s, float* out_o, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sK = sm;             // 2 boxes x 8 KB
  uint8_t* sV = sm + 16384;     // 2 boxes x 8 KB
  uint8_t* sQ = sm + 32768;     // 2 atoms x 1 KB (dims 0-63, 64-127)
  uint8_t* sP = sm + 34816;     // 1 atom [8 g][64 tok]
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 64 * 128; i += 128) {
    const int t = i / 128, d = i % 128;
    *(__nv_bfloat16*)(sK + (d >> 6) * 8192 + sw128(t, d & 63)) = K[i];
    *(__nv_bfloat16*)(sV + (d >> 6) * 8192 + sw128(t, d & 63)) = V[i];
  }
  for (int i = tid; i < 8 * 128; i += 128) {
    const int g = i / 128, d = i % 128;
    *(__nv_bfloat16*)(sQ + (d >> 6) * 1024 + sw128(g, d & 63)) = Q[i];
  }
  for (int i = tid; i < 8 * 64; i += 128) {
    const int g = i / 64, t = i % 64;
    *(__nv_bfloat16*)(sP + sw128(g, t)) = P[i];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> tensor-core reads
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  const uint32_t b = smem_u32(&bar);
  long long t0 = 0, t1 = 0, t2 = 0, t3 = 0, t4 = 0;

  // ---- S^T = K Q^T: A = K tile (K-major, SBO = 1 KB between 8-token groups), B = Q (K-major)
  __syncwarp();
  if (tid == 0) {
    t0 = clock64();
    constexpr uint32_t id_s = idesc(64, 8, 0, 0);
    for (int kk = 0; kk < 8; ++kk) {   // K16 step kk: dims 16 kk .. 16 kk + 15 -> box kk / 4, +32 B per step
      const uint64_t a = sdesc(smem_u32(sK) + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
      const uint64_t bq = sdesc(smem_u32(sQ) + (kk >> 2) * 1024 + (kk & 3) * 32, 16, 1024);
      mma(tm, a, bq, id_s, kk > 0);
    }
    commit(b);
  }
  mbar_wait(b, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) t1 = clock64();
  {
    float v[8];
    ld8(tm + ((uint32_t)(warp * 32) << 16), v);    // lane quadrant of this warp, columns 0..7
    if (tid == 0) t2 = clock64();
    for (int c = 0; c < 8; ++c) out_s[(warp * 32 + lane) * 8 + c] = v[c];
  }
  // ---- O^T = V^T P^T: A = V tile read MN-major (64 dims per 128-byte row, LBO = 8 KB to the
  //      dims-64..127 box, SBO = 1 KB between 8-token groups), B = P (K-major atom)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    t3 = clock64();
    constexpr uint32_t id_o = idesc(128, 8, 1, 0);
    for (int kk = 0; kk < 4; ++kk) {   // K16 step: tokens 16 kk .. : 2 groups of 8 rows = +2 KB per step
      const uint64_t a = sdesc(smem_u32(sV) + kk * 2048, 8192, 1024);
      const uint64_t bp = sdesc(smem_u32(sP) + kk * 32, 16, 1024);
      mma(tm + 8, a, bp, id_o, kk > 0);
    }
    commit(b);
  }
  mbar_wait(b, 1);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) t4 = clock64();
  {
    float v[8];
    ld8(tm + 8 + ((uint32_t)(warp * 32) << 16), v);
    for (int c = 0; c < 8; ++c) out_o[(warp * 32 + lane) * 8 + c] = v[c];
  }
  // ---- warm repeats: S^T again (8 MMAs) and O^T with the P hi / lo pair (8 MMAs), each one round trip
  long long t5 = 0, t6 = 0, t7 = 0, t8 = 0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    t5 = clock64();
    constexpr uint32_t id_s = idesc(64, 8, 0, 0);
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t a = sdesc(smem_u32(sK) + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
      const uint64_t bq = sdesc(smem_u32(sQ) + (kk >> 2) * 1024 + (kk & 3) * 32, 16, 1024);
      mma(tm + 16, a, bq, id_s, kk > 0);
    }
    commit(b);
  }
  mbar_wait(b, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) t6 = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    t7 = clock64();
    constexpr uint32_t id_o = idesc(128, 8, 1, 0);
    for (int kk = 0; kk < 8; ++kk) {   // hi / lo: the same A, two B atoms (here both P)
      const uint64_t a = sdesc(smem_u32(sV) + (kk & 3) * 2048, 8192, 1024);
      const uint64_t bp = sdesc(smem_u32(sP) + (kk & 3) * 32, 16, 1024);
      mma(tm + 24, a, bp, id_o, kk > 0);
    }
    commit(b);
  }
  mbar_wait(b, 1);
  if (tid == 0) t8 = clock64();
  // ---- split chains: S^T as two independent 4-MMA chains (dims 0-63 / 64-127 into two
  //      accumulators), O^T hi and lo into two accumulators; one commit each
  long long t9 = 0, t10 = 0, t11 = 0, t12 = 0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    t9 = clock64();
    constexpr uint32_t id_s = idesc(64, 8, 0, 0);
    for (int j = 0; j < 4; ++j)
      for (int h = 0; h < 2; ++h) {
        const int kk = 4 * h + j;
        const uint64_t a = sdesc(smem_u32(sK) + h * 8192 + j * 32, 16, 1024);
        const uint64_t bq = sdesc(smem_u32(sQ) + h * 1024 + j * 32, 16, 1024);
        mma(tm + 16 + 8 * h, a, bq, id_s, j > 0);
        (void)kk;
      }
    commit(b);
  }
  mbar_wait(b, 0);
  if (tid == 0) t10 = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    t11 = clock64();
    constexpr uint32_t id_o = idesc(128, 8, 1, 0);
    for (int kk = 0; kk < 4; ++kk)
      for (int h = 0; h < 2; ++h) {
        const uint64_t a = sdesc(smem_u32(sV) + kk * 2048, 8192, 1024);
        const uint64_t bp = sdesc(smem_u32(sP) + kk * 32, 16, 1024);
        mma(tm + 8 + 16 * h, a, bp, id_o, kk > 0);
      }
    commit(b);
  }
  mbar_wait(b, 1);
  if (tid == 0) t12 = clock64();
  if (tid == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t4 - t3; cyc[3] = t6 - t5; cyc[4] = t8 - t7;
                  cyc[5] = t10 - t9; cyc[6] = t12 - t11; }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

int main() {
  std::vector<float> k(64 * 128), v(64 * 128), q(8 * 128), p(8 * 64);
  srand(1);
  auto rnd = [] { return bf((rand() / (float)RAND_MAX) * 2.f - 1.f); };
  for (auto& x : k) x = rnd();
  for (auto& x : v) x = rnd();
  for (auto& x : q) x = rnd();
  for (auto& x : p) x = bf(rand() / (float)RAND_MAX);
  auto up = [](const std::vector<float>& h) {
    std::vector<__nv_bfloat16> t(h.size());
    for (size_t i = 0; i < h.size(); ++i) t[i] = __float2bfloat16(h[i]);
    __nv_bfloat16* d; CK(cudaMalloc(&d, t.size() * 2)); CK(cudaMemcpy(d, t.data(), t.size() * 2, cudaMemcpyHostToDevice));
    return d;
  };
  __nv_bfloat16 *dk = up(k), *dv = up(v), *dq = up(q), *dp = up(p);
  float *ds, *dO; long long* dc;
  CK(cudaMalloc(&ds, 128 * 8 * 4)); CK(cudaMalloc(&dO, 128 * 8 * 4)); CK(cudaMalloc(&dc, 64));
  CK(cudaMemset(ds, 0, 128 * 8 * 4));
  CK(cudaFuncSetAttribute(tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024));
  long long best[7] = {1ll << 60, 1ll << 60, 1ll << 60, 1ll << 60, 1ll << 60, 1ll << 60, 1ll << 60};
  for (int it = 0; it < 20; ++it) {
    tile_kernel<<<1, 128, 40 * 1024>>>(dk, dv, dq, dp, ds, dO, dc);
    CK(cudaDeviceSynchronize());
    long long c[7]; CK(cudaMemcpy(c, dc, 56, cudaMemcpyDeviceToHost));
    for (int i = 0; i < 7; ++i) best[i] = c[i] < best[i] ? c[i] : best[i];
  }
  std::vector<float> hs(128 * 8), ho(128 * 8);
  CK(cudaMemcpy(hs.data(), ds, hs.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ho.data(), dO, ho.size() * 4, cudaMemcpyDeviceToHost));
  // reference S[t][g], O[d][g]
  std::vector<double> S(64 * 8), O(128 * 8);
  for (int t = 0; t < 64; ++t) for (int g = 0; g < 8; ++g) { double a = 0; for (int d = 0; d < 128; ++d) a += (double)k[t * 128 + d] * q[g * 128 + d]; S[t * 8 + g] = a; }
  for (int d = 0; d < 128; ++d) for (int g = 0; g < 8; ++g) { double a = 0; for (int t = 0; t < 64; ++t) a += (double)v[t * 128 + d] * p[g * 64 + t]; O[d * 8 + g] = a; }
  // where does accumulator row t (M = 64) land?  try lane = t (rows 0-63) and lane = 32 (t / 16) + t % 16
  double e_lin = 0, e_q16 = 0;
  for (int t = 0; t < 64; ++t) for (int g = 0; g < 8; ++g) {
    e_lin = fmax(e_lin, fabs(hs[t * 8 + g] - S[t * 8 + g]));
    e_q16 = fmax(e_q16, fabs(hs[(32 * (t / 16) + t % 16) * 8 + g] - S[t * 8 + g]));
  }
  double e_o = 0;
  for (int i = 0; i < 128 * 8; ++i) e_o = fmax(e_o, fabs(ho[i] - O[i]));
  printf("S^T (M=64): max |err| lane = row %.3e ; lane = 32 (row / 16) + row %% 16 %.3e\n", e_lin, e_q16);
  printf("O^T (M=128, A MN-major): max |err| %.3e\n", e_o);
  printf("S lanes 0..3 col 0: %f %f %f %f | ref rows 0..3: %f %f %f %f\n", hs[0], hs[8], hs[16], hs[24], S[0], S[8], S[16], S[24]);
  printf("cycles (best of 20): S^T 8 MMAs issue->mbarrier %lld, tcgen05.ld 32x32b.x8 %lld, O^T 4 MMAs issue->mbarrier %lld\n",
         best[0], best[1], best[2]);
  printf("warm repeats: S^T 8 MMAs %lld, O^T 8 MMAs (P hi + lo) %lld\n", best[3], best[4]);
  printf("two accumulators: S^T 2 x 4 MMAs %lld, O^T hi / lo 2 x 4 MMAs %lld\n", best[5], best[6]);
  return 0;
}
