// tcgen05 microbenchmark for a query-rows-as-M decode tile (development tool, not part of the
// product): the contraction of a KV head shared by G = 64 (or 128) query heads (MQA / wide GQA).
//
//   S = Q K^T   tcgen05.mma kind::f16  M = G rows, N = 64 tokens, K = 128 dims (8 x K16)
//               A = Q (K-major, two 128B-swizzled 64-dim boxes), B = the K tile (K-major)
//   O = P V     M = G rows, N = 128 dims, K = 64 tokens (4 x K16, twice: P_hi and P_lo)
//               A = P (K-major, one 128B-swizzled box [rows][64 tokens]), B = the V tile (MN-major)
// The K / V tiles use exactly the TMA boxes of csrc/fwd.cu ([half][token][64 dims], SWIZZLE_128B).
// Checks S and O against a host fp64 reference, reports the TMEM lane of accumulator row r, times
// issue -> commit -> mbarrier for both products and the tcgen05.ld of a 64-column row.
// Then the same two products with A read from TMEM ("TS": tcgen05.mma ... [d], [a_tmem], b_desc):
// Q and P written into TMEM by the row threads (tcgen05.st, two bf16 per 32-bit column, row r on
// the accumulator's lane), which takes the A operand's shared-memory traffic off the tile.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/mb_rows scripts/microbench_tcgen05_rows.cu && /tmp/mb_rows
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__host__ __device__ inline uint32_t sw128(int r, int c) { return r * 128 + ((((c >> 3) ^ (r & 7)) & 7) << 4) + (c & 7) * 2; }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t id, int acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t id, int acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem), "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
               "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
               ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                 "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
                 "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
                 "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(bar), "r"(ph) : "memory");
}
__device__ __forceinline__ void ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                 "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                 "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// M = G query rows.  out_s: [128 lanes][64], out_o: [128 lanes][128], cyc: timings
template <int M>
__global__ void __launch_bounds__(128) rows_kernel(const __nv_bfloat16* K, const __nv_bfloat16* V,
                                                    const __nv_bfloat16* Q, const __nv_bfloat16* P,
                                                    float* out_s, float* out_o, long long* cyc,
                                                    float* out_s2, float* out_o2, int lane_mode) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sK = sm;                  // 2 boxes x 8 KB  [half][token][64]
  uint8_t* sV = sm + 16384;          // 2 boxes x 8 KB
  uint8_t* sQ = sm + 32768;          // 2 boxes x M x 128 B  [half][row][64]
  uint8_t* sP = sQ + 2 * M * 128;    // 1 box [row][64 tokens]
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 64 * 128; i += 128) {
    const int t = i / 128, d = i % 128;
    *(__nv_bfloat16*)(sK + (d >> 6) * 8192 + sw128(t, d & 63)) = K[i];
    *(__nv_bfloat16*)(sV + (d >> 6) * 8192 + sw128(t, d & 63)) = V[i];
  }
  for (int i = tid; i < M * 128; i += 128) {
    const int g = i / 128, d = i % 128;
    *(__nv_bfloat16*)(sQ + (d >> 6) * (M * 128) + sw128(g, d & 63)) = Q[i];
  }
  for (int i = tid; i < M * 64; i += 128) {
    const int g = i / 64, t = i % 64;
    *(__nv_bfloat16*)(sP + sw128(g, t)) = P[i];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  const uint32_t b = smem_u32(&bar);
  long long t0 = 0, t1 = 0, t2 = 0, t3 = 0, t4 = 0;
  if (tid == 0) {
    t0 = clock64();
    constexpr uint32_t id_s = idesc(M, 64, 0, 0);
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t a = sdesc(smem_u32(sQ) + (kk >> 2) * (M * 128) + (kk & 3) * 32, 16, 1024);
      const uint64_t bk = sdesc(smem_u32(sK) + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
      mma(tm, a, bk, id_s, kk > 0);
    }
    commit(b);
  }
  mbar_wait(b, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) t1 = clock64();
  {
    float v[64];
    ld32(tm + ((uint32_t)(warp * 32) << 16), v);
    ld32(tm + 32 + ((uint32_t)(warp * 32) << 16), v + 32);
    if (tid == 0) t2 = clock64();
    for (int c = 0; c < 64; ++c) out_s[(warp * 32 + lane) * 64 + c] = v[c];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    t3 = clock64();
    constexpr uint32_t id_o = idesc(M, 128, 0, 1);
    for (int kk = 0; kk < 8; ++kk) {   // P_hi then P_lo (here the same P twice: O = 2 P V)
      const uint64_t a = sdesc(smem_u32(sP) + (kk & 3) * 32, 16, 1024);
      const uint64_t bv = sdesc(smem_u32(sV) + (kk & 3) * 2048, 8192, 1024);
      mma(tm + 64, a, bv, id_o, kk > 0);
    }
    commit(b);
  }
  mbar_wait(b, 1);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) t4 = clock64();
  {
    float v[128];
    for (int c = 0; c < 4; ++c) ld32(tm + 64 + 32 * c + ((uint32_t)(warp * 32) << 16), v + 32 * c);
    for (int c = 0; c < 128; ++c) out_o[(warp * 32 + lane) * 128 + c] = v[c];
  }
  // ---- TS: A from TMEM.  Q at columns [256, 320) (128 dims packed two per column), P at [320, 352)
  {
    const int r = lane_mode == 0 ? warp * 32 + lane : (lane < 16 ? warp * 16 + lane : -1);   // row of this lane
    uint32_t qa[64], pa[32];
    for (int c = 0; c < 64; ++c) {
      uint32_t w = 0;
      if (r >= 0 && r < M) {
        const uint16_t lo = *reinterpret_cast<const uint16_t*>(&Q[r * 128 + 2 * c]);
        const uint16_t hi = *reinterpret_cast<const uint16_t*>(&Q[r * 128 + 2 * c + 1]);
        w = (uint32_t)lo | ((uint32_t)hi << 16);
      }
      qa[c] = w;
    }
    for (int c = 0; c < 32; ++c) {
      uint32_t w = 0;
      if (r >= 0 && r < M) {
        const uint16_t lo = *reinterpret_cast<const uint16_t*>(&P[r * 64 + 2 * c]);
        const uint16_t hi = *reinterpret_cast<const uint16_t*>(&P[r * 64 + 2 * c + 1]);
        w = (uint32_t)lo | ((uint32_t)hi << 16);
      }
      pa[c] = w;
    }
    const uint32_t la = (uint32_t)(warp * 32) << 16;
    st32(tm + 256 + la, qa);
    st32(tm + 288 + la, qa + 32);
    st32(tm + 320 + la, pa);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  long long t5 = 0, t6 = 0, t7 = 0, t8 = 0;
  if (tid == 0) {
    t5 = clock64();
    constexpr uint32_t id_s = idesc(M, 64, 0, 0);
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t bk = sdesc(smem_u32(sK) + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
      mma_ts(tm + 352 - 352 + 0, tm + 256 + kk * 8, bk, id_s, kk > 0);
    }
    commit(b);
  }
  mbar_wait(b, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) t6 = clock64();
  {
    float v[64];
    ld32(tm + ((uint32_t)(warp * 32) << 16), v);
    ld32(tm + 32 + ((uint32_t)(warp * 32) << 16), v + 32);
    for (int c = 0; c < 64; ++c) out_s2[(warp * 32 + lane) * 64 + c] = v[c];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    t7 = clock64();
    constexpr uint32_t id_o = idesc(M, 128, 0, 1);
    for (int kk = 0; kk < 8; ++kk) {   // twice over the 4 token steps (O = 2 P V, as above)
      const uint64_t bv = sdesc(smem_u32(sV) + (kk & 3) * 2048, 8192, 1024);
      mma_ts(tm + 64, tm + 320 + (kk & 3) * 8, bv, id_o, kk > 0);
    }
    commit(b);
  }
  mbar_wait(b, 1);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) t8 = clock64();
  {
    float v[128];
    for (int c = 0; c < 4; ++c) ld32(tm + 64 + 32 * c + ((uint32_t)(warp * 32) << 16), v + 32 * c);
    for (int c = 0; c < 128; ++c) out_o2[(warp * 32 + lane) * 128 + c] = v[c];
  }
  if (tid == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t4 - t3; cyc[3] = t6 - t5; cyc[4] = t8 - t7; }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

template <int M>
static void run() {
  std::vector<float> k(64 * 128), v(64 * 128), q(M * 128), p(M * 64);
  srand(1 + M);
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
  float *ds, *dO, *ds2, *dO2; long long* dc;
  CK(cudaMalloc(&ds, 128 * 64 * 4)); CK(cudaMalloc(&dO, 128 * 128 * 4)); CK(cudaMalloc(&dc, 64));
  CK(cudaMalloc(&ds2, 128 * 64 * 4)); CK(cudaMalloc(&dO2, 128 * 128 * 4));
  const int smem = 32768 + 2 * M * 128 + M * 128 + 1024;
  CK(cudaFuncSetAttribute(rows_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  long long best[5] = {1ll << 60, 1ll << 60, 1ll << 60, 1ll << 60, 1ll << 60};
  const int lane_mode = M == 64 ? 1 : 0;
  for (int it = 0; it < 20; ++it) {
    rows_kernel<M><<<1, 128, smem>>>(dk, dv, dq, dp, ds, dO, dc, ds2, dO2, lane_mode);
    CK(cudaDeviceSynchronize());
    long long c[5]; CK(cudaMemcpy(c, dc, 40, cudaMemcpyDeviceToHost));
    for (int i = 0; i < 5; ++i) best[i] = c[i] < best[i] ? c[i] : best[i];
  }
  std::vector<float> hs2(128 * 64), ho2(128 * 128);
  CK(cudaMemcpy(hs2.data(), ds2, hs2.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ho2.data(), dO2, ho2.size() * 4, cudaMemcpyDeviceToHost));
  std::vector<float> hs(128 * 64), ho(128 * 128);
  CK(cudaMemcpy(hs.data(), ds, hs.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ho.data(), dO, ho.size() * 4, cudaMemcpyDeviceToHost));
  auto lane_of = [](int r, int mode) { return mode == 0 ? r : 32 * (r / 16) + r % 16; };
  for (int mode = 0; mode < 2; ++mode) {
    double es = 0, eo = 0;
    for (int r = 0; r < M; ++r) {
      const int ln = lane_of(r, mode);
      for (int t = 0; t < 64; ++t) {
        double a = 0;
        for (int d = 0; d < 128; ++d) a += (double)q[r * 128 + d] * k[t * 128 + d];
        es = fmax(es, fabs(hs[ln * 64 + t] - a));
      }
      for (int d = 0; d < 128; ++d) {
        double a = 0;
        for (int t = 0; t < 64; ++t) a += 2.0 * p[r * 64 + t] * v[t * 128 + d];
        eo = fmax(eo, fabs(ho[ln * 128 + d] - a));
      }
    }
    printf("M=%d lane mapping %s: max |err| S %.3e  O %.3e\n", M, mode == 0 ? "lane = row" : "lane = 32 (row / 16) + row % 16",
           es, eo);
  }
  printf("M=%d cycles (best of 20): S 8 MMAs issue->mbarrier %lld, tcgen05.ld 2 x 32x32b.x32 %lld, O 8 MMAs (N=128) %lld\n",
         M, best[0], best[1], best[2]);
  {
    double es = 0, eo = 0;
    for (int r = 0; r < M; ++r) {
      const int ln = lane_of(r, M == 64 ? 1 : 0);
      for (int t = 0; t < 64; ++t) {
        double a = 0;
        for (int d = 0; d < 128; ++d) a += (double)q[r * 128 + d] * k[t * 128 + d];
        es = fmax(es, fabs(hs2[ln * 64 + t] - a));
      }
      for (int d = 0; d < 128; ++d) {
        double a = 0;
        for (int t = 0; t < 64; ++t) a += 2.0 * p[r * 64 + t] * v[t * 128 + d];
        eo = fmax(eo, fabs(ho2[ln * 128 + d] - a));
      }
    }
    printf("M=%d TS (A from TMEM, row r on the accumulator's lane): max |err| S %.3e  O %.3e; cycles S %lld, O %lld\n",
           M, es, eo, best[3], best[4]);
  }
}

int main() {
  run<64>();
  run<128>();
  return 0;
}
