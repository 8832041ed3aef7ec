// tcgen05 throughput microbenchmark (development tool): N_REP back-to-back MMAs of one shape, issued
// by one thread into 2 alternating accumulators, timed issue -> commit -> mbarrier (clock64).
// Shapes of the decode tile: S = Q K^T (M = 64 / 128 rows, N = 64 tokens, K = 16 per MMA) and
// O = P V (M = 64 / 128, N = 128 dims), A from shared memory (SS) or TMEM (TS); B from shared memory
// (K-major for S, MN-major V for O).  Operand contents are irrelevant here (zeros).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/mb_tput scripts/microbench_tcgen05_tput.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(a), "l"(b), "r"(id));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(id));
}

constexpr int N_REP = 128;
#ifndef RANDOM_DATA
#define RANDOM_DATA 1
#endif

template <int M, int N, bool TS, bool VB, int COMMIT_EVERY = 0>
__global__ void tput(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar, bar2;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  // operands: zeros, or pseudo-random bf16 in [-1, 1) (RANDOM_DATA)
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) {
    uint32_t x = RANDOM_DATA ? (uint32_t)i * 2654435761u + 12345u : 0u;
    x ^= x >> 13;
    const uint32_t lo = RANDOM_DATA ? (0x3c00u | (x & 0x7fu) | ((x & 0x100u) << 7)) : 0u;
    const uint32_t hi = RANDOM_DATA ? (0x3c00u | ((x >> 9) & 0x7fu) | ((x & 0x200u) << 6)) : 0u;
    reinterpret_cast<uint32_t*>(sm)[i] = lo | (hi << 16);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)));
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
  if (TS && RANDOM_DATA) {   // the TMEM A region (columns 256..319) of this warp's lanes
    uint32_t r[32];
    for (int c = 0; c < 32; ++c) r[c] = 0x3c003c00u ^ ((uint32_t)(tid * 33 + c) * 0x9e3779b9u & 0x007f007fu);
    for (int h = 0; h < 2; ++h)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                   "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                   ::"r"(tm + 256 + 32 * h + ((uint32_t)(warp * 32) << 16)), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]),
                     "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]),
                     "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]),
                     "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
                     "r"(r[29]), "r"(r[30]), "r"(r[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    constexpr uint32_t id = idesc(M, N, 0, VB ? 1 : 0);
    const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 32768);
    const long long t0 = clock64();
    for (int i = 0; i < N_REP; ++i) {
      const uint64_t b = VB ? sdesc(b0 + (i & 3) * 2048, 8192, 1024) : sdesc(b0 + (i & 3) * 32, 16, 1024);
      const uint32_t d = tm + (i & 1) * 128;
      if (TS) mma_ts(d, tm + 256 + (i & 7) * 8, b, id);
      else mma_ss(d, sdesc(a0 + (i & 3) * 32, 16, 1024), b, id);
      if (COMMIT_EVERY > 0 && (i + 1) % COMMIT_EVERY == 0 && i + 1 < N_REP)   // commits nobody waits on
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
    out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

// the decode tile's issue pattern: per tile 8 S MMAs (M = 64, N = 64) + commit, 4 PV MMAs (M = 128,
// N = 128, B MN-major) + 2 commits, optionally a tcgen05.fence::after_thread_sync before each group
template <bool FENCE>
__global__ void pattern(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar, bar2;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)));
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
  if (tid == 0) {
    constexpr uint32_t id_s = idesc(64, 64, 0, 0), id_o = idesc(128, 128, 0, 1);
    const uint32_t b0 = smem_u32(sm);
    const long long t0 = clock64();
    for (int t = 0; t < 32; ++t) {
      if (FENCE) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int kk = 0; kk < 8; ++kk)
        mma_ts(tm + (t % 3) * 64, tm + 320 + kk * 8, sdesc(b0 + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), id_s);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)) : "memory");
      if (FENCE) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int kk = 0; kk < 4; ++kk)
        mma_ts(tm + 192, tm + 384 + kk * 8, sdesc(b0 + 16384 + kk * 2048, 8192, 1024), id_o);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)) : "memory");
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
    out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

// the 128-token stage of fwd_tc.cu: S (M = 64, N = 128, K-major K halves 16 KB apart) + PV (M = 128,
// N = 128, MN-major V with the 64-dim halves 16 KB apart, 8 steps of 16 tokens)
template <int LBO_V>
__global__ void pattern128(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar, bar2;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)));
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
  if (tid == 0) {
    constexpr uint32_t id_s = idesc(64, 128, 0, 0), id_o = idesc(128, 128, 0, 1);
    const uint32_t sK = smem_u32(sm), sV = sK + 32768;
    long long tS = 0, tP = 0;
    const long long t0 = clock64();
    for (int t = 0; t < 32; ++t) {
      const long long a0 = clock64();
      for (int kk = 0; kk < 8; ++kk)
        mma_ts(tm + (t & 1) * 128, tm + 384 + kk * 8, sdesc(sK + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), id_s);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)) : "memory");
      const long long a1 = clock64();
      for (int kk = 0; kk < 8; ++kk)
        mma_ts(tm + 256, tm + (t & 1) * 128 + kk * 8, sdesc(sV + kk * 2048, LBO_V, 1024), id_o);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)) : "memory");
      const long long a2 = clock64();
      tS += a1 - a0;
      tP += a2 - a1;
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
    out[0] = clock64() - t0;
    out[1] = tS;
    out[2] = tP;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int LBO_V>
void run_pattern128() {
  long long* d; cudaMalloc(&d, 24);
  cudaFuncSetAttribute(pattern128<LBO_V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  long long best[3] = {1ll << 60, 0, 0};
  for (int it = 0; it < 10; ++it) {
    pattern128<LBO_V><<<1, 128, 100 * 1024>>>(d);
    cudaDeviceSynchronize();
    long long c[3]; cudaMemcpy(c, d, 24, cudaMemcpyDeviceToHost);
    if (c[0] < best[0]) best[0] = c[0], best[1] = c[1], best[2] = c[2];
  }
  printf("128-token stage pattern (S 8 x M64 N128, PV 8 x M128 N128, V LBO %d): %.0f cycles per stage "
         "(issue time S %.0f, PV %.0f; floor 8 x 65 + 8 x 66 = 1048)\n",
         LBO_V, best[0] / 32.0, best[1] / 32.0, best[2] / 32.0);
  cudaFree(d);
}

template <bool FENCE>
void run_pattern() {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(pattern<FENCE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  long long best = 1ll << 60;
  for (int it = 0; it < 10; ++it) {
    pattern<FENCE><<<1, 128, 100 * 1024>>>(d);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    best = c < best ? c : best;
  }
  printf("decode-tile pattern (8 S + 4 PV MMAs, 3 commits per tile)%s: %.0f cycles per tile (floor 8 x 45 + 4 x 66 = 624)\n",
         FENCE ? " + fence::after_thread_sync per group" : "", best / 32.0);
  cudaFree(d);
}

static int g_ctas = 1;
template <int M, int N, bool TS, bool VB, int CE = 0>
void run(const char* name) {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(tput<M, N, TS, VB, CE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  long long best = 1ll << 60;
  for (int it = 0; it < 10; ++it) {
    tput<M, N, TS, VB, CE><<<g_ctas, 128, 100 * 1024>>>(d);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    best = c < best ? c : best;
  }
  const double flop = 2.0 * M * N * 16;
  printf("%-34s M=%3d N=%3d %s commit/%2d: %6.1f cycles per MMA, %6.0f flop/cycle (%4.1f %% of 8192)\n", name, M, N, TS ? "TS" : "SS", CE,
         (double)best / N_REP, flop * N_REP / best, 100.0 * flop * N_REP / best / 8192);
  cudaFree(d);
}

int main(int argc, char** argv) {
  if (argc > 1) g_ctas = atoi(argv[1]);
  printf("%d CTAs, %s operands\n", g_ctas, RANDOM_DATA ? "random" : "zero");
  run<64, 64, false, false>("S = Q K^T (B K-major)");
  run<64, 64, true, false>("S = Q K^T (B K-major)");
  run<128, 64, false, false>("S = Q K^T (B K-major)");
  run<128, 64, true, false>("S = Q K^T (B K-major)");
  run<64, 128, false, true>("O = P V (B MN-major)");
  run<64, 128, true, true>("O = P V (B MN-major)");
  run<128, 128, false, true>("O = P V (B MN-major)");
  run<128, 128, true, true>("O = P V (B MN-major)");
  run<128, 256, true, false>("reference M128 N256 (B K-major)");
  run<64, 256, true, false>("reference M64 N256 (B K-major)");
  run_pattern128<8192>();
  run_pattern128<16384>();
  run_pattern<false>();
  run_pattern<true>();
  run<64, 64, true, false, 8>("S, commit after every 8");
  run<128, 128, true, true, 4>("PV, commit after every 4");
  run<128, 128, true, true, 2>("PV, commit after every 2");
  return 0;
}
