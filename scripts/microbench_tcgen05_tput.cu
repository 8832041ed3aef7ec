// tcgen05 throughput microbenchmark (development tool): N_REP back-to-back MMAs of one shape, issued
// by one thread into 2 alternating accumulators, timed issue -> commit -> mbarrier (clock64).
// Shapes of the decode tile: S = Q K^T (M = 64 / 128 rows, N = 64 tokens, K = 16 per MMA) and
// O = P V (M = 64 / 128, N = 128 dims), A from shared memory (SS) or TMEM (TS); B from shared memory
// (K-major for S, MN-major V for O).  Operand contents are irrelevant here (zeros).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/mb_tput scripts/microbench_tcgen05_tput.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

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

template <int M, int N, bool TS, bool VB>
__global__ void tput(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
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
  if (tid == 0) {
    constexpr uint32_t id = idesc(M, N, 0, VB ? 1 : 0);
    const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 32768);
    const long long t0 = clock64();
    for (int i = 0; i < N_REP; ++i) {
      const uint64_t b = VB ? sdesc(b0 + (i & 3) * 2048, 8192, 1024) : sdesc(b0 + (i & 3) * 32, 16, 1024);
      const uint32_t d = tm + (i & 1) * 128;
      if (TS) mma_ts(d, tm + 256 + (i & 7) * 8, b, id);
      else mma_ss(d, sdesc(a0 + (i & 3) * 32, 16, 1024), b, id);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
    out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int M, int N, bool TS, bool VB>
void run(const char* name) {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(tput<M, N, TS, VB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  long long best = 1ll << 60;
  for (int it = 0; it < 10; ++it) {
    tput<M, N, TS, VB><<<1, 128, 100 * 1024>>>(d);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    best = c < best ? c : best;
  }
  const double flop = 2.0 * M * N * 16;
  printf("%-34s M=%3d N=%3d %s: %6.1f cycles per MMA, %6.0f flop/cycle (%4.1f %% of 8192)\n", name, M, N, TS ? "TS" : "SS",
         (double)best / N_REP, flop * N_REP / best, 100.0 * flop * N_REP / best / 8192);
  cudaFree(d);
}

int main() {
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
  return 0;
}
