// tcgen05 contention microbenchmark (development tool): the 128-token stage of fwd_tc.cu (S = 8 MMAs
// M = 64 N = 128 with A from TMEM, PV = 8 MMAs M = 128 N = 128 with A from TMEM, B MN-major) issued
// by one thread for 64 stages, alone and with the two kinds of traffic the real kernel runs beside it:
//   MODE bit 0: one warp streams 64 KB per stage from global memory into a separate shared-memory
//               region with cp.async.bulk (the TMA ring's writes; every SM streams, so DRAM is loaded)
//   MODE bit 1: eight warps read the stage's S buffer (tcgen05.ld 16x256b.x8) and write P_hi / P_lo
//               (two tcgen05.st 16x128b.x8) once per stage, after its S MMAs commit (the softmax's
//               TMEM traffic)
// Prints cycles per stage per mode.  Operand contents are irrelevant (zeros).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/mb_cont scripts/microbench_tcgen05_contention.cu
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
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) { while (!try_wait(bar, par)) {} }

constexpr int kStages = 64;

template <int MODE>
__global__ void __launch_bounds__(320, 1) contention(const uint8_t* __restrict__ src, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t s_done[2], pv_done[2], p_full[2], bulk_bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_done[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&pv_done[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(&p_full[i])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bulk_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  const uint32_t sK = smem_u32(sm), sV = sK + 32768, sBulk = sK + 65536;
  if (warp == 9 && lane == 0) {
    // MMA issuer: S(0), S(1), then PV(s), S(s + 2), PV waits for the stage's "P" (bit 1) like the kernel
    constexpr uint32_t id_s = idesc(64, 128, 0, 0), id_o = idesc(128, 128, 0, 1);
    auto issue_s = [&](int s) {
      for (int kk = 0; kk < 8; ++kk)
        mma_ts(tm + (s & 1) * 128, tm + 384 + kk * 8, sdesc(sK + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), id_s, kk > 0);
      commit(smem_u32(&s_done[s & 1]));
    };
    auto issue_pv = [&](int s) {
      if (MODE & 2) wait(smem_u32(&p_full[s & 1]), (s >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int kk = 0; kk < 8; ++kk)
        mma_ts(tm + 256, tm + (s & 1) * 128 + kk * 8, sdesc(sV + kk * 2048, 16384, 1024), id_o, (s > 0 || kk > 0));
      commit(smem_u32(&pv_done[s & 1]));
    };
    const long long t0 = clock64();
    issue_s(0);
    issue_s(1);
    for (int s = 0; s < kStages; ++s) {
      issue_pv(s);
      if (s + 2 < kStages) issue_s(s + 2);
    }
    wait(smem_u32(&pv_done[(kStages - 1) & 1]), ((kStages - 1) >> 1) & 1);
    out[blockIdx.x] = clock64() - t0;
  } else if (warp == 8 && lane == 0 && (MODE & 1)) {
    // bulk copier: 4 x 16 KB per stage into its own region, waiting for each batch
    const uint8_t* base = src + (size_t)blockIdx.x * (kStages + 8) * 65536;
    for (int s = 0; s < kStages + 8; ++s) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bulk_bar)), "r"(65536) : "memory");
      for (int c = 0; c < 4; ++c)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sBulk + c * 16384), "l"(base + (size_t)s * 65536 + c * 16384), "r"(16384), "r"(smem_u32(&bulk_bar))
                     : "memory");
      wait(smem_u32(&bulk_bar), s & 1);
    }
  } else if (warp < 8 && (MODE & 2)) {
    // "softmax": per stage, read S (16x256b.x8 from this warp's quadrant) and write P_hi / P_lo
    const uint32_t lane_addr = (uint32_t)((warp & 3) * 32) << 16;
    const int hh = warp >> 2;
    for (int s = 0; s < kStages; ++s) {
      wait(smem_u32(&s_done[s & 1]), (s >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t r[32];
      const uint32_t sp = tm + lane_addr + (s & 1) * 128;
      asm volatile(
          "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(sp + 64 * hh)
          : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      uint32_t w[16];
      for (int i = 0; i < 16; ++i) w[i] = r[2 * i] ^ r[2 * i + 1];
      for (int h = 0; h < 2; ++h)
        asm volatile(
            "tcgen05.st.sync.aligned.16x128b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
            ::"r"(sp + (h ? (16u << 16) : 0u) + 32 * hh), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]),
              "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]),
              "r"(w[14]), "r"(w[15])
            : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&p_full[s & 1])) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 9) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int MODE>
void run(const uint8_t* src, int ctas, const char* name) {
  long long* d;
  cudaMalloc(&d, ctas * sizeof(long long));
  const int smem = 128 * 1024 + 1024;
  cudaFuncSetAttribute(contention<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  double best = 1e30;
  for (int it = 0; it < 5; ++it) {
    contention<MODE><<<ctas, 320, smem>>>(src, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    long long h[148];
    cudaMemcpy(h, d, ctas * sizeof(long long), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < ctas; ++i) mx = h[i] > mx ? h[i] : mx;
    best = mx < best ? mx : best;
  }
  printf("%-44s %d CTAs: %.0f cycles per stage (slowest CTA, best of 5; stand-alone floor ~1034)\n", name, ctas,
         best / kStages);
  cudaFree(d);
}

int main() {
  const int ctas = 148;
  uint8_t* src;
  const size_t bytes = (size_t)ctas * (kStages + 8) * 65536;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 0, bytes);
  run<0>(src, ctas, "MMA only");
  run<1>(src, ctas, "MMA + 64 KB/stage bulk copies (DRAM)");
  run<2>(src, ctas, "MMA + softmax TMEM ld/st, P hand-off");
  run<3>(src, ctas, "MMA + bulk copies + TMEM ld/st");
  run<0>(src, 1, "MMA only");
  run<2>(src, 1, "MMA + softmax TMEM ld/st, P hand-off");
  cudaFree(src);
  return 0;
}
