// Development microbenchmark: how fast can ONE SM (and a few SMs) ingest a contiguous
// bf16 KV stream on B200?  Compares TMA box shapes, 1-D bulk copies and plain LDG.128.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/microbench_tma.cu \
//        -L/usr/local/cuda/lib64/stubs -lcuda -o scripts/mb_tma.bin
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int NS = 6, STAGE = 32768;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint32_t b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c)); }
__device__ __forceinline__ void expect(uint32_t b, int n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n) : "memory"); }
__device__ __forceinline__ void arrive(uint32_t b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory"); }
__device__ __forceinline__ void wait(uint32_t b, int ph) {
  uint32_t ok = 0;
  while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}" : "=r"(ok) : "r"(b), "r"(ph) : "memory");
}

// MODE 0: 4D tensor boxes 64 el x 64 rows, SWIZZLE_128B (4 boxes / stage)
// MODE 1: 4D tensor boxes 128 el x 64 rows, no swizzle (2 boxes / stage)
// MODE 2: 1-D bulk copy 16 KB (2 / stage)
// MODE 3: 4D tensor boxes 64 el x 128 rows (2 boxes / stage, 128 tokens... only K)
template <int MODE>
__global__ void __launch_bounds__(224, 1) k_tma(const __grid_constant__ CUtensorMap m0, const __grid_constant__ CUtensorMap m1,
                                                const uint8_t* src, int tiles_per_cta, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  uint32_t base = (sa(sm) + 1023) & ~1023u;
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { for (int i = 0; i < NS; ++i) { bar_init(sa(&full[i]), 1); bar_init(sa(&empty[i]), 1); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  int t0 = blockIdx.x * tiles_per_cta;
  if (warp == NS) {
    if (lane == 0) for (int i = 0; i < tiles_per_cta; ++i) {
      int st = i % NS;
      if (i >= NS) wait(sa(&empty[st]), ((i / NS) - 1) & 1);
      uint32_t fb = sa(&full[st]); expect(fb, STAGE);
      uint32_t dst = base + st * STAGE; int t = (t0 + i) * 64;
      if (MODE == 0) {
        for (int h = 0; h < 4; ++h) {
          const CUtensorMap* mp = h < 2 ? &m0 : &m1;
          asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
            ::"r"(dst + h * 8192), "l"((uint64_t)mp), "r"(fb), "r"((h & 1) * 64), "r"(0), "r"(t), "r"(0) : "memory");
        }
      } else if (MODE == 1) {
        for (int h = 0; h < 2; ++h) {
          const CUtensorMap* mp = h < 1 ? &m0 : &m1;
          asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
            ::"r"(dst + h * 16384), "l"((uint64_t)mp), "r"(fb), "r"(0), "r"(0), "r"(t), "r"(0) : "memory");
        }
      } else if (MODE == 2) {
        for (int h = 0; h < 2; ++h) {
          const uint8_t* g = src + (size_t)h * (1u << 28) + (size_t)t * 256;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(dst + h * 16384), "l"(g), "r"(16384), "r"(fb) : "memory");
        }
      }
    }
  } else {
    float acc = 0.f;
    for (int i = warp, r = 0; i < tiles_per_cta; i += NS, ++r) {
      wait(sa(&full[warp]), r & 1);
      uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(base + warp * STAGE + lane * 4));
      acc += __uint_as_float(v);
      __syncwarp();
      if (lane == 0) arrive(sa(&empty[warp]));
    }
    if (acc == 12345.f) out[0] = acc;
  }
}

// LDG: every thread streams 16-B vectors, 8 in flight per thread
__global__ void __launch_bounds__(512, 1) k_ldg(const uint4* src, size_t n16_per_cta, float* out) {
  const uint4* p = src + blockIdx.x * n16_per_cta;
  uint32_t acc = 0;
  for (size_t i = threadIdx.x; i < n16_per_cta; i += blockDim.x * 8) {
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { size_t k = i + j * blockDim.x; v[j] = k < n16_per_cta ? __ldcs(p + k) : make_uint4(0,0,0,0); }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc ^= v[j].x ^ v[j].w;
  }
  if (acc == 0x12345) out[0] = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;
CUtensorMap mk(void* p, int inner, int box_inner, CUtensorMapSwizzle sw) {
  CUtensorMap m; cuuint64_t dims[4] = {128, 1, 1u << 20, 1}; cuuint64_t str[3] = {256, 256, 256ull << 20};
  cuuint32_t box[4] = {(cuuint32_t)box_inner, 1, 64, 1}, es[4] = {1, 1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); exit(1); }
  return m;
}

template <class F>
float time_graph(F launch, int reps = 50) {
  cudaStream_t st; CK(cudaStreamCreate(&st));
  for (int i = 0; i < 3; ++i) launch(st);
  CK(cudaStreamSynchronize(st));
  cudaGraph_t g; cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < reps; ++i) launch(st);
  CK(cudaStreamEndCapture(st, &g)); CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, st)); CK(cudaStreamSynchronize(st));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  std::vector<float> ts;
  for (int r = 0; r < 5; ++r) { cudaEventRecord(a, st); cudaGraphLaunch(ge, st); cudaEventRecord(b, st); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); ts.push_back(ms * 1e3f / reps); }
  std::sort(ts.begin(), ts.end()); return ts[2];
}

int main() {
  cudaDriverEntryPointQueryResult q; void* fp;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q)); enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
  uint8_t* buf; CK(cudaMalloc(&buf, 2u << 28)); CK(cudaMemset(buf, 0, 2u << 28));
  float* out; CK(cudaMalloc(&out, 16));
  CUtensorMap a0 = mk(buf, 128, 64, CU_TENSOR_MAP_SWIZZLE_128B), a1 = mk(buf + (1u << 28), 128, 64, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap b0 = mk(buf, 128, 128, CU_TENSOR_MAP_SWIZZLE_NONE), b1 = mk(buf + (1u << 28), 128, 128, CU_TENSOR_MAP_SWIZZLE_NONE);
  int smem = NS * STAGE + 1024;
  CK(cudaFuncSetAttribute(k_tma<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int ctas : {1, 3, 8, 148}) {
    for (int tiles : {1, 8, 64}) {
      double bytes = (double)ctas * tiles * STAGE;
      float t0 = time_graph([&](cudaStream_t s) { k_tma<0><<<ctas, 224, smem, s>>>(a0, a1, buf, tiles, out); });
      float t1 = time_graph([&](cudaStream_t s) { k_tma<1><<<ctas, 224, smem, s>>>(b0, b1, buf, tiles, out); });
      float t2 = time_graph([&](cudaStream_t s) { k_tma<2><<<ctas, 224, smem, s>>>(a0, a1, buf, tiles, out); });
      float t3 = time_graph([&](cudaStream_t s) { k_ldg<<<ctas, 512, 0, s>>>((const uint4*)buf, (size_t)tiles * STAGE / 16, out); });
      printf("ctas %3d tiles/cta %3d (%7.0f KB): swz128 %6.2f us (%6.0f GB/s) | box256 %6.2f (%6.0f) | bulk1d %6.2f (%6.0f) | ldg %6.2f (%6.0f)\n",
             ctas, tiles, bytes / 1024, t0, bytes / t0 / 1e3, t1, bytes / t1 / 1e3, t2, bytes / t2 / 1e3, t3, bytes / t3 / 1e3);
    }
  }
  return 0;
}
