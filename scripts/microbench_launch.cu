// Development microbenchmark: per-step cost of tiny kernels replayed back to back in a
// CUDA graph on B200, with / without PDL, with / without thread-block clusters, and the
// cost of the two cross-CTA merge protocols (DSMEM push vs global last-CTA ticket).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/microbench_launch.cu -o /tmp/mb && /tmp/mb
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <int MODE>
__global__ void k_empty(float* out, unsigned* ctr, int s) {
  extern __shared__ float sm[];
  if (MODE & 1) pdl_trigger();
  pdl_wait();
  if (MODE & 2) {  // cluster push: ranks != 0 store 4 KB into rank 0 then arrive; rank 0 waits
    __shared__ __align__(8) uint64_t bar;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0) {
      uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(s - 1));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    if (rank != 0) {
      uint32_t dst = (uint32_t)__cvta_generic_to_shared(sm + threadIdx.x * 4), r;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(dst), "r"(0));
      asm volatile("st.shared::cluster.v4.f32 [%0], {%1,%1,%1,%1};" ::"r"(r), "f"(1.f) : "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar), rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(b), "r"(0));
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
      }
    } else {
      uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar), ok = 0;
      while (!ok) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}" : "=r"(ok) : "r"(b) : "memory");
      }
      out[threadIdx.x] = sm[threadIdx.x * 4];
    }
    return;
  }
  if (MODE & 4) {  // global last-CTA ticket: every CTA writes 4 KB, fence, atomic; last one reads all
    const int cta = blockIdx.x;
    out[1024 + cta * 256 * 4 + threadIdx.x] = 1.f;
    __threadfence();
    __syncthreads();
    __shared__ unsigned last;
    if (threadIdx.x == 0) last = atomicAdd(ctr, 1u) == (unsigned)(s - 1);
    __syncthreads();
    if (last) {
      float acc = 0.f;
      for (int r = 0; r < s; ++r) acc += __ldcg(out + 1024 + r * 256 * 4 + threadIdx.x);
      out[threadIdx.x] = acc;
      if (threadIdx.x == 0) *ctr = 0;
    }
    return;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 1.f;
}

template <int MODE>
float run(int ctas, int cluster, int smem, bool pdl_attr, int steps = 400) {
  float* out; unsigned* ctr;
  CK(cudaMalloc(&out, 1 << 22)); CK(cudaMalloc(&ctr, 4)); CK(cudaMemset(ctr, 0, 4));
  CK(cudaFuncSetAttribute(k_empty<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaStream_t st; CK(cudaStreamCreate(&st));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem; cfg.stream = st;
  cudaLaunchAttribute at[2]; int na = 0;
  if (pdl_attr) { at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[na].val.programmaticStreamSerializationAllowed = 1; ++na; }
  if (cluster > 1) { at[na].id = cudaLaunchAttributeClusterDimension; at[na].val.clusterDim = {(unsigned)cluster, 1, 1}; ++na; }
  cfg.attrs = at; cfg.numAttrs = na;
  for (int i = 0; i < 10; ++i) CK(cudaLaunchKernelEx(&cfg, k_empty<MODE>, out, ctr, ctas));
  CK(cudaStreamSynchronize(st));
  cudaGraph_t g; cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < steps; ++i) CK(cudaLaunchKernelEx(&cfg, k_empty<MODE>, out, ctr, ctas));
  CK(cudaStreamEndCapture(st, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, st)); CK(cudaStreamSynchronize(st));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  std::vector<float> ts;
  for (int r = 0; r < 7; ++r) {
    cudaEventRecord(e0, st); CK(cudaGraphLaunch(ge, st)); cudaEventRecord(e1, st);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); ts.push_back(ms * 1e3f / steps);
  }
  std::sort(ts.begin(), ts.end());
  cudaGraphExecDestroy(ge); cudaGraphDestroy(g); cudaFree(out); cudaFree(ctr); cudaStreamDestroy(st);
  return ts[3];
}

#include <algorithm>
int main() {
  printf("empty 1 CTA, no PDL                : %.2f us\n", run<0>(1, 1, 1024, false));
  printf("empty 1 CTA, PDL attr, no trigger  : %.2f us\n", run<0>(1, 1, 1024, true));
  printf("empty 1 CTA, PDL + early trigger   : %.2f us\n", run<1>(1, 1, 1024, true));
  printf("empty 1 CTA, 200KB smem, PDL+trig  : %.2f us\n", run<1>(1, 1, 200 * 1024, true));
  printf("empty 3 CTA, PDL+trig              : %.2f us\n", run<1>(3, 1, 200 * 1024, true));
  printf("empty 3 CTA cluster3, no PDL       : %.2f us\n", run<0>(3, 3, 200 * 1024, false));
  printf("empty 3 CTA cluster3, PDL+trig     : %.2f us\n", run<1>(3, 3, 200 * 1024, true));
  printf("push  3 CTA cluster3, PDL+trig     : %.2f us\n", run<3>(3, 3, 200 * 1024, true));
  printf("push  8 CTA cluster8, PDL+trig     : %.2f us\n", run<3>(8, 8, 200 * 1024, true));
  printf("ticket 3 CTA, PDL+trig             : %.2f us\n", run<5>(3, 1, 200 * 1024, true));
  printf("ticket 8 CTA, PDL+trig             : %.2f us\n", run<5>(8, 1, 200 * 1024, true));
  printf("ticket 3 CTA, no PDL               : %.2f us\n", run<4>(3, 1, 200 * 1024, false));
  return 0;
}
