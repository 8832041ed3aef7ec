// Latency of the flag / fence operations the peer exchange uses (development tool): one thread,
// dependent chains of loads on a device-memory flag, clock64 per operation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/mb_acq scripts/microbench_sys_acquire.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

template <int kMode>
__device__ __forceinline__ uint32_t ld(const uint32_t* p) {
  uint32_t v;
  if (kMode == 0) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  if (kMode == 1) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  if (kMode == 2) asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  if (kMode == 3) asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int kMode>
__global__ void chain(const uint32_t* flags, long long* out, uint32_t* sink) {
  const uint32_t* p = flags;
  uint32_t acc = 0;
  for (int i = 0; i < 4; ++i) acc += ld<kMode>(p + (acc & 1));      // warm
  const long long t0 = clock64();
  for (int i = 0; i < 64; ++i) acc += ld<kMode>(p + (acc & 1));     // dependent chain
  const long long t1 = clock64();
  *out = (t1 - t0) / 64;
  *sink = acc;
}

__global__ void fences(long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < 64; ++i) asm volatile("fence.acq_rel.sys;" ::: "memory");
  long long t1 = clock64();
  for (int i = 0; i < 64; ++i) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  long long t2 = clock64();
  out[0] = (t1 - t0) / 64;
  out[1] = (t2 - t1) / 64;
}

int main() {
  uint32_t *flags, *sink;
  long long* out;
  cudaMalloc(&flags, 256);
  cudaMalloc(&sink, 4);
  cudaMalloc(&out, 64);
  cudaMemset(flags, 0, 256);
  long long h[4];
  const char* names[4] = {"ld.acquire.sys", "ld.acquire.gpu", "ld.relaxed.sys", "ld.volatile"};
  for (int rep = 0; rep < 2; ++rep) {
    chain<0><<<1, 1>>>(flags, out + 0, sink);
    chain<1><<<1, 1>>>(flags, out + 1, sink);
    chain<2><<<1, 1>>>(flags, out + 2, sink);
    chain<3><<<1, 1>>>(flags, out + 3, sink);
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
  }
  for (int i = 0; i < 4; ++i) printf("%-16s %lld cycles per dependent load\n", names[i], h[i]);
  fences<<<1, 1>>>(out);
  cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  printf("fence.acq_rel.sys %lld cycles, fence.acq_rel.gpu %lld cycles (single thread, nothing outstanding)\n", h[0], h[1]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
