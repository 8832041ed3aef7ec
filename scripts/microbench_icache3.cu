// Development microbenchmark: instruction-cache capacity seen by one warp per SM across launches.
// Kernel = N straight-line FFMA groups (one block of code, ~N * 1.25 instructions of 16 B).  Each of
// 148 CTAs (one per SM) times the block; launches 2..4 repeat the kernel on a warm GPU.
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c) :: "memory");
  return c;
}
__device__ __forceinline__ void pin(float& x) { asm volatile("mov.b32 %0, %0;" : "+f"(x)); }

template <int N>
__global__ void k(float* out, long long* t) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  float a = threadIdx.x, b = 1.0001f, c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f, c4 = 0.f, c5 = 0.f, c6 = 0.f, c7 = 0.f;
  long long t0 = clk();
  pin(a);
#pragma unroll
  for (int i = 0; i < N; i += 8) {
    c0 = fmaf(a, b, c0); c1 = fmaf(a, b + 1, c1); c2 = fmaf(a, b + 2, c2); c3 = fmaf(a, b + 3, c3);
    c4 = fmaf(a, b + 4, c4); c5 = fmaf(a, b + 5, c5); c6 = fmaf(a, b + 6, c6); c7 = fmaf(a, b + 7, c7);
    a += 1e-7f;
  }
  pin(c0); pin(c1); pin(c2); pin(c3); pin(c4); pin(c5); pin(c6); pin(c7);
  long long t1 = clk();
  if (threadIdx.x == 0) t[smid] = t1 - t0;
  out[blockIdx.x * 32 + threadIdx.x] = c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7;
}

static long long med(long long* t) {
  std::vector<long long> v;
  for (int s = 0; s < 256; ++s) if (t[s]) v.push_back(t[s]);
  std::sort(v.begin(), v.end());
  return v.empty() ? 0 : v[v.size() / 2];
}

template <int N>
void run(float* out, long long* t) {
  long long c[4];
  for (int l = 0; l < 4; ++l) {
    cudaMemset(t, 0, 256 * 8);
    k<N><<<148, 32>>>(out, t);
    cudaDeviceSynchronize();
    c[l] = med(t);
  }
  const double instr = N * 1.125;
  printf("N=%5d (~%5.1f KB): cycles per launch %lld %lld %lld %lld  -> IPC warm-launch %.2f\n", N,
         instr * 16 / 1024, c[0], c[1], c[2], c[3], instr / c[3]);
}

int main() {
  float* out; long long* t;
  cudaMalloc(&out, 148 * 32 * 4);
  cudaMallocManaged(&t, 256 * 8);
  run<256>(out, t);
  run<512>(out, t);
  run<768>(out, t);
  run<1024>(out, t);
  run<1280>(out, t);
  run<1536>(out, t);
  run<1792>(out, t);
  run<2048>(out, t);
  run<3072>(out, t);
  return 0;
}
