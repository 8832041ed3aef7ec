// Development microbenchmark: does the SM instruction cache survive from one launch of a kernel
// to the next launch of the same kernel on the same SM, and what does a cold constant-bank
// (kernel parameter) read cost?  148 CTAs (one per SM), each times a ~21 KB straight-line FFMA
// block (pass 1), then the same block again (pass 2, warm), and a read of a far kernel-parameter
// word.  Printed per launch: median cycles over SMs.
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

struct Big { float pad[1000]; };   // 4 KB of kernel parameters: the last word sits far away

template <int N>
__device__ __forceinline__ void block(float& c0, float& c1, float& c2, float& c3, float a, float b) {
#pragma unroll
  for (int i = 0; i < N; i += 4) {
    c0 = fmaf(a, b, c0); c1 = fmaf(a, b + 1, c1); c2 = fmaf(a, b + 2, c2); c3 = fmaf(a, b + 3, c3);
    a += 1e-7f;
  }
}

__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c) :: "memory");
  return c;
}
__device__ __forceinline__ void pin(float& x) { asm volatile("mov.b32 %0, %0;" : "+f"(x)); }

__global__ void k(float* out, long long* t, const __grid_constant__ Big big) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  float a = threadIdx.x, b = 1.0001f, c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
  long long t0 = clk();
  pin(a);
  block<1024>(c0, c1, c2, c3, a, b);
  pin(c0); pin(c1); pin(c2); pin(c3);
  long long t1 = clk();
  pin(a);
  block<1024>(c0, c1, c2, c3, a, b);      // identical instructions at other addresses: still cold
  pin(c0); pin(c1); pin(c2); pin(c3);
  long long t1b = clk();
  // dependent FMULs with constant-bank operands (SASS c[0x0][...]): the first touches a cold line
  float x = c0;
  pin(x);
  x = x * big.pad[999];
  pin(x);
  long long t2 = clk();
  x = x * big.pad[998];                                                 // same line: warm
  pin(x);
  long long t3 = clk();
  float far = x, near = 0.f;
  c0 += far + near;
  if (threadIdx.x == 0) {
    t[smid * 4 + 0] = t1 - t0;
    t[smid * 4 + 1] = t2 - t1b;
    t[smid * 4 + 2] = t3 - t2;
    t[smid * 4 + 3] = t1b - t1;
  }
  out[blockIdx.x * 32 + threadIdx.x] = c0 + c1 + c2 + c3;
}

// the same straight-line block in a 2-iteration loop: iteration 0 cold, iteration 1 warm
__global__ void kloop(float* out, long long* t) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  float a = threadIdx.x, b = 1.0001f, c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
  long long tt[3];
  tt[0] = clk();
#pragma unroll 1
  for (int rep = 0; rep < 2; ++rep) {
    pin(a);
    block<1024>(c0, c1, c2, c3, a, b);
    pin(c0); pin(c1); pin(c2); pin(c3);
    tt[rep + 1] = clk();
  }
  if (threadIdx.x == 0) { t[smid * 4 + 0] = tt[1] - tt[0]; t[smid * 4 + 1] = tt[2] - tt[1]; }
  out[blockIdx.x * 32 + threadIdx.x] = c0 + c1 + c2 + c3;
}

static long long med(std::vector<long long> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; }

int main() {
  float* out; long long* t;
  cudaMalloc(&out, 148 * 32 * 4);
  cudaMallocManaged(&t, 256 * 4 * 8);
  Big big; for (int i = 0; i < 1000; ++i) big.pad[i] = 0.f;
  for (int launch = 0; launch < 4; ++launch) {
    cudaMemset(t, 0, 256 * 4 * 8);
    k<<<148, 32>>>(out, t, big);
    cudaDeviceSynchronize();
    std::vector<long long> code, code2, farc, nearc;
    for (int s = 0; s < 256; ++s) if (t[s * 4]) { code.push_back(t[s * 4]); farc.push_back(t[s * 4 + 1]); nearc.push_back(t[s * 4 + 2]); code2.push_back(t[s * 4 + 3]); }
    printf("launch %d: %zu SMs, straight-line 1024 FFMA block A %lld cyc, block B %lld cyc, far param read %lld cyc, near %lld cyc\n",
           launch, code.size(), med(code), med(code2), med(farc), med(nearc));
  }
  // back to back without a host sync in between
  for (int launch = 0; launch < 3; ++launch) k<<<148, 32>>>(out, t, big);
  cudaDeviceSynchronize();
  std::vector<long long> code;
  for (int s = 0; s < 256; ++s) if (t[s * 4]) code.push_back(t[s * 4]);
  printf("back-to-back 3rd launch: straight-line %lld cyc\n", med(code));
  for (int launch = 0; launch < 3; ++launch) {
    cudaMemset(t, 0, 256 * 4 * 8);
    kloop<<<148, 32>>>(out, t);
    cudaDeviceSynchronize();
    std::vector<long long> c1, c2;
    for (int s = 0; s < 256; ++s) if (t[s * 4]) { c1.push_back(t[s * 4]); c2.push_back(t[s * 4 + 1]); }
    printf("loop launch %d: iteration 0 (cold) %lld cyc, iteration 1 (warm) %lld cyc\n", launch, med(c1), med(c2));
  }
  return 0;
}
