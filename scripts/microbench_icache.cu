// Development microbenchmark: cost of executing cold straight-line code on B200.
// One CTA runs an unrolled block of N independent FFMAs twice (cold pass, warm pass) and records clock64.
#include <cstdio>
#include <cuda_runtime.h>
template <int N, int U>
__global__ void k(float* out, long long* t) {
  float a = threadIdx.x, b = 1.0001f, c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
  long long t0 = clock64();
#pragma unroll 1
  for (int rep = 0; rep < 2; ++rep) {
#pragma unroll U
    for (int i = 0; i < N; i += 4) {
      c0 = fmaf(a, b, c0); c1 = fmaf(a, b + 1, c1); c2 = fmaf(a, b + 2, c2); c3 = fmaf(a, b + 3, c3);
      a += 1e-7f;
    }
    if (rep == 0) t[1] = clock64() - t0;
  }
  t[0] = clock64() - t0;
  out[threadIdx.x] = c0 + c1 + c2 + c3;
}
int main() {
  float* out; long long* t; cudaMalloc(&out, 4096); cudaMallocManaged(&t, 64);
  k<1024, 256><<<1, 32>>>(out, t); cudaDeviceSynchronize();
  k<1024, 256><<<1, 32>>>(out, t); cudaDeviceSynchronize();
  printf("N=1024 fully unrolled (~21 KB): pass1 %lld cyc, pass2 %lld cyc\n", t[1], t[0] - t[1]);
  k<1024, 16><<<1, 32>>>(out, t); cudaDeviceSynchronize();
  k<1024, 16><<<1, 32>>>(out, t); cudaDeviceSynchronize();
  printf("N=1024 unroll 16 (~1.3 KB body): pass1 %lld cyc, pass2 %lld cyc\n", t[1], t[0] - t[1]);
  k<1024, 4><<<1, 32>>>(out, t); cudaDeviceSynchronize();
  k<1024, 4><<<1, 32>>>(out, t); cudaDeviceSynchronize();
  printf("N=1024 unroll 4: pass1 %lld cyc, pass2 %lld cyc\n", t[1], t[0] - t[1]);
  k<1024, 64><<<1, 32>>>(out, t); cudaDeviceSynchronize();
  k<1024, 64><<<1, 32>>>(out, t); cudaDeviceSynchronize();
  printf("N=1024 unroll 64 (~5 KB body): pass1 %lld cyc, pass2 %lld cyc\n", t[1], t[0] - t[1]);
  return 0;
}
