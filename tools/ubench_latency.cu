// Microbenchmarks of the latencies that bound the sweep's per-item pipeline
// (dependent DFMA, L2-hit load, ld.acquire.gpu, st.release.gpu, bar.sync).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, double a, double b, int n, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_chase(const unsigned* next, int n, long long* cyc, unsigned* sink) {
  unsigned p = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = __ldcg(next + p);
  long long t1 = clock64();
  *sink = p;
  *cyc = t1 - t0;
}
__global__ void k_acq(unsigned* next, int n, long long* cyc, unsigned* sink) {
  unsigned p = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(p) : "l"(next + p) : "memory");
  long long t1 = clock64();
  *sink = p;
  *cyc = t1 - t0;
}
__global__ void k_rel(unsigned* flags, int n, long long* cyc) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    flags[1024 + i] = i;  // a prior plain store to order
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + i), "r"(i) : "memory");
  }
  long long t1 = clock64();
  *cyc = t1 - t0;
}
__global__ void k_fence(unsigned* flags, int n, long long* cyc) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    flags[1024 + i] = i;
    __threadfence();
    flags[i] = i;
  }
  long long t1 = clock64();
  *cyc = t1 - t0;
}
__global__ void k_bar(int n, long long* cyc) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* d;
  long long* c;
  unsigned *nx, *sink, *flags;
  cudaMalloc(&d, 1024 * 8);
  cudaMalloc(&c, 8);
  cudaMalloc(&sink, 4);
  cudaMalloc(&flags, 1 << 20);
  const int N = 1 << 16;
  unsigned* h = new unsigned[N];
  for (int i = 0; i < N; ++i) h[i] = (i * 4099 + 77) % N;  // pseudo-random cycle-ish chase
  cudaMalloc(&nx, N * 4);
  cudaMemcpy(nx, h, N * 4, cudaMemcpyHostToDevice);
  long long cyc;
  auto rep = [&](const char* name, int n) {
    cudaDeviceSynchronize();
    cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %8.1f cycles/op\n", name, double(cyc) / n);
  };
  k_dfma<<<1, 1>>>(d, 1.0000001, 1e-9, 4096, c); k_dfma<<<1, 1>>>(d, 1.0000001, 1e-9, 4096, c); rep("dfma dependent (1 thread)", 4096);
  k_dfma<<<1, 256>>>(d, 1.0000001, 1e-9, 4096, c); rep("dfma dependent (256 thr)", 4096);
  k_chase<<<1, 1>>>(nx, 2000, c, sink); k_chase<<<1, 1>>>(nx, 2000, c, sink); rep("ld.cg L2-hit chase", 2000);
  k_acq<<<1, 1>>>(nx, 2000, c, sink); rep("ld.acquire.gpu chase", 2000);
  k_rel<<<1, 1>>>(flags, 2000, c); k_rel<<<1, 1>>>(flags, 2000, c); rep("st + st.release.gpu", 2000);
  k_fence<<<1, 1>>>(flags, 2000, c); rep("st + threadfence + st", 2000);
  k_bar<<<1, 320>>>(2000, c); rep("bar.sync (320 thr)", 2000);
  return 0;
}
