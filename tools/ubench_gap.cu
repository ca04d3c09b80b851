// Device-side gap between consecutive kernels of one stream: a small
// "dual-space" kernel (148 x 256 threads, static smem) followed by a
// "sweep-like" kernel (148 x 576 threads, ~200 KB dynamic smem), each spinning
// for a set time. Each kernel stamps %globaltimer at the first CTA's entry and
// the last CTA's exit; the gap is B.entry - A.exit. Variants: cooperative vs
// regular launches, carveout preference on the small kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/ubench_gap.cu -o /tmp/ubench_gap
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// stamps[0] = min entry, stamps[1] = max exit
__global__ void k_small(unsigned long long* st, unsigned ns) {
  __shared__ double red[8];
  const unsigned long long t0 = gt();
  if (threadIdx.x == 0) atomicMin(st, t0);
  while (gt() - t0 < ns) {
  }
  if (threadIdx.x < 8) red[threadIdx.x] = 0;
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(st + 1, gt());
}
__global__ void __launch_bounds__(576, 1) k_big(unsigned long long* st, unsigned ns) {
  extern __shared__ double sm[];
  const unsigned long long t0 = gt();
  if (threadIdx.x == 0) atomicMin(st, t0);
  sm[threadIdx.x] = 0;
  while (gt() - t0 < ns) {
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(st + 1, gt());
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int G = p.multiProcessorCount;
  const size_t big = 200 * 1024;
  cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(big));
  unsigned long long* st;
  cudaMalloc(&st, 64 * sizeof(unsigned long long));
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const unsigned long long init[2] = {~0ull, 0ull};
  for (int variant = 0; variant < 5; ++variant) {
    // 0: both cooperative; 1: both regular; 2: small regular, big cooperative;
    // 3: small cooperative, big regular; 4: as 0 with max-shared carveout on the small kernel
    if (variant == 4) cudaFuncSetAttribute(k_small, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    const bool cs = variant == 0 || variant == 3 || variant == 4, cb = variant == 0 || variant == 2 || variant == 4;
    double gap_ab = 0, gap_ba = 0;
    const int reps = 200;
    for (int r = 0; r < reps + 10; ++r) {
      for (int q = 0; q < 3; ++q) cudaMemcpyAsync(st + 2 * q, init, sizeof(init), cudaMemcpyHostToDevice, s);
      unsigned ns_small = 10000, ns_big = 100000;
      unsigned long long* a = st;
      unsigned long long* b = st + 2;
      unsigned long long* c = st + 4;
      void* aa[] = {&a, &ns_small};
      void* ab[] = {&b, &ns_big};
      void* ac[] = {&c, &ns_small};
      if (cs) cudaLaunchCooperativeKernel((void*)k_small, G, 256, aa, 0, s);
      else k_small<<<G, 256, 0, s>>>(a, ns_small);
      if (cb) cudaLaunchCooperativeKernel((void*)k_big, G, 576, ab, big, s);
      else k_big<<<G, 576, big, s>>>(b, ns_big);
      if (cs) cudaLaunchCooperativeKernel((void*)k_small, G, 256, ac, 0, s);
      else k_small<<<G, 256, 0, s>>>(c, ns_small);
      unsigned long long h[6];
      cudaMemcpyAsync(h, st, sizeof(h), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      if (r >= 10) {
        gap_ab += (h[2] - h[1]) * 1e-3;
        gap_ba += (h[4] - h[3]) * 1e-3;
      }
    }
    static const char* names[5] = {"coop/coop", "reg/reg", "reg small/coop big", "coop small/reg big",
                                   "coop/coop + carveout"};
    std::printf("%-24s small->big gap %.2f us, big->small gap %.2f us\n", names[variant], gap_ab / reps,
                gap_ba / reps);
  }
  return 0;
}
