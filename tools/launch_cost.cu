// Host cost of a cooperative vs a regular launch (one block per SM, empty
// body with one grid-wide atomic), and GPU back-to-back rate.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_empty(unsigned* c) { if (threadIdx.x == 0) atomicAdd(c, 1u); }
int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  unsigned* c;
  cudaMalloc(&c, 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  void* args[] = {&c};
  for (int coop = 0; coop < 2; ++coop) {
    for (int it = 0; it < 2; ++it) {
      cudaStreamSynchronize(s);
      auto t0 = std::chrono::steady_clock::now();
      const int n = 2000;
      for (int i = 0; i < n; ++i) {
        if (coop) cudaLaunchCooperativeKernel((void*)k_empty, p.multiProcessorCount, 256, args, 0, s);
        else k_empty<<<p.multiProcessorCount, 256, 0, s>>>(c);
      }
      auto t1 = std::chrono::steady_clock::now();
      cudaStreamSynchronize(s);
      auto t2 = std::chrono::steady_clock::now();
      if (it) printf("%s: host %.2f us/launch, total %.2f us/launch\n", coop ? "cooperative" : "regular",
                     std::chrono::duration<double, std::micro>(t1 - t0).count() / n,
                     std::chrono::duration<double, std::micro>(t2 - t0).count() / n);
    }
  }
  return 0;
}
