// Device -> host bandwidth of the box's link for a 9.9 MB result (the C3
// primal point): kernel stores into mapped pinned memory (zero-copy; 8- and
// 16-byte stores, one CTA per SM) against cudaMemcpyAsync from device memory
// (copy engine), and both together split in halves.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/ubench_pcie.cu -o /tmp/ubench_pcie
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_write16(double2* __restrict__ dst, const double2* __restrict__ src, size_t n2) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += size_t(gridDim.x) * blockDim.x) dst[i] = src[i];
}
__global__ void k_write8(double* __restrict__ dst, const double* __restrict__ src, size_t n) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) dst[i] = src[i];
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const size_t n = 1238980;  // doubles (C3 x and u)
  const size_t bytes = n * sizeof(double);
  double *h, *hd, *d;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  cudaHostGetDevicePointer(&hd, h, 0);
  cudaMalloc(&d, bytes);
  cudaMemset(d, 0, bytes);
  cudaStream_t s, s2;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto&& f) {
    for (int i = 0; i < 3; ++i) f();
    cudaStreamSynchronize(s);
    const int reps = 20;
    cudaEventRecord(a, s);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::printf("%-34s %7.1f us  %6.1f GB/s\n", name, 1e3 * ms / reps, bytes / (1e6 * ms / reps));
  };
  for (int threads : {256, 512, 1024})
    for (int blocks : {p.multiProcessorCount, 2 * p.multiProcessorCount}) {
      char nm[64];
      std::snprintf(nm, sizeof nm, "zero-copy 16B, %d x %d", blocks, threads);
      run(nm, [&] { k_write16<<<blocks, threads, 0, s>>>(reinterpret_cast<double2*>(hd), reinterpret_cast<double2*>(d), n / 2); });
    }
  run("zero-copy 8B, 148 x 512", [&] { k_write8<<<p.multiProcessorCount, 512, 0, s>>>(hd, d, n); });
  run("cudaMemcpyAsync D2H", [&] { cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s); });
  run("2 x cudaMemcpyAsync halves", [&] {
    cudaMemcpyAsync(h, d, bytes / 2, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(h + n / 2, d + n / 2, bytes - bytes / 2, cudaMemcpyDeviceToHost, s);
  });
  run("H2D cudaMemcpyAsync", [&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s); });
  return 0;
}
