// Latency of reading a 2 KB scalar block back to the host after a kernel:
// D2H memcpy to pinned memory vs a kernel writing mapped pinned memory,
// measured as back-to-back stream time and as host round trips.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_work(double* S) { if (threadIdx.x == 0 && blockIdx.x == 0) S[0] += 1.0; }
__global__ void k_pub(const double* S, double* h, int n) {
  for (int t = threadIdx.x; t < n; t += blockDim.x) h[t] = S[t];
}
__global__ void k_pub_v(const double2* S, double2* h, int n2) {
  for (int t = threadIdx.x; t < n2; t += blockDim.x) h[t] = S[t];
}
int main() {
  const int n = 256;  // 2 KB
  double *S, *hp, *hm, *dm;
  cudaMalloc(&S, n * 8);
  cudaMemset(S, 0, n * 8);
  cudaMallocHost(&hp, n * 8);
  cudaHostAlloc(&hm, n * 8, cudaHostAllocMapped);
  cudaHostGetDevicePointer((void**)&dm, hm, 0);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 4; ++mode) {
    const char* name[] = {"work only", "work + D2H memcpy", "work + mapped pub (scalar)", "work + mapped pub (double2)"};
    for (int rep = 0; rep < 2; ++rep) {
      const int it = 200;
      cudaStreamSynchronize(s);
      cudaEventRecord(a, s);
      for (int i = 0; i < it; ++i) {
        k_work<<<148, 256, 0, s>>>(S);
        if (mode == 1) cudaMemcpyAsync(hp, S, n * 8, cudaMemcpyDeviceToHost, s);
        if (mode == 2) k_pub<<<1, 256, 0, s>>>(S, dm, n);
        if (mode == 3) k_pub_v<<<1, 128, 0, s>>>((const double2*)S, (double2*)dm, n / 2);
      }
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      // host round trip: enqueue, wait, per iteration
      auto t0 = std::chrono::steady_clock::now();
      for (int i = 0; i < it; ++i) {
        k_work<<<148, 256, 0, s>>>(S);
        if (mode == 1) cudaMemcpyAsync(hp, S, n * 8, cudaMemcpyDeviceToHost, s);
        if (mode == 2) k_pub<<<1, 256, 0, s>>>(S, dm, n);
        if (mode == 3) k_pub_v<<<1, 128, 0, s>>>((const double2*)S, (double2*)dm, n / 2);
        cudaStreamSynchronize(s);
      }
      auto t1 = std::chrono::steady_clock::now();
      if (rep)
        printf("%-30s stream %.2f us/iter, host round trip %.2f us/iter\n", name[mode], 1e3 * ms / it,
               std::chrono::duration<double, std::micro>(t1 - t0).count() / it);
    }
  }
  return 0;
}
