// Host-side launch, copy and round-trip costs on one B200 (the floor under a
// small query):  nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a
//   tools/launch_cost.cu -o /tmp/launch_cost && /tmp/launch_cost
#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>
template <int N> struct P { char b[N]; };
template <int N> __global__ void k(const __grid_constant__ P<N> p, int* out) { if (threadIdx.x == 0 && blockIdx.x == 0 && p.b[0] == 7) *out = 1; }
template <int N> double cost(cudaStream_t s, int* d) {
  P<N> p{}; 
  for (int i = 0; i < 100; ++i) k<N><<<148, 256, 0, s>>>(p, d);
  cudaStreamSynchronize(s);
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < 1000; ++i) k<N><<<148, 256, 0, s>>>(p, d);
  auto t1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(s);
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / 1000;
}
int main() {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int* d; cudaMalloc(&d, 4096);
  unsigned long long* h; cudaMallocHost(&h, 4096);
  printf("launch host cost us: 64B %.2f  1KB %.2f  4KB %.2f  6KB %.2f  12KB %.2f\n", cost<64>(s, d), cost<1024>(s, d), cost<4096>(s, d), cost<6144>(s, d), cost<12288>(s,d));
  // H2D small pinned, D2H small pinned, event record
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < 1000; ++i) cudaMemcpyAsync(d, h, 192, cudaMemcpyHostToDevice, s);
  auto t1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(s);
  cudaEvent_t e; cudaEventCreate(&e);
  auto t2 = std::chrono::steady_clock::now();
  for (int i = 0; i < 1000; ++i) cudaEventRecord(e, s);
  auto t3 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(s);
  auto t4 = std::chrono::steady_clock::now();
  for (int i = 0; i < 1000; ++i) cudaMemsetAsync(d, 0, 64, s);
  auto t5 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(s);
  // round trip: launch tiny kernel + D2H + poll
  double rt = 0;
  for (int i = 0; i < 1000; ++i) {
    auto a = std::chrono::steady_clock::now();
    k<64><<<148, 256, 0, s>>>(P<64>{}, d);
    cudaMemcpyAsync(h, d, 64, cudaMemcpyDeviceToHost, s);
    while (cudaStreamQuery(s) == cudaErrorNotReady) {}
    rt += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - a).count();
  }
  double rt2 = 0;
  for (int i = 0; i < 1000; ++i) {
    auto a = std::chrono::steady_clock::now();
    k<64><<<148, 256, 0, s>>>(P<64>{}, d);
    cudaMemcpyAsync(h, d, 64, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    rt2 += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - a).count();
  }
  printf("H2D 192B %.2f us, event %.2f us, memset %.2f us, roundtrip poll %.2f us, roundtrip sync %.2f us\n",
    std::chrono::duration<double, std::micro>(t1 - t0).count() / 1000, std::chrono::duration<double, std::micro>(t3 - t2).count() / 1000,
    std::chrono::duration<double, std::micro>(t5 - t4).count() / 1000, rt / 1000, rt2 / 1000);
}
