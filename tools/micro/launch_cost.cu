// Launch-overhead microbenchmark: empty kernels with small vs 6 KB
// __grid_constant__ parameter blocks, and the per-call runtime calls the
// C-ABI makes (cudaGetDeviceCount / cudaSetDevice / cudaMemsetAsync).
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
struct Small { unsigned v[16]; };
struct Big { unsigned v[1560]; };
__global__ void k_small(const __grid_constant__ Small p, unsigned *o) { if (threadIdx.x == 0 && p.v[0] == 7) *o = 1; }
__global__ void k_big(const __grid_constant__ Big p, unsigned *o) { if (threadIdx.x == 0 && p.v[0] == 7) *o = 1; }
template <class F> double per_call_us(F f, int n) {
  for (int i = 0; i < 20; ++i) f();
  cudaDeviceSynchronize();
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) f();
  cudaDeviceSynchronize();
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / n;
}
int main() {
  unsigned *o; cudaMalloc(&o, 64);
  Small s{}; Big b{};
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  printf("small param launch: %.2f us\n", per_call_us([&] { k_small<<<8, 128, 0, st>>>(s, o); }, 2000));
  printf("6 KB param launch:  %.2f us\n", per_call_us([&] { k_big<<<8, 128, 0, st>>>(b, o); }, 2000));
  printf("memsetAsync 4B:     %.2f us\n", per_call_us([&] { cudaMemsetAsync(o, 0, 4, st); }, 2000));
  printf("getDeviceCount+set: %.2f us\n", per_call_us([&] { int n; cudaGetDeviceCount(&n); cudaSetDevice(0); }, 2000));
  printf("launch+sync small:  %.2f us\n", per_call_us([&] { k_small<<<8, 128, 0, st>>>(s, o); cudaStreamSynchronize(st); }, 2000));
  printf("launch+sync big:    %.2f us\n", per_call_us([&] { k_big<<<8, 128, 0, st>>>(b, o); cudaStreamSynchronize(st); }, 2000));
  return 0;
}
