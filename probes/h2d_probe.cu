// Host->device transfer options for pageable numpy-like sources (1 GiB).
#include <cuda_runtime.h>
#include <omp.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <vector>
using clk = std::chrono::steady_clock;
static double ms(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }
int main() {
  const size_t N = size_t(1) << 30;
  char* src = (char*)aligned_alloc(4096, N);
  memset(src, 1, N);  // touch
  char* dev; cudaMalloc(&dev, N);
  char* pin; cudaMallocHost(&pin, N);
  cudaStream_t st; cudaStreamCreate(&st);
  for (int nt : {1, 2, 4, 8, 16}) {
    auto t0 = clk::now();
#pragma omp parallel for num_threads(nt)
    for (int i = 0; i < 64; ++i) memcpy(pin + i * (N / 64), src + i * (N / 64), N / 64);
    auto t1 = clk::now();
    printf("memcpy threads=%2d : %.1f GB/s\n", nt, N / ms(t0, t1) / 1e6);
  }
  for (int rep = 0; rep < 2; ++rep) {
    auto t0 = clk::now();
    cudaMemcpyAsync(dev, src, N, cudaMemcpyHostToDevice, st); cudaStreamSynchronize(st);
    auto t1 = clk::now();
    printf("pageable cudaMemcpyAsync: %.1f GB/s\n", N / ms(t0, t1) / 1e6);
  }
  for (int rep = 0; rep < 2; ++rep) {
    auto t0 = clk::now();
    cudaError_t e = cudaHostRegister(src, N, cudaHostRegisterDefault);
    auto t1 = clk::now();
    cudaMemcpyAsync(dev, src, N, cudaMemcpyHostToDevice, st); cudaStreamSynchronize(st);
    auto t2 = clk::now();
    cudaHostUnregister(src);
    auto t3 = clk::now();
    printf("register %.1f ms (%s), dma %.1f ms, unregister %.1f ms\n", ms(t0, t1), cudaGetErrorString(e), ms(t1, t2), ms(t2, t3));
  }
  // chunked register of 16 MB pieces (per-atom block size)
  {
    auto t0 = clk::now();
    for (size_t off = 0; off < N; off += (16 << 20)) cudaHostRegister(src + off, 16 << 20, 0);
    auto t1 = clk::now();
    for (size_t off = 0; off < N; off += (16 << 20)) cudaHostUnregister(src + off);
    auto t2 = clk::now();
    printf("register 64x16MB %.1f ms, unregister %.1f ms\n", ms(t0, t1), ms(t1, t2));
  }
  // staged pipeline: 4 slots x 32 MB, 8 threads
  {
    const size_t S = 32 << 20; cudaEvent_t ev[4]; for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    for (int nt : {4, 8, 16}) {
      auto t0 = clk::now();
      for (size_t c = 0, k = 0; c < N; c += S, ++k) {
        int s = k % 4; if (k >= 4) cudaEventSynchronize(ev[s]);
#pragma omp parallel for num_threads(nt)
        for (int i = 0; i < nt; ++i) memcpy(pin + s * S + i * (S / nt), src + c + i * (S / nt), S / nt);
        cudaMemcpyAsync(dev + c, pin + s * S, S, cudaMemcpyHostToDevice, st); cudaEventRecord(ev[s], st);
      }
      cudaStreamSynchronize(st);
      printf("staged 32MB slots threads=%d: %.1f GB/s\n", nt, N / ms(t0, clk::now()) / 1e6);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
