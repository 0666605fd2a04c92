// Repeatability of the host stack-gather staging pattern (32 atoms x 121 x 8000).
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
  const int na = 32, nl = 121, ng = 8000;
  std::vector<double*> blocks(na);
  for (auto& b : blocks) { b = (double*)malloc(size_t(nl) * ng * 16); memset(b, 1, size_t(nl) * ng * 16); }
  const size_t col = size_t(na) * nl * 16, piece = size_t(nl) * 16, S = 32 << 20;
  const int per = S / col;
  char* slot[4]; cudaEvent_t ev[4];
  for (int i = 0; i < 4; ++i) { cudaMallocHost((void**)&slot[i], S); cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming); }
  char* dev; cudaMalloc(&dev, col * ng);
  cudaStream_t st; cudaStreamCreate(&st);
  for (int nt : {4, 8, 12, 16}) for (int sched = 0; sched < 2; ++sched) {
    double best = 1e9, worst = 0;
    for (int rep = 0; rep < 5; ++rep) {
      auto t0 = clk::now();
      int used = 0, s = 0;
      for (int g0 = 0; g0 < ng; g0 += per) {
        int nc = std::min(per, ng - g0);
        if (used >= 4) cudaEventSynchronize(ev[s]);
        if (sched == 0) {
#pragma omp parallel for num_threads(nt) schedule(static)
          for (long idx = 0; idx < long(nc) * na; ++idx) {
            long g = idx / na, a = idx % na;
            memcpy(slot[s] + g * col + a * piece, blocks[a] + 2 * (g0 + g) * nl, piece);
          }
        } else {
#pragma omp parallel for num_threads(nt) schedule(dynamic, 64)
          for (long idx = 0; idx < long(nc) * na; ++idx) {
            long g = idx / na, a = idx % na;
            memcpy(slot[s] + g * col + a * piece, blocks[a] + 2 * (g0 + g) * nl, piece);
          }
        }
        cudaMemcpyAsync(dev + g0 * col, slot[s], nc * col, cudaMemcpyHostToDevice, st);
        cudaEventRecord(ev[s], st);
        s = (s + 1) % 4; ++used;
      }
      cudaStreamSynchronize(st);
      double t = ms(t0, clk::now());
      best = std::min(best, t); worst = std::max(worst, t);
    }
    printf("threads=%2d sched=%s  best %.1f ms  worst %.1f ms  (%.1f GB/s best)\n", nt, sched ? "dyn" : "static", best, worst, col * ng / best / 1e6);
  }
  // DMA only
  for (int rep = 0; rep < 3; ++rep) {
    auto t0 = clk::now();
    for (int g0 = 0, s = 0; g0 < ng; g0 += per, s = (s + 1) % 4) cudaMemcpyAsync(dev + g0 * col, slot[s], std::min(per, ng - g0) * col, cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);
    printf("dma only %.1f ms\n", ms(t0, clk::now()));
  }
}
