// Host memory bandwidth vs PCIe DMA: is the pinned-host e2e path bound by the
// host's DRAM rather than by PCIe?  Measures (1) host copy / NT-store fill
// bandwidth on all threads, (2) H2D + D2H duplex DMA alone, (3) the duplex DMA
// while the host threads run a Hermitian mirror (the k-point lanes' host work).
//   nvcc -O3 -Xcompiler -fopenmp -Xcompiler -march=native probes/host_contention.cu -o /tmp/hc && /tmp/hc
#include <cuda_runtime.h>
#include <emmintrin.h>
#include <omp.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// conj-transpose the strict lower triangle of an n x n complex128 matrix into
// the upper one in 64 x 64 tiles, non-temporal stores (as hsb_api.cu HostMirror)
static void mirror(double* m, long n, int threads) {
  const long tb = 64, nt = (n + tb - 1) / tb;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
  for (long t = 0; t < nt * nt; ++t) {
    const long I = t / nt, J = t % nt;
    if (J <= I) continue;
    for (long c = J * tb; c < std::min(n, J * tb + tb); ++c)
      for (long r = I * tb; r < std::min(c, I * tb + tb); ++r)
        _mm_stream_pd(m + 2 * (r + c * n),
                      _mm_xor_pd(_mm_load_pd(m + 2 * (c + r * n)), _mm_set_pd(-0.0, 0.0)));
  }
  _mm_sfence();
}

int main() {
  const size_t G = size_t(1) << 30;
  const int T = omp_get_max_threads();
  char *h_src, *h_dst, *d_a, *d_b;
  cudaHostAlloc(&h_src, G, cudaHostAllocDefault);
  cudaHostAlloc(&h_dst, G, cudaHostAllocDefault);
  cudaMalloc(&d_a, G);
  cudaMalloc(&d_b, G);
  memset(h_src, 1, G);
  memset(h_dst, 1, G);
  const long n = 8000;
  double* mat;
  cudaHostAlloc(&mat, n * n * 16, cudaHostAllocDefault);
  memset(mat, 0, n * n * 16);
  cudaStream_t s1, s2;
  cudaStreamCreate(&s1);
  cudaStreamCreate(&s2);

  // (1) host copy bandwidth (read + write counted)
  for (int rep = 0; rep < 3; ++rep) {
    double t0 = now();
#pragma omp parallel for num_threads(T)
    for (long i = 0; i < 1024; ++i) memcpy(h_dst + i * (G / 1024), h_src + i * (G / 1024), G / 1024);
    double t = now() - t0;
    printf("host memcpy %d threads: %.1f GB/s (read+write)\n", T, 2.0 * G / t / 1e9);
  }
  for (int rep = 0; rep < 2; ++rep) {
    double t0 = now();
    mirror(mat, n, T);
    double t = now() - t0;
    printf("host mirror 8000^2, %d threads: %.1f ms (%.1f GB/s read+write)\n", T, t * 1e3,
           2.0 * 8 * n * n / t / 1e9);
  }
  // (2) duplex DMA alone
  auto duplex = [&]() {
    cudaDeviceSynchronize();
    double t0 = now();
    cudaMemcpyAsync(d_a, h_src, G, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(h_dst, d_b, G, cudaMemcpyDeviceToHost, s2);
    cudaDeviceSynchronize();
    return now() - t0;
  };
  for (int rep = 0; rep < 3; ++rep) printf("duplex DMA alone: %.1f ms (%.1f GB/s)\n", duplex() * 1e3, 2.0 * G / duplex() / 1e9);
  // (2b) the pipeline's shapes: H2D as 64 DMAs of 16 MB, D2H as 2-D copies of
  // 256-column lower-triangle panels of an 8000^2 complex128 matrix
  auto shaped = [&](bool h2d, bool d2h, bool d2h_2d) {
    cudaDeviceSynchronize();
    double t0 = now();
    if (h2d)
      for (int i = 0; i < 64; ++i)
        cudaMemcpyAsync(d_a + i * (G / 64), h_src + i * (G / 64), G / 64, cudaMemcpyHostToDevice, s1);
    if (d2h)
      for (long a = 0; a < n; a += 256) {
        const long b = std::min(n, a + 256);
        if (d2h_2d)
          cudaMemcpy2DAsync(reinterpret_cast<char*>(mat) + (a * n + a) * 16, n * 16, d_b + (a * n + a) * 16, n * 16,
                            (n - a) * 16, b - a, cudaMemcpyDeviceToHost, s2);
        else
          for (long c = a; c < b; ++c)
            cudaMemcpyAsync(reinterpret_cast<char*>(mat) + (c * n + a) * 16, d_b + (c * n + a) * 16, (n - a) * 16,
                            cudaMemcpyDeviceToHost, s2);
      }
    cudaDeviceSynchronize();
    return now() - t0;
  };
  for (int rep = 0; rep < 2; ++rep) {
    printf("shaped H2D alone %.1f ms | lower-tri 2D D2H alone %.1f ms | both %.1f ms | both, 1-D D2H %.1f ms\n",
           shaped(true, false, true) * 1e3, shaped(false, true, true) * 1e3, shaped(true, true, true) * 1e3,
           shaped(true, true, false) * 1e3);
  }
  // (3) duplex DMA while host threads mirror continuously
  for (int th : {T, T / 2, 4}) {
    std::atomic<bool> stop{false};
    std::atomic<int> mirrors{0};
    std::thread bg([&] {
      while (!stop) {
        mirror(mat, n, th);
        ++mirrors;
      }
    });
    std::this_thread::sleep_for(std::chrono::milliseconds(50));
    double best = 1e9;
    for (int rep = 0; rep < 4; ++rep) best = std::min(best, duplex());
    const double t0 = now();
    const int m0 = mirrors;
    std::this_thread::sleep_for(std::chrono::milliseconds(300));
    const double mrate = (mirrors - m0) / (now() - t0);
    stop = true;
    bg.join();
    printf("duplex DMA with a %d-thread mirror running: %.1f ms (%.1f GB/s); mirrors %.1f/s\n", th, best * 1e3,
           2.0 * G / best / 1e9, mrate);
  }
  return 0;
}
