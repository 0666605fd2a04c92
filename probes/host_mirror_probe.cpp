// Host-side Hermitian mirror throughput: fill the strict upper triangle of an
// n x n column-major complex128 matrix from its lower triangle (conjugate
// transpose), in square tiles, with OpenMP threads.  Decides whether H / S can
// cross PCIe as lower triangles only and be completed on the host.
//   g++ -O3 -march=native -fopenmp probes/host_mirror_probe.cpp -o /tmp/hm && /tmp/hm 8000
#include <emmintrin.h>
#include <omp.h>

#include <chrono>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

using cd = std::complex<double>;

static void mirror(cd* m, long n, int tb, int threads) {
  const long nt = (n + tb - 1) / tb;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
  for (long p = 0; p < nt * (nt + 1) / 2; ++p) {
    long J = 0, rem = p;  // tile (I, J), I >= J in a lower-triangular enumeration
    while (rem >= nt - J) rem -= nt - J++;
    const long I = J + rem;
    const long i0 = I * tb, j0 = J * tb;
    const long i1 = std::min(n, i0 + tb), j1 = std::min(n, j0 + tb);
    // upper tile (J, I): m[j + i * n] (j < i) = conj(m[i + j * n])
    for (long i = i0; i < i1; ++i)
      for (long j = j0; j < std::min(j1, i); ++j) m[j + i * n] = std::conj(m[i + j * n]);
  }
}

// same, with 16-byte non-temporal stores (no read-for-ownership of the
// destination lines)
static void mirror_nt(cd* m, long n, int tb, int threads) {
  const long nt = (n + tb - 1) / tb;
  const __m128d sign = _mm_set_pd(-0.0, 0.0);
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
  for (long p = 0; p < nt * (nt + 1) / 2; ++p) {
    long J = 0, rem = p;
    while (rem >= nt - J) rem -= nt - J++;
    const long I = J + rem;
    const long i0 = I * tb, j0 = J * tb;
    const long i1 = std::min(n, i0 + tb), j1 = std::min(n, j0 + tb);
    double* d = reinterpret_cast<double*>(m);
    for (long i = i0; i < i1; ++i)
      for (long j = j0; j < std::min(j1, i); ++j)
        _mm_stream_pd(d + 2 * (j + i * n), _mm_xor_pd(_mm_load_pd(d + 2 * (i + j * n)), sign));
    _mm_sfence();
  }
}

int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : 8000;
  std::printf("hardware threads %d\n", omp_get_max_threads());
  std::vector<cd> m(static_cast<size_t>(n) * n);
  for (size_t i = 0; i < m.size(); ++i) m[i] = cd(i * 1e-9, -1.0 * i);
  std::vector<cd> dst(m.size());
  auto t0 = std::chrono::steady_clock::now();
  std::memcpy(dst.data(), m.data(), m.size() * 16);
  double mc = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("memcpy 1 thread: %.1f GB/s\n", m.size() * 16 / mc / 1e9);
  for (int nt = 0; nt < 2; ++nt)
  for (int tb : {32, 64, 128})
    for (int th : {1, 4, 8, 16, 32, 64}) {
      if (th > omp_get_max_threads()) continue;
      auto f = nt ? mirror_nt : mirror;
      f(m.data(), n, tb, th);
      auto a = std::chrono::steady_clock::now();
      const int reps = 3;
      for (int r = 0; r < reps; ++r) f(m.data(), n, tb, th);
      double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count() / reps;
      std::printf("%s tile %3d threads %2d: %.2f ms per %ld^2 matrix (%.1f GB/s of read+write)\n", nt ? "stream" : "plain ", tb, th, s * 1e3,
                  n, static_cast<double>(n) * n * 16 / s / 1e9);
    }
  return 0;
}
