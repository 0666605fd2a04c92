// ptx.cuh — inline-PTX helpers shared by the DMMA kernels (mbarrier, TMA,
// DMMA.8x8x4) and the lower-triangle tile decoder.
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace hsb {

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ double flip_sign(double x, unsigned long long mask) {
  return __longlong_as_double(__double_as_longlong(x) ^ mask);
}

// Decode blockIdx into (tile row, tile col) for the lower-triangle schedule,
// column-major: column block j holds tiles (j..T-1, j).  With the mirrored
// epilogue, column block c of the output is final once tile columns 0..c
// are done, so completed columns stream out in order (done_cnt).
__device__ __forceinline__ void tri_tile(int t, int T, int& bi, int& bj) {
  // tiles before column j: S(j) = j*T - j*(j-1)/2
  const double b = 2.0 * T + 1.0;
  int j = static_cast<int>((b - sqrt(b * b - 8.0 * t)) * 0.5);
  if (j < 0) j = 0;
  while (j > 0 && j * T - (j * (j - 1)) / 2 > t) --j;
  while ((j + 1) * T - ((j + 1) * j) / 2 <= t) ++j;
  bj = j;
  bi = j + (t - (j * T - (j * (j - 1)) / 2));
}

}  // namespace hsb
