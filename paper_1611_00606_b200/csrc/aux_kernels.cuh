// aux_kernels.cuh — launchers for the small / memory-bound kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>

#include "zrk.cuh"

namespace hsb {

// Per-device one-time setup (constant uploads, kernel attributes): both are
// per device, so a process driving several GPUs must run it on each.
struct PerDeviceOnce {
  static constexpr int kMaxDev = 64;
  std::mutex mu;
  std::atomic<bool> done[kMaxDev] = {};
  cudaError_t status[kMaxDev] = {};
};
template <class F>
cudaError_t per_device_once(PerDeviceOnce& o, F&& fn) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= PerDeviceOnce::kMaxDev) return cudaErrorInvalidDevice;
  if (o.done[dev].load(std::memory_order_acquire)) return o.status[dev];
  std::lock_guard<std::mutex> g(o.mu);
  if (!o.done[dev].load(std::memory_order_relaxed)) {
    o.status[dev] = fn();
    o.done[dev].store(true, std::memory_order_release);
  }
  return o.status[dev];
}

constexpr size_t kPotrfSmemMax = 200 * 1024;  // packed lower triangle up to n = 158

cudaError_t launch_zrk(const ZrkParams& p, bool conj, int grid_x, int grid_z, cudaStream_t st);
// 3M (Gauss) variant, persistent: ntiles tiles per batch x nbatch batches
cudaError_t launch_zrk3m(const ZrkParams& p, bool conj, int pmode, int ntiles, int nbatch, cudaStream_t st);
// per-atom planes of count n x n column-major complex blocks (atom stride bstride
// complex): out[(b * n + c) * kp + k] = Re x -/+ Im x (minus: Re - Im), zero for
// k in [n, kp)
cudaError_t launch_sum_planes_batched(const double* x, int n, int64_t bstride, int64_t count, bool minus,
                                     double* out, int kp, cudaStream_t st);
cudaError_t launch_potrf_route(const double* t_aa, double* q, int32_t* info, int n_atoms, int n,
                               bool force_nonhpd, double* gscratch, cudaStream_t st);
cudaError_t launch_half_mirror(const double* t, double* out, int n, int64_t count, double scale,
                               cudaStream_t st);
// out_a = T_a^H for count consecutive n x n complex matrices
cudaError_t launch_conj_transpose(const double* t, double* out, int n, int64_t count, cudaStream_t st);
// out_a = t_a diag(1 / u_a) for per-atom n x n blocks (u: count * n entries)
cudaError_t launch_scale_cols_inv(const double* t, double* out, const double* u, int n, int64_t count,
                                  cudaStream_t st);
cudaError_t launch_diag_scale(const double* src, int64_t lds, double* dst, int64_t ldd, const double* u,
                              int64_t rows, int64_t cols, cudaStream_t st);
cudaError_t launch_mirror(double* c, int64_t ldc, int n, cudaStream_t st);
// out[i] = sum over n_slots slots (stride complex elements apart) of slot[i], complex
cudaError_t launch_sum_slots(const double* slots, int n_slots, int64_t stride, int64_t count, double* out,
                             cudaStream_t st);
cudaError_t launch_fill_i32(int32_t* p, int64_t n, int32_t v, cudaStream_t st);
// device-side Loop 2 routing (offsets of R / gather lists) + info export to mapped host memory
cudaError_t launch_route_atoms(const int32_t* info, int na, int nl, int32_t* offs, int32_t* info_host,
                               cudaStream_t st);
// small int32 copies by a kernel (e.g. into mapped host memory: no copy-engine queue)
cudaError_t launch_copy_i32(const int32_t* src, int32_t* dst, int n, cudaStream_t st);
cudaError_t launch_sum_planes(const double* x, int64_t ldx, int64_t rows, int64_t cols, double* minus,
                              double* plus, int64_t ldp, cudaStream_t st);
cudaError_t launch_gather_rows(const double* src, int64_t lds, double* dst, int64_t ldd, const int32_t* src_off,
                               const int32_t* dst_off, int n_blocks, int n_l, int64_t cols, cudaStream_t st);
cudaError_t launch_stack_blocks(const double* raw, double* dst, int n_atoms, int rows, int64_t cols,
                                cudaStream_t st);
cudaError_t launch_first_nonfinite(const double* v, int n_blocks, int64_t doubles_per_block, int* flag,
                                   cudaStream_t st);
cudaError_t launch_transpose(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int64_t cols,
                             bool conj, cudaStream_t st);

}  // namespace hsb
