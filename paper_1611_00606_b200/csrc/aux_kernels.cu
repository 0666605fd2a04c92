// aux_kernels.cu — the memory-bound and per-atom small kernels around the
// DMMA contractions: batched Cholesky routing (Loop 2 potrf), T staging
// (Loop 1 1/2 T_BB), U-norm row scaling, Hermitian mirror, row gathers and
// operand transposes.  All are HBM- or latency-bound; none is GEMM-shaped.
#include <cuda_runtime.h>
#include <stdint.h>

#include "aux_kernels.cuh"

namespace hsb {

// --------------------------------------------------------------------------
// Batched lower Cholesky with failure-as-data (kernels.potrf_lower,
// kernels.py:296-325; routing in builder.build_phase2, builder.py:162-185).
// One CTA per atom.  The lower triangle of T_AA is factored right-looking in
// packed shared memory; on success Q = C (dense, zero strict upper), on
// failure Q = hermitian_mirror(T_AA) (the hemm operand, kernels.py:223-231)
// and info = 1-based order of the first non-positive leading minor.
// Subtraction order per element is ascending k, like the reference.
// --------------------------------------------------------------------------
__device__ __forceinline__ int pk(int n, int i, int j) {  // packed lower, column-major, i >= j
  return j * n - (j * (j - 1)) / 2 + (i - j);
}

__global__ void potrf_route_kernel(const double2* __restrict__ t_aa, double2* __restrict__ q,
                                   int32_t* __restrict__ info, int n, int force_nonhpd,
                                   double2* __restrict__ gscratch) {
  extern __shared__ double2 sm_pk[];
  const int a = blockIdx.x;
  const double2* T = t_aa + static_cast<int64_t>(a) * n * n;
  double2* Q = q + static_cast<int64_t>(a) * n * n;
  double2* L = gscratch ? gscratch + static_cast<int64_t>(a) * n * (n + 1) / 2 : sm_pk;
  __shared__ int s_info;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nwarps = nth >> 5;

  if (tid == 0) s_info = force_nonhpd ? -1 : 0;
  if (!force_nonhpd) {
    for (int j = 0; j < n; ++j)
      for (int i = j + tid; i < n; i += nth) L[pk(n, i, j)] = T[i + j * n];
  }
  __syncthreads();
  if (!force_nonhpd) {
    for (int j = 0; j < n; ++j) {
      const double d = L[pk(n, j, j)].x;
      if (!(d > 0.0)) {  // NaN or non-positive minor
        if (tid == 0) s_info = j + 1;
        break;
      }
      const double ljj = sqrt(d);
      __syncthreads();  // everyone has read d before it is overwritten
      if (tid == 0) L[pk(n, j, j)] = make_double2(ljj, 0.0);
      for (int i = j + 1 + tid; i < n; i += nth) {
        double2 v = L[pk(n, i, j)];
        L[pk(n, i, j)] = make_double2(v.x / ljj, v.y / ljj);
      }
      __syncthreads();
      // trailing update  L(r,c) -= L(r,j) * conj(L(c,j)),  j < c <= r
      for (int c = j + 1 + warp; c < n; c += nwarps) {
        const double2 lc = L[pk(n, c, j)];
        for (int r = c + lane; r < n; r += 32) {
          const double2 lr = L[pk(n, r, j)];
          double2 v = L[pk(n, r, c)];
          // lr * conj(lc)
          v.x -= lr.x * lc.x + lr.y * lc.y;
          v.y -= lr.y * lc.x - lr.x * lc.y;
          L[pk(n, r, c)] = v;
        }
      }
      __syncthreads();
    }
  }
  __syncthreads();
  const int inf = s_info;
  if (tid == 0) info[a] = inf;
  for (int idx = tid; idx < n * n; idx += nth) {
    const int i = idx % n, j = idx / n;
    double2 v;
    if (inf == 0) {
      v = (i >= j) ? L[pk(n, i, j)] : make_double2(0.0, 0.0);
    } else if (i > j) {
      v = T[i + j * n];
    } else if (i < j) {
      const double2 w = T[j + i * n];
      v = make_double2(w.x, -w.y);
    } else {
      v = make_double2(T[i + i * n].x, 0.0);
    }
    Q[idx] = v;
  }
}

// P[a] = scale * hermitian_mirror(T[a])   (Loop 1: 1/2 T_BB, kernels.hemm_left)
__global__ void half_mirror_kernel(const double2* __restrict__ t, double2* __restrict__ out, int n,
                                   int64_t count, double scale) {
  const int64_t nn = static_cast<int64_t>(n) * n;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < count * nn;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t a = idx / nn;
    const int r = static_cast<int>(idx % nn);
    const int i = r % n, j = r / n;
    const double2* T = t + a * nn;
    double2 v;
    if (i > j) {
      v = T[i + j * n];
    } else if (i < j) {
      const double2 w = T[j + i * n];
      v = make_double2(w.x, -w.y);
    } else {
      v = make_double2(T[i + i * n].x, 0.0);
    }
    out[idx] = make_double2(scale * v.x, scale * v.y);
  }
}

// out_a = T_a^H (column-major n x n blocks)
__global__ void conj_transpose_kernel(const double2* __restrict__ t, double2* __restrict__ out, int n,
                                      int64_t count) {
  const int64_t nn = static_cast<int64_t>(n) * n;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < count * nn;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t a = idx / nn;
    const int r = static_cast<int>(idx % nn);
    const int i = r % n, j = r / n;
    const double2 w = t[a * nn + j + static_cast<int64_t>(i) * n];
    out[idx] = make_double2(w.x, -w.y);
  }
}

// out_a[k, r] = t_a[k, r] / u[a n + r]: per-atom n x n blocks with column r
// divided by the atom's u_r (correctly rounded), so that L^H R yields rows
// scaled by 1/u (the INT8 engine's H = A^H V1 + (UB)^H (U^-1 V2) regrouping)
__global__ void scale_cols_inv_kernel(const double2* __restrict__ t, double2* __restrict__ out,
                                      const double* __restrict__ u, int n, int64_t count) {
  const int64_t nn = static_cast<int64_t>(n) * n;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < count * nn;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t a = idx / nn;
    const int r = static_cast<int>((idx - a * nn) / n);
    const double d = u[a * n + r];
    const double2 w = t[idx];
    out[idx] = make_double2(w.x / d, w.y / d);
  }
}

// dst[r, g] = u[r] * src[r, g]   (kernels.diag_scale, kernels.py:328-339)
__global__ void diag_scale_kernel(const double2* __restrict__ src, int64_t lds,
                                  double2* __restrict__ dst, int64_t ldd,
                                  const double* __restrict__ u, int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = idx % rows, c = idx / rows;
    const double2 v = src[r + c * lds];
    const double w = u[r];
    dst[r + c * ldd] = make_double2(w * v.x, w * v.y);
  }
}

// Sum planes for the 3M contraction (zrk3m_kernel.cu): for a complex k x n
// operand X, minus = Re X - Im X (its role as the conjugated left factor) and
// plus = Re X + Im X (right factor), both k x n real, leading dimension ldp.
// Computed once per operand here instead of once per output tile inside the
// contraction, where the adds would share the FP64 pipe with DMMA.
__global__ void sum_planes_kernel(const double2* __restrict__ x, int64_t ldx, int64_t rows, int64_t cols,
                                  double* __restrict__ minus, double* __restrict__ plus, int64_t ldp) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = idx % rows, c = idx / rows;
    const double2 v = x[r + c * ldx];
    minus[r + c * ldp] = v.x - v.y;
    plus[r + c * ldp] = v.x + v.y;
  }
}

__global__ void sum_planes_batched_kernel(const double2* __restrict__ x, int n, int64_t bstride, int64_t count,
                                          int minus, double* __restrict__ out, int kp) {
  const int64_t total = count * n * kp;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(idx % kp);
    const int64_t bc = idx / kp, b = bc / n, c = bc - b * n;
    double v = 0.0;
    if (k < n) {
      const double2 w = x[b * bstride + c * static_cast<int64_t>(n) + k];
      v = minus ? w.x - w.y : w.x + w.y;
    }
    out[idx] = v;
  }
}

// In-place Hermitian mirror (matcore.hermitian_mirror, matcore.py:89-105):
// 32 x 32 tile pairs staged through shared memory so both the lower-tile read
// and the upper-tile write are coalesced.
__global__ void mirror_kernel(double2* __restrict__ c, int64_t ldc, int n) {
  __shared__ double2 tile[32][33];
  // blockIdx.x enumerates lower tile pairs (bi >= bj)
  const int t = blockIdx.x;
  int bi = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while (bi * (bi + 1) / 2 > t) --bi;
  while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
  const int bj = t - bi * (bi + 1) / 2;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int k = ty; k < 32; k += 8) {
    const int row = bi * 32 + tx, col = bj * 32 + k;
    if (row < n && col < n) tile[k][tx] = c[row + col * ldc];  // tile[col][row]
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    // write element (row' = bj*32+tx, col' = bi*32+k) = conj(C[col', row'])
    const int row = bj * 32 + tx, col = bi * 32 + k;
    if (row < n && col < n) {
      if (row < col) {
        const double2 v = tile[tx][k];
        c[row + col * ldc] = make_double2(v.x, -v.y);
      } else if (row == col) {
        c[row + col * ldc] = make_double2(tile[tx][k].x, 0.0);
      }
    }
  }
}

// Copy per-atom row blocks: dst[dst_off[a] + l, g] = src[src_off[a] + l, g]
__global__ void gather_rows_kernel(const double2* __restrict__ src, int64_t lds,
                                   double2* __restrict__ dst, int64_t ldd,
                                   const int32_t* __restrict__ src_off,
                                   const int32_t* __restrict__ dst_off, int n_l, int64_t cols) {
  const int a = blockIdx.y;
  const int64_t so = src_off[a], d0 = dst_off[a];
  const int64_t total = static_cast<int64_t>(n_l) * cols;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t l = idx % n_l, g = idx / n_l;
    dst[d0 + l + g * ldd] = src[so + l + g * lds];
  }
}

// dst (cols x rows, ldd) = op(src (rows x cols, lds)), op = transpose or
// conjugate transpose; stages 'N'/'T'/'C' gemm operands into the reduction-
// major layout the DMMA kernel reads.
__global__ void transpose_kernel(const double2* __restrict__ src, int64_t lds, double2* __restrict__ dst,
                                 int64_t ldd, int64_t rows, int64_t cols, int conj) {
  __shared__ double2 tile[32][33];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32, c0 = static_cast<int64_t>(blockIdx.y) * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int k = ty; k < 32; k += 8) {
    const int64_t r = r0 + tx, c = c0 + k;
    if (r < rows && c < cols) tile[k][tx] = src[r + c * lds];
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int64_t r = c0 + tx, c = r0 + k;  // dst row = src col
    if (r < cols && c < rows) {
      double2 v = tile[tx][k];
      if (conj) v.y = -v.y;
      dst[r + c * ldd] = v;
    }
  }
}

// dst (stacked, column g = [atom 0 rows | atom 1 rows | ...], ld = n_atoms*rows)
//   <- raw (atom-major: n_atoms contiguous rows x cols column-major blocks)
// i.e. matcore.stack (matcore.py:68-86) on the device, after contiguous DMAs.
__global__ void stack_blocks_kernel(const double2* __restrict__ raw, double2* __restrict__ dst, int n_atoms,
                                    int rows, int64_t cols) {
  const int64_t total = static_cast<int64_t>(n_atoms) * rows * cols;
  const int64_t K = static_cast<int64_t>(n_atoms) * rows;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t l = idx % rows;
    const int64_t rest = idx / rows;
    const int64_t g = rest % cols, a = rest / cols;
    dst[g * K + a * rows + l] = raw[idx];
  }
}

// *flag = min over blocks holding a NaN/Inf of the block index (flag starts at
// 0x7f7f7f7f).  Device counterpart of the finiteness test in
// probgen.validate_instance (probgen.py:155-161) for pinned uploads.
__global__ void first_nonfinite_kernel(const unsigned long long* __restrict__ v, int64_t per_block,
                                       int64_t total, int* __restrict__ flag) {
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if ((v[idx] & 0x7ff0000000000000ull) == 0x7ff0000000000000ull) atomicMin(flag, static_cast<int>(idx / per_block));
  }
}

// ------------------------------------------------------------------ launchers
static inline int grid_for(int64_t total, int threads, int max_blocks) {
  int64_t b = (total + threads - 1) / threads;
  if (b > max_blocks) b = max_blocks;
  if (b < 1) b = 1;
  return static_cast<int>(b);
}

cudaError_t launch_potrf_route(const double* t_aa, double* q, int32_t* info, int n_atoms, int n,
                               bool force_nonhpd, double* gscratch, cudaStream_t st) {
  const size_t packed = static_cast<size_t>(n) * (n + 1) / 2 * 16;
  const bool use_smem = packed <= kPotrfSmemMax;
  size_t smem = use_smem ? packed : 0;
  if (use_smem) {
    cudaError_t e = cudaFuncSetAttribute(potrf_route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kPotrfSmemMax));
    if (e != cudaSuccess) return e;
  }
  potrf_route_kernel<<<n_atoms, 1024, smem, st>>>(
      reinterpret_cast<const double2*>(t_aa), reinterpret_cast<double2*>(q), info, n, force_nonhpd ? 1 : 0,
      use_smem ? nullptr : reinterpret_cast<double2*>(gscratch));
  return cudaGetLastError();
}

cudaError_t launch_half_mirror(const double* t, double* out, int n, int64_t count, double scale,
                               cudaStream_t st) {
  const int64_t total = count * n * n;
  half_mirror_kernel<<<grid_for(total, 256, 148 * 16), 256, 0, st>>>(
      reinterpret_cast<const double2*>(t), reinterpret_cast<double2*>(out), n, count, scale);
  return cudaGetLastError();
}

cudaError_t launch_conj_transpose(const double* t, double* out, int n, int64_t count, cudaStream_t st) {
  const int64_t total = count * static_cast<int64_t>(n) * n;
  if (total <= 0) return cudaSuccess;
  conj_transpose_kernel<<<grid_for(total, 256, 148 * 16), 256, 0, st>>>(reinterpret_cast<const double2*>(t),
                                                                         reinterpret_cast<double2*>(out), n, count);
  return cudaGetLastError();
}

cudaError_t launch_scale_cols_inv(const double* t, double* out, const double* u, int n, int64_t count,
                                  cudaStream_t st) {
  const int64_t total = count * static_cast<int64_t>(n) * n;
  if (total <= 0) return cudaSuccess;
  scale_cols_inv_kernel<<<grid_for(total, 256, 148 * 16), 256, 0, st>>>(
      reinterpret_cast<const double2*>(t), reinterpret_cast<double2*>(out), u, n, count);
  return cudaGetLastError();
}

cudaError_t launch_diag_scale(const double* src, int64_t lds, double* dst, int64_t ldd, const double* u,
                              int64_t rows, int64_t cols, cudaStream_t st) {
  diag_scale_kernel<<<grid_for(rows * cols, 256, 148 * 32), 256, 0, st>>>(
      reinterpret_cast<const double2*>(src), lds, reinterpret_cast<double2*>(dst), ldd, u, rows, cols);
  return cudaGetLastError();
}

cudaError_t launch_sum_planes(const double* x, int64_t ldx, int64_t rows, int64_t cols, double* minus,
                              double* plus, int64_t ldp, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  sum_planes_kernel<<<grid_for(rows * cols, 256, 148 * 32), 256, 0, st>>>(reinterpret_cast<const double2*>(x), ldx,
                                                                          rows, cols, minus, plus, ldp);
  return cudaGetLastError();
}

cudaError_t launch_sum_planes_batched(const double* x, int n, int64_t bstride, int64_t count, bool minus,
                                     double* out, int kp, cudaStream_t st) {
  const int64_t total = count * n * kp;
  if (total <= 0) return cudaSuccess;
  sum_planes_batched_kernel<<<grid_for(total, 256, 148 * 16), 256, 0, st>>>(
      reinterpret_cast<const double2*>(x), n, bstride, count, minus ? 1 : 0, out, kp);
  return cudaGetLastError();
}

// out[i] = sum_r slots[r * stride + i] (complex): the owner's half of the fused
// multi-GPU scatter (hsb_peer_out).  16-byte loads of every slot in flight,
// summed in rank order (deterministic).  HBM-bound: (n_slots + 1) * 16 B per
// element.
__global__ void sum_slots_kernel(const double2* __restrict__ slots, int n_slots, int64_t stride, int64_t count,
                                 double2* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double2 acc = __ldg(slots + i);
    for (int r = 1; r < n_slots; ++r) {
      const double2 v = __ldg(slots + r * stride + i);
      acc.x += v.x;
      acc.y += v.y;
    }
    out[i] = acc;
  }
}

cudaError_t launch_sum_slots(const double* slots, int n_slots, int64_t stride, int64_t count, double* out,
                             cudaStream_t st) {
  if (count <= 0 || n_slots <= 0) return cudaSuccess;
  sum_slots_kernel<<<grid_for(count, 256, 148 * 16), 256, 0, st>>>(reinterpret_cast<const double2*>(slots), n_slots,
                                                                   stride, count, reinterpret_cast<double2*>(out));
  return cudaGetLastError();
}

__global__ void fill_i32_kernel(int32_t* p, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = v;
}
// Loop 2 routing on the device (the HPD / non-HPD split of builder.py:135-160):
// from every atom's potrf info, the row offset of its product in R = [Y_hpd ;
// X_nh] and the gather lists of the non-HPD atoms, all in atom order.  info
// is also exported to mapped host memory, so the host learns the split
// without a copy-engine transfer queued behind other streams' bulk copies.
// One block; chunked block-wide scan over the atoms.
__global__ void route_atoms_kernel(const int32_t* __restrict__ info, int na, int nl, int32_t* __restrict__ offs,
                                   int32_t* __restrict__ info_host) {
  __shared__ int s_warp[32];
  __shared__ int s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  int cnt = 0;
  for (int i = tid; i < na; i += blockDim.x) cnt += info[i] == 0;
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(~0u, cnt, o);
  if (lane == 0) s_warp[warp] = cnt;
  if (tid == 0) s_base = 0;
  __syncthreads();
  int n_hpd = 0;
  for (int w = 0; w < nw; ++w) n_hpd += s_warp[w];
  __syncthreads();
  for (int c0 = 0; c0 < na; c0 += blockDim.x) {
    const int i = c0 + tid;
    const int v = i < na ? info[i] : 1;
    const bool hpd = i < na && v == 0;
    const unsigned m = __ballot_sync(~0u, hpd);
    if (lane == 0) s_warp[warp] = __popc(m);
    __syncthreads();
    int ih = s_base + __popc(m & ((1u << lane) - 1));  // HPD atoms before atom i
    for (int w = 0; w < warp; ++w) ih += s_warp[w];
    if (i < na) {
      info_host[i] = v;
      if (hpd) {
        offs[i] = ih * nl;
      } else {
        const int in = i - ih;  // non-HPD atoms before atom i
        offs[i] = (n_hpd + in) * nl;
        offs[na + in] = i * nl;  // A_nh source rows
        offs[2 * na + in] = in * nl;  // A_nh destination rows
      }
    }
    __syncthreads();
    if (tid == 0)
      for (int w = 0; w < nw; ++w) s_base += s_warp[w];
    __syncthreads();
  }
}
cudaError_t launch_route_atoms(const int32_t* info, int na, int nl, int32_t* offs, int32_t* info_host,
                               cudaStream_t st) {
  route_atoms_kernel<<<1, 1024, 0, st>>>(info, na, nl, offs, info_host);
  return cudaGetLastError();
}

__global__ void copy_i32_kernel(const int32_t* __restrict__ src, int32_t* __restrict__ dst, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[i];
}
cudaError_t launch_copy_i32(const int32_t* src, int32_t* dst, int n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  copy_i32_kernel<<<grid_for(n, 256, 64), 256, 0, st>>>(src, dst, n);
  return cudaGetLastError();
}

cudaError_t launch_fill_i32(int32_t* p, int64_t n, int32_t v, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  fill_i32_kernel<<<grid_for(n, 256, 1024), 256, 0, st>>>(p, n, v);
  return cudaGetLastError();
}

cudaError_t launch_mirror(double* c, int64_t ldc, int n, cudaStream_t st) {
  const int64_t nt = (n + 31) / 32;
  const int64_t pairs = nt * (nt + 1) / 2;
  mirror_kernel<<<static_cast<unsigned>(pairs), dim3(32, 8), 0, st>>>(reinterpret_cast<double2*>(c), ldc, n);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const double* src, int64_t lds, double* dst, int64_t ldd, const int32_t* src_off,
                               const int32_t* dst_off, int n_blocks, int n_l, int64_t cols, cudaStream_t st) {
  if (n_blocks == 0) return cudaSuccess;
  const int gx = grid_for(static_cast<int64_t>(n_l) * cols, 256, 256);
  gather_rows_kernel<<<dim3(gx, n_blocks), 256, 0, st>>>(reinterpret_cast<const double2*>(src), lds,
                                                         reinterpret_cast<double2*>(dst), ldd, src_off, dst_off,
                                                         n_l, cols);
  return cudaGetLastError();
}

cudaError_t launch_stack_blocks(const double* raw, double* dst, int n_atoms, int rows, int64_t cols,
                                cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(n_atoms) * rows * cols;
  stack_blocks_kernel<<<grid_for(total, 256, 148 * 32), 256, 0, st>>>(reinterpret_cast<const double2*>(raw),
                                                                       reinterpret_cast<double2*>(dst), n_atoms,
                                                                       rows, cols);
  return cudaGetLastError();
}

cudaError_t launch_first_nonfinite(const double* v, int n_blocks, int64_t doubles_per_block, int* flag,
                                   cudaStream_t st) {
  cudaError_t e = launch_fill_i32(flag, 1, 0x7f7f7f7f, st);
  if (e != cudaSuccess) return e;
  const int64_t total = static_cast<int64_t>(n_blocks) * doubles_per_block;
  first_nonfinite_kernel<<<grid_for(total, 256, 148 * 16), 256, 0, st>>>(
      reinterpret_cast<const unsigned long long*>(v), doubles_per_block, total, flag);
  return cudaGetLastError();
}

cudaError_t launch_transpose(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int64_t cols,
                             bool conj, cudaStream_t st) {
  dim3 grid(static_cast<unsigned>((rows + 31) / 32), static_cast<unsigned>((cols + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(reinterpret_cast<const double2*>(src), lds,
                                                 reinterpret_cast<double2*>(dst), ldd, rows, cols, conj ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace hsb
