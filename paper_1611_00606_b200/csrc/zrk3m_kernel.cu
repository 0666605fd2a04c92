// zrk3m_kernel.cu — the segmented complex rank-k update of zrk.cuh with the
// 3-multiplication (Gauss) complex product, persistent over output tiles.
//
// The 4M kernel (zrk_kernel.cu) spends 4 real MACs per complex MAC, the
// reference's 8-flop model (kernels.py:66-85).  Here the three real products
//
//     P = Lr^T Rr,   Q = Li^T Ri,   W = (Lr -/+ Li)^T (Rr + Ri)
//
// give  L^H R = (P + Q) + i (W - P + Q)      (CONJ,  W uses Lr - Li)
//       L^T R = (P - Q) + i (W - P - Q)      (plain, W uses Lr + Li)
// for 3 real MACs per complex MAC: 25 % less DMMA work for the same result
// (Higham, "Stability of a method for multiplying complex matrices with
// three real matrix multiplications", SIMAX 13 (1992): the error bound grows
// by a small constant factor, far inside the north star's 1e-10).
//
// Same TMA operand layout as the 4M kernel (64-row x 16-real boxes, 128B
// swizzle), so the host encodes identical descriptors.  Differences:
//   * one CTA per SM, persistent: CTA b processes work items b, b + grid, ...
//     (work item = tile x batch).  The producer warp streams straight into
//     the next tile while the consumers run the epilogue of the current one;
//   * 8 consumer warps (2 x 4), each owning a 32 x 16 complex sub-tile held as
//     4 x 2 DMMA.8x8x4 accumulator triples (P, Q, W): 96 registers;
//   * a DMMA k-step covers 4 complex k; lane (g, t) loads the double2
//     (re, im) of complex k = 2t + s, s = 0, 1 within the 8-complex chunk.
//     With the 128B swizzle (chunk ^= row & 7) the 8 lanes of a quarter-warp
//     (rows g, g+1; chunks {s, 2+s, 4+s, 6+s} ^ g) hit 8 distinct 16-byte
//     chunks: conflict-free LDS.128;
//   * 12 pipeline stages x 16 KB.
//
// PMODE (plane mode): 2 -- the host precomputes Re-Im of every left operand and
// Re+Im of every right operand (sum_planes_kernel), loaded by TMA beside the
// complex tiles (+8 KB per stage, 8 stages), so the main loop is LDS + DMMA
// only; 1 -- left planes only: the batched per-atom products (V products),
// whose left operands are the small T blocks, get them as per-atom planes
// padded to an even k (so the 3-D TMA view's atom stride is 16-byte aligned;
// +4 KB per stage, 9 stages), and form only the right operand's sum in
// registers (2 of the 6 DADD per k step); 0 -- both sums in registers (DADD
// shares the FP64 pipe with DMMA: ncu 90 % vs 96 % DMMA-active on the H launch).
#include <algorithm>

#include "aux_kernels.cuh"
#include "ptx.cuh"
#include "zrk.cuh"

namespace hsb {

constexpr int k3ConsumerWarps = 8;  // 2 (rows) x 4 (cols) warps of 32 x 16
constexpr int k3Threads = (k3ConsumerWarps + 1) * 32;
constexpr int kPlaneTileBytes = kBM * 8 * 8;  // 64 rows x 8 complex k, one double each
template <int PMODE>
struct Cfg3 {
  static constexpr int load_bytes = kStageBytes + PMODE * kPlaneTileBytes;  // TMA bytes per stage
  static constexpr int stage_bytes = load_bytes;
  static constexpr int stages = PMODE == 2 ? 8 : PMODE == 1 ? 9 : 12;  // PMODE 1: 180 KB, room for a residue block beside it
  static constexpr int smem = stages * stage_bytes + 1024 /*align*/ + 256 /*barriers*/;
};

__device__ __forceinline__ void dmma_nv(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void work_tile(const ZrkParams& p, int w, int ntiles, int& tm, int& tn, int& z) {
  z = w / ntiles;
  const int t = w - z * ntiles;
  if (p.tile_list) {
    const int2 tt = p.tile_list[t];
    tm = tt.x;
    tn = tt.y;
  } else if (p.triangle) {
    tri_tile(t, p.tiles_m, tm, tn);
  } else {
    tm = t % p.tiles_m;
    tn = t / p.tiles_m;
  }
}

template <bool CONJ, int PMODE>
__global__ void __launch_bounds__(k3Threads, 1) zrk3m_kernel(const __grid_constant__ ZrkParams p, int ntiles,
                                                              int nwork) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;  // 128B swizzle atom = 1024 B
  const double2* tiles = reinterpret_cast<const double2*>(smem_raw + (base - raw));
  using C3 = Cfg3<PMODE>;
  constexpr bool LPLANE = PMODE >= 1, RPLANE = PMODE == 2;
  constexpr int kSt = C3::stages;
  constexpr int kSB = C3::stage_bytes;
  const uint32_t bar_base = base + kSt * kSB;  // full[s] then empty[s]
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (kSt + s); };

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSt; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), k3ConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == k3ConsumerWarps) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      for (int s = 0; s < p.nseg; ++s) {
        prefetch_tmap(&p.lmap[s]);
        prefetch_tmap(&p.rmap[s]);
        if (LPLANE) prefetch_tmap(&p.lsum[s]);
        if (RPLANE) prefetch_tmap(&p.rsum[s]);
      }
      int stage = 0;
      uint32_t phase = 1;  // fresh empty barriers read as "released"
      for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
        int tm, tn, z;
        work_tile(p, w, ntiles, tm, tn, z);
        const int row0 = tm * kBM, col0 = tn * kBN;
        for (int s = 0; s < p.nseg; ++s) {
          const SegDesc sd = p.seg[s];
          for (int kc = 0; kc < sd.kchunks; ++kc) {
            mbar_wait(empty_bar(stage), phase);
            const uint32_t fb = full_bar(stage);
            mbar_expect_tx(fb, C3::load_bytes);
            const uint32_t dst = base + stage * kSB;
            const int k0 = kc * kBK;
            if (sd.lbpos == 1)
              tma_load_3d(dst, &p.lmap[s], k0, z, row0, fb);
            else
              tma_load_3d(dst, &p.lmap[s], k0, row0, z, fb);
            if (sd.rbpos == 1)
              tma_load_3d(dst + kTileBytes, &p.rmap[s], k0, z, col0, fb);
            else
              tma_load_3d(dst + kTileBytes, &p.rmap[s], k0, col0, z, fb);
            if (LPLANE) {  // k in complex units
              if (p.lplane3d)
                tma_load_3d(dst + kStageBytes, &p.lsum[s], kc * 8, row0, z, fb);
              else
                tma_load_2d(dst + kStageBytes, &p.lsum[s], kc * 8, row0, fb);
            }
            if (RPLANE)  // plain operands only (z == 0): 2-D planes
              tma_load_2d(dst + kStageBytes + kPlaneTileBytes, &p.rsum[s], kc * 8, col0, fb);
            if (++stage == kSt) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int g = lane >> 2;  // DMMA group id   (row of A / col of B / row of C)
  const int t = lane & 3;   // thread in group (k index)
  const int wm = warp & 1, wn = warp >> 1;
  // double2 offsets inside one 64-row x 8-complex swizzled tile
  const int offa0 = (wm * 32 + g) * 8 + (((2 * t) ^ g) & 7);
  const int offa1 = (wm * 32 + g) * 8 + (((2 * t + 1) ^ g) & 7);
  const int offb0 = (wn * 16 + g) * 8 + (((2 * t) ^ g) & 7);
  const int offb1 = (wn * 16 + g) * 8 + (((2 * t + 1) ^ g) & 7);
  constexpr int kTile2 = kTileBytes / 16;  // double2 per operand tile

  const bool lower_only = p.flags & kLowerOnly;
  const bool mirror = p.flags & kMirror;
  const bool zero_imag = p.flags & kZeroImagDiag;
  const bool has_beta = (p.beta_re != 0.0) || (p.beta_im != 0.0);
  const int64_t ldc = p.ldc;

  int stage = 0;
  uint32_t phase = 0;
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
    int tm, tn, z;
    work_tile(p, w, ntiles, tm, tn, z);

    double cp[4][2][2], cq[4][2][2], cw[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) cp[i][j][e] = cq[i][j][e] = cw[i][j][e] = 0.0;

    for (int it = 0; it < p.total_chunks; ++it) {
      mbar_wait(full_bar(stage), phase);
      const double2* As = tiles + stage * (kSB / 16);
      const double2* Bs = As + kTile2;
      // plane tiles: 64 rows x 4 double2 (complex k = 2t, 2t+1 of this lane)
      double2 sa[4], sb[2];
      if (LPLANE) {
        const double2* Ps = Bs + kTile2;
#pragma unroll
        for (int i = 0; i < 4; ++i) sa[i] = Ps[(wm * 32 + i * 8 + g) * 4 + t];
      }
      if (RPLANE) {
        const double2* Qs = Bs + kTile2 + kPlaneTileBytes / 16;
#pragma unroll
        for (int j = 0; j < 2; ++j) sb[j] = Qs[(wn * 16 + j * 8 + g) * 4 + t];
      }
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int oa = s ? offa1 : offa0;
        const int ob = s ? offb1 : offb0;
        double2 a[4], b[2];
        double as[4], bs[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[oa + i * 64];
#pragma unroll
        for (int j = 0; j < 2; ++j) b[j] = Bs[ob + j * 64];
        if (LPLANE) {
#pragma unroll
          for (int i = 0; i < 4; ++i) as[i] = s ? sa[i].y : sa[i].x;
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) as[i] = CONJ ? a[i].x - a[i].y : a[i].x + a[i].y;
        }
        if (RPLANE) {
#pragma unroll
          for (int j = 0; j < 2; ++j) bs[j] = s ? sb[j].y : sb[j].x;
        } else {
#pragma unroll
          for (int j = 0; j < 2; ++j) bs[j] = b[j].x + b[j].y;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            dmma_nv(cp[i][j][0], cp[i][j][1], a[i].x, b[j].x);
            dmma_nv(cq[i][j][0], cq[i][j][1], a[i].y, b[j].y);
            dmma_nv(cw[i][j][0], cw[i][j][1], as[i], bs[j]);
          }
      }
      // Release the stage only once this warp's reads of it are complete: the
      // scheduler sinks DMMAs (and so the waits on their LDS operands) below
      // the arrive, and the arrive does not wait for LDS in flight, so the
      // producer's next TMA could overwrite rows not yet read (rare wrong A
      // rows in one warp's sub-tile, probes/stress_dmma_phys.py).  The proxy
      // fence orders this thread's generic-proxy reads before the async-proxy
      // (TMA) writes that follow the release.
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_bar(stage));
      if (++stage == kSt) {
        stage = 0;
        phase ^= 1u;
      }
    }

    // ------------------------------------------------------------ epilogue
    double* C = p.c + 2 * (p.c_rowoff ? static_cast<int64_t>(p.c_rowoff[z]) : z * p.c_bstride);
    double cmax[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // per column: max |Re| + |Im| of this lane's rows
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = tm * kBM + wm * 32 + i * 8 + g;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = tn * kBN + wn * 16 + j * 8 + 2 * t + e;
          if (row >= p.m || col >= p.n) continue;
          if (lower_only && row < col) continue;
          const double P = cp[i][j][e], Q = cq[i][j][e], W = cw[i][j][e];
          const double xr = CONJ ? P + Q : P - Q;
          const double xi = CONJ ? (W - P) + Q : (W - P) - Q;
          double vr = p.alpha_re * xr - p.alpha_im * xi;
          double vi = p.alpha_re * xi + p.alpha_im * xr;
          double2* dst = reinterpret_cast<double2*>(C) + row + col * ldc;
          if (has_beta) {
            const double2 o = *dst;
            vr += p.beta_re * o.x - p.beta_im * o.y;
            vi += p.beta_re * o.y + p.beta_im * o.x;
          }
          if (row == col && (zero_imag || mirror)) vi = 0.0;
          *dst = make_double2(vr, vi);
          if (mirror && row > col) reinterpret_cast<double2*>(C)[col + row * ldc] = make_double2(vr, -vi);
          cmax[j][e] = fmax(cmax[j][e], fabs(vr) + fabs(vi));
        }
      }
    }
    if (p.col_exp) {
      // the 8 lanes of a column (g = 0..7) hold its 32 rows of this warp: reduce
      // over g, then one atomicMax of the frexp exponent per column and warp
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double m = cmax[j][e];
          m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 4));
          m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 8));
          m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 16));
          const int col = tn * kBN + wn * 16 + j * 8 + 2 * t + e;
          if (g == 0 && col < p.n) {
            int ex = 0;
            frexp(m, &ex);
            atomicMax(p.col_exp + col, ex);
          }
        }
    }
    if (p.done_cnt) {
      // all consumer stores of this tile precede the count: EVERY storing
      // thread fences (its stores performed at device scope, where the copy
      // engine reads them) before the named barrier over the consumer warps;
      // a barrier alone orders issue, not completion -- with only thread 0
      // fencing, a host download of a "final" column block occasionally read
      // stores still in flight (probes/stress_host_outputs.py)
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"n"(k3ConsumerWarps * 32) : "memory");
      if (threadIdx.x == 0) {
        __threadfence_system();
        atomicAdd_system(p.done_cnt + tn, 1);
        if (tm != tn) atomicAdd_system(p.done_cnt + tm, 1);
      }
    }
  }
}

// ------------------------------------------------------------------ launcher
template <bool CONJ, int PMODE>
static cudaError_t launch3(const ZrkParams& p, int ntiles, int nwork, int n_sm, cudaStream_t st) {
  static PerDeviceOnce attr;  // the attribute is per device
  auto kern = zrk3m_kernel<CONJ, PMODE>;
  cudaError_t e = per_device_once(
      attr, [&] { return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg3<PMODE>::smem); });
  if (e != cudaSuccess) return e;
  const int grid = std::min(nwork, n_sm);
  kern<<<dim3(grid), dim3(k3Threads), Cfg3<PMODE>::smem, st>>>(p, ntiles, nwork);
  return cudaGetLastError();
}

cudaError_t launch_zrk3m(const ZrkParams& p, bool conj, int pmode, int ntiles, int nbatch, cudaStream_t st) {
  int dev = 0, n_sm = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  const int64_t nwork = static_cast<int64_t>(ntiles) * nbatch;
  if (nwork > 0x7fffffff) return cudaErrorInvalidConfiguration;
  if (pmode == 2 && nbatch != 1) return cudaErrorInvalidValue;
  const int nw = static_cast<int>(nwork);
  switch (pmode * 2 + (conj ? 1 : 0)) {
    case 0: return launch3<false, 0>(p, ntiles, nw, n_sm, st);
    case 1: return launch3<true, 0>(p, ntiles, nw, n_sm, st);
    case 2: return launch3<false, 1>(p, ntiles, nw, n_sm, st);
    case 3: return launch3<true, 1>(p, ntiles, nw, n_sm, st);
    case 4: return launch3<false, 2>(p, ntiles, nw, n_sm, st);
    case 5: return launch3<true, 2>(p, ntiles, nw, n_sm, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hsb
