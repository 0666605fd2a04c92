// zrk_kernel.cu — the TMA-fed, warp-specialised FP64 DMMA kernel declared in
// zrk.cuh.  One CTA = one 64 x 64 complex output tile; warp 4 is the TMA
// producer (one elected lane), warps 0-3 each own a 32 x 32 complex sub-tile
// held in registers as 4 x 4 DMMA.8x8x4 accumulator pairs (real, imag).
#include "aux_kernels.cuh"
#include "ptx.cuh"
#include "zrk.cuh"

namespace hsb {

// Offset (in doubles) of element (row, k) in a 64 x 16 double tile written by
// TMA with CU_TENSOR_MAP_SWIZZLE_128B: the 16-byte chunk index (k/2) is XORed
// with (row mod 8).  Fragment loads (8 rows x 4 k per DMMA operand) therefore
// hit 8 distinct chunks per half-warp: conflict-free.
__device__ __forceinline__ int swz(int row, int k) {
  return row * 16 + ((((k >> 1) ^ row) & 7) << 1) + (k & 1);
}

template <bool CONJ>
__global__ void __launch_bounds__(kThreads, 2) zrk_kernel(const __grid_constant__ ZrkParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;  // 128B swizzle atom = 1024 B
  double* tiles = reinterpret_cast<double*>(smem_raw + (base - raw));
  const uint32_t bar_base = base + kStages * kStageBytes;  // full[s] then empty[s]
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (kStages + s); };

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  int tm, tn;
  if (p.triangle) {
    tri_tile(blockIdx.x, p.tiles_m, tm, tn);
  } else {
    tm = blockIdx.x % p.tiles_m;
    tn = blockIdx.x / p.tiles_m;
  }
  const int z = blockIdx.z;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      for (int s = 0; s < p.nseg; ++s) {
        prefetch_tmap(&p.lmap[s]);
        prefetch_tmap(&p.rmap[s]);
      }
      int stage = 0;
      uint32_t phase = 1;  // fresh empty barriers read as "released"
      const int row0 = tm * kBM, col0 = tn * kBN;
      for (int s = 0; s < p.nseg; ++s) {
        const SegDesc sd = p.seg[s];
        for (int kc = 0; kc < sd.kchunks; ++kc) {
          mbar_wait(empty_bar(stage), phase);
          const uint32_t fb = full_bar(stage);
          mbar_expect_tx(fb, kStageBytes);
          const uint32_t dst = base + stage * kStageBytes;
          const int k0 = kc * kBK;
          if (sd.lbpos == 1)
            tma_load_3d(dst, &p.lmap[s], k0, z, row0, fb);
          else
            tma_load_3d(dst, &p.lmap[s], k0, row0, z, fb);
          if (sd.rbpos == 1)
            tma_load_3d(dst + kTileBytes, &p.rmap[s], k0, z, col0, fb);
          else
            tma_load_3d(dst + kTileBytes, &p.rmap[s], k0, col0, z, fb);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
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
  const unsigned long long odd_mask = (t & 1) ? 0x8000000000000000ull : 0ull;

  double cr[4][4][2], ci[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      cr[i][j][0] = cr[i][j][1] = 0.0;
      ci[i][j][0] = ci[i][j][1] = 0.0;
    }

  // per-thread swizzled offsets for the 4 k-steps (row part added per fragment)
  int offk[4], offkx[4];
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    offk[ks] = swz(g, ks * 4 + t) - g * 16;
    offkx[ks] = swz(g, ks * 4 + (t ^ 1)) - g * 16;
  }
  const int arow = (wm * 32 + g) * 16;  // + f * 8 * 16
  const int brow = (wn * 32 + g) * 16;

  int stage = 0;
  uint32_t phase = 0;
  for (int it = 0; it < p.total_chunks; ++it) {
    mbar_wait(full_bar(stage), phase);
    const double* As = tiles + stage * (kStageBytes / 8);
    const double* Bs = As + kTileBytes / 8;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      double a[4], b[4], bx[4];
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        a[f] = As[arow + f * 128 + offk[ks]];
        b[f] = Bs[brow + f * 128 + offk[ks]];
        bx[f] = Bs[brow + f * 128 + offkx[ks]];
      }
      if (CONJ) {
        // Re += Lt^T Rt ; Im += Lt^T Rs,  Rs = (Im R, -Re R) pairs
#pragma unroll
        for (int f = 0; f < 4; ++f) bx[f] = flip_sign(bx[f], odd_mask);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            dmma(cr[i][j][0], cr[i][j][1], a[i], b[j]);
            dmma(ci[i][j][0], ci[i][j][1], a[i], bx[j]);
          }
      } else {
        // Re += Ln^T Rt (Ln = (Re L, -Im L)) ; Im += Lt^T Rw (Rw = (Im R, Re R))
        double an[4];
#pragma unroll
        for (int f = 0; f < 4; ++f) an[f] = flip_sign(a[f], odd_mask);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            dmma(cr[i][j][0], cr[i][j][1], an[i], b[j]);
            dmma(ci[i][j][0], ci[i][j][1], a[i], bx[j]);
          }
      }
    }
    // this warp's shared-memory reads complete before the stage is released to
    // the TMA producer (see zrk3m_kernel.cu: the arrive does not wait for LDS)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_bar(stage));
    if (++stage == kStages) {
      stage = 0;
      phase ^= 1u;
    }
  }

  // -------------------------------------------------------------- epilogue
  double* C = p.c + 2 * (p.c_rowoff ? static_cast<int64_t>(p.c_rowoff[z]) : z * p.c_bstride);
  const int64_t ldc = p.ldc;
  const bool lower_only = p.flags & kLowerOnly;
  const bool mirror = p.flags & kMirror;
  const bool zero_imag = p.flags & kZeroImagDiag;
  const bool has_beta = (p.beta_re != 0.0) || (p.beta_im != 0.0);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = tm * kBM + wm * 32 + i * 8 + g;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = tn * kBN + wn * 32 + j * 8 + 2 * t + e;
        if (row >= p.m || col >= p.n) continue;
        if (lower_only && row < col) continue;
        const double xr = cr[i][j][e], xi = ci[i][j][e];
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
        if (mirror && row > col) {
          reinterpret_cast<double2*>(C)[col + row * ldc] = make_double2(vr, -vi);
        }
      }
    }
  }
  if (p.done_cnt) {
    // all consumer stores of this tile precede the count (bar.sync orders them
    // CTA-wide; the system-scope fence makes them visible to the host/DMA)
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
    if (threadIdx.x == 0) {
      __threadfence_system();
      atomicAdd_system(p.done_cnt + tn, 1);
      if (tm != tn) atomicAdd_system(p.done_cnt + tm, 1);
    }
  }
}

// ------------------------------------------------------------------ launcher
cudaError_t launch_zrk(const ZrkParams& p, bool conj, int grid_x, int grid_z, cudaStream_t st) {
  static PerDeviceOnce attr[2];  // the attribute is per device
  auto kern = conj ? zrk_kernel<true> : zrk_kernel<false>;
  cudaError_t e = per_device_once(
      attr[conj], [&] { return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes); });
  if (e != cudaSuccess) return e;
  kern<<<dim3(grid_x, 1, grid_z), dim3(kThreads), kSmemBytes, st>>>(p);
  return cudaGetLastError();
}

}  // namespace hsb
