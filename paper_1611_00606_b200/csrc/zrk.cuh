// zrk.cuh — segmented complex128 rank-k update on FP64 DMMA tensor cores.
//
// One kernel family serves every dense contraction of Algorithm 1
// (builder.py:73-208):
//
//     C  <-  alpha * SUM_s  op(L_s)^T R_s  +  beta * C
//
// where each segment s is a pair of K_s x M / K_s x N complex128 column-major
// operands (reduction dimension first, i.e. "A^H B" shaped exactly like
// kernels.herk / her2k / gemm('C','N') in kernels.py:195-281), op = conj for
// 'C' (CONJ=true) and identity for 'T'.  Segments accumulate into the same
// register accumulators, so  H1 = Z^H B + B^H Z  (her2k, executor.py:148-182)
// is two segments, S = A^H A + (UB)^H (UB) is two segments, and the fused
// H = Z^H B + B^H Z + Y^H Y + A_nh^H X_nh is four.
//
// Complex arithmetic is mapped onto real DMMA.8x8x4 by viewing each complex
// K x N matrix as the real 2K x N matrix of its interleaved (re, im) pairs
// (the raw memory of a numpy complex128 F-order array):
//     Re(L^H R) = Lt^T Rt,   Im(L^H R) = Lt^T Rs,  Rs[2p] = Im R[p], Rs[2p+1] = -Re R[p]
// so a complex MAC costs exactly 4 real MACs (= the reference's 8-flop model,
// kernels.py:66-85) and both products share the A fragment.
//
// Output tiles are 64 x 64; in triangle mode only tiles on or below the
// diagonal are launched (plan_tiles(triangular=True), executor.py:66-84) and
// the epilogue writes i >= j only (kernels._update_lower, kernels.py:234-253),
// optionally mirroring conj(C_ij) into C_ji (matcore.hermitian_mirror,
// matcore.py:89-105) so no separate mirror pass is needed.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace hsb {

constexpr int kBM = 64;            // output tile rows   (complex)
constexpr int kBN = 64;            // output tile cols   (complex)
constexpr int kBK = 16;            // reduction chunk    (reals = 8 complex), 128 B rows
constexpr int kStages = 6;         // TMA pipeline depth
constexpr int kConsumerWarps = 4;  // 2 x 2 warps of 32 x 32
constexpr int kThreads = (kConsumerWarps + 1) * 32;  // + 1 TMA producer warp
constexpr int kMaxSeg = 4;
constexpr int kTileBytes = kBM * kBK * 8;            // 8 KB per operand tile
constexpr int kStageBytes = 2 * kTileBytes;          // 16 KB per stage
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;

// epilogue flags (superset of the ABI flags in include/hsb200.h)
constexpr uint32_t kLowerOnly = 0x1u;    // write i >= j only
constexpr uint32_t kMirror = 0x2u;       // also write C_ji = conj(C_ij), real diagonal
constexpr uint32_t kZeroImagDiag = 0x4u; // Im(C_ii) := 0 (herk/her2k tail)

struct SegDesc {
  int32_t kchunks;  // reduction chunks of kBK reals
  int32_t lbpos;    // batch coordinate slot of the L map: 1 -> dim1, 2 -> dim2
  int32_t rbpos;
  int32_t pad;
};

struct ZrkParams {
  CUtensorMap lmap[kMaxSeg];  // 3-D maps over the real view, box {16, 64|1, 1|64}
  CUtensorMap rmap[kMaxSeg];
  CUtensorMap lsum[kMaxSeg];  // 3M with planes: 2-D maps over Re-Im of L / Re+Im of R,
  CUtensorMap rsum[kMaxSeg];  // box {8 complex k, 64 cols}, no swizzle (zrk3m_kernel.cu);
                              // batched left operands (lplane3d): 3-D {kp, cols, batch}, box {8, 64, 1}
  int32_t lplane3d;           // 1: lsum maps are 3-D per-atom planes (batch coordinate last)
  SegDesc seg[kMaxSeg];
  int32_t nseg;
  int32_t total_chunks;
  int32_t m, n;             // output extent (complex)
  int32_t tiles_m, tiles_n; // rect mode grid
  int32_t triangle;         // 1: blockIdx.x enumerates lower-triangle tiles
  uint32_t flags;
  double alpha_re, alpha_im, beta_re, beta_im;
  double* c;                // interleaved complex128, column-major
  int64_t ldc;              // complex elements
  int64_t c_bstride;        // complex elements between batch outputs
  const int32_t* c_rowoff;  // optional per-batch row offset (complex), overrides c_bstride
  const int2* tile_list;    // optional (triangle mode, 3M kernel): work order as (tile row,
                            // tile col), grouped for L2 reuse of the operand panels
  int32_t* col_exp;         // optional (3M kernel, rect mode): atomicMax of the exponent of
                            // each output column's max |Re| + |Im| (ozaki_colexp_kernel's)
  int* done_cnt;            // optional (triangle mode): per 64-column block, tiles finished
                            // writing into it; host-visible (mapped pinned memory).  A block
                            // is final when its count reaches tiles_m.
};

// Host-side description of one operand (complex view).
struct OperandView {
  const double* base;   // interleaved complex128
  int64_t k;            // reduction length (complex rows)
  int64_t cols;         // columns (M or N extent)
  int64_t ld;           // complex elements between columns
  int64_t batch;        // >= 1
  int64_t bstride;      // complex elements between batches
  int32_t bpos;         // 1: dims (2k, batch, cols); 2: dims (2k, cols, batch)
  const double* rscale = nullptr;  // INT8 engine only: real row factors (x[r, c] * rscale[r])
};

}  // namespace hsb
