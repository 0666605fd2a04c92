// ozaki.cuh — FP64-accurate complex Hermitian rank-k updates on the INT8
// tensor cores (tcgen05.mma kind::i8), by the Chinese-remainder ("Ozaki
// scheme II") integer emulation of a floating-point product.
//
// For C = sum_s L_s^H R_s over complex K_s x N operands (the S and H
// contractions of Algorithm 1, builder.py:91-208):
//
//  1. column scaling: e^L_m = exponent of max over all segments and k of
//     |Re L| + |Im L| in column m (ozaki_colexp_kernel); same for R.
//  2. integer operands: x' = rint(Re X * 2^(b - e_col)), y' = rint(Im X * ...),
//     |x'| + |y'| <= 2^b, i.e. a Gaussian integer z' = x' + i y'.
//  3. split complex arithmetic: every modulus p_i is odd with all prime
//     factors = 1 (mod 4), so -1 has a square root j_i mod p_i and
//        Z_p[i] -> Z_p x Z_p,  z = x + i y -> (x + j y, x - j y)
//     is a ring isomorphism (phi1, phi2); conjugation swaps the components.
//     Two planes per modulus, phi1(z') and phi2(z') as symmetric int8
//     residues (ozaki_residue_kernel), and two real products per modulus,
//     exact in int32 (tcgen05 INT8 GEMM, TMEM accumulators, ozaki_gemm_kernel):
//        L^H R:  phi1(C) = phi2(L)^T phi1(R),  phi2(C) = phi1(L)^T phi2(R)
//        L^T R:  phi1(C) = phi1(L)^T phi1(R),  phi2(C) = phi2(L)^T phi2(R)
//     reduced mod p_i in the epilogue and stored as int8 residues: 2 integer
//     GEMMs per modulus instead of the 3 of a Gauss/3M split.
//  4. reconstruction (ozaki_crt_kernel): Re C = (phi1 + phi2) / 2,
//     Im C = (phi1 - phi2) / (2 j) mod p_i, the constants folded into the
//     explicit CRT weights; scaled by 2^(e^L_m + e^R_n - 2b); alpha/beta,
//     Im(diag) = 0, mirror.
//
// Exactness: every step after the rounding in (2) is exact integer
// arithmetic as long as |Re C'|, |Im C'| < M/2 = prod p_i / 2, which fixes b
// from K_tot: the host picks the fewest moduli with b >= 53 (17 moduli at
// C3 / C4), so every operand keeps a full FP64 mantissa relative to its
// column's max -- the largest entries of each column are exact -- and the only
// error is the rounding of entries smaller than their column max: measured
// ~1e-16 relative Frobenius, the FP64 DMMA engine's level (tests/).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace hsb {

constexpr int kOzMaxMod = 20;
constexpr int kOzMinMod = 11;
constexpr int kOzDefaultBits = 53;  // operand bits by default: a full FP64 mantissa
constexpr int kOzMaxBits = 55;      // |x'| <= 2^55 keeps the residue quotients exact
constexpr int kOzMaxSeg = 4;
constexpr int kOzBM = 256;   // output tile rows   (CTA pair: 128 TMEM lanes each)
constexpr int kOzBN = 256;   // output tile cols   (TMEM columns per accumulator)
constexpr int kOzBK = 128;   // k bytes per stage  (128B swizzle row)
// pairwise coprime, descending, every prime factor = 1 (mod 4)
// (221 = 13 * 17, 205 = 5 * 41); the first n_mod are used.  17 moduli
// (M ~ 2^124.2) give b >= 53-bit operands up to K_tot ~ 2^15.
__host__ __device__ constexpr int oz_mod(int i) {
  switch (i) {
    case 0: return 241;  case 1: return 233;  case 2: return 229;  case 3: return 221;
    case 4: return 205;  case 5: return 197;  case 6: return 193;  case 7: return 181;
    case 8: return 173;  case 9: return 157;  case 10: return 149; case 11: return 137;
    case 12: return 113; case 13: return 109; case 14: return 101; case 15: return 97;
    case 16: return 89;  case 17: return 73;  case 18: return 61;  default: return 53;
  }
}
// j_i: a square root of -1 modulo oz_mod(i), symmetric representative
__host__ __device__ constexpr int oz_sqrtm1(int i) {
  switch (i) {
    case 0: return 64;   case 1: return 89;   case 2: return 107;  case 3: return 21;
    case 4: return 32;   case 5: return 14;   case 6: return 81;   case 7: return 19;
    case 8: return 80;   case 9: return 28;   case 10: return 44;  case 11: return 37;
    case 12: return 15;  case 13: return 33;  case 14: return 10;  case 15: return 22;
    case 16: return 34;  case 17: return 27;  case 18: return 11;  default: return 23;
  }
}

// k extent of a residue plane row (bytes): the reduction length rounded up to
// kOzKpadAlign so every 128-byte TMA row segment of a GEMM operand box is one
// L2 line (HSB_OZ_KPAD for experiments; TMA needs a multiple of 16)
int64_t oz_kpad(int64_t k);

// planes of a residue buffer: [plane][modulus][col][kpad] int8
enum OzPlane { kOzPhi1 = 0, kOzPhi2 = 1 };
constexpr int kOzPlanes = 2;
constexpr int kOzProds = 2;   // integer GEMMs per modulus: phi1(C), phi2(C)

constexpr int kOzMaxSlab = 16;
constexpr int kOzTileBytes = 256 * 256;  // one tile of int8 residues, column-major

// The reduction (the concatenated segments, in 128-byte k chunks) is split into
// slabs of ~16 KB of k: each work item covers one slab of one tile, so the
// operand panels the tiles in flight stream (256 rows x slab) stay L2-resident
// even for long reductions (C4: 46464 bytes of k; DRAM 878 -> 345 GB per H
// GEMM).  Slab s > 0 of a tile adds its residues into slab s-1's in place
// (mod p): its epilogue warps wait on a per-(product, modulus, tile) counter
// that slab s-1's warps bump -- work is claimed in order, so the counted item
// was claimed earlier by a resident CTA pair and the wait always ends.
struct OzGemmParams {
  // maps[prod][seg][side]: 3-D int8 maps {k, cols, modulus}, box {128, 128, 1}
  CUtensorMap map[kOzProds][kOzMaxSeg][2];
  int32_t seg_chunk0[kOzMaxSeg + 1];    // first global k chunk of each segment (+ total)
  int32_t seg_ksteps_last[kOzMaxSeg];   // 32-byte MMA k steps of a segment's last chunk (0: all 4;
                                        // the rest of the chunk is zero padding)
  int32_t slab_chunk0[kOzMaxSlab + 1];  // first global k chunk of each slab (+ total)
  int32_t nseg, nslab;
  int32_t n_mod;
  int32_t n;            // output is n x n (triangle)
  int32_t ntiles;       // tiles of this launch: tile_list[tile0 .. tile0 + ntiles)
  int32_t tile0;
  const int2* tile_list;  // (tile row, tile col) of the 256 x 256 tiles on or below the diagonal
  int8_t* res;          // residues [prod][modulus][tile][256 x 256 col-major]
  int64_t mod_stride;   // bytes between moduli (all tiles of the triangle * kOzTileBytes)
  int64_t prod_stride;  // bytes between products (mod_stride * n_mod)
  int32_t* counter;     // work-stealing counter (zeroed by the launcher)
  int32_t* slab_cnt;    // nslab > 1: per (prod, modulus, tile), epilogue warps finished (zeroed)
  int32_t tiles_total;  // tiles of the whole triangle (slab_cnt / residue indexing)
  // The MMA's A operand (map[..][..][0], TMEM lanes) covers tile column tn,
  // its B operand (map[..][..][1]) tile row tm; residue tiles are stored with
  // the rows of one column contiguous.  Output columns < n and rows < nrows are
  // valid.  Rectangular batched mode (the per-atom V products, contract.cu,
  // rect_gtiles > 0): tile t = (tm, tn) = (atom0 + t / gtiles, t % gtiles); the
  // A operand's k coordinate is shifted by (tm * a_k_per_tm) & ~15 (the atom's
  // rows of the stack, 16-byte aligned for TMA).  Triangle mode: 0, nrows = n.
  int32_t a_k_per_tm;
  int32_t nrows;
  int32_t rect_atom0, rect_gtiles;
  // wide mode (long reductions): work item t = wide_list[t] = (tile row tm,
  // tile col tn, tile index of (tm, tn), tile index of (tm + 1, tn) or -1): the
  // pair computes both row tiles against one shared column panel, one TMEM
  // accumulator each (ntiles = number of wide items)
  const int4* wide_list;
};

struct OzCrtParams {
  const int8_t* res;
  int64_t mod_stride, prod_stride;
  const int32_t* tile_index;  // T x T: tile_list position of tile (tm, tn), tm >= tn
  int32_t T;                  // tiles per side
  int32_t n0;                 // first output column of this launch (grid.y columns follow)
  int32_t n_mod;
  int32_t n;
  int32_t b;                 // operand integer bits
  int32_t conj;              // 1: L^H R ; 0: L^T R
  const int32_t* el;         // column exponents of the left / right operands
  const int32_t* er;
  double alpha_re, alpha_im, beta_re, beta_im;
  double* c;                 // interleaved complex128, column-major
  int64_t ldc;
  uint32_t flags;            // kLowerOnly | kMirror | kZeroImagDiag (zrk.cuh)
  // peer output (hsb_peer_out): element (m, n) goes to slot `rank` of the owner of
  // column n: peer[n / cpr] + ((rank * cpr + n % cpr) * pld + m), instead of c
  double2* const* peer;
  int32_t P, rank;
  int64_t cpr, pld;
};

// V products of the fused H (contract.cu run_ozaki_hv): per-atom left blocks
// L1 = [T_AA | T_AB], L2 = [T_AB^H | T_BB] (256 x 256 per atom, rows shifted by
// (nl a) mod 16, zero padded; T_AA, T_BB completed from their lower
// triangles), so that [V1_a; V2_a] = L1_a^H A_a + L2_a^H B_a.
cudaError_t launch_ozaki_vblocks(const double* taa, const double* tab, const double* tbb, int nl, int64_t na,
                                 double* l1, double* l2, cudaStream_t st);
struct OzVcrtParams {
  const int8_t* res;           // [prod][modulus][tile][256 x 256]: column g_local, row r
  int64_t mod_stride, prod_stride;
  int32_t n_mod;
  int32_t bsum;                // b_left + b_right of the product
  int32_t gtiles, atom0, natoms;
  int32_t nl, ng;
  const int32_t* et;           // [atom * 256 + r] exponents of the L columns
  const int32_t* el;           // [g] exponents of the A / B columns
  double* v1;                  // rows nl * a + r       (r <  nl), leading dimension ldv
  double* v2;                  // rows nl * a + r - nl  (r >= nl)
  int64_t ldv;
  int32_t* er;                 // [g] atomicMax of the V column exponents
};
cudaError_t launch_ozaki_vcrt(const OzVcrtParams& p, cudaStream_t st);

// rscale (optional): the operand is diag(rscale) x (S's U-normed B without a
// materialised copy; the product rounds exactly as diag_scale_kernel's)
cudaError_t launch_ozaki_colexp(const double* x, int64_t ldx, int64_t k, int64_t cols, int32_t* exp_out,
                                cudaStream_t st, const double* rscale = nullptr);
cudaError_t launch_ozaki_init_exp(int32_t* e, int64_t n, cudaStream_t st);
// e[c] = exponent of the column max over a, diag(u) b and (with_b) b (written, not max-ed)
cudaError_t launch_ozaki_colexp_ab(const double* a, const double* b, int64_t ld, int64_t k, int64_t cols,
                                   const double* u, int32_t* exp_out, cudaStream_t st, bool with_b);
// one residue-plane source: x (ldx, k rows of complex) scaled per column by
// 2^(b - col_exp), optionally by rscale per row, into out[plane][mod][col][kpad]
constexpr int kOzResMaxSrc = 4;
struct OzResSrc {
  const double* x;
  int64_t ldx, k;
  const int32_t* col_exp;
  const double* rscale;
  int8_t* out;
  int64_t kpad;
};
// up to kOzResMaxSrc sources of the same column count in one launch
cudaError_t launch_ozaki_residues_batch(const OzResSrc* srcs, int nsrc, int64_t cols, int b, int n_mod,
                                        cudaStream_t st);
cudaError_t launch_ozaki_residues(const double* x, int64_t ldx, int64_t k, int64_t cols, const int32_t* col_exp,
                                  int b, int n_mod, int8_t* out, int64_t kpad, cudaStream_t st, const double* rscale = nullptr);
cudaError_t launch_ozaki_gemm(const OzGemmParams& p, cudaStream_t st);
cudaError_t launch_ozaki_crt(const OzCrtParams& p, cudaStream_t st);
// the reconstruction table of n_mod moduli: w[part][i][limb], fl(M); 0 on success
int oz_crt_table_host(int n_mod, double* w, double* m);
cudaError_t launch_ozaki_crt_cols(const OzCrtParams& p, int64_t ncols, cudaStream_t st);

}  // namespace hsb
