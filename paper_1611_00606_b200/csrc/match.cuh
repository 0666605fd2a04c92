// match.cuh — matching-coefficient kernel parameters (see match_kernel.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace hsb {

constexpr int kMaxL = 31;  // one lane per m in the Y_lm recurrence

struct MatchParams {
  const int32_t* gvec;    // device, n_g x 3 integer G (reciprocal-lattice coordinates)
  const double* tau;      // device, n_atoms x 3 Cartesian positions
  const int32_t* type_of; // device, n_atoms
  const double* rmt;      // device, n_types
  const double* radial;   // device, n_types x (lmax+1) x 4: u, u', udot, udot' at R_t
  double kpt[3];          // k in reciprocal-lattice coordinates
  double recip[9];        // reciprocal lattice vectors as rows (1/bohr)
  double pre;             // 4 pi / sqrt(Omega)
  int64_t n_g;
  int64_t ld;             // complex elements between output columns (>= n_atoms * N_L)
  int32_t n_atoms, n_types, lmax, pad;
};

cudaError_t launch_match_coeffs(const MatchParams& p, double* A, double* B, cudaStream_t st);

// Matching coefficients plus the INT8 engine's left operands of S and H in one
// pass: each CTA owns whole G columns, so it also takes the
// column's exponent e = max over A and fl(u B) (|Re| + |Im|) and writes the
// residue planes of A and of UB = diag(u) B at b bits, n_mod moduli
// ([plane][modulus][col][kpad] int8), exactly as ozaki_colexp_ab +
// ozaki_residue_kernel would from the stored stacks.
struct MatchRes {
  const double* u;   // device, n_atoms * N_L row norms
  int32_t* col_exp;  // device, n_g: the shared left exponent
  int8_t* res_a;     // planes of A
  int8_t* res_ub;    // planes of UB
  int64_t kpad;
  int32_t b, n_mod;
};
cudaError_t launch_match_coeffs_res(const MatchParams& p, double* A, double* B, const MatchRes& r, cudaStream_t st);
size_t match_smem_bytes(const MatchParams& p);

}  // namespace hsb
