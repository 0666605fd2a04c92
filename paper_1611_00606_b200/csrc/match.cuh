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
size_t match_smem_bytes(const MatchParams& p);

}  // namespace hsb
