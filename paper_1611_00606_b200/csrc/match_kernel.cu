// match_kernel.cu — FLAPW matching coefficients A^alpha_lm(k+G), B^alpha_lm(k+G).
//
// North-star part (1); no reference implementation exists (A, B are random
// inputs in probgen.py:131-132).  Definition: PAPER.md:226-241 (Rayleigh
// expansion of exp(i K.r) matched in value and slope at the muffin-tin
// radius), conventions of SURVEY.md 8(a) row A0, restated on the CPU in
// oracle/matching.py:
//
//   c_lm = (4 pi / sqrt(Omega)) i^l exp(i K.tau_alpha) conj(Y_lm(K^))
//   A    = c [ j_l(KR) udot'_l - K j_l'(KR) udot_l ] / D_l
//   B    = c [ K j_l'(KR) u_l  - j_l(KR) u'_l      ] / D_l,   D_l = u udot' - udot u'
//
// One CTA per kMatchCols G columns.  The per-column special functions are
// computed once into shared memory (Y_lm by the normalised associated-Legendre
// recurrence, one lane per m; j_l by upward recurrence for x >= lmax+1,
// Miller's downward recurrence below that, a 3-term series for x < 1e-3;
// structure phases by sincos), then all threads stream the n_atoms * N_L rows
// of the columns of A and B with coalesced 16-byte stores: the kernel is
// HBM-write bound (2 * K * 16 bytes per column).
#include <cuda_runtime.h>
#include <stdint.h>

#include "match.cuh"
#include "ozaki_res.cuh"

namespace hsb {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// j_0..j_{nmax} at x >= 0 into j[] (nmax <= kMaxL + 1).
__device__ void spherical_bessel(double x, int nmax, double* j) {
  if (x == 0.0) {
    j[0] = 1.0;
    for (int l = 1; l <= nmax; ++l) j[l] = 0.0;
    return;
  }
  if (x < 1e-3) {  // j_l = x^l/(2l+1)!! [1 - x^2/(2(2l+3)) + x^4/(8(2l+3)(2l+5)) - ...]
    double xl = 1.0, df = 1.0;  // x^l, (2l+1)!!
    const double x2 = x * x;
    for (int l = 0; l <= nmax; ++l) {
      if (l > 0) {
        xl *= x;
        df *= (2 * l + 1);
      }
      const double a3 = 2 * l + 3, a5 = 2 * l + 5, a7 = 2 * l + 7;
      const double s = 1.0 - x2 / (2.0 * a3) * (1.0 - x2 / (4.0 * a5) * (1.0 - x2 / (6.0 * a7)));
      j[l] = xl / df * s;
    }
    return;
  }
  double sn, cs;
  sincos(x, &sn, &cs);
  const double j0 = sn / x;
  const double j1 = sn / (x * x) - cs / x;
  if (x >= nmax) {  // upward recurrence is stable for l < x
    j[0] = j0;
    if (nmax >= 1) j[1] = j1;
    for (int l = 1; l < nmax; ++l) j[l + 1] = (2 * l + 1) / x * j[l] - j[l - 1];
    return;
  }
  // Miller: downward from well above max(nmax, x), normalised by the larger of j0, j1
  const int start = nmax + 24 + static_cast<int>(x);
  double fp1 = 0.0, f = 1e-280;
  for (int l = start; l > nmax; --l) {  // f = f_l, fp1 = f_{l+1}
    const double fm1 = (2 * l + 1) / x * f - fp1;
    fp1 = f;
    f = fm1;
    if (fabs(f) > 1e250) {
      f *= 1e-250;
      fp1 *= 1e-250;
    }
  }
  // now f = f_nmax, fp1 = f_{nmax+1}
  j[nmax] = f;
  double cur = f, nxt = fp1;
  for (int l = nmax; l > 0; --l) {
    const double prev = (2 * l + 1) / x * cur - nxt;
    nxt = cur;
    cur = prev;
    j[l - 1] = cur;
    if (fabs(cur) > 1e250) {
      for (int q = l - 1; q <= nmax; ++q) j[q] *= 1e-250;
      cur *= 1e-250;
      nxt *= 1e-250;
    }
  }
  const double scale = (fabs(j0) >= fabs(j1)) ? j0 / j[0] : j1 / j[1];
  for (int l = 0; l <= nmax; ++l) j[l] *= scale;
}

// kMatchCols G columns per CTA: the special functions of the kMatchCols
// columns are computed concurrently (warps 4..7: Y_lm, one column at a time each;
// warps 0..3: radial factors and structure phases of all of them), then all
// threads stream the kMatchCols columns.  At C3 (K = 3872 rows) one column is
// only 124 KB of stores, so one column per CTA left the HBM 43 % idle behind
// the per-column prologue.
constexpr int kMatchCols = 8;
constexpr int kMatchThreads = 256;

// NM = 0: A and B only; NM > 0: also the residue planes of A and UB (MatchRes)
template <int NM>
__global__ void __launch_bounds__(kMatchThreads) match_coeffs_kernel(MatchParams p, double2* __restrict__ A,
                                                                      double2* __restrict__ B, MatchRes res) {
  extern __shared__ double smem_d[];
  const int lmax = p.lmax, nlm = (lmax + 1) * (lmax + 1), nl1 = lmax + 1;
  double2* ys = reinterpret_cast<double2*>(smem_d);                     // [col][nlm]: pre i^l conj(Y_lm)
  double2* phase = ys + kMatchCols * nlm;                               // [col][n_atoms]
  double* fa = reinterpret_cast<double*>(phase + kMatchCols * p.n_atoms);  // [col][n_types * (lmax+1)]
  double* fb = fa + kMatchCols * p.n_types * nl1;
  unsigned char* lidx = reinterpret_cast<unsigned char*>(fb + kMatchCols * p.n_types * nl1);  // nlm

  const int64_t g0 = static_cast<int64_t>(blockIdx.x) * kMatchCols;
  const int ncols = static_cast<int>(p.n_g - g0 < kMatchCols ? p.n_g - g0 : kMatchCols);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto kvec = [&](int c, double& kx, double& ky, double& kz) {
    const int* gv = p.gvec + 3 * (g0 + c);
    const double f0 = p.kpt[0] + gv[0], f1 = p.kpt[1] + gv[1], f2 = p.kpt[2] + gv[2];
    kx = f0 * p.recip[0] + f1 * p.recip[3] + f2 * p.recip[6];
    ky = f0 * p.recip[1] + f1 * p.recip[4] + f2 * p.recip[7];
    kz = f0 * p.recip[2] + f1 * p.recip[5] + f2 * p.recip[8];
  };

  if (warp < 4) {
    // ---- radial factors per (column, type, l)
    for (int i = tid; i < ncols * p.n_types; i += 128) {
      const int c = i / p.n_types, t = i - c * p.n_types;
      double kx, ky, kz;
      kvec(c, kx, ky, kz);
      const double kn = sqrt(kx * kx + ky * ky + kz * kz);
      double j[kMaxL + 2];
      spherical_bessel(kn * p.rmt[t], lmax + 1, j);
      for (int l = 0; l <= lmax; ++l) {
        const double dj = (l == 0) ? -j[1] : (l * j[l - 1] - (l + 1) * j[l + 1]) / (2 * l + 1);
        const double* r = p.radial + (t * nl1 + l) * 4;  // u, u', udot, udot'
        const double d = r[0] * r[3] - r[2] * r[1];
        fa[(c * p.n_types + t) * nl1 + l] = (j[l] * r[3] - kn * dj * r[2]) / d;
        fb[(c * p.n_types + t) * nl1 + l] = (kn * dj * r[0] - j[l] * r[1]) / d;
      }
    }
    // ---- structure phases per (column, atom)
    for (int i = tid; i < ncols * p.n_atoms; i += 128) {
      const int c = i / p.n_atoms, a = i - c * p.n_atoms;
      double kx, ky, kz;
      kvec(c, kx, ky, kz);
      const double* tau = p.tau + 3 * a;
      double sn, cs;
      sincos(kx * tau[0] + ky * tau[1] + kz * tau[2], &sn, &cs);
      phase[c * p.n_atoms + a] = make_double2(cs, sn);
    }
    for (int L = tid; L < nlm; L += 128) {
      int l = 0;
      while ((l + 1) * (l + 1) <= L) ++l;
      lidx[L] = static_cast<unsigned char>(l);
    }
  } else {
    // ---- spherical harmonics: warp 4 + w handles columns w, w + 4, ...; lane m
    // runs the l recurrence for m
    for (int c = warp - 4; c < ncols; c += 4) {
    const int m = lane;
    if (m <= lmax) {
      double kx, ky, kz;
      kvec(c, kx, ky, kz);
      const double rho = sqrt(kx * kx + ky * ky);
      const double kn = sqrt(kx * kx + ky * ky + kz * kz);
      const double ct = kn > 0.0 ? kz / kn : 1.0;
      const double st = kn > 0.0 ? rho / kn : 0.0;
      const double cp = rho > 0.0 ? kx / rho : 1.0, sp = rho > 0.0 ? ky / rho : 0.0;
      double2 em = make_double2(1.0, 0.0);  // e^{i m phi}
      for (int q = 0; q < m; ++q) em = cmul(em, make_double2(cp, sp));
      double pmm = 0.28209479177387814;  // P_mm, normalised, Condon-Shortley phase; 1/sqrt(4 pi)
      for (int q = 1; q <= m; ++q) pmm *= -sqrt((2.0 * q + 1.0) / (2.0 * q)) * st;
      double plm2 = 0.0, plm1 = pmm;
      double2* yc = ys + c * nlm;
      for (int l = m; l <= lmax; ++l) {
        double plm;
        if (l == m) {
          plm = pmm;
        } else if (l == m + 1) {
          plm = sqrt(2.0 * m + 3.0) * ct * pmm;
        } else {
          const double a = sqrt((4.0 * l * l - 1.0) / (double(l) * l - double(m) * m));
          const double b = sqrt((double(l - 1) * (l - 1) - double(m) * m) / (4.0 * (l - 1) * (l - 1) - 1.0));
          plm = a * (ct * plm1 - b * plm2);
        }
        if (l > m) {
          plm2 = plm1;
          plm1 = plm;
        }
        // Y_lm = plm e^{i m phi};  Y_{l,-m} = (-1)^m conj(Y_lm)
        const double2 y = make_double2(plm * em.x, plm * em.y);
        const int lr = l & 3;  // i^l
        const double2 il = lr == 0 ? make_double2(1, 0) : lr == 1 ? make_double2(0, 1)
                         : lr == 2 ? make_double2(-1, 0) : make_double2(0, -1);
        const double2 cy = cmul(il, make_double2(y.x, -y.y));  // i^l conj(Y_lm)
        yc[l * l + l + m] = make_double2(p.pre * cy.x, p.pre * cy.y);
        if (m > 0) {
          const double sgn = (m & 1) ? -1.0 : 1.0;  // conj(Y_{l,-m}) = (-1)^m Y_lm
          const double2 cyn = cmul(il, make_double2(sgn * y.x, sgn * y.y));
          yc[l * l + l - m] = make_double2(p.pre * cyn.x, p.pre * cyn.y);
        }
      }
    }
    }
  }
  __syncthreads();

  // ---- stream the columns: rows (atom, L), 16-byte coalesced stores
  const int64_t K = static_cast<int64_t>(p.n_atoms) * nlm;
  __shared__ double red[kMatchThreads / 32];
  for (int c = 0; c < ncols; ++c) {
    double2* colA = A + (g0 + c) * p.ld;
    double2* colB = B + (g0 + c) * p.ld;
    const double2* yc = ys + c * nlm;
    const double2* ph = phase + c * p.n_atoms;
    const double* fac = fa + c * p.n_types * nl1;
    const double* fbc = fb + c * p.n_types * nl1;
    auto coeffs = [&](int64_t r, double2& va, double2& vb) {
      const int a = static_cast<int>(r / nlm), L = static_cast<int>(r - static_cast<int64_t>(a) * nlm);
      const int t = p.type_of[a], l = lidx[L];
      const double2 base = cmul(yc[L], ph[a]);
      const double ca = fac[t * nl1 + l], cb = fbc[t * nl1 + l];
      va = make_double2(base.x * ca, base.y * ca);
      vb = make_double2(base.x * cb, base.y * cb);
    };
    double mx = 0.0;
    for (int64_t r = tid; r < K; r += kMatchThreads) {
      double2 va, vb;
      coeffs(r, va, vb);
      colA[r] = va;
      colB[r] = vb;
      if constexpr (NM > 0) {  // fl(u b), as diag_scale_kernel rounds it
        const double u = __ldg(res.u + r);
        mx = fmax(mx, fmax(fabs(va.x) + fabs(va.y), fabs(u * vb.x) + fabs(u * vb.y)));
      }
    }
    if constexpr (NM > 0) {
      // the column's exponent (frexp of the max: max < 2^e), then its residues
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) red[warp] = mx;
      __syncthreads();
      double m = red[0];
#pragma unroll
      for (int w = 1; w < kMatchThreads / 32; ++w) m = fmax(m, red[w]);
      int e = 0;
      frexp(m, &e);
      if (tid == 0) res.col_exp[g0 + c] = e;
      const int sh = res.b - e;
      const double s1 = pow2i(sh / 2), s2 = pow2i(sh - sh / 2);
      const int64_t mod_stride = p.n_g * res.kpad, plane_stride = NM * mod_stride;
      for (int64_t r0 = 4 * tid; r0 < res.kpad; r0 += 4 * kMatchThreads) {
        uint32_t al[4], ah[4], bl[4], bh[4], ul[4], uh[4], vl[4], vh[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          double ar = 0.0, ai = 0.0, ur = 0.0, ui = 0.0;
          if (r0 + j < K) {
            double2 va, vb;
            coeffs(r0 + j, va, vb);
            const double u = __ldg(res.u + r0 + j);
            ar = rint((va.x * s1) * s2);
            ai = rint((va.y * s1) * s2);
            ur = rint(((u * vb.x) * s1) * s2);
            ui = rint(((u * vb.y) * s1) * s2);
          }
          oz_split(ar, al[j], ah[j]);
          oz_split(ai, bl[j], bh[j]);
          oz_split(ur, ul[j], uh[j]);
          oz_split(ui, vl[j], vh[j]);
        }
        const int64_t off = (g0 + c) * res.kpad + r0;
        oz_residue_planes_global<NM>(al, ah, bl, bh, res.res_a + off, plane_stride, mod_stride);
        oz_residue_planes_global<NM>(ul, uh, vl, vh, res.res_ub + off, plane_stride, mod_stride);
      }
      __syncthreads();  // red[] is rewritten by the next column
    }
  }
}

size_t match_smem_bytes(const MatchParams& p) {
  const size_t nlm = static_cast<size_t>(p.lmax + 1) * (p.lmax + 1);
  return kMatchCols * (nlm * 16 + static_cast<size_t>(p.n_atoms) * 16 +
                       2 * static_cast<size_t>(p.n_types) * (p.lmax + 1) * 8) +
         nlm + 16;
}

template <int NM>
static cudaError_t launch_match(const MatchParams& p, double* A, double* B, const MatchRes& r, cudaStream_t st) {
  const size_t smem = match_smem_bytes(p);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(match_coeffs_kernel<NM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const int64_t blocks = (p.n_g + kMatchCols - 1) / kMatchCols;
  if (blocks <= 0) return cudaSuccess;
  match_coeffs_kernel<NM><<<static_cast<unsigned>(blocks), kMatchThreads, smem, st>>>(
      p, reinterpret_cast<double2*>(A), reinterpret_cast<double2*>(B), r);
  return cudaGetLastError();
}

cudaError_t launch_match_coeffs(const MatchParams& p, double* A, double* B, cudaStream_t st) {
  return launch_match<0>(p, A, B, MatchRes{}, st);
}

cudaError_t launch_match_coeffs_res(const MatchParams& p, double* A, double* B, const MatchRes& r, cudaStream_t st) {
  if (r.kpad % 16 != 0 || r.kpad < static_cast<int64_t>(p.n_atoms) * (p.lmax + 1) * (p.lmax + 1))
    return cudaErrorInvalidValue;
  switch (r.n_mod) {
#define HSB_MATCH_RES(NM) \
  case NM:                \
    return launch_match<NM>(p, A, B, r, st);
    HSB_MATCH_RES(15) HSB_MATCH_RES(16) HSB_MATCH_RES(17) HSB_MATCH_RES(18) HSB_MATCH_RES(19) HSB_MATCH_RES(20)
#undef HSB_MATCH_RES
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace hsb
