// ozaki_res.cuh — device helpers of the INT8 engine's operand residues,
// shared by the residue kernel (ozaki.cu) and the matching-coefficient kernel
// that emits A's and UB's residue planes directly (match_kernel.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ozaki.cuh"

namespace hsb {

// 2^e for |e| <= 1022 from the exponent bits
__device__ __forceinline__ double pow2i(int e) { return __longlong_as_double(static_cast<long long>(e + 1023) << 52); }

// ---- residues by byte dot products (IDP4A) --------------------------------
// An operand integer x' (|x'| <= 2^55, exact in FP64) is split once per element
// into two 32-bit words, x' = (hi - 2^31) 2^32 + lo with lo, hi unsigned, i.e.
// eight unsigned bytes; then for every modulus
//     x' mod p  =  sum_d byte_d (2^(8d) mod p)  -  (2^63 mod p)        (mod p)
// is two dp4a.u32.s32 against packed symmetric weights, and the split-complex
// planes phi1,2 = x' +- j y' fold j into y's weights: X + Y and X - Y with
// |X|, |Y| <= 8 * 255 * 120 + 120 < 2^18.  Each is reduced to its symmetric
// residue by an exact integer quotient (oz_sym_reduce).  Per element and
// modulus ~11 integer instructions, no FP64 or conversion-pipe work (the
// FP64 magic-quotient form issued ~32).
__host__ __device__ constexpr int oz_pow2_mod(int e, int p) {
  int r = 1 % p;
  for (int i = 0; i < e; ++i) r = (2 * r) % p;
  return r;
}
__host__ __device__ constexpr int oz_symrep(long long v, int p) {
  long long r = v % p;
  if (r < 0) r += p;
  return static_cast<int>(r > p / 2 ? r - p : r);
}
// packed int8 weights of bytes d0 .. d0+3: (mult * 2^(8d)) mod p, symmetric
__host__ __device__ constexpr uint32_t oz_wpack(int i, int mult, int d0) {
  uint32_t w = 0;
  for (int d = 0; d < 4; ++d)
    w |= (static_cast<uint32_t>(oz_symrep(static_cast<long long>(mult) * oz_pow2_mod(8 * (d0 + d), oz_mod(i)),
                                          oz_mod(i))) & 0xffu) << (8 * d);
  return w;
}
// -(mult * 2^63) mod p, symmetric: the bias of hi
__host__ __device__ constexpr int oz_bias(int i, int mult) {
  return oz_symrep(-static_cast<long long>(mult) * oz_pow2_mod(63, oz_mod(i)), oz_mod(i));
}
// rn(2^32 / p): the quotient multiplier of oz_sym_reduce
__host__ __device__ constexpr long long oz_qmul(int i) { return ((1ll << 32) + oz_mod(i) / 2) / oz_mod(i); }

__device__ __forceinline__ int dp4a_us(uint32_t a, uint32_t b, int c) {
  int d;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
// symmetric residue of |v| < 2^19 modulo p: q = floor((v m + 2^31) / 2^32) =
// rn(v / p) exactly (m = rn(2^32 / p) errs by <= 1/2, so v m / 2^32 is within
// |v| 2^-33 <= 2^-14 of v / p, which is >= 1/(2p) > 2^-9 from any half-integer)
template <int I>
__device__ __forceinline__ int oz_sym_reduce(int v) {
  const int q = static_cast<int>((static_cast<long long>(v) * oz_qmul(I) + (1ll << 31)) >> 32);
  return v - oz_mod(I) * q;
}
// exact x' = (hi - 2^31) 2^32 + lo of an exactly-integer double |x| <= 2^55:
// h = floor(x 2^-32) by a round-down add of the 1.5 * 2^52 magic constant (x 2^-32
// is exact), l = x - h 2^32 in [0, 2^32) exactly, both read from the low
// mantissa word.  (Round-to-nearest would give l = +2^31 on ties, which does
// not fit the word.)
__device__ __forceinline__ void oz_split(double x, uint32_t& lo, uint32_t& hi) {
  constexpr double M = 6755399441055744.0;  // 1.5 * 2^52
  const double hm = __dadd_rd(x * 2.3283064365386963e-10, M);  // M + floor(x 2^-32)
  lo = static_cast<uint32_t>(__double2loint(fma(-(hm - M), 4294967296.0, x) + M));
  hi = static_cast<uint32_t>(__double2loint(hm)) + 0x80000000u;
}
template <int I>
__device__ __forceinline__ void oz_planes(uint32_t xl, uint32_t xh, uint32_t yl, uint32_t yh, int& u, int& w) {
  const int X = dp4a_us(xh, oz_wpack(I, 1, 4), dp4a_us(xl, oz_wpack(I, 1, 0), oz_bias(I, 1)));
  const int Y = dp4a_us(yh, oz_wpack(I, oz_sqrtm1(I), 4), dp4a_us(yl, oz_wpack(I, oz_sqrtm1(I), 0), oz_bias(I, oz_sqrtm1(I))));
  u = oz_sym_reduce<I>(X + Y);  // phi1 = x' + j y'
  w = oz_sym_reduce<I>(X - Y);  // phi2 = x' - j y'
}
// residues of 4 consecutive rows, every modulus, written straight to the
// planes [plane][modulus][col][kpad] (o0 = plane 0, modulus 0, this column and row)
template <int NM, int I = 0>
__device__ __forceinline__ void oz_residue_planes_global(const uint32_t (&xl)[4], const uint32_t (&xh)[4],
                                                         const uint32_t (&yl)[4], const uint32_t (&yh)[4],
                                                         int8_t* o0, int64_t plane_stride, int64_t mod_stride) {
  if constexpr (I < NM) {
    int u[4], w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) oz_planes<I>(xl[j], xh[j], yl[j], yh[j], u[j], w[j]);
    const auto pack = [](const int* v) {
      return __byte_perm(__byte_perm(v[0], v[1], 0x40), __byte_perm(v[2], v[3], 0x40), 0x5410);
    };
    *reinterpret_cast<uint32_t*>(o0) = pack(u);
    *reinterpret_cast<uint32_t*>(o0 + plane_stride) = pack(w);
    oz_residue_planes_global<NM, I + 1>(xl, xh, yl, yh, o0 + mod_stride, plane_stride, mod_stride);
  }
}

}  // namespace hsb
