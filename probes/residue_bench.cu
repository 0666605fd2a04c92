// residue_bench.cu — variants of the INT8 engine's residue kernel
// (csrc/ozaki.cu ozaki_residue_kernel) on the C3 operand shape: bit-identical
// output against the library kernel's formulation, and CUDA-event times.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I. probes/residue_bench.cu -o probes/residue_bench
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "paper_1611_00606_b200/csrc/ozaki.cuh"

using namespace hsb;

__constant__ double c_inv[kOzMaxMod];

__device__ __forceinline__ double pow2i(int e) { return __longlong_as_double(static_cast<long long>(e + 1023) << 52); }
__device__ __forceinline__ int sym_mod_magic(double v, double p, double inv_p) {
  constexpr double M = 6755399441055744.0;
  const double q = fma(v, inv_p, M) - M;
  return static_cast<int>(__double2loint(fma(-p, q, v) + M));
}
__device__ __forceinline__ int sym_mod_small(int v, int p, float inv_p) {
  return v - p * __float2int_rn(__int2float_rn(v) * inv_p);
}
__device__ __forceinline__ uint32_t pack4(int a, int b, int c, int d) {
  return __byte_perm(__byte_perm(a, b, 0x40), __byte_perm(c, d, 0x40), 0x5410);
}

// V0/V1: the library formulation, KPT consecutive k per thread
template <int NM, int KPT, int MINB>
__global__ void __launch_bounds__(128, MINB) res_dp(const double2* __restrict__ x, int64_t ldx, int64_t k, int64_t cols,
                                                    const int32_t* __restrict__ col_exp, int b, int8_t* __restrict__ out,
                                                    int64_t kpad) {
  const int64_t k0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * KPT;
  if (k0 >= kpad) return;
  const int64_t mod_stride = cols * kpad;
  const int64_t plane_stride = NM * mod_stride;
  for (int64_t c = blockIdx.y; c < cols; c += gridDim.y) {
    const int sh = b - __ldg(col_exp + c);
    const double s1 = pow2i(sh / 2), s2 = pow2i(sh - sh / 2);
    double xr[KPT], xi[KPT];
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      if (k0 + j < k) {
        const double2 v = x[c * ldx + k0 + j];
        xr[j] = rint((v.x * s1) * s2);
        xi[j] = rint((v.y * s1) * s2);
      } else {
        xr[j] = xi[j] = 0.0;
      }
    }
    int8_t* o0 = out + c * kpad + k0;
    int8_t* o1 = o0 + plane_stride;
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      const double p = oz_mod(i), inv = c_inv[i];
      const int jm = oz_sqrtm1(i);
      const float invf = 1.0f / oz_mod(i);
      int u[KPT], w[KPT];
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const int rr = sym_mod_magic(xr[j], p, inv);
        const int t = jm * sym_mod_magic(xi[j], p, inv);
        u[j] = sym_mod_small(rr + t, oz_mod(i), invf);
        w[j] = sym_mod_small(rr - t, oz_mod(i), invf);
      }
      if constexpr (KPT == 8) {
        *reinterpret_cast<int2*>(o0) = make_int2(pack4(u[0], u[1], u[2], u[3]), pack4(u[4], u[5], u[6], u[7]));
        *reinterpret_cast<int2*>(o1) = make_int2(pack4(w[0], w[1], w[2], w[3]), pack4(w[4], w[5], w[6], w[7]));
      } else {
        *reinterpret_cast<uint32_t*>(o0) = pack4(u[0], u[1], u[2], u[3]);
        *reinterpret_cast<uint32_t*>(o1) = pack4(w[0], w[1], w[2], w[3]);
      }
      o0 += mod_stride;
      o1 += mod_stride;
    }
  }
}

// V2: FP32 arithmetic per modulus.  x' = xh 2^22 + xl (|xh|, |xl| <= 2^21,
// exact floats); x' mod p = (xh mod p) c + xl mod p with c = 2^22 mod p.
// q = rn(v * fl(1/p)) through the 1.5 * 2^23 magic constant (one rounding of
// the exact product); |v| <= 2^22 keeps the error below 1/(4p), half the
// distance of v/p from a half-integer.  The result's float bits + magic hold
// the int8 two's complement in the low byte.
__device__ __forceinline__ float fmod_sym(float v, float p, float inv) {
  constexpr float M = 12582912.0f;
  const float q = __fadd_rn(__fmaf_rn(v, inv, M), -M);
  return __fmaf_rn(-p, q, v);
}
template <int NM, int KPT, int MINB>
__global__ void __launch_bounds__(128, MINB) res_sp(const double2* __restrict__ x, int64_t ldx, int64_t k, int64_t cols,
                                                    const int32_t* __restrict__ col_exp, int b, int8_t* __restrict__ out,
                                                    int64_t kpad) {
  const int64_t k0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * KPT;
  if (k0 >= kpad) return;
  const int64_t mod_stride = cols * kpad;
  const int64_t plane_stride = NM * mod_stride;
  for (int64_t c = blockIdx.y; c < cols; c += gridDim.y) {
    const int sh = b - __ldg(col_exp + c);
    const double s1 = pow2i(sh / 2), s2 = pow2i(sh - sh / 2);
    float xh[KPT], xl[KPT], yh[KPT], yl[KPT];
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      double2 v = make_double2(0.0, 0.0);
      if (k0 + j < k) v = x[c * ldx + k0 + j];
      const double a = rint((v.x * s1) * s2), bb = rint((v.y * s1) * s2);
      const double ah = rint(a * 0x1p-22), bh = rint(bb * 0x1p-22);
      xh[j] = static_cast<float>(ah);
      xl[j] = static_cast<float>(fma(-ah, 0x1p22, a));
      yh[j] = static_cast<float>(bh);
      yl[j] = static_cast<float>(fma(-bh, 0x1p22, bb));
    }
    int8_t* o0 = out + c * kpad + k0;
    int8_t* o1 = o0 + plane_stride;
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      const float p = oz_mod(i), inv = 1.0f / oz_mod(i);
      const float jm = oz_sqrtm1(i);
      const float c22 = static_cast<float>(((1 << 22) % oz_mod(i) + oz_mod(i) / 2) % oz_mod(i) - oz_mod(i) / 2);
      int u[KPT], w[KPT];
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const float rr = fmod_sym(__fmaf_rn(fmod_sym(xh[j], p, inv), c22, xl[j]), p, inv);
        const float ri = fmod_sym(__fmaf_rn(fmod_sym(yh[j], p, inv), c22, yl[j]), p, inv);
        u[j] = __float_as_int(fmod_sym(__fmaf_rn(jm, ri, rr), p, inv) + 12582912.0f);
        w[j] = __float_as_int(fmod_sym(__fmaf_rn(-jm, ri, rr), p, inv) + 12582912.0f);
      }
      if constexpr (KPT == 8) {
        *reinterpret_cast<int2*>(o0) = make_int2(pack4(u[0], u[1], u[2], u[3]), pack4(u[4], u[5], u[6], u[7]));
        *reinterpret_cast<int2*>(o1) = make_int2(pack4(w[0], w[1], w[2], w[3]), pack4(w[4], w[5], w[6], w[7]));
      } else {
        *reinterpret_cast<uint32_t*>(o0) = pack4(u[0], u[1], u[2], u[3]);
        *reinterpret_cast<uint32_t*>(o1) = pack4(w[0], w[1], w[2], w[3]);
      }
      o0 += mod_stride;
      o1 += mod_stride;
    }
  }
}

int main() {
  constexpr int NM = 13;
  const int64_t k = 3872, cols = 8000, kpad = (k + 15) / 16 * 16;
  const int b = 41;
  std::vector<double> hx(2 * k * cols);
  std::mt19937_64 rng(3);
  std::normal_distribution<double> nd;
  for (auto& v : hx) v = nd(rng) * std::exp(nd(rng) * 3);
  std::vector<int32_t> he(cols);
  for (int64_t c = 0; c < cols; ++c) {
    double m = 0;
    for (int64_t r = 0; r < k; ++r) m = std::max(m, std::fabs(hx[2 * (c * k + r)]) + std::fabs(hx[2 * (c * k + r) + 1]));
    int ex;
    std::frexp(m, &ex);
    he[c] = ex;
  }
  double inv[kOzMaxMod];
  for (int i = 0; i < kOzMaxMod; ++i) inv[i] = 1.0 / oz_mod(i);
  cudaMemcpyToSymbol(c_inv, inv, sizeof(inv));
  double2* dx;
  int32_t* de;
  int8_t *d0, *d1;
  const size_t ob = 2ull * NM * cols * kpad;
  cudaMalloc(&dx, hx.size() * 8);
  cudaMalloc(&de, cols * 4);
  cudaMalloc(&d0, ob);
  cudaMalloc(&d1, ob);
  cudaMemcpy(dx, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(de, he.data(), cols * 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto grid = [&](int kpt) { return dim3(static_cast<unsigned>((kpad / kpt + 127) / 128), static_cast<unsigned>(cols)); };
  auto time_it = [&](auto launch) {
    for (int r = 0; r < 3; ++r) launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 20;
  };
  const double bytes = 16.0 * k * cols + ob;
  float t = time_it([&] { res_dp<NM, 8, 3><<<grid(8), 128>>>(dx, k, k, cols, de, b, d0, kpad); });
  printf("dp  KPT 8 minB 3: %.3f ms  %.2f TB/s\n", t, bytes / t / 1e9);
  std::vector<int8_t> ref(ob), got(ob);
  cudaMemcpy(ref.data(), d0, ob, cudaMemcpyDeviceToHost);
  auto check = [&](const char* name, float tt) {
    cudaMemcpy(got.data(), d1, ob, cudaMemcpyDeviceToHost);
    size_t bad = 0;
    for (size_t i = 0; i < ob; ++i) {
      // residue classes must agree (representatives may differ by p)
      const int64_t plane = i / (NM * cols * kpad), mod = (i / (cols * kpad)) % NM;
      (void)plane;
      const int p = oz_mod(static_cast<int>(mod));
      if (((ref[i] - got[i]) % p + p) % p != 0) ++bad;
    }
    printf("%-18s %.3f ms  %.2f TB/s  mismatches %zu\n", name, tt, bytes / tt / 1e9, bad);
    cudaMemset(d1, 0, ob);
  };
  check("dp KPT 4 minB 6", time_it([&] { res_dp<NM, 4, 6><<<grid(4), 128>>>(dx, k, k, cols, de, b, d1, kpad); }));
  check("dp KPT 4 minB 4", time_it([&] { res_dp<NM, 4, 4><<<grid(4), 128>>>(dx, k, k, cols, de, b, d1, kpad); }));
  check("sp KPT 8 minB 3", time_it([&] { res_sp<NM, 8, 3><<<grid(8), 128>>>(dx, k, k, cols, de, b, d1, kpad); }));
  check("sp KPT 8 minB 4", time_it([&] { res_sp<NM, 8, 4><<<grid(8), 128>>>(dx, k, k, cols, de, b, d1, kpad); }));
  check("sp KPT 4 minB 6", time_it([&] { res_sp<NM, 4, 6><<<grid(4), 128>>>(dx, k, k, cols, de, b, d1, kpad); }));
  check("sp KPT 4 minB 8", time_it([&] { res_sp<NM, 4, 8><<<grid(4), 128>>>(dx, k, k, cols, de, b, d1, kpad); }));
  // copy floor: read x, write the residue bytes
  printf("(HBM floor at 6.5 TB/s: %.3f ms)\n", bytes / 6.5e12 * 1e3);
  return 0;
}
