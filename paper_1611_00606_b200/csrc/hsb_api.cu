// hsb_api.cu — the C ABI (include/hsb200.h): device context, TMA descriptor
// encoding, the kernel-level entry points and the native build_hs pipeline.
//
// The pipeline re-hosts Algorithm 1 as implemented by
// builder.build_hs (/root/reference/pkg/src/hsgen/builder.py:211-224) on one
// device, with every K x N_G operand kept in the stacked layout of
// matcore.stack (matcore.py:68-86):
//
//   potrf_route (Loop 2 potrf)      T_AA -> Q_a (Cholesky factor | mirror(T_AA)), info
//   half_mirror + zrk batched       Z_a = T_AB^H A_a + (1/2 T_BB) B_a          (Loop 1)
//   diag_scale                      UB = diag(u) B                              (U norm)
//   zrk triangle, 2 segments        S = A^H A + UB^H UB, mirrored               (S1, S2)
//   zrk batched (routed offsets)    [Y_hpd ; X_nh] = Q_a^H A_a                 (Loop 2)
//   zrk triangle, 2-4 segments      H = Z^H B + B^H Z + Y^H Y + A_nh^H X_nh     (H1, H3, H2)
//
// With HSB_OPT_UNFUSED the large updates run as one launch per reference
// section, in the reference's order, followed by a separate mirror.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/hsb200.h"
#include "aux_kernels.cuh"
#include "zrk.cuh"

using namespace hsb;

struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
};

struct hsb_ctx {
  int device = 0;
  std::string err;
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  std::map<std::string, DevBuf> bufs;
  void* pinned = nullptr;  // small pinned host scratch (routing info / offsets)
  size_t pinned_bytes = 0;
};

static thread_local std::string g_create_err;

namespace {

hsb_status fail(hsb_ctx* ctx, hsb_status st, const std::string& msg) {
  if (ctx) ctx->err = msg;
  else g_create_err = msg;
  return st;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(ctx, HSB_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define CKS(expr)                     \
  do {                                \
    hsb_status s_ = (expr);           \
    if (s_ != HSB_OK) return s_;      \
  } while (0)

hsb_status ws(hsb_ctx* ctx, const char* name, size_t bytes, void** out) {
  DevBuf& b = ctx->bufs[name];
  if (b.bytes < bytes) {
    if (b.ptr) cudaFree(b.ptr);
    b.ptr = nullptr;
    b.bytes = 0;
    cudaError_t e = cudaMalloc(&b.ptr, bytes ? bytes : 16);
    if (e != cudaSuccess) {
      b.ptr = nullptr;
      cudaGetLastError();
      return fail(ctx, HSB_ERR_NOMEM, std::string("device allocation of ") + std::to_string(bytes) +
                                          " bytes for '" + name + "' failed: " + cudaGetErrorString(e));
    }
    b.bytes = bytes;
  }
  *out = b.ptr;
  return HSB_OK;
}

hsb_status pinned(hsb_ctx* ctx, size_t bytes, void** out) {
  if (ctx->pinned_bytes < bytes) {
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    ctx->pinned = nullptr;
    ctx->pinned_bytes = 0;
    if (cudaMallocHost(&ctx->pinned, bytes) != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, HSB_ERR_NOMEM, "pinned host allocation failed");
    }
    ctx->pinned_bytes = bytes;
  }
  *out = ctx->pinned;
  return HSB_OK;
}

// ----------------------------------------------------------- TMA descriptors
hsb_status encode_operand(hsb_ctx* ctx, CUtensorMap* map, const OperandView& v) {
  if (reinterpret_cast<uintptr_t>(v.base) % 16 != 0)
    return fail(ctx, HSB_ERR_INPUT, "operand base address must be 16-byte aligned");
  cuuint64_t dims[3], strides[2];
  cuuint32_t box[3], estr[3] = {1, 1, 1};
  const cuuint64_t col_stride = static_cast<cuuint64_t>(v.ld) * 16;
  const cuuint64_t bat_stride =
      static_cast<cuuint64_t>(v.batch > 1 ? v.bstride : std::max<int64_t>(1, v.ld * std::max<int64_t>(1, v.cols))) * 16;
  dims[0] = static_cast<cuuint64_t>(2 * v.k);
  box[0] = kBK;
  if (v.bpos == 1) {
    dims[1] = static_cast<cuuint64_t>(v.batch);
    dims[2] = static_cast<cuuint64_t>(v.cols);
    strides[0] = bat_stride;
    strides[1] = col_stride;
    box[1] = 1;
    box[2] = kBM;
  } else {
    dims[1] = static_cast<cuuint64_t>(v.cols);
    dims[2] = static_cast<cuuint64_t>(v.batch);
    strides[0] = col_stride;
    strides[1] = bat_stride;
    box[1] = kBM;
    box[2] = 1;
  }
  CUresult r = ctx->encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(v.base), dims, strides,
                           box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(ctx, HSB_ERR_CUDA, "cuTensorMapEncodeTiled failed (code " + std::to_string(static_cast<int>(r)) +
                                       ") for k=" + std::to_string(v.k) + " cols=" + std::to_string(v.cols) +
                                       " ld=" + std::to_string(v.ld));
  return HSB_OK;
}

struct Seg {
  OperandView l, r;
};

struct ZrkCall {
  std::vector<Seg> segs;
  int64_t m = 0, n = 0;
  bool triangle = false;
  bool conj = true;
  uint32_t flags = 0;
  double alpha_re = 1, alpha_im = 0, beta_re = 0, beta_im = 0;
  double* c = nullptr;
  int64_t ldc = 0;
  int64_t batch = 1;
  int64_t c_bstride = 0;
  const int32_t* c_rowoff = nullptr;
};

hsb_status run_zrk(hsb_ctx* ctx, cudaStream_t st, const ZrkCall& z, int* launches) {
  if (z.m <= 0 || z.n <= 0 || z.batch <= 0) return HSB_OK;
  if (z.segs.size() > static_cast<size_t>(kMaxSeg)) return fail(ctx, HSB_ERR_UNSUPPORTED, "too many segments");
  if (z.triangle && z.m != z.n) return fail(ctx, HSB_ERR_DIMENSION, "triangle mode needs a square output");
  if (z.m > (int64_t{1} << 30) || z.n > (int64_t{1} << 30))
    return fail(ctx, HSB_ERR_UNSUPPORTED, "output dimension too large");
  ZrkParams p;
  std::memset(&p, 0, sizeof(p));
  int nseg = 0, total = 0;
  for (const Seg& s : z.segs) {
    if (s.l.k <= 0) continue;
    if (s.l.k != s.r.k) return fail(ctx, HSB_ERR_DIMENSION, "segment operands disagree in reduction length");
    CKS(encode_operand(ctx, &p.lmap[nseg], s.l));
    CKS(encode_operand(ctx, &p.rmap[nseg], s.r));
    const int64_t chunks = (2 * s.l.k + kBK - 1) / kBK;
    if (chunks > (int64_t{1} << 30)) return fail(ctx, HSB_ERR_UNSUPPORTED, "reduction too long");
    p.seg[nseg].kchunks = static_cast<int32_t>(chunks);
    p.seg[nseg].lbpos = s.l.bpos;
    p.seg[nseg].rbpos = s.r.bpos;
    total += static_cast<int>(chunks);
    ++nseg;
  }
  p.nseg = nseg;
  p.total_chunks = total;
  p.m = static_cast<int32_t>(z.m);
  p.n = static_cast<int32_t>(z.n);
  p.tiles_m = static_cast<int32_t>((z.m + kBM - 1) / kBM);
  p.tiles_n = static_cast<int32_t>((z.n + kBN - 1) / kBN);
  p.triangle = z.triangle ? 1 : 0;
  p.flags = z.flags;
  p.alpha_re = z.alpha_re;
  p.alpha_im = z.alpha_im;
  p.beta_re = z.beta_re;
  p.beta_im = z.beta_im;
  p.c = z.c;
  p.ldc = z.ldc;
  p.c_bstride = z.c_bstride;
  p.c_rowoff = z.c_rowoff;
  int64_t grid_x = z.triangle ? static_cast<int64_t>(p.tiles_m) * (p.tiles_m + 1) / 2
                              : static_cast<int64_t>(p.tiles_m) * p.tiles_n;
  if (grid_x > 0x7fffffff || z.batch > 65535) return fail(ctx, HSB_ERR_UNSUPPORTED, "grid too large");
  CK(launch_zrk(p, z.conj, static_cast<int>(grid_x), static_cast<int>(z.batch), st));
  if (launches) ++*launches;
  return HSB_OK;
}

// plain stacked operand: k x cols, leading dimension ld
OperandView plain(const double* base, int64_t k, int64_t cols, int64_t ld) {
  OperandView v;
  v.base = base;
  v.k = k;
  v.cols = cols;
  v.ld = ld;
  v.batch = 1;
  v.bstride = 0;
  v.bpos = 2;
  return v;
}
// per-atom row blocks of a stacked K x cols array (rows a*n_l .. a*n_l+n_l-1)
OperandView atom_rows(const double* stacked, int64_t n_atoms, int64_t n_l, int64_t cols, int64_t ld) {
  OperandView v;
  v.base = stacked;
  v.k = n_l;
  v.cols = cols;
  v.ld = ld;
  v.batch = n_atoms;
  v.bstride = n_l;
  v.bpos = 1;
  return v;
}
// n_atoms contiguous n_l x n_l matrices
OperandView atom_mats(const double* base, int64_t n_atoms, int64_t n_l) {
  OperandView v;
  v.base = base;
  v.k = n_l;
  v.cols = n_l;
  v.ld = n_l;
  v.batch = n_atoms;
  v.bstride = n_l * n_l;
  v.bpos = 2;
  return v;
}

}  // namespace

// =============================================================================
extern "C" {

int32_t hsb_abi_version(void) { return 1; }

hsb_status hsb_ctx_create(int32_t device, hsb_ctx** out) {
  hsb_ctx* ctx = nullptr;
  if (!out) return fail(nullptr, HSB_ERR_INPUT, "out is NULL");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(nullptr, HSB_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  if (device < 0 || device >= n) return fail(nullptr, HSB_ERR_INPUT, "device index out of range");
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return fail(nullptr, HSB_ERR_CUDA, "device query failed");
  if (prop.major != 10 || prop.minor != 0)
    return fail(nullptr, HSB_ERR_UNSUPPORTED,
                "libhsb200 is built for sm_100a (B200); device is sm_" + std::to_string(prop.major) +
                    std::to_string(prop.minor));
  if (cudaSetDevice(device) != cudaSuccess) return fail(nullptr, HSB_ERR_CUDA, "cudaSetDevice failed");
  ctx = new hsb_ctx();
  ctx->device = device;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  e = cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) {
    delete ctx;
    return fail(nullptr, HSB_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  }
  ctx->encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  *out = ctx;
  return HSB_OK;
}

void hsb_ctx_destroy(hsb_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  for (auto& kv : ctx->bufs)
    if (kv.second.ptr) cudaFree(kv.second.ptr);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  delete ctx;
}

const char* hsb_last_error(const hsb_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

hsb_status hsb_ctx_trim(hsb_ctx* ctx) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
  cudaSetDevice(ctx->device);
  CK(cudaDeviceSynchronize());
  for (auto& kv : ctx->bufs)
    if (kv.second.ptr) cudaFree(kv.second.ptr);
  ctx->bufs.clear();
  return HSB_OK;
}

// ----------------------------------------------------------------- kernels
hsb_status hsb_zherk(hsb_ctx* ctx, void* stream, int64_t n, int64_t k, double alpha, const double* a, int64_t lda,
                     double beta, double* c, int64_t ldc, uint32_t flags) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
  if (n < 0 || k < 0) return fail(ctx, HSB_ERR_DIMENSION, "negative dimension");
  if (n == 0) return HSB_OK;
  if (ldc < n || (k > 0 && lda < k)) return fail(ctx, HSB_ERR_DIMENSION, "leading dimension too small");
  cudaSetDevice(ctx->device);
  ZrkCall z;
  if (alpha != 0.0 && k > 0) z.segs.push_back({plain(a, k, n, lda), plain(a, k, n, lda)});
  z.m = z.n = n;
  z.triangle = true;
  z.conj = true;
  z.flags = kLowerOnly | kZeroImagDiag | (flags & HSB_MIRROR ? kMirror : 0u);
  z.alpha_re = alpha;
  z.beta_re = beta;
  z.c = c;
  z.ldc = ldc;
  return run_zrk(ctx, static_cast<cudaStream_t>(stream), z, nullptr);
}

hsb_status hsb_zher2k(hsb_ctx* ctx, void* stream, int64_t n, int64_t k, double alpha_re, double alpha_im,
                      const double* zp, int64_t ldz, const double* b, int64_t ldb, double beta, double* c,
                      int64_t ldc, uint32_t flags) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
  if (n < 0 || k < 0) return fail(ctx, HSB_ERR_DIMENSION, "negative dimension");
  if (n == 0) return HSB_OK;
  if (ldc < n || (k > 0 && (ldz < k || ldb < k))) return fail(ctx, HSB_ERR_DIMENSION, "leading dimension too small");
  cudaSetDevice(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool zero = (alpha_re == 0.0 && alpha_im == 0.0) || k == 0;
  const uint32_t mir = (flags & HSB_MIRROR) ? kMirror : 0u;
  if (zero || alpha_im == 0.0) {
    // alpha real: alpha Z^H B + alpha B^H Z in one pass (two segments)
    ZrkCall z;
    if (!zero) {
      z.segs.push_back({plain(zp, k, n, ldz), plain(b, k, n, ldb)});
      z.segs.push_back({plain(b, k, n, ldb), plain(zp, k, n, ldz)});
    }
    z.m = z.n = n;
    z.triangle = true;
    z.flags = kLowerOnly | kZeroImagDiag | mir;
    z.alpha_re = alpha_re;
    z.beta_re = beta;
    z.c = c;
    z.ldc = ldc;
    return run_zrk(ctx, st, z, nullptr);
  }
  // complex alpha: two passes sharing C (alpha Z^H B, then conj(alpha) B^H Z)
  ZrkCall z1;
  z1.segs.push_back({plain(zp, k, n, ldz), plain(b, k, n, ldb)});
  z1.m = z1.n = n;
  z1.triangle = true;
  z1.flags = kLowerOnly;
  z1.alpha_re = alpha_re;
  z1.alpha_im = alpha_im;
  z1.beta_re = beta;
  z1.c = c;
  z1.ldc = ldc;
  CKS(run_zrk(ctx, st, z1, nullptr));
  ZrkCall z2 = z1;
  z2.segs.clear();
  z2.segs.push_back({plain(b, k, n, ldb), plain(zp, k, n, ldz)});
  z2.alpha_im = -alpha_im;
  z2.beta_re = 1.0;
  z2.flags = kLowerOnly | kZeroImagDiag | mir;
  return run_zrk(ctx, st, z2, nullptr);
}

hsb_status hsb_zgemm(hsb_ctx* ctx, void* stream, char opa, char opb, int64_t m, int64_t n, int64_t k,
                     double alpha_re, double alpha_im, const double* a, int64_t lda, const double* b, int64_t ldb,
                     double beta_re, double beta_im, double* c, int64_t ldc, uint32_t flags) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
  auto valid_op = [](char o) { return o == 'N' || o == 'T' || o == 'C'; };
  if (!valid_op(opa) || !valid_op(opb)) return fail(ctx, HSB_ERR_INPUT, "op must be one of N, T, C");
  if (m < 0 || n < 0 || k < 0) return fail(ctx, HSB_ERR_DIMENSION, "negative dimension");
  if (m == 0 || n == 0) return HSB_OK;
  if (ldc < m) return fail(ctx, HSB_ERR_DIMENSION, "ldc too small");
  if ((flags & HSB_LOWER_ONLY) && m != n) return fail(ctx, HSB_ERR_DIMENSION, "lower-only gemm needs square C");
  cudaSetDevice(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool zero = (alpha_re == 0.0 && alpha_im == 0.0) || k == 0;
  // Stage op(A) as a reduction-major k x m operand L with C = op'(L)^T R:
  //   opa 'C': L = A, conj  | 'T': L = A, plain | 'N': L = A^T (transpose), plain
  //   opb 'N': R = B        | 'T': R = B^T      | 'C': R = conj(B^T)
  // 'C' on A and a plain op on another operand cannot share one kernel mode,
  // so opa 'N'/'T' run in the non-conjugating mode.
  const double* L = a;
  int64_t ldl = lda;
  const double* R = b;
  int64_t ldr = ldb;
  bool conj = (opa == 'C');
  if (!zero) {
    if (opa == 'N') {
      if (lda < m) return fail(ctx, HSB_ERR_DIMENSION, "lda too small");
      void* t;
      CKS(ws(ctx, "gemm_lt", static_cast<size_t>(k) * m * 16, &t));
      CK(launch_transpose(a, lda, static_cast<double*>(t), k, m, k, false, st));
      L = static_cast<double*>(t);
      ldl = k;
    } else if (lda < k) {
      return fail(ctx, HSB_ERR_DIMENSION, "lda too small");
    }
    if (opb == 'N') {
      if (ldb < k) return fail(ctx, HSB_ERR_DIMENSION, "ldb too small");
    } else {
      if (ldb < n) return fail(ctx, HSB_ERR_DIMENSION, "ldb too small");
      void* t;
      CKS(ws(ctx, "gemm_rt", static_cast<size_t>(k) * n * 16, &t));
      CK(launch_transpose(b, ldb, static_cast<double*>(t), k, n, k, opb == 'C', st));
      R = static_cast<double*>(t);
      ldr = k;
    }
  }
  ZrkCall z;
  if (!zero) z.segs.push_back({plain(L, k, m, ldl), plain(R, k, n, ldr)});
  z.m = m;
  z.n = n;
  z.triangle = (flags & HSB_LOWER_ONLY) != 0;
  z.conj = conj;
  z.flags = ((flags & HSB_LOWER_ONLY) ? kLowerOnly : 0u) | ((flags & HSB_MIRROR) ? kMirror : 0u);
  z.alpha_re = alpha_re;
  z.alpha_im = alpha_im;
  z.beta_re = beta_re;
  z.beta_im = beta_im;
  z.c = c;
  z.ldc = ldc;
  return run_zrk(ctx, st, z, nullptr);
}

hsb_status hsb_hermitian_mirror(hsb_ctx* ctx, void* stream, int64_t n, double* c, int64_t ldc) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
  if (n < 0 || ldc < n) return fail(ctx, HSB_ERR_DIMENSION, "bad mirror dimensions");
  if (n == 0) return HSB_OK;
  cudaSetDevice(ctx->device);
  CK(launch_mirror(c, ldc, static_cast<int>(n), static_cast<cudaStream_t>(stream)));
  return HSB_OK;
}

// ----------------------------------------------------------------- pipeline
hsb_status hsb_build_hs(hsb_ctx* ctx, void* stream, const hsb_problem* p, uint32_t opts, const hsb_output* out,
                        hsb_timings* tm, int32_t* atom_info) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
  if (!p || !out) return fail(ctx, HSB_ERR_INPUT, "problem/output is NULL");
  const int64_t na = p->n_atoms, nl = p->n_l, ng = p->n_g;
  if (na < 1 || nl < 1 || ng < 1) return fail(ctx, HSB_ERR_INPUT, "dimensions must be positive");
  if (out->ld < ng) return fail(ctx, HSB_ERR_DIMENSION, "output leading dimension < n_g");
  if (na > 65535) return fail(ctx, HSB_ERR_UNSUPPORTED, "more than 65535 atoms");
  const int64_t K = na * nl;
  if (K > (int64_t{1} << 31)) return fail(ctx, HSB_ERR_UNSUPPORTED, "stack too tall");
  cudaSetDevice(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool unfused = opts & HSB_OPT_UNFUSED;
  const bool force_nonhpd = opts & HSB_OPT_FORCE_NONHPD;
  int launches = 0;

  enum { E_START, E_H2D, E_POTRF, E_LOOP1, E_H1, E_S1, E_UNORM, E_S2, E_SMIR, E_LOOP2, E_H2, E_H3, E_HMIR,
         E_D2H, E_N };
  cudaEvent_t ev[E_N];
  for (int i = 0; i < E_N; ++i) CK(cudaEventCreate(&ev[i]));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < E_N; ++i) cudaEventDestroy(e[i]);
    }
  } guard{ev};

  CK(cudaEventRecord(ev[E_START], st));

  // ---------------------------------------------------------------- inputs
  const double *A, *B, *TAA, *TAB, *TBB, *U;
  const size_t stack_bytes = static_cast<size_t>(K) * ng * 16;
  const size_t tblk_bytes = static_cast<size_t>(nl) * nl * 16;
  if (p->location == HSB_LOC_HOST) {
    if (!p->a_blocks || !p->b_blocks || !p->t_aa || !p->t_ab || !p->t_bb || !p->u_norms)
      return fail(ctx, HSB_ERR_INPUT, "host block arrays are NULL");
    void *a, *b, *taa, *tab, *tbb, *u;
    CKS(ws(ctx, "in_a", stack_bytes, &a));
    CKS(ws(ctx, "in_b", stack_bytes, &b));
    CKS(ws(ctx, "in_taa", tblk_bytes * na, &taa));
    CKS(ws(ctx, "in_tab", tblk_bytes * na, &tab));
    CKS(ws(ctx, "in_tbb", tblk_bytes * na, &tbb));
    CKS(ws(ctx, "in_u", static_cast<size_t>(K) * 8, &u));
    for (int64_t i = 0; i < na; ++i) {
      CK(cudaMemcpy2DAsync(static_cast<char*>(a) + i * nl * 16, K * 16, p->a_blocks[i], nl * 16, nl * 16, ng,
                           cudaMemcpyHostToDevice, st));
      CK(cudaMemcpy2DAsync(static_cast<char*>(b) + i * nl * 16, K * 16, p->b_blocks[i], nl * 16, nl * 16, ng,
                           cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(static_cast<char*>(taa) + i * tblk_bytes, p->t_aa[i], tblk_bytes, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(static_cast<char*>(tab) + i * tblk_bytes, p->t_ab[i], tblk_bytes, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(static_cast<char*>(tbb) + i * tblk_bytes, p->t_bb[i], tblk_bytes, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(static_cast<char*>(u) + i * nl * 8, p->u_norms[i], nl * 8, cudaMemcpyHostToDevice, st));
    }
    A = static_cast<double*>(a);
    B = static_cast<double*>(b);
    TAA = static_cast<double*>(taa);
    TAB = static_cast<double*>(tab);
    TBB = static_cast<double*>(tbb);
    U = static_cast<double*>(u);
  } else if (p->location == HSB_LOC_DEVICE) {
    A = p->a_stack;
    B = p->b_stack;
    TAA = p->t_aa_dev;
    TAB = p->t_ab_dev;
    TBB = p->t_bb_dev;
    U = p->u_dev;
    if (!A || !B || !TAA || !TAB || !TBB || !U) return fail(ctx, HSB_ERR_INPUT, "device arrays are NULL");
  } else {
    return fail(ctx, HSB_ERR_INPUT, "unknown problem location");
  }
  CK(cudaEventRecord(ev[E_H2D], st));

  double *H, *S;
  int64_t ldo;
  const size_t out_bytes = static_cast<size_t>(ng) * ng * 16;
  if (out->location == HSB_LOC_HOST) {
    void *h, *s;
    CKS(ws(ctx, "out_h", out_bytes, &h));
    CKS(ws(ctx, "out_s", out_bytes, &s));
    H = static_cast<double*>(h);
    S = static_cast<double*>(s);
    ldo = ng;
  } else {
    H = out->h;
    S = out->s;
    ldo = out->ld;
  }
  if (!out->h || !out->s) return fail(ctx, HSB_ERR_INPUT, "output pointers are NULL");

  // ------------------------------------------------------ scratch buffers
  void *q, *info_d, *pbb, *zbuf, *ub, *rbuf, *offs_d, *potrf_scr = nullptr;
  CKS(ws(ctx, "q", tblk_bytes * na, &q));
  CKS(ws(ctx, "info", static_cast<size_t>(na) * 4 * 4, &info_d));
  CKS(ws(ctx, "pbb", tblk_bytes * na, &pbb));
  CKS(ws(ctx, "z", stack_bytes, &zbuf));
  CKS(ws(ctx, "ub", stack_bytes, &ub));
  CKS(ws(ctx, "r", stack_bytes, &rbuf));
  CKS(ws(ctx, "offs", static_cast<size_t>(na) * 3 * 4, &offs_d));
  if (static_cast<size_t>(nl) * (nl + 1) / 2 * 16 > kPotrfSmemMax)
    CKS(ws(ctx, "potrf_scr", static_cast<size_t>(na) * nl * (nl + 1) / 2 * 16, &potrf_scr));
  void* hostbuf;
  CKS(pinned(ctx, static_cast<size_t>(na) * 4 * 4, &hostbuf));
  int32_t* info_h = static_cast<int32_t*>(hostbuf);
  int32_t* offs_h = info_h + na;  // 3 * na entries: r row offset, anh src, anh dst

  // --------------------------------------------------- Loop 2, part 1: potrf
  CK(launch_potrf_route(TAA, static_cast<double*>(q), static_cast<int32_t*>(info_d), static_cast<int>(na),
                        static_cast<int>(nl), force_nonhpd, static_cast<double*>(potrf_scr), st));
  ++launches;
  CK(cudaMemcpyAsync(info_h, info_d, na * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(ev[E_POTRF], st));

  // ---------------------------------------------------------------- Loop 1
  CK(launch_half_mirror(TBB, static_cast<double*>(pbb), static_cast<int>(nl), na, 0.5, st));
  ++launches;
  {
    ZrkCall z;
    z.segs.push_back({atom_mats(TAB, na, nl), atom_rows(A, na, nl, ng, K)});
    z.segs.push_back({atom_mats(static_cast<double*>(pbb), na, nl), atom_rows(B, na, nl, ng, K)});
    z.m = nl;
    z.n = ng;
    z.c = static_cast<double*>(zbuf);
    z.ldc = K;
    z.batch = na;
    z.c_bstride = nl;
    CKS(run_zrk(ctx, st, z, &launches));
  }
  CK(cudaEventRecord(ev[E_LOOP1], st));
  double* Z = static_cast<double*>(zbuf);
  double* UB = static_cast<double*>(ub);

  if (unfused) {
    // H1: lower(Z^H B + B^H Z), beta = 0 (builder.h_cross, builder.py:91-104)
    ZrkCall h1;
    h1.segs.push_back({plain(Z, K, ng, K), plain(B, K, ng, K)});
    h1.segs.push_back({plain(B, K, ng, K), plain(Z, K, ng, K)});
    h1.m = h1.n = ng;
    h1.triangle = true;
    h1.flags = kLowerOnly | kZeroImagDiag;
    h1.c = H;
    h1.ldc = ldo;
    CKS(run_zrk(ctx, st, h1, &launches));
    CK(cudaEventRecord(ev[E_H1], st));
    // S1 (builder.build_s, builder.py:107-132)
    ZrkCall s1;
    s1.segs.push_back({plain(A, K, ng, K), plain(A, K, ng, K)});
    s1.m = s1.n = ng;
    s1.triangle = true;
    s1.flags = kLowerOnly | kZeroImagDiag;
    s1.c = S;
    s1.ldc = ldo;
    CKS(run_zrk(ctx, st, s1, &launches));
    CK(cudaEventRecord(ev[E_S1], st));
  } else {
    CK(cudaEventRecord(ev[E_H1], st));
    CK(cudaEventRecord(ev[E_S1], st));
  }
  // U norm
  CK(launch_diag_scale(B, K, UB, K, U, K, ng, st));
  ++launches;
  CK(cudaEventRecord(ev[E_UNORM], st));
  if (unfused) {
    ZrkCall s2;
    s2.segs.push_back({plain(UB, K, ng, K), plain(UB, K, ng, K)});
    s2.m = s2.n = ng;
    s2.triangle = true;
    s2.flags = kLowerOnly | kZeroImagDiag;
    s2.beta_re = 1.0;
    s2.c = S;
    s2.ldc = ldo;
    CKS(run_zrk(ctx, st, s2, &launches));
    CK(cudaEventRecord(ev[E_S2], st));
    CK(launch_mirror(S, ldo, static_cast<int>(ng), st));
    ++launches;
    CK(cudaEventRecord(ev[E_SMIR], st));
  } else {
    ZrkCall s;
    s.segs.push_back({plain(A, K, ng, K), plain(A, K, ng, K)});
    s.segs.push_back({plain(UB, K, ng, K), plain(UB, K, ng, K)});
    s.m = s.n = ng;
    s.triangle = true;
    s.flags = kLowerOnly | kMirror;
    s.c = S;
    s.ldc = ldo;
    CKS(run_zrk(ctx, st, s, &launches));
    CK(cudaEventRecord(ev[E_S2], st));
    CK(cudaEventRecord(ev[E_SMIR], st));
  }

  // ------------------------------------------- routing (host, overlaps S)
  CK(cudaEventSynchronize(ev[E_POTRF]));
  int64_t n_hpd = 0, n_nh = 0;
  for (int64_t i = 0; i < na; ++i) (info_h[i] == 0 ? n_hpd : n_nh)++;
  {
    int64_t ih = 0, in = 0;
    for (int64_t i = 0; i < na; ++i) {
      if (info_h[i] == 0) {
        offs_h[i] = static_cast<int32_t>(ih * nl);
        ++ih;
      } else {
        offs_h[i] = static_cast<int32_t>((n_hpd + in) * nl);
        offs_h[na + in] = static_cast<int32_t>(i * nl);    // A_nh source rows
        offs_h[2 * na + in] = static_cast<int32_t>(in * nl);  // A_nh dest rows
        ++in;
      }
    }
  }
  if (atom_info) std::memcpy(atom_info, info_h, na * 4);
  CK(cudaMemcpyAsync(offs_d, offs_h, na * 3 * 4, cudaMemcpyHostToDevice, st));
  const int32_t* offs_dev = static_cast<int32_t*>(offs_d);

  // ---------------------------------------------------- Loop 2, part 2
  double* R = static_cast<double*>(rbuf);  // [Y_hpd ; X_nh]
  double* ANH = nullptr;
  {
    ZrkCall z;
    z.segs.push_back({atom_mats(static_cast<double*>(q), na, nl), atom_rows(A, na, nl, ng, K)});
    z.m = nl;
    z.n = ng;
    z.c = R;
    z.ldc = K;
    z.batch = na;
    z.c_rowoff = offs_dev;
    CKS(run_zrk(ctx, st, z, &launches));
    if (n_nh > 0) {
      void* anh;
      CKS(ws(ctx, "anh", static_cast<size_t>(n_nh) * nl * ng * 16, &anh));
      ANH = static_cast<double*>(anh);
      CK(launch_gather_rows(A, K, ANH, n_nh * nl, offs_dev + na, offs_dev + 2 * na, static_cast<int>(n_nh),
                            static_cast<int>(nl), ng, st));
      ++launches;
    }
  }
  CK(cudaEventRecord(ev[E_LOOP2], st));
  const int64_t k_hpd = n_hpd * nl, k_nh = n_nh * nl;
  const double* Y = R;
  const double* XNH = R + 2 * k_hpd;

  if (unfused) {
    if (n_nh > 0) {  // H2: gemm('C','N', beta = 1) (builder.py:187-194), lower tiles
      ZrkCall h2;
      h2.segs.push_back({plain(ANH, k_nh, ng, k_nh), plain(XNH, k_nh, ng, K)});
      h2.m = h2.n = ng;
      h2.triangle = true;
      h2.flags = kLowerOnly;
      h2.beta_re = 1.0;
      h2.c = H;
      h2.ldc = ldo;
      CKS(run_zrk(ctx, st, h2, &launches));
    }
    CK(cudaEventRecord(ev[E_H2], st));
    if (n_hpd > 0) {  // H3: herk(beta = 1) (builder.py:195-200)
      ZrkCall h3;
      h3.segs.push_back({plain(Y, k_hpd, ng, K), plain(Y, k_hpd, ng, K)});
      h3.m = h3.n = ng;
      h3.triangle = true;
      h3.flags = kLowerOnly | kZeroImagDiag;
      h3.beta_re = 1.0;
      h3.c = H;
      h3.ldc = ldo;
      CKS(run_zrk(ctx, st, h3, &launches));
    }
    CK(cudaEventRecord(ev[E_H3], st));
    CK(launch_mirror(H, ldo, static_cast<int>(ng), st));
    ++launches;
    CK(cudaEventRecord(ev[E_HMIR], st));
  } else {
    ZrkCall h;
    h.segs.push_back({plain(Z, K, ng, K), plain(B, K, ng, K)});
    h.segs.push_back({plain(B, K, ng, K), plain(Z, K, ng, K)});
    if (n_hpd > 0) h.segs.push_back({plain(Y, k_hpd, ng, K), plain(Y, k_hpd, ng, K)});
    if (n_nh > 0) h.segs.push_back({plain(ANH, k_nh, ng, k_nh), plain(XNH, k_nh, ng, K)});
    h.m = h.n = ng;
    h.triangle = true;
    h.flags = kLowerOnly | kMirror;
    h.c = H;
    h.ldc = ldo;
    CKS(run_zrk(ctx, st, h, &launches));
    CK(cudaEventRecord(ev[E_H2], st));
    CK(cudaEventRecord(ev[E_H3], st));
    CK(cudaEventRecord(ev[E_HMIR], st));
  }

  // --------------------------------------------------------------- outputs
  if (out->location == HSB_LOC_HOST) {
    CK(cudaMemcpy2DAsync(out->h, out->ld * 16, H, ldo * 16, ng * 16, ng, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpy2DAsync(out->s, out->ld * 16, S, ldo * 16, ng * 16, ng, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaEventRecord(ev[E_D2H], st));
  CK(cudaEventSynchronize(ev[E_D2H]));

  if (tm) {
    auto el = [&](int a, int b) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[a], ev[b]);
      return ms * 1e-3;
    };
    std::memset(tm, 0, sizeof(*tm));
    tm->h2d = el(E_START, E_H2D);
    const double t_potrf = el(E_H2D, E_POTRF);
    tm->loop1 = el(E_POTRF, E_LOOP1);
    tm->unorm = el(E_S1, E_UNORM);
    tm->loop2 = t_potrf + el(E_SMIR, E_LOOP2);
    const double fS = 4.0 * K * double(ng) * ng;  // S1 == S2 model flops
    const double fH1 = 8.0 * K * double(ng) * ng, fH2 = 8.0 * k_nh * double(ng) * ng,
                 fH3 = 4.0 * k_hpd * double(ng) * ng;
    if (unfused) {
      tm->h1 = el(E_LOOP1, E_H1);
      tm->s1 = el(E_H1, E_S1);
      tm->s2 = el(E_UNORM, E_S2) + el(E_S2, E_SMIR);
      tm->h2 = el(E_LOOP2, E_H2);
      tm->h3 = el(E_H2, E_H3) + el(E_H3, E_HMIR);
    } else {
      const double ts = el(E_UNORM, E_S2);
      tm->s1 = ts * 0.5;
      tm->s2 = ts * 0.5;
      const double th = el(E_LOOP2, E_H2);
      const double fh = fH1 + fH2 + fH3;
      tm->h1 = th * fH1 / fh;
      tm->h2 = th * fH2 / fh;
      tm->h3 = th * fH3 / fh;
    }
    tm->d2h = el(E_HMIR, E_D2H);
    tm->total = el(E_START, E_D2H);
    tm->n_hpd = static_cast<int32_t>(n_hpd);
    tm->n_nonhpd = static_cast<int32_t>(n_nh);
    tm->launches = launches;
  }
  return HSB_OK;
}

}  // extern "C"
