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
#include <omp.h>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif

#include <condition_variable>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>

#include "host_ctx.cuh"

using namespace hsb_host;

// =============================================================================
extern "C" {

int32_t hsb_abi_version(void) { return 8; }

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
  if (ctx->m_stage) cudaFreeHost(ctx->m_stage);
  if (ctx->m_stage_done) cudaEventDestroy(ctx->m_stage_done);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->done_cnt) cudaFreeHost(ctx->done_cnt);
  delete ctx;
}

const char* hsb_last_error(const hsb_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

hsb_status hsb_ctx_set_complex_mult(hsb_ctx* ctx, int32_t algo) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
  if (algo != HSB_CPLX_4M && algo != HSB_CPLX_3M) return fail(ctx, HSB_ERR_INPUT, "unknown complex product form");
  std::lock_guard<std::mutex> g(ctx->call_mu);
  ctx->cplx = algo;
  return HSB_OK;
}

hsb_status hsb_ctx_set_engine(hsb_ctx* ctx, int32_t engine, int32_t min_bits) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
  if (engine != HSB_ENGINE_DMMA && engine != HSB_ENGINE_INT8 && engine != HSB_ENGINE_AUTO)
    return fail(ctx, HSB_ERR_INPUT, "unknown engine");
  if (min_bits != 0 && (min_bits < 30 || min_bits > kOzMaxBits))
    return fail(ctx, HSB_ERR_INPUT, "min_bits must be 0 (default 53, a full FP64 mantissa) or in [30, 55]");
  std::lock_guard<std::mutex> g(ctx->call_mu);
  ctx->engine_setting = engine;
  ctx->oz_min_bits = min_bits ? min_bits : kOzDefaultBits;
  return HSB_OK;
}

hsb_status hsb_oz_crt_table(int32_t n_mod, double* weights, double* m) {
  if (!weights || !m) return fail(nullptr, HSB_ERR_INPUT, "NULL output");
  if (oz_crt_table_host(n_mod, weights, m) != 0) return fail(nullptr, HSB_ERR_INPUT, "n_mod out of range");
  return HSB_OK;
}

hsb_status hsb_ipc_handle(hsb_ctx* ctx, void* dev_ptr, uint8_t handle[64]) {
  if (!ctx || !dev_ptr || !handle) return fail(ctx, HSB_ERR_INPUT, "NULL argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handle size");
  cudaSetDevice(ctx->device);
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, dev_ptr));
  std::memcpy(handle, &h, 64);
  return HSB_OK;
}

hsb_status hsb_ipc_open(hsb_ctx* ctx, const uint8_t handle[64], void** dev_ptr) {
  if (!ctx || !dev_ptr || !handle) return fail(ctx, HSB_ERR_INPUT, "NULL argument");
  cudaSetDevice(ctx->device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  CK(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return HSB_OK;
}

hsb_status hsb_ipc_close(hsb_ctx* ctx, void* dev_ptr) {
  if (!ctx || !dev_ptr) return fail(ctx, HSB_ERR_INPUT, "NULL argument");
  cudaSetDevice(ctx->device);
  CK(cudaIpcCloseMemHandle(dev_ptr));
  return HSB_OK;
}

hsb_status hsb_ctx_trim(hsb_ctx* ctx) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
  CtxCall call_guard(ctx, false);
  cudaSetDevice(ctx->device);
  CK(cudaDeviceSynchronize());
  for (auto& kv : ctx->bufs)
    if (kv.second.ptr) cudaFree(kv.second.ptr);
  ctx->bufs.clear();
  ctx->tile_list_T = 0;
  ctx->oz_tiles_n = 0;
  return HSB_OK;
}

// ----------------------------------------------------------------- kernels
hsb_status hsb_zherk(hsb_ctx* ctx, void* stream, int64_t n, int64_t k, double alpha, const double* a, int64_t lda,
                     double beta, double* c, int64_t ldc, uint32_t flags) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
  CtxCall call_guard(ctx, false);
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
  CtxCall call_guard(ctx, false);
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
  CtxCall call_guard(ctx, false);
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
  CtxCall call_guard(ctx, false);
  if (n < 0 || ldc < n) return fail(ctx, HSB_ERR_DIMENSION, "bad mirror dimensions");
  if (n == 0) return HSB_OK;
  cudaSetDevice(ctx->device);
  CK(launch_mirror(c, ldc, static_cast<int>(n), static_cast<cudaStream_t>(stream)));
  return HSB_OK;
}

hsb_status hsb_sum_slots(hsb_ctx* ctx, void* stream, const double* slots, int32_t n_slots, int64_t slot_stride,
                         int64_t count, double* out) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
  CtxCall call_guard(ctx, false);
  if (n_slots < 1 || count < 0 || slot_stride < count) return fail(ctx, HSB_ERR_DIMENSION, "bad slot dimensions");
  if (count == 0) return HSB_OK;
  if (!slots || !out) return fail(ctx, HSB_ERR_INPUT, "slot/output pointers are NULL");
  cudaSetDevice(ctx->device);
  CK(launch_sum_slots(slots, n_slots, slot_stride, count, out, static_cast<cudaStream_t>(stream)));
  return HSB_OK;
}

// ----------------------------------------------------------------- pipeline
namespace {

ZrkCall tri_call(double* c, int64_t ldc, int64_t n, uint32_t flags, double beta) {
  ZrkCall z;
  z.m = z.n = n;
  z.triangle = true;
  z.flags = flags;
  z.beta_re = beta;
  z.c = c;
  z.ldc = ldc;
  return z;
}

}  // namespace

// probgen.validate_instance value checks of the small host inputs
// (probgen.py:155-168): finiteness of T_AA, T_AB, T_BB, u (fields in that
// order, atoms in order), then T_AA / T_BB Hermitian within
// 1e-14 (1 + ||T||_F) (matcore.hermitian_defect, matcore.py:108-114), then
// u > 0.  Host threads, no Python (the k-point lanes run it concurrently).
// Hermitian outputs cross PCIe as lower triangles (each downloaded column
// range [c0, c1) carries rows >= c0) and are completed on the host: once a
// range has landed (its event), rows [c0, c1) of the columns >= c1 are the
// conjugate transpose of the arrived panel.  Those rows of later columns are
// never written by a later download (it starts at its own c0 >= c1), so the
// host threads and the DMA engine touch disjoint bytes.  Halves the D2H bytes
// (the e2e bound of the pinned-host path) for ~1 GB/s-per-core host work.
// Split of the upper triangles between PCIe and the host mirror: column c
// (in its 64-column download block) crosses PCIe from row d2h_row0(c) on, and
// the host threads fill rows < d2h_row0(c).  frac = 0: lower triangles only.
// Host DRAM carries the DMA writes plus the mirror's reads and writes, PCIe
// the DMA: moving part of the upper triangles to the DMA engine balances the
// two (the pinned-host e2e path is bound by their sum).
constexpr double kD2hUpperHostIn = 0.0, kD2hUpperDevIn = 0.2;  // measured: profiles/d2h_split_r02.txt
static int64_t d2h_row0(int64_t c, double frac) {
  const int64_t a = c & ~int64_t{63};
  return static_cast<int64_t>((1.0 - frac) * static_cast<double>(a)) & ~int64_t{7};
}
static double d2h_upper_frac(bool host_in) {
  const char* e = std::getenv("HSB_D2H_UPPER");  // experiments / tests: a fraction in [0, 1]
  if (e && *e) return std::min(std::max(std::atof(e), 0.0), 1.0);
  // host inputs also read host DRAM (the A / B uploads): more of the upper
  // triangles over PCIe
  return host_in ? kD2hUpperHostIn : kD2hUpperDevIn;
}

struct HostMirror {
  struct Job {
    cudaEvent_t ev;
    double* m;
    int64_t ld, n, c0, c1;
    double frac;
  };
  // a worker thread waits for each range's event and mirrors it, so the
  // caller keeps issuing downloads meanwhile
  std::deque<Job> q;
  std::mutex mu;
  std::condition_variable cv;
  std::thread worker;
  bool closing = false;
  cudaError_t err = cudaSuccess;
  int device = 0;
  int threads = mirror_threads();
  static int mirror_threads() {
    static const int n = [] {
      const char* e = std::getenv("HSB_MIRROR_THREADS");
      const int v = e ? std::atoi(e) : 0;
      // default: half the cores -- the mirror shares the host's DRAM with the
      // lanes' DMA traffic, and more threads slow the uploads (probes/host_contention.cu)
      return v > 0 ? v : std::max(1, omp_get_max_threads() / 2);
    }();
    return n;
  }
  ~HostMirror() { finish(); }
  cudaError_t push(cudaStream_t cs, double* m, int64_t ld, int64_t n, int64_t c0, int64_t c1, double frac) {
    if (c1 >= n) return cudaSuccess;  // nothing above the diagonal blocks
    cudaEvent_t e;
    cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (r != cudaSuccess) return r;
    r = cudaEventRecord(e, cs);
    if (r != cudaSuccess) {
      cudaEventDestroy(e);
      return r;
    }
    if (!worker.joinable()) {
      cudaGetDevice(&device);
      worker = std::thread([this] { loop(); });
    }
    std::lock_guard<std::mutex> lk(mu);
    q.push_back({e, m, ld, n, c0, c1, frac});
    cv.notify_one();
    return cudaSuccess;
  }
  void loop() {
    cudaSetDevice(device);
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [this] { return closing || !q.empty(); });
        if (q.empty()) return;
        j = q.front();
        q.pop_front();
      }
      cudaError_t e = cudaEventSynchronize(j.ev);
      cudaEventDestroy(j.ev);
      if (e != cudaSuccess) {
        std::lock_guard<std::mutex> lk(mu);
        if (err == cudaSuccess) err = e;
        continue;
      }
      run(j, threads);
    }
  }
  static void run(const Job& j, int threads) {
    constexpr int64_t tb = 64;
    const int64_t ntj = (j.n - j.c1 + tb - 1) / tb, nti = (j.c1 - j.c0 + tb - 1) / tb;
    double* m = j.m;
    const int64_t ld = j.ld;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
    for (int64_t t = 0; t < ntj * nti; ++t) {
      const int64_t j0 = j.c1 + (t / nti) * tb, i0 = j.c0 + (t % nti) * tb;
      const int64_t j1 = std::min(j.n, j0 + tb), i1 = std::min(j.c1, i0 + tb);
      // (r, c) upper  <-  conj (c, r) lower; destination runs are contiguous
      // in r and written with non-temporal stores (no read-for-ownership)
      for (int64_t c = j0; c < j1; ++c)
        for (int64_t r = i0, r1 = std::min(i1, d2h_row0(c, j.frac)); r < r1; ++r) {  // rows >= r1: DMA'd
#if defined(__SSE2__)
          const __m128d sign = _mm_set_pd(-0.0, 0.0);
          _mm_stream_pd(m + 2 * (r + c * ld), _mm_xor_pd(_mm_load_pd(m + 2 * (c + r * ld)), sign));
#else
          m[2 * (r + c * ld)] = m[2 * (c + r * ld)];
          m[2 * (r + c * ld) + 1] = -m[2 * (c + r * ld) + 1];
#endif
        }
#if defined(__SSE2__)
      _mm_sfence();
#endif
    }
  }
  // wait until every queued range is mirrored
  cudaError_t finish() {
    if (worker.joinable()) {
      {
        std::lock_guard<std::mutex> lk(mu);
        closing = true;
        cv.notify_one();
      }
      worker.join();
    }
    return err;
  }
};

static hsb_status validate_small_inputs(hsb_ctx* ctx, const hsb_problem* p) {
  const int64_t na = p->n_atoms, nl = p->n_l;
  enum { FIN_TAA, FIN_TAB, FIN_TBB, FIN_U, HERM_TAA, HERM_TBB, POS_U, NCHK };
  int64_t first[NCHK];
  for (auto& f : first) f = na;
  const double* const* tf[3] = {p->t_aa, p->t_ab, p->t_bb};
#pragma omp parallel for schedule(dynamic, 4) num_threads(std::max(1, std::min(8, omp_get_max_threads())))
  for (int64_t a = 0; a < na; ++a) {
    bool bad[NCHK] = {};
    for (int f = 0; f < 3; ++f) {
      const double* t = tf[f][a];
      for (int64_t i = 0; i < 2 * nl * nl; ++i)
        if (!std::isfinite(t[i])) {
          bad[FIN_TAA + f] = true;
          break;
        }
    }
    const double* u = p->u_norms[a];
    for (int64_t i = 0; i < nl; ++i) {
      if (!std::isfinite(u[i])) bad[FIN_U] = true;
      if (!(u[i] > 0)) bad[POS_U] = true;
    }
    for (int f = 0; f < 2; ++f) {
      const double* t = f == 0 ? p->t_aa[a] : p->t_bb[a];  // column-major complex
      double defect = 0, fro = 0;
      for (int64_t j = 0; j < nl; ++j)
        for (int64_t i = 0; i < nl; ++i) {
          const double xr = t[2 * (i + j * nl)], xi = t[2 * (i + j * nl) + 1];
          const double yr = t[2 * (j + i * nl)], yi = -t[2 * (j + i * nl) + 1];
          defect = std::max(defect, std::hypot(xr - yr, xi - yi));
          fro += xr * xr + xi * xi;
        }
      for (int64_t i = 0; i < nl; ++i) defect = std::max(defect, std::fabs(t[2 * (i + i * nl) + 1]));
      if (defect > 1e-14 * (1.0 + std::sqrt(fro))) bad[f == 0 ? HERM_TAA : HERM_TBB] = true;
    }
    for (int c = 0; c < NCHK; ++c)
      if (bad[c]) {
#pragma omp critical(hsb_validate)
        first[c] = std::min(first[c], a);
      }
  }
  static const char* name[NCHK] = {"t_aa", "t_ab", "t_bb", "u_norms", "t_aa", "t_bb", "u_norms"};
  static const char* what[NCHK] = {"contains non-finite entries", "contains non-finite entries",
                                   "contains non-finite entries", "contains non-finite entries",
                                   "is not Hermitian within 1e-14", "is not Hermitian within 1e-14",
                                   "has non-positive entries"};
  for (int c = 0; c < NCHK; ++c)
    if (first[c] < na)
      return fail(ctx, HSB_ERR_INVARIANT,
                  std::string(name[c]) + "[" + std::to_string(first[c]) + "] " + what[c]);
  return HSB_OK;
}

static hsb_status build_hs_core(hsb_ctx* ctx, void* stream, const hsb_problem* p, uint32_t opts,
                                const hsb_output* out, hsb_timings* tm, int32_t* atom_info);

hsb_status hsb_build_hs(hsb_ctx* ctx, void* stream, const hsb_problem* p, uint32_t opts, const hsb_output* out,
                        hsb_timings* tm, int32_t* atom_info) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
  CtxCall call_guard(ctx, true);
  ctx->oz_prepared = {};
  return build_hs_core(ctx, stream, p, opts, out, tm, atom_info);
}

static hsb_status build_hs_core(hsb_ctx* ctx, void* stream, const hsb_problem* p, uint32_t opts,
                                const hsb_output* out, hsb_timings* tm, int32_t* atom_info) {
  if (!p || !out) return fail(ctx, HSB_ERR_INPUT, "problem/output is NULL");
  const int64_t na = p->n_atoms, nl = p->n_l, ng = p->n_g;
  if (na < 1 || nl < 1 || ng < 1) return fail(ctx, HSB_ERR_INPUT, "dimensions must be positive");
  if (out->ld < ng) return fail(ctx, HSB_ERR_DIMENSION, "output leading dimension < n_g");
  if (!out->peer && (!out->h || !out->s)) return fail(ctx, HSB_ERR_INPUT, "output pointers are NULL");
  if (na > 65535) return fail(ctx, HSB_ERR_UNSUPPORTED, "more than 65535 atoms");
  const int64_t K = na * nl;
  if (K > (int64_t{1} << 31)) return fail(ctx, HSB_ERR_UNSUPPORTED, "stack too tall");
  if (p->location != HSB_LOC_HOST && p->location != HSB_LOC_DEVICE)
    return fail(ctx, HSB_ERR_INPUT, "unknown problem location");
  if ((opts & HSB_OPT_VALIDATE) && p->location == HSB_LOC_HOST) {
    if (!p->t_aa || !p->t_ab || !p->t_bb || !p->u_norms) return fail(ctx, HSB_ERR_INPUT, "host block arrays are NULL");
    CKS(validate_small_inputs(ctx, p));
  }
  if ((opts & HSB_OPT_LOWER_ONLY) && (out->location != HSB_LOC_DEVICE || out->peer))
    return fail(ctx, HSB_ERR_INPUT, "HSB_OPT_LOWER_ONLY needs device outputs");
  // fused paths: the final H / S epilogues mirror (FULL) unless lower triangles were asked for
  const uint32_t out_mirror = (opts & HSB_OPT_LOWER_ONLY) ? kZeroImagDiag : kMirror;
  cudaSetDevice(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!ctx->copy_stream) CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  cudaStream_t cs = ctx->copy_stream;
  const bool unfused = opts & HSB_OPT_UNFUSED;
  const bool force_nonhpd = opts & HSB_OPT_FORCE_NONHPD;
  const bool host_in = p->location == HSB_LOC_HOST;
  // Host inputs + fused launches: upload B, start U norm and the (UB)^H(UB)
  // half of S, and stage A on the copy stream meanwhile.
  const bool overlap_upload = host_in && !unfused;
  const hsb_peer_out* peer = out->peer;
  if (peer) {
    if (unfused || ctx->engine != HSB_ENGINE_INT8 || out->location != HSB_LOC_DEVICE)
      return fail(ctx, HSB_ERR_UNSUPPORTED, "peer output needs the fused INT8 engine and device outputs");
    if (peer->n_ranks < 1 || peer->rank < 0 || peer->rank >= peer->n_ranks || peer->ld < ng ||
        peer->cols_per_rank * peer->n_ranks < ng || !peer->h_slots || !peer->s_slots)
      return fail(ctx, HSB_ERR_INPUT, "inconsistent hsb_peer_out");
  }
  // INT8 engine + pinned host S: S runs in column groups whose downloads
  // start as each group is final (events), overlapping the rest of S and H
  std::vector<std::pair<cudaEvent_t, int64_t>> s_chunks;
  struct ChunkDel {
    std::vector<std::pair<cudaEvent_t, int64_t>>& v;
    ~ChunkDel() {
      for (auto& c : v) cudaEventDestroy(c.first);
    }
  } s_chunks_del{s_chunks};
  const bool chunk_s = !unfused && ctx->engine == HSB_ENGINE_INT8 && out->location == HSB_LOC_HOST &&
                       host_is_pinned(out->s);
  int launches = 0;
  double h2d_bytes = 0, d2h_bytes = 0;  // PCIe bytes this call moves (host in / out)
  Timeline tl;
  HostClock hc;  // host-side phase stamps, printed when HSB_DEBUG_TIMING is set
  GpuTrace tr;    // absolute GPU timeline, printed when HSB_TRACE is set
  tr.who = ctx;
  // ordering against the previous pipelined call (hsb_output.h2d_after ...):
  // wait until it has recorded the event, then make the stream wait on it
  struct OrderGuard {  // never leave the next call waiting (early returns)
    int32_t* f;
    ~OrderGuard() {
      if (f) __atomic_store_n(f, 2, __ATOMIC_RELEASE);
    }
  } order_guard{out->order_out};
  auto order_wait = [&](void* ev, int32_t level, cudaStream_t s) -> cudaError_t {
    if (!ev) return cudaSuccess;
    if (out->order_in)
      while (__atomic_load_n(out->order_in, __ATOMIC_ACQUIRE) < level)
        std::this_thread::sleep_for(std::chrono::microseconds(20));
    return cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(ev), 0);
  };
  auto order_done = [&](void* ev, int32_t level, cudaStream_t s) -> cudaError_t {
    if (ev) {
      const cudaError_t e = cudaEventRecord(static_cast<cudaEvent_t>(ev), s);
      if (e != cudaSuccess) return e;
    }
    if (out->order_out) __atomic_store_n(out->order_out, level, __ATOMIC_RELEASE);
    return cudaSuccess;
  };
  if (host_in) CK(order_wait(out->h2d_after, 1, st));
  CK(tl.mark(st, "start"));
  tr.mark(st, "start");

  // ------------------------------------------------------------ buffers
  const size_t stack_bytes = static_cast<size_t>(K) * ng * 16;
  const size_t tblk_bytes = static_cast<size_t>(nl) * nl * 16;
  const double *A, *B, *TAA, *TAB, *TBB, *U;
  void *a_in = nullptr, *b_in = nullptr;
  if (host_in) {
    if (!p->a_blocks || !p->b_blocks || !p->t_aa || !p->t_ab || !p->t_bb || !p->u_norms)
      return fail(ctx, HSB_ERR_INPUT, "host block arrays are NULL");
    void *taa, *tab, *tbb, *u;
    CKS(ws(ctx, "in_a", stack_bytes, &a_in));
    CKS(ws(ctx, "in_b", stack_bytes, &b_in));
    CKS(ws(ctx, "in_taa", tblk_bytes * na, &taa));
    CKS(ws(ctx, "in_tab", tblk_bytes * na, &tab));
    CKS(ws(ctx, "in_tbb", tblk_bytes * na, &tbb));
    CKS(ws(ctx, "in_u", static_cast<size_t>(K) * 8, &u));
    A = static_cast<double*>(a_in);
    B = static_cast<double*>(b_in);
    TAA = static_cast<double*>(taa);
    TAB = static_cast<double*>(tab);
    TBB = static_cast<double*>(tbb);
    U = static_cast<double*>(u);
  } else {
    A = p->a_stack;
    B = p->b_stack;
    TAA = p->t_aa_dev;
    TAB = p->t_ab_dev;
    TBB = p->t_bb_dev;
    U = p->u_dev;
    if (!A || !B || !TAA || !TAB || !TBB || !U) return fail(ctx, HSB_ERR_INPUT, "device arrays are NULL");
  }
  double *H, *S;
  int64_t ldo;
  const size_t out_bytes = static_cast<size_t>(ng) * ng * 16;
  if (out->location == HSB_LOC_HOST) {
    void *h, *s;
    // host inputs: the pinned blocks land in these buffers first (raw_b in
    // out_s, raw_a in out_h; see stage_stack), so they hold a stack as well
    const size_t ob = host_in ? std::max(out_bytes, stack_bytes) : out_bytes;
    CKS(ws(ctx, "out_h", ob, &h));
    CKS(ws(ctx, "out_s", ob, &s));
    H = static_cast<double*>(h);
    S = static_cast<double*>(s);
    ldo = ng;
  } else {
    H = out->h;
    S = out->s;
    ldo = out->ld;
  }
  void *q, *info_d, *pbb, *zbuf, *ub, *rbuf, *offs_d, *potrf_scr = nullptr, *hostbuf;
  CKS(ws(ctx, "q", tblk_bytes * na, &q));
  CKS(ws(ctx, "info", static_cast<size_t>(na) * 4, &info_d));
  CKS(ws(ctx, "pbb", tblk_bytes * na, &pbb));
  CKS(ws(ctx, "z", stack_bytes, &zbuf));
  // the INT8 engine's fused paths scale B by u on the fly (UB not materialised)
  const bool u_fused = !unfused && ctx->engine == HSB_ENGINE_INT8;
  ub = nullptr;
  if (!u_fused) CKS(ws(ctx, "ub", stack_bytes, &ub));
  CKS(ws(ctx, "r", stack_bytes, &rbuf));
  CKS(ws(ctx, "offs", static_cast<size_t>(na) * 3 * 4, &offs_d));
  if (static_cast<size_t>(nl) * (nl + 1) / 2 * 16 > kPotrfSmemMax)
    CKS(ws(ctx, "potrf_scr", static_cast<size_t>(na) * nl * (nl + 1) / 2 * 16, &potrf_scr));
  CKS(pinned(ctx, (static_cast<size_t>(na) * 4 + 2) * 4, &hostbuf));
  // info and the non-finite flags come back through mapped host memory, written
  // by kernels: a copy-engine transfer would queue behind other streams' bulk
  // downloads (k-point lanes) and stall this call's compute stream
  int32_t* info_h = static_cast<int32_t*>(hostbuf);
  int32_t* hostbuf_dev = nullptr;
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hostbuf_dev), hostbuf, 0));
  double* Z = static_cast<double*>(zbuf);
  double* UB = static_cast<double*>(ub);
  double* R = static_cast<double*>(rbuf);  // [Y_hpd ; X_nh]
  int32_t* flag_h = info_h + na;  // first non-finite atom of A / B (pinned uploads)
  flag_h[0] = flag_h[1] = -1;

  // dma_done: recorded on s once the DMAs have landed, before the restack
  // kernels (which may wait for SMs held by another call's kernels)
  auto stage_stack = [&](int m, cudaStream_t s, const std::function<cudaError_t()>& dma_done) -> hsb_status {
    // A (m = 0) or B (m = 1) into the stacked layout.  Pinned blocks: one
    // contiguous DMA per atom into an atom-major buffer, then a device
    // restack (HBM speed).  Pageable blocks: host threads gather stacked
    // columns into pinned slots, checking finiteness on the fly
    // (probgen.validate_instance, probgen.py:155-161).
    const double* const* blocks = m == 0 ? p->a_blocks : p->b_blocks;
    double* dst = static_cast<double*>(m == 0 ? a_in : b_in);
    bool all_pinned = true;
    for (int64_t i = 0; i < na && all_pinned; ++i) all_pinned = host_is_pinned(blocks[i]);
    int64_t bad = -1;
    if (all_pinned) {
      void* raw;
      // atom-major landing buffer; with host outputs it aliases an output
      // buffer written only after the restack: B's (stream order on st:
      // restack, U norm, then S) in out_s, A's (restacked on the copy stream
      // before the compute stream waits for it) in out_h
      const bool alias = out->location == HSB_LOC_HOST;
      CKS(ws(ctx, alias ? (m == 0 ? "out_h" : "out_s") : (m == 0 ? "raw_a" : "raw_b"),
             alias ? std::max(out_bytes, stack_bytes) : stack_bytes, &raw));
      const size_t blk = static_cast<size_t>(nl) * ng * 16;
      for (int64_t i = 0; i < na; ++i)
        CK(cudaMemcpyAsync(static_cast<char*>(raw) + i * blk, blocks[i], blk, cudaMemcpyHostToDevice, s));
      h2d_bytes += static_cast<double>(blk) * na;
      if (dma_done) CK(dma_done());
      CK(launch_stack_blocks(static_cast<double*>(raw), dst, static_cast<int>(na), static_cast<int>(nl), ng, s));
      ++launches;
      void* flag;
      CKS(ws(ctx, m == 0 ? "bad_a" : "bad_b", 8, &flag));
      CK(launch_first_nonfinite(static_cast<double*>(raw), static_cast<int>(na), static_cast<int64_t>(nl) * ng * 2,
                                static_cast<int*>(flag), s));
      ++launches;
      CK(launch_copy_i32(static_cast<int32_t*>(flag), hostbuf_dev + na + m, 1, s));  // checked after the final sync
      ++launches;
      hc.mark(m == 0 ? "h2d A pinned" : "h2d B pinned");
      return HSB_OK;
    }
    CK(ctx->stager.h2d_stack(dst, blocks, na, nl, ng, s, &bad));
    h2d_bytes += static_cast<double>(stack_bytes);
    if (dma_done) CK(dma_done());
    hc.mark(m == 0 ? "h2d A stack" : "h2d B stack");
    if (bad >= 0) {
      cudaStreamSynchronize(st);
      cudaStreamSynchronize(cs);
      return fail(ctx, HSB_ERR_INVARIANT, std::string(m == 0 ? "a_blocks" : "b_blocks") + "[" +
                                              std::to_string(bad) + "] contains non-finite entries");
    }
    return HSB_OK;
  };

  // ------------------------------------------------------------- uploads
  cudaEvent_t ev_b_up;  // B stack uploaded
  CK(cudaEventCreateWithFlags(&ev_b_up, cudaEventDisableTiming));
  struct EvDel0 {
    cudaEvent_t e;
    ~EvDel0() { cudaEventDestroy(e); }
  } ev_b_up_del{ev_b_up};
  if (host_in) {
    std::vector<Copy2D> jobs;  // T blocks and u: the potrf / Loop 1 operands
    for (int64_t i = 0; i < na; ++i) {
      jobs.push_back({const_cast<double*>(TAA) + i * nl * nl * 2, tblk_bytes, p->t_aa[i], tblk_bytes, tblk_bytes, 1});
      jobs.push_back({const_cast<double*>(TAB) + i * nl * nl * 2, tblk_bytes, p->t_ab[i], tblk_bytes, tblk_bytes, 1});
      jobs.push_back({const_cast<double*>(TBB) + i * nl * nl * 2, tblk_bytes, p->t_bb[i], tblk_bytes, tblk_bytes, 1});
      jobs.push_back({const_cast<double*>(U) + i * nl, static_cast<size_t>(nl) * 8, p->u_norms[i],
                      static_cast<size_t>(nl) * 8, static_cast<size_t>(nl) * 8, 1});
    }
    CK(ctx->stager.h2d(jobs, st));
    for (const auto& j : jobs) h2d_bytes += static_cast<double>(j.width) * j.height;
    hc.mark("h2d T,u");
    CKS(stage_stack(1, st, [&] {
      tr.mark(st, "h2d_b");
      return cudaEventRecord(ev_b_up, st);
    }));
    if (!overlap_upload) CKS(stage_stack(0, st, [&] { return order_done(out->h2d_done, 1, st); }));
    CK(tl.mark(st, "h2d"));
  }
  CK(order_wait(out->compute_after, 2, st));

  // ------------------------------------------- Loop 2, part 1: Cholesky routing
  // On the fused INT8 path with the side preparation (the default) nothing on
  // the device waits for the routing -- H = A^H V1 + (UB)^H W2 covers HPD and
  // non-HPD atoms alike; only the split counts need it -- so the 32-CTA,
  // latency-bound potrf runs on the copy stream after S's operand preparation,
  // beside the S contraction, instead of ahead of everything on the compute
  // stream; the host collects the counts after enqueueing H.
  cudaEvent_t ev_info;
  CK(cudaEventCreateWithFlags(&ev_info, cudaEventDisableTiming));
  struct EvDel {
    cudaEvent_t e;
    ~EvDel() {
      if (e) cudaEventDestroy(e);
    }
  } ev_info_del{ev_info};
  auto routing = [&](cudaStream_t s_) -> hsb_status {
    CK(launch_potrf_route(TAA, static_cast<double*>(q), static_cast<int32_t*>(info_d), static_cast<int>(na),
                          static_cast<int>(nl), force_nonhpd, static_cast<double*>(potrf_scr), s_));
    ++launches;
    CK(launch_route_atoms(static_cast<int32_t*>(info_d), static_cast<int>(na), static_cast<int>(nl),
                          static_cast<int32_t*>(offs_d), hostbuf_dev, s_));
    ++launches;
    CK(cudaEventRecord(ev_info, s_));
    return HSB_OK;
  };
  static const bool no_defer_routing = std::getenv("HSB_NO_DEFER_ROUTING") != nullptr;  // A/B experiments
  const bool defer_routing = !unfused && !overlap_upload && ctx->engine == HSB_ENGINE_INT8 && !no_defer_routing &&
                             !(std::getenv("HSB_INT8_V") != nullptr) && !(std::getenv("HSB_NO_SIDE_PREP") != nullptr);
  if (!defer_routing) CKS(routing(st));
  CK(tl.mark(st, "loop2"));
  bool side_prep_used = false;  // set by the fused branch below

  auto loop1 = [&]() -> hsb_status {  // Z_a = T_AB^H A_a + (1/2 T_BB)^H B_a (builder.py:73-88)
    CK(launch_half_mirror(TBB, static_cast<double*>(pbb), static_cast<int>(nl), na, 0.5, st));
    ++launches;
    ZrkCall z;
    z.segs.push_back({atom_mats(TAB, na, nl), atom_rows(A, na, nl, ng, K)});
    z.segs.push_back({atom_mats(static_cast<double*>(pbb), na, nl), atom_rows(B, na, nl, ng, K)});
    z.m = nl;
    z.n = ng;
    z.c = Z;
    z.ldc = K;
    z.batch = na;
    z.c_bstride = nl;
    CKS(run_zrk(ctx, st, z, &launches));
    CK(tl.mark(st, "loop1"));
    return HSB_OK;
  };
  // Fused path: H = sum_a X_a^H M_a X_a with X_a = [A_a; B_a] and the
  // Hermitian M_a = [[T_AA, T_AB], [T_AB^H, T_BB]] (Eq. 7; the
  // reference's Loop 1 / H1 / Loop 2 / H2 / H3 regroup these four terms):
  // V1_a = T_AA A_a + T_AB B_a and V2_a = T_AB^H A_a + T_BB B_a (batched, into the
  // Z and R stacks), then H = A^H V1 + B^H V2 over the lower triangle, a
  // reduction of 2K instead of the 3K of Z^H B + B^H Z + Y^H Y.  The same
  // product covers HPD and non-HPD T_AA alike; potrf_route still runs for the
  // reference's split counts.  T_AA and T_BB are read from their lower
  // triangles (kernels.py:223-231, 296-307), as in the reference.
  // INT8 engine, HSB_INT8_V=1 (experimental): the V products run on the INT8
  // tensor cores inside the H phase (run_ozaki_hv), sharing H's left residues
  // of A and B.  Measured slower than the DMMA V products so far (C3: 4.6 vs
  // 3.3 ms; its modular GEMM is epilogue-bound at K = 2 n_l), so off by default.
  static const bool int8_v_env = std::getenv("HSB_INT8_V") != nullptr;
  const bool int8_v = int8_v_env && !unfused && ctx->engine == HSB_ENGINE_INT8 && 2 * nl <= 256;
  // INT8 engine, fused paths: shared left exponent / A residues (oz_left below)
  const bool oz_share = !unfused && ctx->engine == HSB_ENGINE_INT8 && !int8_v;
  // ... and H regrouped as A^H V1 + (UB)^H W2 with W2 = U^-1 V2 (the rows of V2
  // divided by u: B^H V2 = B^H U U^-1 V2), so H's left operands are exactly S's
  // (A and UB, one shared exponent): their residue planes serve both
  // contractions and B's own residue pass disappears.  W2 comes out of the V
  // products directly: the columns of V2's left blocks (T_AB, T_BB) are divided
  // by u first (per-atom 121 x 121 blocks; one correctly rounded division each).
  static const bool no_h_ub = std::getenv("HSB_NO_H_UB") != nullptr;  // A/B experiments
  const bool h_via_ub = oz_share && u_fused && !no_h_ub;
  int32_t* oz_er_v = nullptr;  // H's right exponents from the V products' epilogue
  auto vloop = [&]() -> hsb_status {
    if (int8_v) return HSB_OK;
    void *taa_full, *tab_h;
    CKS(ws(ctx, "taa_full", tblk_bytes * na, &taa_full));
    CKS(ws(ctx, "tab_h", tblk_bytes * na, &tab_h));
    CK(launch_half_mirror(TAA, static_cast<double*>(taa_full), static_cast<int>(nl), na, 1.0, st));
    CK(launch_half_mirror(TBB, static_cast<double*>(pbb), static_cast<int>(nl), na, 1.0, st));
    CK(launch_conj_transpose(TAB, static_cast<double*>(tab_h), static_cast<int>(nl), na, st));
    launches += 3;
    const double* v2_l0 = TAB;                              // (T_AB^H)^H
    const double* v2_l1 = static_cast<const double*>(pbb);  // T_BB^H = T_BB
    if (h_via_ub) {  // W2 = U^-1 V2: V2's left blocks with their columns divided by u
      void *tab_s, *tbb_s;
      CKS(ws(ctx, "tab_u", tblk_bytes * na, &tab_s));
      CKS(ws(ctx, "tbb_u", tblk_bytes * na, &tbb_s));
      CK(launch_scale_cols_inv(TAB, static_cast<double*>(tab_s), U, static_cast<int>(nl), na, st));
      CK(launch_scale_cols_inv(static_cast<const double*>(pbb), static_cast<double*>(tbb_s), U,
                               static_cast<int>(nl), na, st));
      launches += 2;
      v2_l0 = static_cast<const double*>(tab_s);
      v2_l1 = static_cast<const double*>(tbb_s);
    }
    // INT8 engine: the V products' epilogue also yields H's right column
    // exponents (max over V1 and V2), so no separate exponent pass reads them
    static const bool no_vexp = std::getenv("HSB_NO_VEXP") != nullptr;  // A/B experiments
    if (oz_share && ctx->cplx == HSB_CPLX_3M && !no_vexp) {
      void* erb;
      CKS(ws(ctx, "oz_exp_r", static_cast<size_t>(ng) * 4, &erb));
      oz_er_v = static_cast<int32_t*>(erb);
      CK(hsb::launch_ozaki_init_exp(oz_er_v, ng, st));
      ++launches;
    }
    for (int half = 0; half < 2; ++half) {  // zrk form: sum_s L_s^H R_s
      ZrkCall z;
      z.col_exp = oz_er_v;
      const double* l0 = half == 0 ? static_cast<const double*>(taa_full) : v2_l0;  // T_AA | (T_AB^H)^H
      const double* l1 = half == 0 ? static_cast<const double*>(tab_h) : v2_l1;     // (T_AB)^H^H | T_BB
      z.segs.push_back({atom_mats(l0, na, nl), atom_rows(A, na, nl, ng, K)});
      z.segs.push_back({atom_mats(l1, na, nl), atom_rows(B, na, nl, ng, K)});
      z.m = nl;
      z.n = ng;
      z.c = half == 0 ? Z : R;
      z.ldc = K;
      z.batch = na;
      z.c_bstride = nl;
      CKS(run_zrk(ctx, st, z, &launches));
    }
    CK(tl.mark(st, "loop1"));
    return HSB_OK;
  };
  // INT8 engine (fused paths): UB is never materialised -- its column exponents
  // and residues read B and scale each row by u on the fly, rounding the product
  // exactly as diag_scale_kernel does
  auto ub_view = [&]() {
    OperandView v = plain(u_fused ? B : UB, K, ng, K);
    if (u_fused) v.rscale = U;
    return v;
  };
  auto unorm = [&]() -> hsb_status {  // UB = diag(u) B (builder.py:124-127)
    if (u_fused) return HSB_OK;
    CK(launch_diag_scale(B, K, UB, K, U, K, ng, st));
    ++launches;
    CK(tl.mark(st, "unorm"));
    return HSB_OK;
  };

  // INT8 engine, fused paths: one left exponent per column over A and UB (and B
  // when H's left side is B) (ozaki_colexp_ab, one pass over A and B) shared by
  // S = A^H A + (UB)^H (UB) and the left side of H = A^H V1 + (UB)^H W2, so the
  // residue planes of A and UB are computed once for both contractions; H's
  // right side (V1, W2) gets its own exponents.
  // The planes are sized for the 2K reduction (oz_ktot) of both calls.
  int32_t* oz_el = nullptr;
  int8_t* oz_res_a = nullptr;
  int8_t* oz_res_ub = nullptr;  // S's UB planes, when prepared ahead (oz_left(with_ub))
  auto oz_left = [&](cudaStream_t s_, bool with_ub) -> hsb_status {  // A and B resident
    if (!oz_share || oz_el) return HSB_OK;
    int n_mod = 0, bits = 0;
    CKS(oz_choose(ctx, 2 * K, &n_mod, &bits));
    const int64_t kpad = hsb::oz_kpad(K);
    const size_t pbytes = static_cast<size_t>(hsb::kOzPlanes) * n_mod * ng * kpad;
    const hsb_ctx::OzPrepared& pre = ctx->oz_prepared;
    if (h_via_ub && pre.a == A && pre.k == K && pre.ng == ng && pre.n_mod == n_mod && pre.bits == bits) {
      // the matching kernel already wrote the exponents and the A / UB planes
      void *eb, *rb, *ubb;
      CKS(ws(ctx, "oz_exp_l", static_cast<size_t>(ng) * 4, &eb));
      CKS(ws(ctx, "oz_res_a", pbytes, &rb));
      CKS(ws(ctx, "oz_res2", pbytes, &ubb));
      oz_el = static_cast<int32_t*>(eb);
      oz_res_a = static_cast<int8_t*>(rb);
      oz_res_ub = static_cast<int8_t*>(ubb);
      return HSB_OK;
    }
    void *eb, *rb;
    CKS(ws(ctx, "oz_exp_l", static_cast<size_t>(ng) * 4, &eb));
    CKS(ws(ctx, "oz_res_a", pbytes, &rb));
    oz_el = static_cast<int32_t*>(eb);
    oz_res_a = static_cast<int8_t*>(rb);
    CK(hsb::launch_ozaki_colexp_ab(A, B, K, K, ng, U, oz_el, s_, !h_via_ub));
    hsb::OzResSrc rs[2] = {{A, K, K, oz_el, nullptr, oz_res_a, kpad}, {}};
    if (with_ub) {
      // the buffer H's contraction uses for its third operand (V2) afterwards,
      // in stream order behind S: no extra workspace
      void* ubb;
      CKS(ws(ctx, "oz_res2", pbytes, &ubb));
      oz_res_ub = static_cast<int8_t*>(ubb);
      rs[1] = {B, K, K, oz_el, U, oz_res_ub, kpad};
    }
    CK(hsb::launch_ozaki_residues_batch(rs, with_ub ? 2 : 1, ng, bits, n_mod, s_));  // A and UB: one launch
    launches += 2;
    return HSB_OK;
  };
  auto oz_use_left = [&](ZrkCall& z, const int32_t* er) {
    if (!oz_share) return;
    z.oz_el = oz_el;
    z.oz_er = er ? er : oz_el;
    z.oz_pre.push_back({A, 0, oz_res_a});
    if (oz_res_ub && (!er || h_via_ub)) z.oz_pre.push_back({B, 0, oz_res_ub, U});  // S (and H via UB)
    z.oz_ktot = 2 * K;
  };

  // ------------------------------------------------------ Loop 1, U norm, S
  if (overlap_upload) {
    CKS(unorm());
    ZrkCall s2 = tri_call(S, ldo, ng, kLowerOnly, 0.0);
    s2.segs.push_back({ub_view(), ub_view()});
    s2.tl = &tl, s2.sect = "s2", s2.core = "s2_core";
    CKS(run_zrk(ctx, st, s2, &launches));
    CK(tl.mark(st, "s2"));
    // A rides the copy engine while (UB)^H(UB) runs -- after B's DMAs, so the
    // two uploads do not split the PCIe bandwidth B is waited on
    CK(cudaStreamWaitEvent(cs, ev_b_up, 0));
    CKS(stage_stack(0, cs, [&] {
      tr.mark(cs, "h2d_a");
      return order_done(out->h2d_done, 1, cs);
    }));
    cudaEvent_t ev_a;
    CK(cudaEventCreateWithFlags(&ev_a, cudaEventDisableTiming));
    EvDel ev_a_del{ev_a};
    CK(cudaEventRecord(ev_a, cs));
    CK(cudaStreamWaitEvent(st, ev_a, 0));
    CK(tl.mark(st, "h2d"));
    ZrkCall s1 = tri_call(S, ldo, ng, kLowerOnly | out_mirror, 1.0);
    s1.segs.push_back({plain(A, K, ng, K), plain(A, K, ng, K)});
    s1.tl = &tl, s1.sect = "s1", s1.core = "s1_core";
    if (chunk_s) s1.chunk_events = &s_chunks;
    CKS(oz_left(st, false));
    oz_use_left(s1, nullptr);
    CKS(run_zrk(ctx, st, s1, &launches));
    CK(tl.mark(st, "s1"));
    CKS(vloop());
  } else if (unfused) {
    CKS(loop1());
    ZrkCall h1 = tri_call(H, ldo, ng, kLowerOnly | kZeroImagDiag, 0.0);  // builder.h_cross (builder.py:91-104)
    h1.segs.push_back({plain(Z, K, ng, K), plain(B, K, ng, K)});
    h1.segs.push_back({plain(B, K, ng, K), plain(Z, K, ng, K)});
    CKS(run_zrk(ctx, st, h1, &launches));
    CK(tl.mark(st, "h1"));
    ZrkCall s1 = tri_call(S, ldo, ng, kLowerOnly | kZeroImagDiag, 0.0);  // builder.build_s (builder.py:107-132)
    s1.segs.push_back({plain(A, K, ng, K), plain(A, K, ng, K)});
    CKS(run_zrk(ctx, st, s1, &launches));
    CK(tl.mark(st, "s1"));
    CKS(unorm());
    ZrkCall s2 = tri_call(S, ldo, ng, kLowerOnly | kZeroImagDiag, 1.0);
    s2.segs.push_back({plain(UB, K, ng, K), plain(UB, K, ng, K)});
    CKS(run_zrk(ctx, st, s2, &launches));
    if (!(opts & HSB_OPT_LOWER_ONLY)) {
      CK(launch_mirror(S, ldo, static_cast<int>(ng), st));
      ++launches;
    }
    CK(tl.mark(st, "s2"));
  } else {
    // INT8 engine: S's operand preparation (exponents, A and UB residues) does
    // not depend on the V products; it runs on the copy stream, overlapping the
    // DMMA V products (they leave registers and shared memory for it on every SM)
    static const bool no_side = std::getenv("HSB_NO_SIDE_PREP") != nullptr;  // A/B experiments
    const bool side_prep = oz_share && u_fused && !int8_v && !no_side;
    side_prep_used = side_prep;
    cudaEvent_t ev_prep_in = nullptr, ev_prep_out = nullptr;
    if (side_prep) {
      CK(cudaEventCreateWithFlags(&ev_prep_in, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ev_prep_out, cudaEventDisableTiming));
    }
    EvDel ev_prep_in_del{ev_prep_in}, ev_prep_out_del{ev_prep_out};
    if (side_prep) {
      CK(cudaEventRecord(ev_prep_in, st));
      CK(cudaStreamWaitEvent(cs, ev_prep_in, 0));
    }
    CKS(vloop());
    if (side_prep) {
      CKS(oz_left(cs, true));
      CK(cudaEventRecord(ev_prep_out, cs));
      if (defer_routing) CKS(routing(cs));  // after the event: S does not wait for it
      CK(cudaStreamWaitEvent(st, ev_prep_out, 0));
    }
    CKS(unorm());
    ZrkCall s = tri_call(S, ldo, ng, kLowerOnly | out_mirror, 0.0);
    s.segs.push_back({plain(A, K, ng, K), plain(A, K, ng, K)});
    s.segs.push_back({ub_view(), ub_view()});
    s.tl = &tl, s.sect = "s", s.core = "s_core";
    if (chunk_s) s.chunk_events = &s_chunks;
    s.peer = peer;
    CKS(oz_left(st, false));
    oz_use_left(s, nullptr);
    CKS(run_zrk(ctx, st, s, &launches));
    CK(tl.mark(st, "s"));
  }
  cudaEvent_t ev_s;  // S final
  CK(cudaEventCreateWithFlags(&ev_s, cudaEventDisableTiming));
  EvDel ev_s_del{ev_s};
  CK(cudaEventRecord(ev_s, st));
  tr.mark(st, "s_done");
  if (out->s_ready) CK(cudaEventRecord(static_cast<cudaEvent_t>(out->s_ready), st));

  // ------------------------------------------- routing (host, overlaps S)
  hc.mark("enqueue to S");
  if (defer_routing && !side_prep_used) CKS(routing(st));  // (no side preparation ran: on the compute stream)
  int64_t n_hpd = 0, n_nh = 0;
  auto await_routing = [&]() -> hsb_status {
    CK(cudaEventSynchronize(ev_info));
    hc.mark("routing wait");
    n_hpd = n_nh = 0;
    std::atomic_thread_fence(std::memory_order_acquire);
    for (int64_t i = 0; i < na; ++i) (info_h[i] == 0 ? n_hpd : n_nh)++;
    if (atom_info) std::memcpy(atom_info, info_h, na * 4);
    return HSB_OK;
  };
  if (!defer_routing) CKS(await_routing());
  const int32_t* offs_dev = static_cast<int32_t*>(offs_d);

  // ------------------------------------------- Loop 2, part 2 (builder.py:162-185)
  // (unfused path only: the fused H uses V1, V2)
  double* ANH = nullptr;
  if (unfused) {
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
  CK(tl.mark(st, "loop2"));
  const int64_t k_hpd = n_hpd * nl, k_nh = n_nh * nl;
  const double* Y = R;
  const double* XNH = R + 2 * k_hpd;
  // Stream H to pinned host memory while the H contraction runs (fused path)
  const int64_t ntiles = (ng + kBN - 1) / kBN;
  const bool stream_h = !unfused && out->location == HSB_LOC_HOST && host_is_pinned(out->h);
  // lower-triangle downloads + host mirror: the streamed (chunked) paths only
  const bool lower_d2h = stream_h && chunk_s && !(opts & HSB_OPT_FULL_D2H);
  HostMirror mirror;

  // -------------------------------------------------- H (builder.py:91-104, 187-200)
  if (unfused) {
    if (n_nh > 0) {  // H2: gemm('C','N', beta = 1), lower tiles (the mirror rebuilds the rest)
      ZrkCall h2 = tri_call(H, ldo, ng, kLowerOnly, 1.0);
      h2.segs.push_back({plain(ANH, k_nh, ng, k_nh), plain(XNH, k_nh, ng, K)});
      CKS(run_zrk(ctx, st, h2, &launches));
    }
    CK(tl.mark(st, "h2"));
    if (n_hpd > 0) {  // H3: herk(beta = 1)
      ZrkCall h3 = tri_call(H, ldo, ng, kLowerOnly | kZeroImagDiag, 1.0);
      h3.segs.push_back({plain(Y, k_hpd, ng, K), plain(Y, k_hpd, ng, K)});
      CKS(run_zrk(ctx, st, h3, &launches));
    }
    if (!(opts & HSB_OPT_LOWER_ONLY)) {
      CK(launch_mirror(H, ldo, static_cast<int>(ng), st));
      ++launches;
    }
    CK(tl.mark(st, "h3"));
  } else {
    ZrkCall h = tri_call(H, ldo, ng, kLowerOnly | out_mirror, 0.0);
    h.segs.push_back({plain(A, K, ng, K), plain(Z, K, ng, K)});  // A^H V1
    if (h_via_ub)
      h.segs.push_back({ub_view(), plain(R, K, ng, K)});  // (UB)^H W2
    else
      h.segs.push_back({plain(B, K, ng, K), plain(R, K, ng, K)});  // B^H V2
    h.tl = &tl, h.sect = "h", h.core = "h_core";
    h.peer = peer;
    h.peer_is_h = true;
    if (stream_h) {  // per-column-block completion counters in mapped host memory
      const size_t nb = static_cast<size_t>(ntiles);
      if (ctx->done_cnt_len < nb) {
        if (ctx->done_cnt) cudaFreeHost(ctx->done_cnt);
        ctx->done_cnt = nullptr;
        ctx->done_cnt_len = 0;
        CK(cudaHostAlloc(reinterpret_cast<void**>(&ctx->done_cnt), nb * sizeof(int), cudaHostAllocMapped));
        ctx->done_cnt_len = nb;
      }
      std::memset(ctx->done_cnt, 0, nb * sizeof(int));
      int* dptr = nullptr;
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dptr), ctx->done_cnt, 0));
      h.done_cnt = dptr;
    }
    tr.mark(st, "loop2_done");
    if (int8_v) {
      HvCall hv;
      hv.A = A;
      hv.B = B;
      hv.TAA = TAA;
      hv.TAB = TAB;
      hv.TBB = TBB;
      hv.V1 = Z;
      hv.V2 = R;
      hv.K = K;
      hv.ng = ng;
      hv.nl = nl;
      hv.na = na;
      hv.tl = &tl;
      hv.vsect = "loop1";
      CKS(run_ozaki_hv(ctx, st, hv, h, &launches));
    } else {
      if (oz_share) {  // H's right exponents: V1, V2 only
        int32_t* er = oz_er_v;
        if (!er) {  // 4M V products: a separate pass
          void* erb;
          CKS(ws(ctx, "oz_exp_r", static_cast<size_t>(ng) * 4, &erb));
          er = static_cast<int32_t*>(erb);
          CK(hsb::launch_ozaki_init_exp(er, ng, st));
          CK(hsb::launch_ozaki_colexp(Z, K, K, ng, er, st));
          CK(hsb::launch_ozaki_colexp(R, K, K, ng, er, st));
          launches += 3;
        }
        oz_use_left(h, er);
      }
      CKS(run_zrk(ctx, st, h, &launches));
    }
    CK(tl.mark(st, "h"));
    tr.mark(st, "h_done");
    if (defer_routing) CKS(await_routing());
  }
  CK(order_done(out->compute_done, 2, st));

  // --------------------------------------------------------------- outputs
  if (out->location == HSB_LOC_HOST) {
    // S is final at ev_s: its download runs on the copy stream, concurrently
    // with the H contraction; H follows on the compute stream.
    const size_t row = static_cast<size_t>(ng) * 16;
    // columns [c0, c1) of a final matrix to the host, on the copy stream.
    // lower_d2h: one copy per 64-column block [a, b) of rows >= d2h_row0(a), and a
    // host mirror job for rows [a, b) of the columns >= b (below their d2h_row0)
    // once it has landed
    // HSB_LOWER_D2H (experiments): which matrices cross as lower triangles ("hs", "s", "h", "-")
    static const std::string lower_which = [] {
      const char* e = std::getenv("HSB_LOWER_D2H");
      return std::string(e ? e : "hs");
    }();
    const double upper_frac = d2h_upper_frac(host_in);
    auto download = [&](double* dst, const double* src, int64_t c0, int64_t c1) -> hsb_status {
      const bool lower = lower_d2h && lower_which.find(dst == out->h ? 'h' : 's') != std::string::npos;
      const int64_t step = lower ? 64 : c1 - c0;  // (c0 is a multiple of 64: d2h_row0's blocks)
      for (int64_t a = c0; a < c1; a += step) {
        const int64_t b = std::min(c1, a + step), r0 = lower ? d2h_row0(a, upper_frac) : 0;
        CK(cudaMemcpy2DAsync(reinterpret_cast<char*>(dst) + (a * out->ld + r0) * 16, out->ld * 16,
                             reinterpret_cast<const char*>(src) + (a * ldo + r0) * 16, ldo * 16, (ng - r0) * 16,
                             b - a, cudaMemcpyDeviceToHost, cs));
        d2h_bytes += 16.0 * (ng - r0) * (b - a);
        if (lower) CK(mirror.push(cs, dst, out->ld, ng, a, b, upper_frac));
      }
      return HSB_OK;
    };
    if (!s_chunks.empty()) {
      // column groups of S download as soon as each is final
      int64_t c0 = 0;
      for (const auto& c : s_chunks) {
        CK(cudaStreamWaitEvent(cs, c.first, 0));
        if (c.second > c0) {
          CKS(download(out->s, S, c0, c.second));
        }
        tr.mark(cs, "d2h_s " + std::to_string(c.second));
        c0 = c.second;
      }
    } else {
      CK(cudaStreamWaitEvent(cs, ev_s, 0));
      d2h_bytes += 16.0 * ng * ng;
      CK(ctx->stager.d2h({{out->s, static_cast<size_t>(out->ld) * 16, S, static_cast<size_t>(ldo) * 16, row,
                           static_cast<size_t>(ng)}},
                         cs));
    }
    if (stream_h) {
      // poll the tile counters; a column block is final when all T tiles that
      // write into it are done (column-major tile order makes this a prefix)
      cudaEvent_t ev_h;
      CK(cudaEventCreateWithFlags(&ev_h, cudaEventDisableTiming));
      EvDel ev_h_del{ev_h};
      CK(cudaEventRecord(ev_h, st));
      volatile int* cnt = ctx->done_cnt;
      const int64_t T = ntiles;
      const int64_t batch = std::max<int64_t>(1, T / 16);
      int64_t sent = 0;
      while (sent < T) {
        int64_t c = sent;
        while (c < T && cnt[c] >= T) ++c;
        const bool kernel_done = cudaEventQuery(ev_h) == cudaSuccess;
        if (kernel_done) c = T;  // everything is final (also guards a counter mismatch)
        if (c - sent >= batch || (c == T && c > sent)) {
          std::atomic_thread_fence(std::memory_order_acquire);
          const int64_t c0 = sent * kBN, c1 = std::min<int64_t>(c * kBN, ng);
          CKS(download(out->h, H, c0, c1));
          tr.mark(cs, "d2h_h " + std::to_string(c1));
          sent = c;
        } else {
          std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
      }
      hc.mark("stream H");
    } else {
      d2h_bytes += 16.0 * ng * ng;
      CK(ctx->stager.d2h({{out->h, static_cast<size_t>(out->ld) * 16, H, static_cast<size_t>(ldo) * 16, row,
                           static_cast<size_t>(ng)}},
                         st));
    }
  }
  cudaEvent_t ev_cs;
  CK(cudaEventCreateWithFlags(&ev_cs, cudaEventDisableTiming));
  EvDel ev_cs_del{ev_cs};
  CK(cudaEventRecord(ev_cs, cs));
  CK(cudaStreamWaitEvent(st, ev_cs, 0));
  CK(tl.mark(st, "d2h"));
  hc.mark("enqueue H + d2h");
  if (!tm && !host_in && out->location == HSB_LOC_DEVICE) return HSB_OK;  // asynchronous: stream order
  CK(cudaEventSynchronize(tl.marks.back().second));
  CK(mirror.finish());
  hc.mark("final sync");
  hc.report();
  tr.report();
  for (int m = 0; m < 2; ++m)
    if (flag_h[m] >= 0 && flag_h[m] < na)  // pinned uploads are scanned on the device; outputs are discarded
      return fail(ctx, HSB_ERR_INVARIANT, std::string(m == 0 ? "a_blocks" : "b_blocks") + "[" +
                                              std::to_string(flag_h[m]) + "] contains non-finite entries");

  if (tm) {
    std::memset(tm, 0, sizeof(*tm));
    tm->h2d = tl.total("h2d");
    tm->loop1 = tl.total("loop1");
    tm->loop2 = tl.total("loop2");
    tm->unorm = tl.total("unorm");
    const double fS = 4.0 * K * double(ng) * ng;
    // (the routing may have been collected after H was enqueued: recount)
    const double fH1 = 8.0 * K * double(ng) * ng, fH2 = 8.0 * n_nh * nl * double(ng) * ng,
                 fH3 = 4.0 * n_hpd * nl * double(ng) * ng;
    const double ts = tl.total("s") + tl.total("s_core");  // fused S: split S1/S2 by model flops (equal)
    tm->s1 = tl.total("s1") + tl.total("s1_core") + ts * 0.5;
    tm->s2 = tl.total("s2") + tl.total("s2_core") + ts * 0.5;
    tm->s_core = tl.total("s_core") + tl.total("s1_core") + tl.total("s2_core");
    tm->h_core = tl.total("h_core");
    const double th = tl.total("h") + tl.total("h_core"), fh = fH1 + fH2 + fH3;
    tm->h1 = tl.total("h1") + th * fH1 / fh;
    tm->h2 = tl.total("h2") + th * fH2 / fh;
    tm->h3 = tl.total("h3") + th * fH3 / fh;
    (void)fS;
    tm->d2h = tl.total("d2h");
    tm->total = tl.span();
    tm->n_hpd = static_cast<int32_t>(n_hpd);
    tm->n_nonhpd = static_cast<int32_t>(n_nh);
    tm->launches = launches;
    tm->h2d_bytes = h2d_bytes;
    tm->d2h_bytes = d2h_bytes;
  }
  return HSB_OK;
}

// validate the physical inputs and upload them into the context's workspace;
// the caller's host arrays may be reused once this returns
static hsb_status match_setup(hsb_ctx* ctx, cudaStream_t st, const hsb_phys* ph, int64_t ld, MatchParams* mp_out) {
  if (!ph) return fail(ctx, HSB_ERR_INPUT, "NULL argument");
  if (ph->n_atoms < 1 || ph->n_g < 1 || ph->n_types < 1 || ph->lmax < 0)
    return fail(ctx, HSB_ERR_INPUT, "dimensions must be positive");
  if (ph->lmax > kMaxL) return fail(ctx, HSB_ERR_UNSUPPORTED, "lmax above 31");
  if (ph->n_g > 0x7fffffff) return fail(ctx, HSB_ERR_UNSUPPORTED, "too many G vectors");
  const int64_t nlm = static_cast<int64_t>(ph->lmax + 1) * (ph->lmax + 1);
  if (ld < ph->n_atoms * nlm) return fail(ctx, HSB_ERR_DIMENSION, "ld < n_atoms * (lmax+1)^2");
  if (!(ph->omega > 0.0)) return fail(ctx, HSB_ERR_INPUT, "cell volume must be positive");
  if (!ph->gvec || !ph->tau || !ph->type_of || !ph->rmt || !ph->radial)
    return fail(ctx, HSB_ERR_INPUT, "NULL input array");
  for (int64_t a = 0; a < ph->n_atoms; ++a)
    if (ph->type_of[a] < 0 || ph->type_of[a] >= ph->n_types) return fail(ctx, HSB_ERR_INPUT, "type index out of range");
  const size_t gb = ph->n_g * 3 * 4, tb = ph->n_atoms * 3 * 8, yb = ph->n_atoms * 4, rb = ph->n_types * 8,
               db = ph->n_types * (ph->lmax + 1) * 4 * 8;
  void *g, *t, *y, *r, *d;
  CKS(ws(ctx, "m_gvec", gb, &g));
  CKS(ws(ctx, "m_tau", tb, &t));
  CKS(ws(ctx, "m_type", yb, &y));
  CKS(ws(ctx, "m_rmt", rb, &r));
  CKS(ws(ctx, "m_radial", db, &d));
  // the small inputs go through a pinned staging buffer: the copies are truly
  // asynchronous (no host stall between back-to-back calls); the buffer is
  // reused once the previous call's copies have run (event)
  const size_t sizes[5] = {gb, tb, yb, rb, db};
  const void* srcs[5] = {ph->gvec, ph->tau, ph->type_of, ph->rmt, ph->radial};
  void* dsts[5] = {g, t, y, r, d};
  size_t total = 0, offs[5];
  for (int i = 0; i < 5; ++i) {
    offs[i] = total;
    total += (sizes[i] + 255) / 256 * 256;
  }
  if (ctx->m_stage_done) CK(cudaEventSynchronize(ctx->m_stage_done));
  else CK(cudaEventCreateWithFlags(&ctx->m_stage_done, cudaEventDisableTiming));
  if (ctx->m_stage_bytes < total) {
    if (ctx->m_stage) cudaFreeHost(ctx->m_stage);
    ctx->m_stage = nullptr;
    ctx->m_stage_bytes = 0;
    CK(cudaHostAlloc(&ctx->m_stage, total, cudaHostAllocDefault));
    ctx->m_stage_bytes = total;
  }
  for (int i = 0; i < 5; ++i) {
    std::memcpy(static_cast<char*>(ctx->m_stage) + offs[i], srcs[i], sizes[i]);
    CK(cudaMemcpyAsync(dsts[i], static_cast<char*>(ctx->m_stage) + offs[i], sizes[i], cudaMemcpyHostToDevice, st));
  }
  CK(cudaEventRecord(ctx->m_stage_done, st));
  MatchParams mp;
  std::memset(&mp, 0, sizeof(mp));
  mp.gvec = static_cast<int32_t*>(g);
  mp.tau = static_cast<double*>(t);
  mp.type_of = static_cast<int32_t*>(y);
  mp.rmt = static_cast<double*>(r);
  mp.radial = static_cast<double*>(d);
  for (int i = 0; i < 3; ++i) mp.kpt[i] = ph->kpt[i];
  for (int i = 0; i < 9; ++i) mp.recip[i] = ph->recip[i];
  mp.pre = 4.0 * 3.14159265358979323846 / std::sqrt(ph->omega);
  mp.n_g = ph->n_g;
  mp.ld = ld;
  mp.n_atoms = static_cast<int32_t>(ph->n_atoms);
  mp.n_types = ph->n_types;
  mp.lmax = ph->lmax;
  if (match_smem_bytes(mp) > 200 * 1024) return fail(ctx, HSB_ERR_UNSUPPORTED, "too many atoms for one column CTA");
  *mp_out = mp;
  return HSB_OK;
}

hsb_status hsb_match_coeffs(hsb_ctx* ctx, void* stream, const hsb_phys* ph, double* a_stack, double* b_stack,
                            int64_t ld) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
  CtxCall call_guard(ctx, false);
  if (!ph || !a_stack || !b_stack) return fail(ctx, HSB_ERR_INPUT, "NULL argument");
  cudaSetDevice(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  MatchParams mp;
  CKS(match_setup(ctx, st, ph, ld, &mp));
  CK(launch_match_coeffs(mp, a_stack, b_stack, st));
  return HSB_OK;
}

hsb_status hsb_build_hs_physical(hsb_ctx* ctx, void* stream, const hsb_phys* ph, const hsb_problem* p,
                                 uint32_t opts, const hsb_output* out, hsb_timings* tm, int32_t* atom_info) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
  CtxCall call_guard(ctx, true);
  ctx->oz_prepared = {};
  if (!ph || !p || !out) return fail(ctx, HSB_ERR_INPUT, "NULL argument");
  if (p->location != HSB_LOC_DEVICE || !p->a_stack || !p->b_stack || !p->u_dev)
    return fail(ctx, HSB_ERR_INPUT, "the physical build needs device stacks (outputs of the matching kernel) and u");
  const int64_t nlm = static_cast<int64_t>(ph->lmax + 1) * (ph->lmax + 1);
  if (p->n_atoms != ph->n_atoms || p->n_l != nlm || p->n_g != ph->n_g)
    return fail(ctx, HSB_ERR_DIMENSION, "problem dimensions disagree with the physical inputs");
  cudaSetDevice(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t K = p->n_atoms * p->n_l, ng = p->n_g;
  double* A = const_cast<double*>(static_cast<const double*>(p->a_stack));
  double* B = const_cast<double*>(static_cast<const double*>(p->b_stack));
  MatchParams mp;
  CKS(match_setup(ctx, st, ph, K, &mp));
  // INT8 engine, fused path: the matching kernel also emits S's and H's left
  // operands (exponents, A and UB residue planes)
  static const bool no_res = std::getenv("HSB_NO_MATCH_RES") != nullptr;  // A/B experiments
  if (ctx->engine == HSB_ENGINE_INT8 && !(opts & HSB_OPT_UNFUSED) && !no_res) {
    int n_mod = 0, bits = 0;
    CKS(oz_choose(ctx, 2 * K, &n_mod, &bits));
    const int64_t kpad = hsb::oz_kpad(K);
    const size_t pbytes = static_cast<size_t>(hsb::kOzPlanes) * n_mod * ng * kpad;
    void *eb, *rb, *ubb;
    CKS(ws(ctx, "oz_exp_l", static_cast<size_t>(ng) * 4, &eb));
    CKS(ws(ctx, "oz_res_a", pbytes, &rb));
    CKS(ws(ctx, "oz_res2", pbytes, &ubb));
    MatchRes r;
    r.u = static_cast<const double*>(p->u_dev);
    r.col_exp = static_cast<int32_t*>(eb);
    r.res_a = static_cast<int8_t*>(rb);
    r.res_ub = static_cast<int8_t*>(ubb);
    r.kpad = kpad;
    r.b = bits;
    r.n_mod = n_mod;
    CK(launch_match_coeffs_res(mp, A, B, r, st));
    ctx->oz_prepared = {A, K, ng, n_mod, bits};
  } else {
    CK(launch_match_coeffs(mp, A, B, st));
  }
  const hsb_status s = build_hs_core(ctx, stream, p, opts, out, tm, atom_info);
  ctx->oz_prepared = {};
  return s;
}

}  // extern "C"
