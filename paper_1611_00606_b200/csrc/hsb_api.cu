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
#include <atomic>
#include <thread>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/hsb200.h"
#include "aux_kernels.cuh"
#include "match.cuh"
#include "ozaki.cuh"
#include "staging.cuh"
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
  hsb::Stager stager;                 // pinned-slot host<->device transfers
  int* done_cnt = nullptr;            // mapped pinned per-column-block tile counters
  size_t done_cnt_len = 0;
  cudaStream_t copy_stream = nullptr;  // overlaps S download with the H contraction
  int64_t tile_list_T = 0;             // tile rows of the cached grouped triangle order
  std::vector<int2> tile_list_host;    // its host copy (source of an async upload)
  int32_t engine = HSB_ENGINE_DMMA;    // triangle contractions: FP64 DMMA or INT8 CRT emulation
  int32_t oz_min_bits = 39;            // INT8 engine: operand integer bits (accuracy ~2^-bits)
  int64_t oz_tiles_n = 0;              // cached INT8-engine tile list (n of the output)
  std::vector<int2> oz_tiles_host;
  std::vector<int32_t> oz_tile_index_host;
  int32_t cplx = HSB_CPLX_3M;          // complex product form of the zrk kernels
};

static thread_local std::string g_create_err;

// Host wall-clock phase stamps for diagnosing the host-buffer path.
struct HostClock {
  using clk = std::chrono::steady_clock;
  bool on = std::getenv("HSB_DEBUG_TIMING") != nullptr;
  clk::time_point t0 = clk::now(), last = t0;
  std::string log;
  void mark(const char* what) {
    if (!on) return;
    auto now = clk::now();
    log += std::string(what) + " " + std::to_string(std::chrono::duration<double, std::milli>(now - last).count()) + " ms; ";
    last = now;
  }
  void report() {
    if (on) std::fprintf(stderr, "[hsb timing] %s\n", log.c_str());
  }
};

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

// 2-D TMA map over one real sum plane (k x cols, leading dimension ldp doubles),
// box {8 complex k, 64 cols}, no swizzle (zrk3m_kernel.cu, PLANES).
hsb_status encode_plane(hsb_ctx* ctx, CUtensorMap* map, const double* base, int64_t k, int64_t cols, int64_t ldp) {
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(cols)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldp) * 8};
  cuuint32_t box[2] = {8, static_cast<cuuint32_t>(kBM)}, estr[2] = {1, 1};
  CUresult r = ctx->encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(ctx, HSB_ERR_CUDA, "cuTensorMapEncodeTiled failed for a sum plane (code " +
                                       std::to_string(static_cast<int>(r)) + ")");
  return HSB_OK;
}

struct Seg {
  OperandView l, r;
};

// Section timeline on the compute stream: each mark closes the interval since
// the previous mark and charges it to a section tag.
struct Timeline {
  std::vector<std::pair<std::string, cudaEvent_t>> marks;
  ~Timeline() {
    for (auto& m : marks) cudaEventDestroy(m.second);
  }
  cudaError_t mark(cudaStream_t st, const char* tag) {
    cudaEvent_t e;
    cudaError_t err = cudaEventCreate(&e);
    if (err != cudaSuccess) return err;
    marks.push_back({tag, e});
    return cudaEventRecord(e, st);
  }
  double total(const char* tag) const {
    double s = 0;
    for (size_t i = 1; i < marks.size(); ++i)
      if (marks[i].first == tag) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, marks[i - 1].second, marks[i].second);
        s += ms * 1e-3;
      }
    return s;
  }
  double span() const {
    float ms = 0.f;
    if (marks.size() > 1) cudaEventElapsedTime(&ms, marks.front().second, marks.back().second);
    return ms * 1e-3;
  }
};

cudaError_t timeline_mark(Timeline* tl, cudaStream_t st, const char* tag) { return tl->mark(st, tag); }

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
  int* done_cnt = nullptr;
  // optional: mark the contraction kernel alone on this timeline, charging the
  // work before it to `sect` and the kernel itself to `core`
  Timeline* tl = nullptr;
  const char* sect = nullptr;
  const char* core = nullptr;
  // optional (INT8 engine): run in column groups and record, after each, an
  // event and the end column of the columns that are final
  std::vector<std::pair<cudaEvent_t, int64_t>>* chunk_events = nullptr;
  // optional (INT8 engine): scatter the result into peer receive slots
  const hsb_peer_out* peer = nullptr;
  bool peer_is_h = false;
};

// Lower-triangle tile order for the persistent 3M kernel.  The 148 CTAs run
// consecutive list entries concurrently and advance through k in near
// lockstep, so the operand panels they share stay in L2.  Column-major tile
// order puts ~148 distinct row panels in flight at once (each streamed from
// HBM: 117 GB per C3 H launch); kTileGroup x kTileGroup blocks of tiles
// (column groups left to right, row groups top to bottom, i >= j) put 2 x 12.
// Column groups still complete left to right, which the H download stream
// relies on (done_cnt prefix).
constexpr int kTileGroup = 12;
hsb_status tile_order(hsb_ctx* ctx, int64_t T, cudaStream_t st, const int2** out) {
  void* buf;
  CKS(ws(ctx, "tile_list", static_cast<size_t>(T * (T + 1) / 2) * sizeof(int2), &buf));
  if (ctx->tile_list_T != T) {
    std::vector<int2>& v = ctx->tile_list_host;
    v.clear();
    v.reserve(static_cast<size_t>(T * (T + 1) / 2));
    for (int64_t j0 = 0; j0 < T; j0 += kTileGroup)
      for (int64_t i0 = j0; i0 < T; i0 += kTileGroup)
        for (int64_t j = j0; j < std::min<int64_t>(j0 + kTileGroup, T); ++j)
          for (int64_t i = std::max(i0, j); i < std::min<int64_t>(i0 + kTileGroup, T); ++i)
            v.push_back(make_int2(static_cast<int>(i), static_cast<int>(j)));
    CK(cudaMemcpyAsync(buf, v.data(), v.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
    ctx->tile_list_T = T;
  }
  *out = static_cast<const int2*>(buf);
  return HSB_OK;
}

// ---------------------------------------------------------------- INT8 engine
// Lower-triangle C = alpha sum_s op(L_s)^T R_s + beta C on the INT8 tensor
// cores (ozaki.cuh): column exponents, residue planes of every distinct
// operand, one persistent tcgen05 GEMM launch over (product, modulus, tile),
// CRT reconstruction + mirror.
hsb_status oz_encode(hsb_ctx* ctx, CUtensorMap* map, const int8_t* planes, int64_t k, int64_t cols, int64_t kpad,
                     int n_mod, int box_rows) {
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(n_mod)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(kpad), static_cast<cuuint64_t>(kpad * cols)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(kOzBK), static_cast<cuuint32_t>(box_rows), 1}, es[3] = {1, 1, 1};
  CUresult r = ctx->encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(planes), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(ctx, HSB_ERR_CUDA, "cuTensorMapEncodeTiled failed for residue planes (code " +
                                       std::to_string(static_cast<int>(r)) + ")");
  return HSB_OK;
}

// 256 x 256 tiles (tile row tm >= tile col tn) of the lower triangle, in
// groups of 6 x 6 tiles for L2 reuse
hsb_status oz_tiles(hsb_ctx* ctx, int64_t n, cudaStream_t st, const int2** out, int* count,
                    const int32_t** index) {
  const int64_t T = (n + kOzBN - 1) / kOzBN;
  std::vector<int2>& v = ctx->oz_tiles_host;
  std::vector<int32_t>& ix = ctx->oz_tile_index_host;
  if (ctx->oz_tiles_n != n) {
    v.clear();
    for (int64_t j0 = 0; j0 < T; j0 += 6)
      for (int64_t i0 = j0; i0 < T; i0 += 6)
        for (int64_t j = j0; j < std::min<int64_t>(j0 + 6, T); ++j)
          for (int64_t i = std::max(i0, j); i < std::min<int64_t>(i0 + 6, T); ++i)
            v.push_back(make_int2(static_cast<int>(i), static_cast<int>(j)));
    ix.assign(static_cast<size_t>(T * T), -1);
    for (size_t t = 0; t < v.size(); ++t) ix[static_cast<size_t>(v[t].x * T + v[t].y)] = static_cast<int32_t>(t);
  }
  void *buf, *ibuf;
  CKS(ws(ctx, "oz_tiles", v.size() * sizeof(int2), &buf));
  CKS(ws(ctx, "oz_tile_index", ix.size() * sizeof(int32_t), &ibuf));
  if (ctx->oz_tiles_n != n) {
    CK(cudaMemcpyAsync(buf, v.data(), v.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ibuf, ix.data(), ix.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    ctx->oz_tiles_n = n;
  }
  *out = static_cast<const int2*>(buf);
  *count = static_cast<int>(v.size());
  *index = static_cast<const int32_t*>(ibuf);
  return HSB_OK;
}

hsb_status run_ozaki(hsb_ctx* ctx, cudaStream_t st, const ZrkCall& z, int* launches) {
  const int64_t n = z.m;
  std::vector<Seg> segs;
  int64_t ktot = 0;
  for (const Seg& s : z.segs)
    if (s.l.k > 0) {
      if (s.l.k != s.r.k) return fail(ctx, HSB_ERR_DIMENSION, "segment operands disagree in reduction length");
      segs.push_back(s);
      ktot += s.l.k;
    }
  if (segs.size() > static_cast<size_t>(kOzMaxSeg)) return fail(ctx, HSB_ERR_UNSUPPORTED, "too many segments");
  // moduli: the fewest with b >= oz_min_bits.  With |x'| + |y'| <= 2^b per
  // element, |Re'| = |sum x'x' + y'y'| and |Im'| = |sum x'_L y'_R - y'_L x'_R|
  // are both <= K 2^2b; the explicit CRT needs |X| < M/2, kept with one bit of
  // margin: 2b <= log2 M - 2 - log2 K.
  int n_mod = 0, b = 0;
  {
    double log2m = 0;
    for (int i = 0; i < kOzMaxMod; ++i) {
      log2m += std::log2(static_cast<double>(oz_mod(i)));
      const int bi = static_cast<int>(std::floor((log2m - 2.0 - std::log2(static_cast<double>(std::max<int64_t>(ktot, 1)))) / 2.0));
      if (i + 1 >= 11 && (bi >= ctx->oz_min_bits || i + 1 == kOzMaxMod)) {
        n_mod = i + 1;
        b = std::min(bi, ctx->oz_min_bits + 4);
        break;
      }
    }
  }
  if (b < 30) return fail(ctx, HSB_ERR_UNSUPPORTED, "reduction too long for the INT8 engine's moduli");
  // exponents: one array for both sides (m == n), max over every operand
  void* ebuf;
  CKS(ws(ctx, "oz_exp", static_cast<size_t>(n) * sizeof(int32_t), &ebuf));
  int32_t* e = static_cast<int32_t*>(ebuf);
  CK(launch_ozaki_init_exp(e, n, st));
  {
    std::vector<const OperandView*> seen;
    auto colexp = [&](const OperandView& v) -> hsb_status {
      for (const OperandView* q : seen)
        if (q->base == v.base && q->k == v.k && q->ld == v.ld) return HSB_OK;
      seen.push_back(&v);
      CK(launch_ozaki_colexp(v.base, v.ld, v.k, v.cols, e, st));
      return HSB_OK;
    };
    for (const Seg& s : segs) {
      CKS(colexp(s.l));
      CKS(colexp(s.r));
    }
  }
  // residue planes of each distinct operand
  struct Src {
    const double* base;
    int64_t k, ld;
    int8_t* planes;
    int64_t kpad;
  };
  std::vector<Src> srcs;
  auto planes_of = [&](const OperandView& v, Src* out) -> hsb_status {
    for (const Src& q : srcs)
      if (q.base == v.base && q.k == v.k && q.ld == v.ld) {
        *out = q;
        return HSB_OK;
      }
    Src q{v.base, v.k, v.ld, nullptr, (v.k + 15) / 16 * 16};
    const std::string name = "oz_res" + std::to_string(srcs.size());
    void* buf;
    CKS(ws(ctx, name.c_str(), static_cast<size_t>(4) * n_mod * n * q.kpad, &buf));
    q.planes = static_cast<int8_t*>(buf);
    CK(launch_ozaki_residues(v.base, v.ld, v.k, n, e, b, n_mod, q.planes, q.kpad, st));
    srcs.push_back(q);
    *out = q;
    return HSB_OK;
  };
  OzGemmParams gp;
  std::memset(&gp, 0, sizeof(gp));
  // products: P = re.re, Q = im.im, W = (re -/+ im)(re + im)
  const int lp[3] = {kOzRe, kOzIm, z.conj ? kOzMinus : kOzPlus};
  const int rp[3] = {kOzRe, kOzIm, kOzPlus};
  for (size_t si = 0; si < segs.size(); ++si) {
    Src L, R;
    CKS(planes_of(segs[si].l, &L));
    CKS(planes_of(segs[si].r, &R));
    const int64_t pl = static_cast<int64_t>(n_mod) * n * L.kpad, pr = static_cast<int64_t>(n_mod) * n * R.kpad;
    for (int pi = 0; pi < 3; ++pi) {
      CKS(oz_encode(ctx, &gp.map[pi][si][0], L.planes + lp[pi] * pl, L.k, n, L.kpad, n_mod, 128));
      CKS(oz_encode(ctx, &gp.map[pi][si][1], R.planes + rp[pi] * pr, R.k, n, R.kpad, n_mod, 128));
    }
    gp.seg_chunk0[si + 1] = gp.seg_chunk0[si] + static_cast<int32_t>((segs[si].l.k + kOzBK - 1) / kOzBK);
  }
  gp.nseg = static_cast<int32_t>(segs.size());
  // slabs of ~16 KB of k (see ozaki.cuh), balanced
  const int32_t total_chunks = gp.seg_chunk0[gp.nseg];
  constexpr int32_t kSlabChunks = 16384 / kOzBK;
  gp.nslab = std::max(1, std::min<int32_t>(kOzMaxSlab, (total_chunks + kSlabChunks - 1) / kSlabChunks));
  for (int sl = 0; sl <= gp.nslab; ++sl)
    gp.slab_chunk0[sl] = static_cast<int32_t>(static_cast<int64_t>(total_chunks) * sl / gp.nslab);
  gp.n_mod = n_mod;
  gp.n = static_cast<int32_t>(n);
  const int32_t* tile_index = nullptr;
  int total_tiles = 0;
  CKS(oz_tiles(ctx, n, st, &gp.tile_list, &total_tiles, &tile_index));
  gp.mod_stride = static_cast<int64_t>(total_tiles) * kOzTileBytes;
  gp.slab_stride = gp.mod_stride * n_mod;
  gp.prod_stride = gp.slab_stride * gp.nslab;
  void* rbuf;
  CKS(ws(ctx, "oz_out", static_cast<size_t>(3 * gp.prod_stride), &rbuf));
  gp.res = static_cast<int8_t*>(rbuf);
  void* cbuf;
  CKS(ws(ctx, "oz_counter", 16, &cbuf));
  gp.counter = static_cast<int32_t*>(cbuf);
  if (gp.nseg == 0) CK(cudaMemsetAsync(rbuf, 0, static_cast<size_t>(3 * gp.prod_stride), st));

  OzCrtParams cp;
  cp.res = gp.res;
  cp.mod_stride = gp.mod_stride;
  cp.slab_stride = gp.slab_stride;
  cp.prod_stride = gp.prod_stride;
  cp.tile_index = tile_index;
  cp.T = static_cast<int32_t>((n + kOzBN - 1) / kOzBN);
  cp.nslab = gp.nslab;
  cp.n_mod = n_mod;
  cp.n = static_cast<int32_t>(n);
  cp.b = b;
  cp.conj = z.conj ? 1 : 0;
  cp.el = e;
  cp.er = e;
  cp.alpha_re = z.alpha_re;
  cp.alpha_im = z.alpha_im;
  cp.beta_re = z.beta_re;
  cp.beta_im = z.beta_im;
  cp.c = z.c;
  cp.ldc = z.ldc;
  cp.flags = z.flags;
  cp.peer = nullptr;
  cp.P = cp.rank = 0;
  cp.cpr = cp.pld = 0;
  if (z.peer) {
    cp.peer = reinterpret_cast<double2* const*>(z.peer_is_h ? z.peer->h_slots : z.peer->s_slots);
    cp.P = z.peer->n_ranks;
    cp.rank = z.peer->rank;
    cp.cpr = z.peer->cols_per_rank;
    cp.pld = z.peer->ld;
  }

  // With a host download waiting on per-column counters (done_cnt), the
  // product runs in column groups of 6 tiles (contiguous in the tile list):
  // once groups 0..g are done their columns are final (the mirror of an
  // entry of an earlier group lands in a later column), so their download
  // overlaps the remaining groups.  Otherwise one GEMM + one CRT launch.
  const int64_t T = (n + kOzBN - 1) / kOzBN;
  const int64_t T64 = (n + kBN - 1) / kBN;  // the host's 64-column blocks
  const std::vector<int2>& tl_host = ctx->oz_tiles_host;
  const int64_t group = (z.done_cnt || z.chunk_events) ? 6 : T;
  int t0 = 0;
  for (int64_t j0 = 0; j0 < T; j0 += group) {
    const int64_t j1 = std::min<int64_t>(j0 + group, T);
    int t1 = t0;
    while (t1 < total_tiles && tl_host[static_cast<size_t>(t1)].y < j1) ++t1;
    if (gp.nseg > 0 && t1 > t0) {
      gp.tile0 = t0;
      gp.ntiles = t1 - t0;
      if (z.tl) CK(timeline_mark(z.tl, st, z.sect));
      CK(launch_ozaki_gemm(gp, st));
      if (z.tl) CK(timeline_mark(z.tl, st, z.core));
    }
    const int64_t c0 = j0 * kOzBN, c1 = std::min<int64_t>(j1 * kOzBN, n);
    cp.n0 = static_cast<int32_t>(c0);
    CK(launch_ozaki_crt_cols(cp, c1 - c0, st));
    if (z.done_cnt) {
      const int64_t b0 = c0 / kBN, b1 = (j1 == T) ? T64 : c1 / kBN;
      CK(launch_fill_i32(z.done_cnt + b0, b1 - b0, static_cast<int32_t>(T64), st));
    }
    if (z.chunk_events) {
      cudaEvent_t ev;
      CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      z.chunk_events->push_back({ev, c1});
      CK(cudaEventRecord(ev, st));
    }
    t0 = t1;
  }
  if (launches) *launches += 3 + 2 * static_cast<int>(segs.size()) + static_cast<int>(srcs.size());
  return HSB_OK;
}

hsb_status run_zrk(hsb_ctx* ctx, cudaStream_t st, const ZrkCall& z, int* launches) {
  if (z.peer && !(ctx->engine == HSB_ENGINE_INT8 && z.triangle && z.batch == 1 && z.m == z.n))
    return fail(ctx, HSB_ERR_UNSUPPORTED, "peer output needs the INT8 engine on a triangle call");
  if (ctx->engine == HSB_ENGINE_INT8 && z.triangle && z.batch == 1 && z.m == z.n && z.m > 0) {
    bool plain = true;
    for (const Seg& s : z.segs) plain = plain && s.l.batch == 1 && s.r.batch == 1;
    if (plain) return run_ozaki(ctx, st, z, launches);
  }
  if (z.m <= 0 || z.n <= 0 || z.batch <= 0) return HSB_OK;
  if (z.segs.size() > static_cast<size_t>(kMaxSeg)) return fail(ctx, HSB_ERR_UNSUPPORTED, "too many segments");
  if (z.triangle && z.m != z.n) return fail(ctx, HSB_ERR_DIMENSION, "triangle mode needs a square output");
  if (z.m > (int64_t{1} << 30) || z.n > (int64_t{1} << 30))
    return fail(ctx, HSB_ERR_UNSUPPORTED, "output dimension too large");
  ZrkParams p;
  std::memset(&p, 0, sizeof(p));
  // 3M on plain (unbatched) operands: Re-Im / Re+Im planes of each distinct
  // operand, computed once here and fed to the kernel by TMA
  const bool g3 = ctx->cplx == HSB_CPLX_3M;
  bool planes = g3 && z.batch == 1;
  for (const Seg& s : z.segs)
    if (s.l.batch != 1 || s.r.batch != 1) planes = false;
  struct PlaneSrc {
    const double* base;
    int64_t k, cols, ld, ldp;
    double* minus;
    double* plus;
  };
  std::vector<PlaneSrc> srcs;
  auto plane_of = [&](const OperandView& v, bool minus, const double** out, int64_t* ldp) -> hsb_status {
    for (const PlaneSrc& q : srcs)
      if (q.base == v.base && q.k == v.k && q.cols == v.cols && q.ld == v.ld) {
        *out = minus ? q.minus : q.plus;
        *ldp = q.ldp;
        return HSB_OK;
      }
    PlaneSrc q{v.base, v.k, v.cols, v.ld, v.k + (v.k & 1), nullptr, nullptr};
    const std::string name = "zplane" + std::to_string(srcs.size());
    void* buf;
    CKS(ws(ctx, name.c_str(), static_cast<size_t>(2 * q.ldp) * q.cols * 8, &buf));
    q.minus = static_cast<double*>(buf);
    q.plus = q.minus + q.ldp * q.cols;
    CK(launch_sum_planes(q.base, q.ld, q.k, q.cols, q.minus, q.plus, q.ldp, st));
    srcs.push_back(q);
    *out = minus ? q.minus : q.plus;
    *ldp = q.ldp;
    return HSB_OK;
  };
  int nseg = 0, total = 0;
  for (const Seg& s : z.segs) {
    if (s.l.k <= 0) continue;
    if (s.l.k != s.r.k) return fail(ctx, HSB_ERR_DIMENSION, "segment operands disagree in reduction length");
    CKS(encode_operand(ctx, &p.lmap[nseg], s.l));
    CKS(encode_operand(ctx, &p.rmap[nseg], s.r));
    if (planes) {
      const double *lp, *rp;
      int64_t ldl, ldr;
      // left factor: Re-Im for L^H R (conj), Re+Im for L^T R
      CKS(plane_of(s.l, z.conj, &lp, &ldl));
      CKS(plane_of(s.r, false, &rp, &ldr));
      CKS(encode_plane(ctx, &p.lsum[nseg], lp, s.l.k, s.l.cols, ldl));
      CKS(encode_plane(ctx, &p.rsum[nseg], rp, s.r.k, s.r.cols, ldr));
    }
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
  p.done_cnt = z.triangle ? z.done_cnt : nullptr;
  int64_t grid_x = z.triangle ? static_cast<int64_t>(p.tiles_m) * (p.tiles_m + 1) / 2
                              : static_cast<int64_t>(p.tiles_m) * p.tiles_n;
  if (grid_x > 0x7fffffff || z.batch > 65535) return fail(ctx, HSB_ERR_UNSUPPORTED, "grid too large");
  if (g3 && z.triangle && z.batch == 1 && p.tiles_m > kTileGroup) CKS(tile_order(ctx, p.tiles_m, st, &p.tile_list));
  if (z.tl) CK(timeline_mark(z.tl, st, z.sect));
  if (g3) {
    if (grid_x * z.batch > 0x7fffffff) return fail(ctx, HSB_ERR_UNSUPPORTED, "grid too large");
    CK(launch_zrk3m(p, z.conj, planes, static_cast<int>(grid_x), static_cast<int>(z.batch), st));
    if (launches) *launches += static_cast<int>(srcs.size());
  } else {
    CK(launch_zrk(p, z.conj, static_cast<int>(grid_x), static_cast<int>(z.batch), st));
  }
  if (z.tl) CK(timeline_mark(z.tl, st, z.core));
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

int32_t hsb_abi_version(void) { return 4; }

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
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->done_cnt) cudaFreeHost(ctx->done_cnt);
  delete ctx;
}

const char* hsb_last_error(const hsb_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

hsb_status hsb_ctx_set_complex_mult(hsb_ctx* ctx, int32_t algo) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
  if (algo != HSB_CPLX_4M && algo != HSB_CPLX_3M) return fail(ctx, HSB_ERR_INPUT, "unknown complex product form");
  ctx->cplx = algo;
  return HSB_OK;
}

hsb_status hsb_ctx_set_engine(hsb_ctx* ctx, int32_t engine, int32_t min_bits) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
  if (engine != HSB_ENGINE_DMMA && engine != HSB_ENGINE_INT8) return fail(ctx, HSB_ERR_INPUT, "unknown engine");
  if (min_bits != 0 && (min_bits < 30 || min_bits > 48))
    return fail(ctx, HSB_ERR_INPUT, "min_bits must be 0 (default 40) or in [30, 48]");
  ctx->engine = engine;
  ctx->oz_min_bits = min_bits ? min_bits : 39;
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

hsb_status hsb_build_hs(hsb_ctx* ctx, void* stream, const hsb_problem* p, uint32_t opts, const hsb_output* out,
                        hsb_timings* tm, int32_t* atom_info) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
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
  Timeline tl;
  HostClock hc;  // host-side phase stamps, printed when HSB_DEBUG_TIMING is set
  CK(tl.mark(st, "start"));

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
  void *q, *info_d, *pbb, *zbuf, *ub, *rbuf, *offs_d, *potrf_scr = nullptr, *hostbuf;
  CKS(ws(ctx, "q", tblk_bytes * na, &q));
  CKS(ws(ctx, "info", static_cast<size_t>(na) * 4, &info_d));
  CKS(ws(ctx, "pbb", tblk_bytes * na, &pbb));
  CKS(ws(ctx, "z", stack_bytes, &zbuf));
  CKS(ws(ctx, "ub", stack_bytes, &ub));
  CKS(ws(ctx, "r", stack_bytes, &rbuf));
  CKS(ws(ctx, "offs", static_cast<size_t>(na) * 3 * 4, &offs_d));
  if (static_cast<size_t>(nl) * (nl + 1) / 2 * 16 > kPotrfSmemMax)
    CKS(ws(ctx, "potrf_scr", static_cast<size_t>(na) * nl * (nl + 1) / 2 * 16, &potrf_scr));
  CKS(pinned(ctx, (static_cast<size_t>(na) * 4 + 2) * 4, &hostbuf));
  int32_t* info_h = static_cast<int32_t*>(hostbuf);
  int32_t* offs_h = info_h + na;  // 3 * na entries: R row offset, A_nh source rows, A_nh dest rows
  double* Z = static_cast<double*>(zbuf);
  double* UB = static_cast<double*>(ub);
  double* R = static_cast<double*>(rbuf);  // [Y_hpd ; X_nh]
  int32_t* flag_h = offs_h + 3 * na;  // first non-finite atom of A / B (pinned uploads)
  flag_h[0] = flag_h[1] = -1;

  auto stage_stack = [&](int m, cudaStream_t s) -> hsb_status {
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
      CKS(ws(ctx, m == 0 ? "raw_a" : "raw_b", stack_bytes, &raw));
      const size_t blk = static_cast<size_t>(nl) * ng * 16;
      for (int64_t i = 0; i < na; ++i)
        CK(cudaMemcpyAsync(static_cast<char*>(raw) + i * blk, blocks[i], blk, cudaMemcpyHostToDevice, s));
      CK(launch_stack_blocks(static_cast<double*>(raw), dst, static_cast<int>(na), static_cast<int>(nl), ng, s));
      ++launches;
      void* flag;
      CKS(ws(ctx, m == 0 ? "bad_a" : "bad_b", 8, &flag));
      CK(launch_first_nonfinite(static_cast<double*>(raw), static_cast<int>(na), static_cast<int64_t>(nl) * ng * 2,
                                static_cast<int*>(flag), s));
      ++launches;
      CK(cudaMemcpyAsync(flag_h + m, flag, 4, cudaMemcpyDeviceToHost, s));  // checked after the final sync
      hc.mark(m == 0 ? "h2d A pinned" : "h2d B pinned");
      return HSB_OK;
    }
    CK(ctx->stager.h2d_stack(dst, blocks, na, nl, ng, s, &bad));
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
    hc.mark("h2d T,u");
    CKS(stage_stack(1, st));
    CK(cudaEventRecord(ev_b_up, st));
    if (!overlap_upload) CKS(stage_stack(0, st));
    CK(tl.mark(st, "h2d"));
  }

  // ------------------------------------------- Loop 2, part 1: Cholesky routing
  CK(launch_potrf_route(TAA, static_cast<double*>(q), static_cast<int32_t*>(info_d), static_cast<int>(na),
                        static_cast<int>(nl), force_nonhpd, static_cast<double*>(potrf_scr), st));
  ++launches;
  CK(cudaMemcpyAsync(info_h, info_d, na * 4, cudaMemcpyDeviceToHost, st));
  cudaEvent_t ev_info;
  CK(cudaEventCreateWithFlags(&ev_info, cudaEventDisableTiming));
  struct EvDel {
    cudaEvent_t e;
    ~EvDel() { cudaEventDestroy(e); }
  } ev_info_del{ev_info};
  CK(cudaEventRecord(ev_info, st));
  CK(tl.mark(st, "loop2"));

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
  auto unorm = [&]() -> hsb_status {  // UB = diag(u) B (builder.py:124-127)
    CK(launch_diag_scale(B, K, UB, K, U, K, ng, st));
    ++launches;
    CK(tl.mark(st, "unorm"));
    return HSB_OK;
  };

  // ------------------------------------------------------ Loop 1, U norm, S
  if (overlap_upload) {
    CKS(unorm());
    ZrkCall s2 = tri_call(S, ldo, ng, kLowerOnly, 0.0);
    s2.segs.push_back({plain(UB, K, ng, K), plain(UB, K, ng, K)});
    s2.tl = &tl, s2.sect = "s2", s2.core = "s2_core";
    CKS(run_zrk(ctx, st, s2, &launches));
    CK(tl.mark(st, "s2"));
    // A rides the copy engine while (UB)^H(UB) runs -- after B's DMAs, so the
    // two uploads do not split the PCIe bandwidth B is waited on
    CK(cudaStreamWaitEvent(cs, ev_b_up, 0));
    CKS(stage_stack(0, cs));
    cudaEvent_t ev_a;
    CK(cudaEventCreateWithFlags(&ev_a, cudaEventDisableTiming));
    EvDel ev_a_del{ev_a};
    CK(cudaEventRecord(ev_a, cs));
    CK(cudaStreamWaitEvent(st, ev_a, 0));
    CK(tl.mark(st, "h2d"));
    ZrkCall s1 = tri_call(S, ldo, ng, kLowerOnly | kMirror, 1.0);
    s1.segs.push_back({plain(A, K, ng, K), plain(A, K, ng, K)});
    s1.tl = &tl, s1.sect = "s1", s1.core = "s1_core";
    if (chunk_s) s1.chunk_events = &s_chunks;
    CKS(run_zrk(ctx, st, s1, &launches));
    CK(tl.mark(st, "s1"));
    CKS(loop1());
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
    CK(launch_mirror(S, ldo, static_cast<int>(ng), st));
    ++launches;
    CK(tl.mark(st, "s2"));
  } else {
    CKS(loop1());
    CKS(unorm());
    ZrkCall s = tri_call(S, ldo, ng, kLowerOnly | kMirror, 0.0);
    s.segs.push_back({plain(A, K, ng, K), plain(A, K, ng, K)});
    s.segs.push_back({plain(UB, K, ng, K), plain(UB, K, ng, K)});
    s.tl = &tl, s.sect = "s", s.core = "s_core";
    if (chunk_s) s.chunk_events = &s_chunks;
    s.peer = peer;
    CKS(run_zrk(ctx, st, s, &launches));
    CK(tl.mark(st, "s"));
  }
  cudaEvent_t ev_s;  // S final
  CK(cudaEventCreateWithFlags(&ev_s, cudaEventDisableTiming));
  EvDel ev_s_del{ev_s};
  CK(cudaEventRecord(ev_s, st));
  if (out->s_ready) CK(cudaEventRecord(static_cast<cudaEvent_t>(out->s_ready), st));

  // ------------------------------------------- routing (host, overlaps S)
  hc.mark("enqueue to S");
  CK(cudaEventSynchronize(ev_info));
  hc.mark("routing wait");
  int64_t n_hpd = 0, n_nh = 0;
  for (int64_t i = 0; i < na; ++i) (info_h[i] == 0 ? n_hpd : n_nh)++;
  {
    int64_t ih = 0, in = 0;
    for (int64_t i = 0; i < na; ++i) {
      if (info_h[i] == 0) {
        offs_h[i] = static_cast<int32_t>(ih++ * nl);
      } else {
        offs_h[i] = static_cast<int32_t>((n_hpd + in) * nl);
        offs_h[na + in] = static_cast<int32_t>(i * nl);      // A_nh source rows
        offs_h[2 * na + in] = static_cast<int32_t>(in * nl);  // A_nh dest rows
        ++in;
      }
    }
  }
  if (atom_info) std::memcpy(atom_info, info_h, na * 4);
  CK(cudaMemcpyAsync(offs_d, offs_h, na * 3 * 4, cudaMemcpyHostToDevice, st));
  const int32_t* offs_dev = static_cast<int32_t*>(offs_d);

  // ------------------------------------------- Loop 2, part 2 (builder.py:162-185)
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
  CK(tl.mark(st, "loop2"));
  const int64_t k_hpd = n_hpd * nl, k_nh = n_nh * nl;
  const double* Y = R;
  const double* XNH = R + 2 * k_hpd;
  // Stream H to pinned host memory while the H contraction runs (fused path)
  const int64_t ntiles = (ng + kBN - 1) / kBN;
  const bool stream_h = !unfused && out->location == HSB_LOC_HOST && host_is_pinned(out->h);

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
    CK(launch_mirror(H, ldo, static_cast<int>(ng), st));
    ++launches;
    CK(tl.mark(st, "h3"));
  } else {
    ZrkCall h = tri_call(H, ldo, ng, kLowerOnly | kMirror, 0.0);
    h.segs.push_back({plain(Z, K, ng, K), plain(B, K, ng, K)});
    h.segs.push_back({plain(B, K, ng, K), plain(Z, K, ng, K)});
    if (n_hpd > 0) h.segs.push_back({plain(Y, k_hpd, ng, K), plain(Y, k_hpd, ng, K)});
    if (n_nh > 0) h.segs.push_back({plain(ANH, k_nh, ng, k_nh), plain(XNH, k_nh, ng, K)});
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
    CKS(run_zrk(ctx, st, h, &launches));
    CK(tl.mark(st, "h"));
  }

  // --------------------------------------------------------------- outputs
  if (out->location == HSB_LOC_HOST) {
    // S is final at ev_s: its download runs on the copy stream, concurrently
    // with the H contraction; H follows on the compute stream.
    const size_t row = static_cast<size_t>(ng) * 16;
    if (!s_chunks.empty()) {
      // column groups of S download as soon as each is final
      int64_t c0 = 0;
      for (const auto& c : s_chunks) {
        CK(cudaStreamWaitEvent(cs, c.first, 0));
        if (c.second > c0)
          CK(cudaMemcpy2DAsync(reinterpret_cast<char*>(out->s) + c0 * out->ld * 16, out->ld * 16,
                               reinterpret_cast<const char*>(S) + c0 * ldo * 16, ldo * 16, row, c.second - c0,
                               cudaMemcpyDeviceToHost, cs));
        c0 = c.second;
      }
    } else {
      CK(cudaStreamWaitEvent(cs, ev_s, 0));
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
          CK(cudaMemcpy2DAsync(reinterpret_cast<char*>(out->h) + c0 * out->ld * 16, out->ld * 16,
                               reinterpret_cast<const char*>(H) + c0 * ldo * 16, ldo * 16, row, c1 - c0,
                               cudaMemcpyDeviceToHost, cs));
          sent = c;
        } else {
          std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
      }
      hc.mark("stream H");
    } else {
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
  hc.mark("final sync");
  hc.report();
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
    const double fH1 = 8.0 * K * double(ng) * ng, fH2 = 8.0 * k_nh * double(ng) * ng,
                 fH3 = 4.0 * k_hpd * double(ng) * ng;
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
  }
  return HSB_OK;
}

hsb_status hsb_match_coeffs(hsb_ctx* ctx, void* stream, const hsb_phys* ph, double* a_stack, double* b_stack,
                            int64_t ld) {
  if (!ctx) return fail(nullptr, HSB_ERR_INPUT, "ctx is NULL");
  if (!ph || !a_stack || !b_stack) return fail(ctx, HSB_ERR_INPUT, "NULL argument");
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
  cudaSetDevice(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t gb = ph->n_g * 3 * 4, tb = ph->n_atoms * 3 * 8, yb = ph->n_atoms * 4, rb = ph->n_types * 8,
               db = ph->n_types * (ph->lmax + 1) * 4 * 8;
  void *g, *t, *y, *r, *d;
  CKS(ws(ctx, "m_gvec", gb, &g));
  CKS(ws(ctx, "m_tau", tb, &t));
  CKS(ws(ctx, "m_type", yb, &y));
  CKS(ws(ctx, "m_rmt", rb, &r));
  CKS(ws(ctx, "m_radial", db, &d));
  CK(cudaMemcpyAsync(g, ph->gvec, gb, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(t, ph->tau, tb, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(y, ph->type_of, yb, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(r, ph->rmt, rb, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d, ph->radial, db, cudaMemcpyHostToDevice, st));
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
  CK(launch_match_coeffs(mp, a_stack, b_stack, st));
  // the small uploads above come from caller memory: finish them before returning
  CK(cudaStreamSynchronize(st));
  return HSB_OK;
}

}  // extern "C"
