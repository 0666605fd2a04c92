// host_ctx.cuh — internal to libhsb200 (not part of the ABI): the context,
// workspace and error helpers, the section timeline, and the contraction
// dispatcher's call description shared by hsb_api.cu and contract.cu.
#pragma once
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
#include <mutex>
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
  void* m_stage = nullptr;  // pinned staging of the matching kernel's small inputs
  size_t m_stage_bytes = 0;
  cudaEvent_t m_stage_done = nullptr;  // its last uploads consumed (reuse after this)
  hsb::Stager stager;                 // pinned-slot host<->device transfers
  int* done_cnt = nullptr;            // mapped pinned per-column-block tile counters
  size_t done_cnt_len = 0;
  cudaStream_t copy_stream = nullptr;  // overlaps S download with the H contraction
  int64_t tile_list_T = 0;             // tile rows of the cached grouped triangle order
  std::vector<int2> tile_list_host;    // its host copy (source of an async upload)
  int32_t engine_setting = HSB_ENGINE_AUTO;  // hsb_ctx_set_engine
  int32_t engine = HSB_ENGINE_DMMA;    // resolved per call (CtxCall): FP64 DMMA or INT8 CRT emulation
  std::mutex call_mu;                  // one entry point at a time per context (workspace, streams, settings)
  int32_t oz_min_bits = kOzDefaultBits; // INT8 engine: operand integer bits (accuracy ~2^-bits)
  std::vector<int4> oz_wide_host;      // wide INT8 GEMM work items (contract.cu, HSB_OZ_WIDE)
  int64_t oz_tiles_n = 0;              // cached INT8-engine tile list (n of the output)
  std::vector<int2> oz_tiles_host;
  std::vector<int32_t> oz_tile_index_host;
  int32_t cplx = HSB_CPLX_3M;          // complex product form of the zrk kernels
  // INT8 engine: left operands of S and H prepared by the matching kernel for
  // the build hsb_build_hs_physical runs (A stack, shape, moduli, bits); the
  // buffers are the workspace entries oz_exp_l, oz_res_a, oz_res2
  struct OzPrepared {
    const double* a = nullptr;
    int64_t k = 0, ng = 0;
    int32_t n_mod = 0, bits = 0;
  } oz_prepared;
};

// Entry-point guard: serialises calls on one context (its workspace map, copy
// stream and staging are not thread-safe; the reference build is externally
// single-entrant, but its kernels are reentrant) and resolves
// HSB_ENGINE_AUTO: the pipeline (hsb_build_hs) runs the INT8 engine at FP64
// width, the kernel-level BLAS calls run FP64 DMMA (elementwise semantics for
// arbitrary operands).
struct CtxCall {
  std::lock_guard<std::mutex> lock;
  CtxCall(hsb_ctx* ctx, bool pipeline) : lock(ctx->call_mu) {
    ctx->engine = ctx->engine_setting != HSB_ENGINE_AUTO ? ctx->engine_setting
                  : pipeline                              ? HSB_ENGINE_INT8
                                                          : HSB_ENGINE_DMMA;
  }
};

inline thread_local std::string g_create_err;  // errors of hsb_ctx_create (no context yet)

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


namespace hsb_host {


inline hsb_status fail(hsb_ctx* ctx, hsb_status st, const std::string& msg) {
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

// grow-only named device workspace (cudaMalloc); pinned host scratch
hsb_status ws(hsb_ctx* ctx, const char* name, size_t bytes, void** out);
hsb_status pinned(hsb_ctx* ctx, size_t bytes, void** out);

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

inline cudaError_t timeline_mark(Timeline* tl, cudaStream_t st, const char* tag) { return tl->mark(st, tag); }

// Absolute GPU timeline across calls and contexts (HSB_TRACE=1): events on
// any stream, resolved after the call against one process-wide base event
// and printed as "[hsb trace] <ctx> <tag> <ms>".  Diagnostics only.
struct GpuTrace {
  bool on = std::getenv("HSB_TRACE") != nullptr;
  const void* who = nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;
  static cudaEvent_t base() {
    static cudaEvent_t b = [] {
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, 0);
      cudaEventSynchronize(e);
      return e;
    }();
    return b;
  }
  ~GpuTrace() {
    for (auto& m : marks) cudaEventDestroy(m.second);
  }
  void mark(cudaStream_t st, const std::string& tag) {
    if (!on) return;
    base();
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    marks.push_back({tag, e});
    cudaEventRecord(e, st);
  }
  void report() {
    if (!on) return;
    std::string s;
    for (auto& m : marks) {
      float ms = -1.f;
      cudaEventSynchronize(m.second);
      cudaEventElapsedTime(&ms, base(), m.second);
      char buf[160];
      std::snprintf(buf, sizeof buf, "[hsb trace] %p %s %.3f\n", who, m.first.c_str(), ms);
      s += buf;
    }
    std::fputs(s.c_str(), stderr);
  }
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
  int* done_cnt = nullptr;
  // optional (3M DMMA kernel, rectangular calls): column exponents of the
  // output for the INT8 engine, atomicMax-ed into col_exp (initialised by the caller)
  int32_t* col_exp = nullptr;
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
  // optional (INT8 engine): precomputed column exponents of the left / right
  // operands, and residue planes of operands by base pointer and side (0 left,
  // 1 right), prepared with the same moduli and bits (oz_choose)
  const int32_t* oz_el = nullptr;
  const int32_t* oz_er = nullptr;
  struct OzPre {
    const double* base;
    int side;
    int8_t* planes;
    const double* rscale = nullptr;  // the operand's row factors (OperandView::rscale)
  };
  std::vector<OzPre> oz_pre;
  // with oz_el: the reduction length the prepared planes were sized for
  // (oz_choose's moduli and bits), when this call's own is shorter
  int64_t oz_ktot = 0;
};


// plain stacked operand: k x cols, leading dimension ld
inline OperandView plain(const double* base, int64_t k, int64_t cols, int64_t ld) {
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
inline OperandView atom_rows(const double* stacked, int64_t n_atoms, int64_t n_l, int64_t cols, int64_t ld) {
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
inline OperandView atom_mats(const double* base, int64_t n_atoms, int64_t n_l) {
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


// the contraction dispatcher (contract.cu): DMMA 3M / 4M kernels or the INT8 engine
hsb_status run_zrk(hsb_ctx* ctx, cudaStream_t st, const ZrkCall& z, int* launches);
// INT8 engine: moduli count and operand bits for a reduction of length ktot
hsb_status oz_choose(hsb_ctx* ctx, int64_t ktot, int* n_mod, int* b);
// INT8 engine, fused H = A^H V1 + B^H V2 with the V products on the INT8 tensor
// cores as well (hsb_api.cu): A, B are K x ng stacks (ld K) of na atoms of nl
// rows; T_* per-atom nl x nl column-major blocks; V1, V2 receive the K x ng
// products; h is the triangle call (segments filled in here)
struct HvCall {
  const double *A, *B, *TAA, *TAB, *TBB;
  double *V1, *V2;
  int64_t K, ng, nl, na;
  Timeline* tl = nullptr;
  const char* vsect = nullptr;  // timeline tag of the V products
};
hsb_status run_ozaki_hv(hsb_ctx* ctx, cudaStream_t st, const HvCall& c, ZrkCall h, int* launches);

}  // namespace hsb_host
