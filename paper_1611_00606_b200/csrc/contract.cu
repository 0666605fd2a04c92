// contract.cu — the contraction dispatcher behind every dense update of the
// pipeline and of the kernel-level ABI: TMA descriptor encoding, the DMMA
// kernels' tile orders and sum planes, and the INT8 engine's orchestration
// (column exponents, residue planes, modular GEMM, CRT; ozaki.cuh).
#include "host_ctx.cuh"

namespace hsb_host {

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

// side of the tile groups (bands of G tile columns), HSB_OZ_GROUP for experiments;
// the column-group launches of the streamed paths follow the same bands
static int64_t oz_tile_group() {
  static const int64_t g = [] {
    const char* e = std::getenv("HSB_OZ_GROUP");
    const int v = e ? std::atoi(e) : 0;
    return static_cast<int64_t>(v > 0 ? v : 6);
  }();
  return g;
}

// 256 x 256 tiles (tile row tm >= tile col tn) of the lower triangle, in
// groups of 6 x 6 tiles for L2 reuse
hsb_status oz_tiles(hsb_ctx* ctx, int64_t n, cudaStream_t st, const int2** out, int* count,
                    const int32_t** index) {
  const int64_t T = (n + kOzBN - 1) / kOzBN;
  std::vector<int2>& v = ctx->oz_tiles_host;
  std::vector<int32_t>& ix = ctx->oz_tile_index_host;
  const int64_t G = oz_tile_group();
  static const int64_t GR = [] {  // HSB_OZ_GROUP_ROWS: rows of a group (default = G)
    const char* e = std::getenv("HSB_OZ_GROUP_ROWS");
    const int v = e ? std::atoi(e) : 0;
    return static_cast<int64_t>(v);
  }();
  const int64_t gr = GR > 0 ? GR : G;
  if (ctx->oz_tiles_n != n) {
    v.clear();
    for (int64_t j0 = 0; j0 < T; j0 += G)
      for (int64_t i0 = j0; i0 < T; i0 += gr)
        for (int64_t j = j0; j < std::min<int64_t>(j0 + G, T); ++j)
          for (int64_t i = std::max(i0, j); i < std::min<int64_t>(i0 + gr, T); ++i)
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

// moduli: the fewest with b >= oz_min_bits.  With |x'| + |y'| <= 2^b per
// element, |Re C'| = |sum x'x' + y'y'| and |Im C'| = |sum x'_L y'_R - y'_L x'_R|
// are both <= K 2^2b; the CRT needs |X| < M/2, kept with one bit of margin:
// 2b <= log2 M - 2 - log2 K.  b may exceed the request (more bits for the
// entries below their column's max, at no cost) up to kOzMaxBits, the range
// the residue kernel's magic-constant quotients are exact for.
hsb_status oz_choose(hsb_ctx* ctx, int64_t ktot, int* n_mod_out, int* b_out) {
  int n_mod = 0, b = 0;
  double log2m = 0;
  for (int i = 0; i < kOzMaxMod; ++i) {
    log2m += std::log2(static_cast<double>(oz_mod(i)));
    const int bi = static_cast<int>(std::floor((log2m - 2.0 - std::log2(static_cast<double>(std::max<int64_t>(ktot, 1)))) / 2.0));
    if (i + 1 >= kOzMinMod && (bi >= ctx->oz_min_bits || i + 1 == kOzMaxMod)) {
      n_mod = i + 1;
      b = std::min(bi, kOzMaxBits);
      break;
    }
  }
  if (b < 30) return fail(ctx, HSB_ERR_UNSUPPORTED, "reduction too long for the INT8 engine's moduli");
  *n_mod_out = n_mod;
  *b_out = b;
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
  int n_mod = 0, b = 0;
  if (z.oz_el && z.oz_ktot > 0) {
    if (z.oz_ktot < ktot) return fail(ctx, HSB_ERR_UNSUPPORTED, "prepared INT8 planes sized for a shorter reduction");
    ktot = z.oz_ktot;
  }
  CKS(oz_choose(ctx, ktot, &n_mod, &b));
  // exponents: one array for both sides (m == n), max over every operand --
  // unless the caller prepared left / right exponents (run_ozaki_hv)
  const bool pre = z.oz_el != nullptr;
  const int32_t* el = z.oz_el;
  const int32_t* er = z.oz_er;
  int32_t* e = nullptr;
  if (!pre) {
    void* ebuf;
    CKS(ws(ctx, "oz_exp", static_cast<size_t>(n) * sizeof(int32_t), &ebuf));
    e = static_cast<int32_t*>(ebuf);
    el = er = e;
    CK(launch_ozaki_init_exp(e, n, st));
  }
  if (!pre) {
    std::vector<const OperandView*> seen;
    auto colexp = [&](const OperandView& v) -> hsb_status {
      for (const OperandView* q : seen)
        if (q->base == v.base && q->k == v.k && q->ld == v.ld && q->rscale == v.rscale) return HSB_OK;
      seen.push_back(&v);
      CK(launch_ozaki_colexp(v.base, v.ld, v.k, v.cols, e, st, v.rscale));
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
    int side;
    const double* rscale;
  };
  std::vector<Src> srcs;
  std::vector<OzResSrc> pending;  // planes still to compute: one batched launch
  int computed = 0;
  auto planes_of = [&](const OperandView& v, int side, Src* out) -> hsb_status {
    if (!pre || el == er) side = 0;  // one exponent array: both sides share residues
    for (const Src& q : srcs)
      if (q.base == v.base && q.k == v.k && q.ld == v.ld && q.side == side && q.rscale == v.rscale) {
        *out = q;
        return HSB_OK;
      }
    Src q{v.base, v.k, v.ld, nullptr, oz_kpad(v.k), side, v.rscale};
    for (const ZrkCall::OzPre& pz : z.oz_pre)
      if (pz.base == v.base && pz.side == side && pz.rscale == v.rscale) q.planes = pz.planes;
    if (!q.planes) {
      const std::string name = "oz_res" + std::to_string(computed++);
      void* buf;
      CKS(ws(ctx, name.c_str(), static_cast<size_t>(kOzPlanes) * n_mod * n * q.kpad, &buf));
      q.planes = static_cast<int8_t*>(buf);
      pending.push_back({v.base, v.ld, v.k, side ? er : el, v.rscale, q.planes, q.kpad});
    }
    srcs.push_back(q);
    *out = q;
    return HSB_OK;
  };
  OzGemmParams gp;
  std::memset(&gp, 0, sizeof(gp));
  // products phi1(C), phi2(C) (ozaki.cuh): conjugation swaps the left planes
  const int lp[kOzProds] = {z.conj ? kOzPhi2 : kOzPhi1, z.conj ? kOzPhi1 : kOzPhi2};
  const int rp[kOzProds] = {kOzPhi1, kOzPhi2};
  std::vector<Src> seg_l(segs.size()), seg_r(segs.size());
  for (size_t si = 0; si < segs.size(); ++si) {
    CKS(planes_of(segs[si].l, 0, &seg_l[si]));
    CKS(planes_of(segs[si].r, 1, &seg_r[si]));
  }
  for (size_t i = 0; i < pending.size(); i += kOzResMaxSrc)
    CK(launch_ozaki_residues_batch(pending.data() + i, static_cast<int>(std::min<size_t>(kOzResMaxSrc, pending.size() - i)),
                                   n, b, n_mod, st));
  for (size_t si = 0; si < segs.size(); ++si) {
    const Src& L = seg_l[si];
    const Src& R = seg_r[si];
    const int64_t pl = static_cast<int64_t>(n_mod) * n * L.kpad, pr = static_cast<int64_t>(n_mod) * n * R.kpad;
    for (int pi = 0; pi < kOzProds; ++pi) {  // MMA A operand: the right factor (output columns)
      CKS(oz_encode(ctx, &gp.map[pi][si][0], R.planes + rp[pi] * pr, R.k, n, R.kpad, n_mod, 128));
      CKS(oz_encode(ctx, &gp.map[pi][si][1], L.planes + lp[pi] * pl, L.k, n, L.kpad, n_mod, 128));
    }
    gp.seg_chunk0[si + 1] = gp.seg_chunk0[si] + static_cast<int32_t>((segs[si].l.k + kOzBK - 1) / kOzBK);
    static const bool no_kskip = std::getenv("HSB_NO_KSKIP") != nullptr;  // A/B experiments
    if (!no_kskip)
      gp.seg_ksteps_last[si] = static_cast<int32_t>((segs[si].l.k - (gp.seg_chunk0[si + 1] - gp.seg_chunk0[si] - 1) * kOzBK + 31) / 32);
  }
  gp.nseg = static_cast<int32_t>(segs.size());
  // slabs of ~16 KB of k (see ozaki.cuh), balanced
  const int32_t total_chunks = gp.seg_chunk0[gp.nseg];
  static const int32_t kSlabChunks = [] {  // HSB_OZ_SLAB_KB: slab k extent for experiments (default 16)
    const char* e = std::getenv("HSB_OZ_SLAB_KB");
    const int v = e ? std::atoi(e) : 0;
    return static_cast<int32_t>((v > 0 ? v : 16) * 1024 / kOzBK);
  }();
  gp.nslab = std::max(1, std::min<int32_t>(kOzMaxSlab, (total_chunks + kSlabChunks - 1) / kSlabChunks));
  for (int sl = 0; sl <= gp.nslab; ++sl)
    gp.slab_chunk0[sl] = static_cast<int32_t>(static_cast<int64_t>(total_chunks) * sl / gp.nslab);
  gp.n_mod = n_mod;
  gp.n = static_cast<int32_t>(n);
  const int32_t* tile_index = nullptr;
  int total_tiles = 0;
  CKS(oz_tiles(ctx, n, st, &gp.tile_list, &total_tiles, &tile_index));
  gp.mod_stride = static_cast<int64_t>(total_tiles) * kOzTileBytes;
  gp.prod_stride = gp.mod_stride * n_mod;
  gp.tiles_total = total_tiles;
  gp.a_k_per_tm = 0;
  gp.nrows = gp.n;
  void* rbuf;
  CKS(ws(ctx, "oz_out", static_cast<size_t>(kOzProds * gp.prod_stride), &rbuf));
  gp.res = static_cast<int8_t*>(rbuf);
  void* cbuf;
  CKS(ws(ctx, "oz_counter", 16, &cbuf));
  gp.counter = static_cast<int32_t*>(cbuf);
  gp.slab_cnt = nullptr;
  if (gp.nslab > 1) {
    const size_t nc = static_cast<size_t>(kOzProds) * n_mod * total_tiles;
    void* sbuf;
    CKS(ws(ctx, "oz_slab_cnt", nc * sizeof(int32_t), &sbuf));
    gp.slab_cnt = static_cast<int32_t*>(sbuf);
    CK(launch_fill_i32(static_cast<int32_t*>(sbuf), static_cast<int64_t>(nc), 0, st));
  }
  if (gp.nseg == 0) CK(cudaMemsetAsync(rbuf, 0, static_cast<size_t>(kOzProds * gp.prod_stride), st));

  OzCrtParams cp;
  cp.res = gp.res;
  cp.mod_stride = gp.mod_stride;
  cp.prod_stride = gp.prod_stride;
  cp.tile_index = tile_index;
  cp.T = static_cast<int32_t>((n + kOzBN - 1) / kOzBN);
  cp.n_mod = n_mod;
  cp.n = static_cast<int32_t>(n);
  cp.b = b;
  cp.conj = z.conj ? 1 : 0;
  cp.el = el;
  cp.er = er;
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
  // product runs in column groups of G tiles (contiguous in the tile list):
  // once groups 0..g are done their columns are final (the mirror of an
  // entry of an earlier group lands in a later column), so their download
  // overlaps the remaining groups.  Otherwise one GEMM + one CRT launch.
  const int64_t T = (n + kOzBN - 1) / kOzBN;
  const int64_t T64 = (n + kBN - 1) / kBN;  // the host's 64-column blocks
  const std::vector<int2>& tl_host = ctx->oz_tiles_host;
  // (the tile list is ordered in bands of kOzTileGroup columns, see oz_tiles)
  const int64_t group = (z.done_cnt || z.chunk_events) ? oz_tile_group() : T;
  // wide work items (HSB_OZ_WIDE, experiments): consecutive row tiles of one
  // column paired, one launch over the whole triangle
  static const bool wide_env = std::getenv("HSB_OZ_WIDE") != nullptr;
  const bool wide = wide_env && group == T && gp.nseg > 0;
  gp.wide_list = nullptr;
  int nwide = 0;
  if (wide) {
    std::vector<int4>& wl = ctx->oz_wide_host;
    wl.clear();
    for (int t = 0; t < total_tiles;) {
      const int2 a = tl_host[static_cast<size_t>(t)];
      const bool pair = t + 1 < total_tiles && tl_host[static_cast<size_t>(t) + 1].y == a.y &&
                        tl_host[static_cast<size_t>(t) + 1].x == a.x + 1;
      wl.push_back(make_int4(a.x, a.y, t, pair ? t + 1 : -1));
      t += pair ? 2 : 1;
    }
    nwide = static_cast<int>(wl.size());
    void* wbuf;
    CKS(ws(ctx, "oz_wide", wl.size() * sizeof(int4), &wbuf));
    CK(cudaMemcpyAsync(wbuf, wl.data(), wl.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
    gp.wide_list = static_cast<const int4*>(wbuf);
  }
  int t0 = 0;
  for (int64_t j0 = 0; j0 < T; j0 += group) {
    const int64_t j1 = std::min<int64_t>(j0 + group, T);
    int t1 = t0;
    while (t1 < total_tiles && tl_host[static_cast<size_t>(t1)].y < j1) ++t1;
    if (gp.nseg > 0 && t1 > t0) {
      gp.tile0 = wide ? 0 : t0;
      gp.ntiles = wide ? nwide : t1 - t0;
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
  if (launches) *launches += 3 + (pre ? 0 : 2 * static_cast<int>(segs.size())) + (computed + kOzResMaxSrc - 1) / kOzResMaxSrc;
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
  static const bool no_zplanes = std::getenv("HSB_NO_ZPLANES") != nullptr;  // experiments
  bool planes = g3 && z.batch == 1 && !no_zplanes;
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
  // 3M on batched products whose left operands are per-atom square blocks (the V
  // products: T blocks): left planes only, per atom, k padded to even so the
  // 3-D TMA view's atom stride is a multiple of 16 bytes.  Opt-in
  // (HSB_LPLANES=1): the V kernel alone runs 4 % faster (C3 3.38 -> 3.26 ms,
  // ncu), but beside the INT8 engine's side preparation of S's operands the
  // build measured no faster (19.1-19.3 vs 19.1 ms)
  static const bool use_lplanes = std::getenv("HSB_LPLANES") != nullptr;
  bool lplanes = g3 && !planes && z.batch > 1 && use_lplanes;
  for (const Seg& s : z.segs)
    if (s.l.k > 0 && !(s.l.batch == z.batch && s.l.bpos == 2 && s.l.ld == s.l.k && s.l.cols == s.l.k &&
                       s.l.bstride == s.l.k * s.l.k && s.l.k <= 0x7fffffff))
      lplanes = false;
  struct LPlane {
    const double* base;
    double* plane;
  };
  std::vector<LPlane> lsrcs;
  auto lplane_of = [&](const OperandView& v, CUtensorMap* map) -> hsb_status {
    const int64_t kp = v.k + (v.k & 1);
    double* plane = nullptr;
    for (const LPlane& q : lsrcs)
      if (q.base == v.base) plane = q.plane;
    if (!plane) {
      const std::string name = "lplane" + std::to_string(lsrcs.size());
      void* buf;
      CKS(ws(ctx, name.c_str(), static_cast<size_t>(kp) * v.cols * v.batch * 8, &buf));
      plane = static_cast<double*>(buf);
      CK(launch_sum_planes_batched(v.base, static_cast<int>(v.k), v.bstride, v.batch, z.conj, plane,
                                   static_cast<int>(kp), st));
      lsrcs.push_back({v.base, plane});
    }
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(kp), static_cast<cuuint64_t>(v.cols),
                          static_cast<cuuint64_t>(v.batch)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(kp) * 8, static_cast<cuuint64_t>(kp * v.cols) * 8};
    cuuint32_t box[3] = {8, static_cast<cuuint32_t>(kBM), 1}, estr[3] = {1, 1, 1};
    CUresult r = ctx->encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, plane, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(ctx, HSB_ERR_CUDA, "cuTensorMapEncodeTiled failed for a batched plane (code " +
                                         std::to_string(static_cast<int>(r)) + ")");
    return HSB_OK;
  };
  int nseg = 0, total = 0;
  for (const Seg& s : z.segs) {
    if (s.l.k <= 0) continue;
    if (s.l.k != s.r.k) return fail(ctx, HSB_ERR_DIMENSION, "segment operands disagree in reduction length");
    CKS(encode_operand(ctx, &p.lmap[nseg], s.l));
    CKS(encode_operand(ctx, &p.rmap[nseg], s.r));
    if (lplanes) CKS(lplane_of(s.l, &p.lsum[nseg]));
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
  if (z.col_exp && (!g3 || z.triangle)) return fail(ctx, HSB_ERR_UNSUPPORTED, "column exponents need the 3M rect kernel");
  p.col_exp = z.col_exp;
  int64_t grid_x = z.triangle ? static_cast<int64_t>(p.tiles_m) * (p.tiles_m + 1) / 2
                              : static_cast<int64_t>(p.tiles_m) * p.tiles_n;
  if (grid_x > 0x7fffffff || z.batch > 65535) return fail(ctx, HSB_ERR_UNSUPPORTED, "grid too large");
  static const bool no_tile_order = std::getenv("HSB_NO_TILE_ORDER") != nullptr;  // experiments
  if (g3 && z.triangle && z.batch == 1 && p.tiles_m > kTileGroup && !no_tile_order)
    CKS(tile_order(ctx, p.tiles_m, st, &p.tile_list));
  if (z.tl) CK(timeline_mark(z.tl, st, z.sect));
  if (g3) {
    if (grid_x * z.batch > 0x7fffffff) return fail(ctx, HSB_ERR_UNSUPPORTED, "grid too large");
    p.lplane3d = lplanes ? 1 : 0;
    CK(launch_zrk3m(p, z.conj, planes ? 2 : lplanes ? 1 : 0, static_cast<int>(grid_x), static_cast<int>(z.batch),
                    st));
    if (launches) *launches += static_cast<int>(srcs.size() + lsrcs.size());
  } else {
    CK(launch_zrk(p, z.conj, static_cast<int>(grid_x), static_cast<int>(z.batch), st));
  }
  if (z.tl) CK(timeline_mark(z.tl, st, z.core));
  if (launches) ++*launches;
  return HSB_OK;
}

// ---------------------------------------------------------------------------
// Fused H on the INT8 engine with the V products there too:
//   el = exponents of the A / B columns -> left residues of A and B
//   L1_a = [T_AA | T_AB], L2_a = [T_AB^H | T_BB] -> exponents, residues
//   [V1_a; V2_a] = L1_a^H A_a + L2_a^H B_a: rectangular (atom, column tile)
//     modular GEMM (M = 2 nl rows per atom, the A / B residues of H's left
//     side as its right operand) + CRT into the V1 / V2 stacks, whose column
//     maxima give er
//   H = A^H V1 + B^H V2 on the lower triangle with (el, er) and the left
//     residues reused (run_ozaki).
// The V product's reduction (2 nl) is shorter than H's (2 K), so H's moduli
// and bits keep it exact.
hsb_status run_ozaki_hv(hsb_ctx* ctx, cudaStream_t st, const HvCall& c, ZrkCall h, int* launches) {
  const int64_t K = c.K, ng = c.ng, nl = c.nl, na = c.na;
  if (2 * nl > 256) return fail(ctx, HSB_ERR_UNSUPPORTED, "INT8 V products need n_l <= 128");
  int n_mod = 0, b = 0;
  CKS(oz_choose(ctx, 2 * K, &n_mod, &b));
  // left blocks: 256 k rows per atom (the atom's nl rows shifted by (nl a) mod 16,
  // matching the 16-byte aligned start of the right operand's TMA box)
  const int64_t kpad = oz_kpad(K), kpad_t = 256;
  const int64_t tcols = na * 256;
  void *el_b, *er_b, *et_b, *la, *lb, *t1, *t2, *rt1, *rt2;
  CKS(ws(ctx, "oz_exp_l", ng * sizeof(int32_t), &el_b));
  CKS(ws(ctx, "oz_exp_r", ng * sizeof(int32_t), &er_b));
  CKS(ws(ctx, "oz_exp_t", tcols * sizeof(int32_t), &et_b));
  int32_t *el = static_cast<int32_t*>(el_b), *er = static_cast<int32_t*>(er_b), *et = static_cast<int32_t*>(et_b);
  // left side of H (and right side of the V products): A, B
  CK(launch_ozaki_init_exp(el, ng, st));
  CK(launch_ozaki_colexp(c.A, K, K, ng, el, st));
  CK(launch_ozaki_colexp(c.B, K, K, ng, el, st));
  const size_t res_bytes = static_cast<size_t>(kOzPlanes) * n_mod * ng * kpad;
  CKS(ws(ctx, "oz_res_la", res_bytes, &la));
  CKS(ws(ctx, "oz_res_lb", res_bytes, &lb));
  CK(launch_ozaki_residues(c.A, K, K, ng, el, b, n_mod, static_cast<int8_t*>(la), kpad, st));
  CK(launch_ozaki_residues(c.B, K, K, ng, el, b, n_mod, static_cast<int8_t*>(lb), kpad, st));
  // left blocks of the V products
  const size_t tb = static_cast<size_t>(tcols) * kpad_t * 16;
  CKS(ws(ctx, "oz_tblk1", tb, &t1));
  CKS(ws(ctx, "oz_tblk2", tb, &t2));
  CK(launch_ozaki_vblocks(c.TAA, c.TAB, c.TBB, static_cast<int>(nl), na, static_cast<double*>(t1),
                          static_cast<double*>(t2), st));
  CK(launch_ozaki_init_exp(et, tcols, st));
  CK(launch_ozaki_colexp(static_cast<double*>(t1), kpad_t, kpad_t, tcols, et, st));
  CK(launch_ozaki_colexp(static_cast<double*>(t2), kpad_t, kpad_t, tcols, et, st));
  const size_t rt_bytes = static_cast<size_t>(kOzPlanes) * n_mod * tcols * kpad_t;
  CKS(ws(ctx, "oz_res_t1", rt_bytes, &rt1));
  CKS(ws(ctx, "oz_res_t2", rt_bytes, &rt2));
  CK(launch_ozaki_residues(static_cast<double*>(t1), kpad_t, kpad_t, tcols, et, b, n_mod, static_cast<int8_t*>(rt1),
                           kpad_t, st));
  CK(launch_ozaki_residues(static_cast<double*>(t2), kpad_t, kpad_t, tcols, et, b, n_mod, static_cast<int8_t*>(rt2),
                           kpad_t, st));
  int nlaunch = 12;

  // V products in batches of atoms (bounded residue output)
  OzGemmParams gp;
  std::memset(&gp, 0, sizeof(gp));
  const int lp[kOzProds] = {kOzPhi2, kOzPhi1};  // L^H R
  const int rp[kOzProds] = {kOzPhi1, kOzPhi2};
  const int64_t pl_t = static_cast<int64_t>(n_mod) * tcols * kpad_t, pl_x = static_cast<int64_t>(n_mod) * ng * kpad;
  for (int pi = 0; pi < kOzProds; ++pi) {
    // MMA A operand: the stacks' columns g (k shifted to the atom's rows); B: the left blocks
    CKS(oz_encode(ctx, &gp.map[pi][0][0], static_cast<int8_t*>(la) + rp[pi] * pl_x, K, ng, kpad, n_mod, 128));
    CKS(oz_encode(ctx, &gp.map[pi][0][1], static_cast<int8_t*>(rt1) + lp[pi] * pl_t, kpad_t, tcols, kpad_t, n_mod, 128));
    CKS(oz_encode(ctx, &gp.map[pi][1][0], static_cast<int8_t*>(lb) + rp[pi] * pl_x, K, ng, kpad, n_mod, 128));
    CKS(oz_encode(ctx, &gp.map[pi][1][1], static_cast<int8_t*>(rt2) + lp[pi] * pl_t, kpad_t, tcols, kpad_t, n_mod, 128));
  }
  const int32_t seg_chunks = static_cast<int32_t>(kpad_t / kOzBK);
  gp.nseg = 2;
  gp.seg_chunk0[0] = 0;
  gp.seg_chunk0[1] = seg_chunks;
  gp.seg_chunk0[2] = 2 * seg_chunks;
  gp.nslab = 1;
  gp.slab_chunk0[0] = 0;
  gp.slab_chunk0[1] = 2 * seg_chunks;
  gp.n_mod = n_mod;
  const int64_t gtiles = (ng + kOzBN - 1) / kOzBN;
  gp.n = static_cast<int32_t>(ng);
  gp.nrows = 1 << 30;  // every row r of the left blocks is stored (the CRT reads r < 2 nl)
  gp.a_k_per_tm = static_cast<int32_t>(nl);
  gp.rect_gtiles = static_cast<int32_t>(gtiles);
  gp.tile_list = nullptr;
  gp.slab_cnt = nullptr;
  const int64_t per_batch = std::max<int64_t>(1, std::min<int64_t>(na, 2048 / gtiles));
  const int64_t cap_tiles = per_batch * gtiles;
  void *vout, *cbuf;
  CKS(ws(ctx, "oz_vout", static_cast<size_t>(kOzProds) * n_mod * cap_tiles * kOzTileBytes, &vout));
  CKS(ws(ctx, "oz_counter", 16, &cbuf));
  gp.res = static_cast<int8_t*>(vout);
  gp.counter = static_cast<int32_t*>(cbuf);
  CK(launch_ozaki_init_exp(er, ng, st));
  OzVcrtParams vp;
  std::memset(&vp, 0, sizeof(vp));
  vp.res = gp.res;
  vp.n_mod = n_mod;
  vp.bsum = 2 * b;
  vp.gtiles = static_cast<int32_t>(gtiles);
  vp.nl = static_cast<int32_t>(nl);
  vp.ng = static_cast<int32_t>(ng);
  vp.et = et;
  vp.el = el;
  vp.v1 = c.V1;
  vp.v2 = c.V2;
  vp.ldv = K;
  vp.er = er;
  for (int64_t a0 = 0; a0 < na; a0 += per_batch) {
    const int64_t nb = std::min(per_batch, na - a0);
    gp.rect_atom0 = static_cast<int32_t>(a0);
    gp.tile0 = 0;
    gp.ntiles = static_cast<int32_t>(nb * gtiles);
    gp.tiles_total = gp.ntiles;
    gp.mod_stride = static_cast<int64_t>(gp.ntiles) * kOzTileBytes;
    gp.prod_stride = gp.mod_stride * n_mod;
    CK(launch_ozaki_gemm(gp, st));
    vp.mod_stride = gp.mod_stride;
    vp.prod_stride = gp.prod_stride;
    vp.atom0 = static_cast<int32_t>(a0);
    vp.natoms = static_cast<int32_t>(nb);
    CK(launch_ozaki_vcrt(vp, st));
    nlaunch += 3;
  }
  if (c.tl && c.vsect) CK(timeline_mark(c.tl, st, c.vsect));

  // H = A^H V1 + B^H V2 with the prepared exponents and left residues
  h.segs.clear();
  h.segs.push_back({plain(c.A, K, ng, K), plain(c.V1, K, ng, K)});
  h.segs.push_back({plain(c.B, K, ng, K), plain(c.V2, K, ng, K)});
  h.oz_el = el;
  h.oz_er = er;
  h.oz_pre.clear();
  h.oz_pre.push_back({c.A, 0, static_cast<int8_t*>(la)});
  h.oz_pre.push_back({c.B, 0, static_cast<int8_t*>(lb)});
  if (launches) *launches += nlaunch;
  return run_ozaki(ctx, st, h, launches);
}

}  // namespace hsb_host
