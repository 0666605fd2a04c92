// ozaki.cu — kernels of the INT8-tensor-core emulated FP64 contraction
// (scheme in ozaki.cuh): column exponents, split-complex residue planes, the
// tcgen05 kind::i8 modular GEMM over lower-triangle tiles, and the CRT
// reconstruction with the Hermitian mirror.
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <mutex>

#include "aux_kernels.cuh"
#include "ozaki.cuh"
#include "ozaki_res.cuh"
#include "ptx.cuh"
#include "zrk.cuh"

namespace hsb {

__constant__ int32_t oz_mod_rt[kOzMaxMod] = {241, 233, 229, 221, 205, 197, 193, 181, 173, 157,
                                             149, 137, 113, 109, 101, 97,  89,  73,  61,  53};

// ------------------------------------------------------------ small helpers
__device__ __forceinline__ int sym_lo(int p) { return -(p >> 1); }

// symmetric residue of an int32 v (the GEMM accumulator) modulo an odd p < 256:
// t = (v >> 16) (2^16 mod p) + (v & 0xffff) = v (mod p), |t| < 2^22, then
// q = floor((t m + 2^31) / 2^32) = rn(t / p) with m = rn(2^32 / p): the error
// |t| 2^-33 <= 2^-11 stays below the 1/(2p) >= 2^-9 distance of t / p from a
// half-integer.  IMAD.WIDE + IMAD instead of five FP32 operations.
__device__ __forceinline__ int sym_mod_i32q(int v, int p, int c16, long long m) {
  const int t = (v >> 16) * c16 + (v & 0xffff);
  const int q = static_cast<int>((static_cast<long long>(t) * m + (1ll << 31)) >> 32);
  return t - p * q;
}
__device__ __forceinline__ int sym_adj(int r, int p) {
  const int lo = sym_lo(p);
  if (r < lo) r += p;
  if (r > lo + p - 1) r -= p;
  return r;
}

// ------------------------------------------------------------ 1. exponents
__global__ void ozaki_init_exp_kernel(int32_t* e, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    e[i] = INT_MIN / 2;
}

// one warp per column: e = frexp exponent of max_k |Re x| + |Im x| (max < 2^e)
__global__ void ozaki_colexp_kernel(const double2* __restrict__ x, int64_t ldx, int64_t k, int64_t cols,
                                    int32_t* __restrict__ e, const double* __restrict__ rscale) {
  const int warps = blockDim.x >> 5;
  for (int64_t c = static_cast<int64_t>(blockIdx.x) * warps + (threadIdx.x >> 5); c < cols;
       c += static_cast<int64_t>(gridDim.x) * warps) {
    double m = 0.0;
    const double2* col = x + c * ldx;
    for (int64_t r = threadIdx.x & 31; r < k; r += 32) {
      double2 v = col[r];
      if (rscale) {
        const double u = __ldg(rscale + r);
        v = make_double2(u * v.x, u * v.y);
      }
      m = fmax(m, fabs(v.x) + fabs(v.y));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) {
      int ex = 0;
      frexp(m, &ex);  // m = f * 2^ex, f in [0.5, 1): m < 2^ex (m = 0 -> ex = 0)
      atomicMax(e + c, ex);
    }
  }
}

// one warp per column, two stacks with the same shape read once: the exponent of
// max_k over |a|, |b| and |fl(u_k b)| (|Re| + |Im|) -- the left exponent shared by
// S = A^H A + (UB)^H (UB) and the left side of H = A^H V1 + B^H V2, so A's
// residue planes serve both contractions
__global__ void ozaki_colexp_ab_kernel(const double2* __restrict__ a, const double2* __restrict__ b, int64_t ld,
                                       int64_t k, int64_t cols, const double* __restrict__ u,
                                       int32_t* __restrict__ e, int with_b) {
  const int warps = blockDim.x >> 5;
  for (int64_t c = static_cast<int64_t>(blockIdx.x) * warps + (threadIdx.x >> 5); c < cols;
       c += static_cast<int64_t>(gridDim.x) * warps) {
    double m = 0.0;
    const double2* ca = a + c * ld;
    const double2* cb = b + c * ld;
    for (int64_t r = threadIdx.x & 31; r < k; r += 32) {
      const double2 va = ca[r], vb = cb[r];
      const double uk = __ldg(u + r);
      m = fmax(m, fabs(va.x) + fabs(va.y));
      if (with_b) m = fmax(m, fabs(vb.x) + fabs(vb.y));
      m = fmax(m, fabs(uk * vb.x) + fabs(uk * vb.y));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) {
      int ex = 0;
      frexp(m, &ex);
      e[c] = ex;
    }
  }
}

// ------------------------------------------------------------ 2. residues
// 1 / p, correctly rounded (compile-time division)
__constant__ double oz_inv_rt[kOzMaxMod] = {
    1.0 / 241, 1.0 / 233, 1.0 / 229, 1.0 / 221, 1.0 / 205, 1.0 / 197, 1.0 / 193, 1.0 / 181, 1.0 / 173, 1.0 / 157,
    1.0 / 149, 1.0 / 137, 1.0 / 113, 1.0 / 109, 1.0 / 101, 1.0 / 97,  1.0 / 89,  1.0 / 73,  1.0 / 61,  1.0 / 53};

// the planes of modulus I .. NM-1 for this thread's 4 elements, as 32-bit
// shared stores at compile-time offsets (plane q = (product, modulus), 1 KB each)
template <int NM, int I = 0>
__device__ __forceinline__ void oz_residue_planes(const uint32_t (&xl)[4], const uint32_t (&xh)[4],
                                                  const uint32_t (&yl)[4], const uint32_t (&yh)[4], uint32_t* s0) {
  if constexpr (I < NM) {
    int u[4], w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) oz_planes<I>(xl[j], xh[j], yl[j], yh[j], u[j], w[j]);
    const auto pack = [](const int* v) {
      return __byte_perm(__byte_perm(v[0], v[1], 0x40), __byte_perm(v[2], v[3], 0x40), 0x5410);
    };
    s0[I * 256] = pack(u);
    s0[(NM + I) * 256] = pack(w);
    oz_residue_planes<NM, I + 1>(xl, xh, yl, yh, s0);
  }
}

// Block = 8 columns (one per warp) x 128 k; lane l owns k = 4l .. 4l+3 of its
// warp's column (coalesced 16-byte loads).  The planes are assembled in
// shared memory as [plane][modulus][column][128 k] -- 32-bit stores at
// compile-time offsets -- and written by one TMA bulk tensor store of the box
// {128 k, 8 columns, NM moduli, 2 planes} into the [plane][modulus][col][kpad]
// buffer (out-of-range k / columns clipped by the TMA unit): no per-store
// 64-bit address arithmetic, full-line DRAM writes.
// plane 0 = phi1(z') = x' + j y', plane 1 = phi2(z') = x' - j y' (mod p_i)
constexpr int kOzResK = 4;
constexpr int kOzResCols = 8;
constexpr int kOzResKBlk = 128;
// blockIdx.z selects one of up to kOzResMaxSrc operands of one launch (same
// exponent width b, moduli and column count; each with its own map / kpad)
struct OzResBatch {
  CUtensorMap map[kOzResMaxSrc];
  OzResSrc src[kOzResMaxSrc];
  int64_t kpad[kOzResMaxSrc];
  int64_t cols;
  int b;
};
// Two k blocks per CTA (kOzResTiles): both blocks' operand loads are issued
// up front, so the second block's HBM latency hides behind the first block's
// residue arithmetic (the one-block form stalled on its loads: long
// scoreboard 28 % of the samples).  C3: 3.15 -> 3.06 ms per launch list at
// 3 CTAs / SM (80 registers); at 2 CTAs / SM (128 registers) 3.50 ms.
constexpr int kOzResTiles = 2;
template <int NM>
__global__ void __launch_bounds__(256, 3) ozaki_residue_kernel(const __grid_constant__ OzResBatch p) {
  __shared__ __align__(128) uint32_t tile[2 * NM * kOzResCols * kOzResKBlk / 4];
  const OzResSrc& sr = p.src[blockIdx.z];
  const int64_t kpad = p.kpad[blockIdx.z];
  const int kb0 = static_cast<int>(blockIdx.x) * kOzResTiles;
  if (static_cast<int64_t>(kb0) * kOzResKBlk >= kpad) return;  // shorter operand of the batch
  const double2* __restrict__ x = reinterpret_cast<const double2*>(sr.x);
  const double* __restrict__ rscale = sr.rscale;
  const int64_t ldx = sr.ldx, k = sr.k, cols = p.cols;
  const int b = p.b;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = static_cast<int64_t>(blockIdx.y) * kOzResCols + warp;
  double2 raw[kOzResTiles][kOzResK];
  double us[kOzResTiles][kOzResK];
#pragma unroll
  for (int tt = 0; tt < kOzResTiles; ++tt) {
    const int64_t k0 = static_cast<int64_t>(kb0 + tt) * kOzResKBlk + kOzResK * lane;
#pragma unroll
    for (int j = 0; j < kOzResK; ++j) {
      const bool in = c < cols && k0 + j < k;
      raw[tt][j] = in ? x[c * ldx + k0 + j] : make_double2(0.0, 0.0);
      us[tt][j] = (in && rscale) ? __ldg(rscale + k0 + j) : 1.0;
    }
  }
  // x * 2^(b - e) in two exact power-of-two steps (each factor stays finite)
  const int sh = c < cols ? b - __ldg(sr.col_exp + c) : 0;
  const double s1 = pow2i(sh / 2), s2 = pow2i(sh - sh / 2);
#pragma unroll
  for (int tt = 0; tt < kOzResTiles; ++tt) {
    const int kb = kb0 + tt;
    if (static_cast<int64_t>(kb) * kOzResKBlk >= kpad) break;  // block-uniform
    uint32_t xl[kOzResK], xh[kOzResK], yl[kOzResK], yh[kOzResK];
#pragma unroll
    for (int j = 0; j < kOzResK; ++j) {
      double2 v = raw[tt][j];
      if (rscale) v = make_double2(us[tt][j] * v.x, us[tt][j] * v.y);  // fl(u x), as diag_scale_kernel rounds it
      oz_split(rint((v.x * s1) * s2), xl[j], xh[j]);
      oz_split(rint((v.y * s1) * s2), yl[j], yh[j]);
    }
    if (tt > 0) {  // the previous block's TMA store has read the staging tile
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncthreads();
    }
    // (columns past the end store zeros; the TMA store clips them anyway)
    oz_residue_planes<NM>(xl, xh, yl, yh, tile + (warp * kOzResKBlk) / 4 + lane);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> TMA reads
    __syncthreads();
    if (threadIdx.x == 0)
      asm volatile(
          "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];\n\t"
          "cp.async.bulk.commit_group;" ::"l"(reinterpret_cast<uint64_t>(&p.map[blockIdx.z])),
          "r"(kb * kOzResKBlk), "r"(static_cast<int>(blockIdx.y) * kOzResCols), "r"(0), "r"(0), "r"(smem_u32(tile))
          : "memory");
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// ------------------------------------------------------------ 3. INT8 GEMM
// CTA pairs (cluster of 2, tcgen05 cta_group::2): the pair owns a 256 x 256
// output tile; CTA r holds rows 128 r .. 128 r + 127 of the A tile and of the
// B tile in its own shared memory, the leader (rank 0) issues one
// M = 256, N = 256, K = 32 MMA per 32-byte k step and each CTA's TMEM receives
// its 128 rows x 256 int32 columns.  Per SM and 128-byte k chunk that is
// 32 KB of TMA traffic for 4M MACs (half of a 1-CTA 128 x 256 tile's), so six
// 32 KB stages fit in shared memory.
constexpr int kOzHalf = 128;                      // rows of A and of B per CTA
constexpr int kOzABytes = kOzHalf * kOzBK;        // 16 KB
// WIDE (long reductions): each stage holds the column panel's half and two row
// panels' halves; the pair runs two MMAs per k step into its two TMEM
// accumulators (no accumulator double buffering: the epilogue of an item is
// short next to its ~240 k chunks), so a wave of pairs covers twice the tiles
// with a third fewer operand panels streamed and a quarter less L2 -> SM traffic
template <bool WIDE>
struct OzG {
  static constexpr int stages = WIDE ? 4 : 7;
  static constexpr int nb = WIDE ? 2 : 1;                       // row-panel halves per stage
  static constexpr int stage_bytes = (1 + nb) * kOzABytes;      // 32 or 48 KB
  static constexpr int smem = stages * stage_bytes + 1024 + 256;
};
// warp 0 TMA, warp 1 MMA (leader) + TMEM owner, warps 2-9 epilogue: two warps
// per TMEM lane quarter, each draining half of the accumulator's columns into
// registers and releasing the TMEM buffer before it reduces and stores them
// (with the early release, 16 epilogue warps -- round 2's first answer to
// short reductions -- were no faster than 8: 8-way C3 shard GEMMs 4.35 vs
// 4.15 ms, C3 unchanged, and 8 need no register spills of note)
constexpr int kOzEpiWarps = 8;
constexpr int kOzEpiParts = kOzEpiWarps / 4;  // column parts per lane quarter
constexpr int kOzThreads = (2 + kOzEpiWarps) * 32;
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;       // shared::cluster address of the leader's copy

__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(leader_bar)
      : "memory");
}
// K-major operand tile, 128B swizzle: 8-row atoms of 1024 B (SBO); LBO unused
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}
constexpr uint32_t kOzIdesc = (2u << 4)                // D: s32
                              | (1u << 7)              // A: signed int8
                              | (1u << 10)             // B: signed int8
                              | ((kOzBN >> 3) << 17)   // N = 256
                              | ((256 >> 4) << 24);    // M = 256 (pair)
__device__ __forceinline__ void mma_i8_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8, %9, %10, %11, %12}, p;\n\t}\n" ::"r"(
          tmem_d),
      "l"(da), "l"(db), "r"(kOzIdesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0), "r"(0), "r"(0), "r"(0), "r"(0));
}
// arrive on the barrier at this offset in both CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          bar),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
}
// Arrive on a (possibly remote) barrier that hands over no generic-proxy data:
// "TMEM buffer drained" (after tcgen05.fence::before_thread_sync) and "work
// slot read".  Release at CTA scope: the cluster-scope release above waits for
// every outstanding global store of the arriving warp (the epilogue's residue
// stores) -- ncu showed it as the top stall (membar) of short-K GEMMs.
__device__ __forceinline__ void mbar_arrive_remote_cta(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint32_t mapa_peer(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_shared_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// tcgen05.ld without the wait: several loads in flight, one tcgen05.wait::ld
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
        "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
        "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

__device__ __forceinline__ void oz_work(const OzGemmParams& p, int w, int& prod, int& slab, int& mod, int& t,
                                        int& tm, int& tn) {
  t = p.tile0 + w % p.ntiles;
  int r = w / p.ntiles;
  mod = r % p.n_mod;
  r /= p.n_mod;
  slab = r % p.nslab;
  prod = r / p.nslab;
  if (p.rect_gtiles > 0) {  // rectangular mode: (atom, column tile)
    tm = p.rect_atom0 + t / p.rect_gtiles;
    tn = t % p.rect_gtiles;
    return;
  }
  const int2 tt = p.tile_list[t];
  tm = tt.x;
  tn = tt.y;
}

template <bool WIDE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kOzThreads, 1)
    ozaki_gemm_kernel(const __grid_constant__ OzGemmParams p) {
  using G = OzG<WIDE>;
  constexpr int kOzStages = G::stages;
  constexpr int kOzStageBytes = G::stage_bytes;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bars = base + kOzStages * kOzStageBytes;
  auto full = [&](int s) { return bars + 8u * s; };
  auto empty = [&](int s) { return bars + 8u * (kOzStages + s); };
  auto tfull = [&](int s) { return bars + 8u * (2 * kOzStages + s); };
  auto tempty = [&](int s) { return bars + 8u * (2 * kOzStages + 2 + s); };
  const uint32_t tmem_slot = bars + 8u * (2 * kOzStages + 4);
  const uint32_t* tmem_slot_ptr = reinterpret_cast<const uint32_t*>(smem_raw + (tmem_slot - raw));
  // work queue: the leader's producer steals work items from a global counter
  // and hands each to every role of both CTAs through kOzQ smem slots
  constexpr int kOzQ = 4;
  auto wfull = [&](int j) { return bars + 8u * (2 * kOzStages + 5 + j); };
  auto wempty = [&](int j) { return bars + 8u * (2 * kOzStages + 5 + kOzQ + j); };
  auto wslot = [&](int j) { return bars + 8u * (2 * kOzStages + 5 + 2 * kOzQ) + 4u * j; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int nwork = kOzProds * p.nslab * p.n_mod * p.ntiles;
  // consumer side of the queue (every role except the leader's producer)
  auto take = [&](int seq) -> int {
    const int j = seq & (kOzQ - 1);
    mbar_wait_cluster(wfull(j), static_cast<uint32_t>((seq / kOzQ) & 1));
    const int w = static_cast<int>(ld_shared_u32(wslot(j)));
    // the slot is rewritten once every role has arrived, and an arrive does not
    // wait for a load still in flight: branch on the value first (never taken)
    // so the arrive cannot be scheduled ahead of the load's completion
    if (w < 0) __trap();
    __syncwarp();
    if (lane == 0) mbar_arrive_remote_cta(wempty(j) & kPeerMask);  // the leader's copy
    return w;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kOzStages; ++s) {
      mbar_init(full(s), 1);   // leader: its expect_tx covers both CTAs' bytes
      mbar_init(empty(s), 1);  // one multicast MMA commit per use
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tfull(s), 1);
      mbar_init(tempty(s), 2 * kOzEpiWarps);  // epilogue warps x 2 CTAs (leader's copy is used)
    }
    for (int j = 0; j < kOzQ; ++j) {
      mbar_init(wfull(j), 1);
      mbar_init(wempty(j), 2 + 2 * kOzEpiWarps);  // leader: MMA + epilogue warps; peer: producer + epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot_ptr;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    // the whole warp runs the loop (uniform control flow keeps the TMA
    // operands in uniform registers); one elected lane issues
    int stage = 0;
    uint32_t phase = 1;
    for (int seq = 0;; ++seq) {
      int w;
      if (leader) {
        const int j = seq & (kOzQ - 1);
        w = 0;
        const bool me = elect_one();
        if (me) {
          mbar_wait(wempty(j), static_cast<uint32_t>(((seq / kOzQ) & 1) ^ 1));
          w = atomicAdd(p.counter, 1);
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(wslot(j)), "r"(static_cast<uint32_t>(w)) : "memory");
          st_cluster_u32(mapa_peer(wslot(j), 1), static_cast<uint32_t>(w));
          mbar_arrive(wfull(j));
          mbar_arrive_cluster(mapa_peer(wfull(j), 1));
        }
        w = __shfl_sync(0xffffffffu, w, __ffs(__ballot_sync(0xffffffffu, me)) - 1);
      } else {
        w = take(seq);
      }
      if (w >= nwork) break;
      int prod, slab, mod, t, tm, tn;
      oz_work(p, w, prod, slab, mod, t, tm, tn);
      if (WIDE) {
        const int4 wt = p.wide_list[t];
        tm = wt.x;
        tn = wt.y;
      }
      // MMA A operand (TMEM lanes, the epilogue threads) = tile column tn,
      // B operand (TMEM columns) = tile row tm: each thread then holds 32
      // consecutive rows of one output column, stored as 32 contiguous bytes
      const int a0 = tn * 256 + static_cast<int>(rank) * kOzHalf;
      const int b0 = tm * 256 + static_cast<int>(rank) * kOzHalf;
      const int a_kofs = (tm * p.a_k_per_tm) & ~15;
      int seg = 0;
      for (int c = p.slab_chunk0[slab]; c < p.slab_chunk0[slab + 1]; ++c) {
        while (c >= p.seg_chunk0[seg + 1]) ++seg;
        const int kc = c - p.seg_chunk0[seg];
        mbar_wait(empty(stage), phase);
        if (elect_one()) {
          if (leader) mbar_expect_tx(full(stage), 2 * kOzStageBytes);
          const uint32_t dst = base + stage * kOzStageBytes;
          const uint32_t fb = full(stage) & kPeerMask;
          tma_load_3d_pair(dst, &p.map[prod][seg][0], kc * kOzBK + a_kofs, a0, mod, fb);
          tma_load_3d_pair(dst + kOzABytes, &p.map[prod][seg][1], kc * kOzBK, b0, mod, fb);
          if (WIDE)  // the second row tile (rows past the matrix read as zeros)
            tma_load_3d_pair(dst + 2 * kOzABytes, &p.map[prod][seg][1], kc * kOzBK, b0 + 256, mod, fb);
        }
        __syncwarp();
        if (++stage == kOzStages) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 1;
      // descriptors of stage 0; a stage is kOzStageBytes further, a 32-byte k step +2
      const uint64_t da0 = sw128_desc(base), db0 = sw128_desc(base + kOzABytes),
                     db1 = sw128_desc(base + 2 * kOzABytes);
      for (int seq = 0;; ++seq) {
        const int w = take(seq);
        if (w >= nwork) break;
        mbar_wait(tempty(acc), acc_phase);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + acc * kOzBN;  // WIDE: acc stays 0, the second accumulator is d + 256
        uint32_t accum = 0;
        const int slab = (w / p.ntiles / p.n_mod) % p.nslab;
        int seg = 0;
        for (int c = p.slab_chunk0[slab]; c < p.slab_chunk0[slab + 1]; ++c) {
          while (c >= p.seg_chunk0[seg + 1]) ++seg;
          // a segment's last chunk: skip the MMA k steps that only see zero padding
          const int ksteps = (c == p.seg_chunk0[seg + 1] - 1 && p.seg_ksteps_last[seg] > 0) ? p.seg_ksteps_last[seg]
                                                                                             : kOzBK / 32;
          mbar_wait(full(stage), phase);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          if (elect_one()) {
            const uint64_t so = static_cast<uint64_t>((stage * kOzStageBytes) >> 4);
#pragma unroll
            for (int kk = 0; kk < kOzBK / 32; ++kk) {
              if (kk < ksteps) {
                mma_i8_pair(d, da0 + so + 2 * kk, db0 + so + 2 * kk, accum | kk);
                if (WIDE) mma_i8_pair(d + kOzBN, da0 + so + 2 * kk, db1 + so + 2 * kk, accum | kk);
              }
            }
            mma_commit_pair(empty(stage));
          }
          __syncwarp();
          accum = 1;
          if (++stage == kOzStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        if (elect_one()) mma_commit_pair(tfull(acc));
        __syncwarp();
        if (WIDE) {
          acc_phase ^= 1u;
        } else if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1u;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    // warp w owns TMEM lanes 32*(w%4) .. +31 = rows of this CTA's half; residue mod p, int8
    const int q = warp & 3;                        // TMEM lane quarter (warp id mod 4)
    const int part = (warp - 2) / 4;               // columns [part, part + 1) * kOzBN / kOzEpiParts
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int seq = 0;; ++seq) {
      const int w = take(seq);
      if (w >= nwork) break;
      int prod, slab, mod, t, tm, tn;
      oz_work(p, w, prod, slab, mod, t, tm, tn);
      int t0 = t, t1 = -1;
      if (WIDE) {
        const int4 wt = p.wide_list[t];
        tm = wt.x;
        tn = wt.y;
        t0 = wt.z;
        t1 = wt.w;
      }
      const int ip = oz_mod_rt[mod];
      const long long qm = ((1ll << 32) + ip / 2) / ip;  // rn(2^32 / p)
      const int c16 = ((65536 % ip) > ip / 2) ? (65536 % ip) - ip : (65536 % ip);
      mbar_wait(tfull(acc), acc_phase);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // thread = output column tn * 256 + cloc (TMEM lane); registers = rows
      const int cloc = static_cast<int>(rank) * kOzHalf + q * 32 + lane;
      const bool col_ok = tn * 256 + cloc < p.n;
      constexpr int kChunks = kOzBN / 32 / kOzEpiParts;  // 32-column TMEM loads per warp
      uint32_t vv[kChunks][32];
      // drain this warp's columns of one accumulator into registers
      auto drain = [&](int acc_cols, int row_tile) {
        const int nrow = min(kOzBN, p.nrows - row_tile * 256);
#pragma unroll
        for (int cc = 0; cc < kChunks; ++cc)
          if ((part * kChunks + cc) * 32 < nrow)  // warp-uniform
            tmem_ld32_issue(tmem + ((q * 32) << 16) + acc_cols + (part * kChunks + cc) * 32, vv[cc]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      };
      // hand the TMEM buffer back to the MMA issuer (before the reduction and
      // the stores: with short reductions the MMA otherwise waits for the
      // whole epilogue of the item two back)
      auto release = [&]() {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_remote_cta(tempty(acc) & kPeerMask);
      };
      // residues mod p of the drained columns into residue tile `tile` (slab
      // s > 0: added to slab s - 1's in place, once that slab's warps are done)
      auto store = [&](int tile, int row_tile) {
        const int nrow = min(kOzBN, p.nrows - row_tile * 256);
        int8_t* out = p.res + prod * p.prod_stride + mod * p.mod_stride + static_cast<int64_t>(tile) * kOzTileBytes +
                      cloc * 256;
        int32_t* cnt = p.nslab > 1 ? p.slab_cnt + (static_cast<int64_t>(prod) * p.n_mod + mod) * p.tiles_total + tile
                                   : nullptr;
        if (slab > 0) {  // slab s-1 of this tile: all epilogue warps of both CTAs finished
          if (lane == 0)
            while (*reinterpret_cast<volatile int32_t*>(cnt) < 2 * kOzEpiWarps * slab) __nanosleep(256);
          __syncwarp();
          __threadfence();
        }
#pragma unroll
        for (int cc = 0; cc < kChunks; ++cc) {
          const int c = part * kChunks + cc;
          if (c * 32 >= nrow) break;  // warp-uniform
          const uint32_t (&v)[32] = vv[cc];
          if (col_ok) {
            uint32_t w8[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              int r4[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) r4[i] = sym_mod_i32q(static_cast<int32_t>(v[4 * j + i]), ip, c16, qm);
              w8[j] = __byte_perm(__byte_perm(r4[0], r4[1], 0x40), __byte_perm(r4[2], r4[3], 0x40), 0x5410);
            }
            uint4* o = reinterpret_cast<uint4*>(out + c * 32);
            if (slab > 0) {  // the residue of the sum of the slabs
              const uint4 o0 = __ldcg(o), o1 = __ldcg(o + 1);
              const uint32_t ow[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                uint32_t x = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const int a = static_cast<int8_t>(w8[j] >> (8 * i)), b = static_cast<int8_t>(ow[j] >> (8 * i));
                  x |= (static_cast<uint32_t>(sym_adj(a + b, ip)) & 0xffu) << (8 * i);
                }
                w8[j] = x;
              }
            }
            // one 256-bit store: the thread's 32 rows are one full 32-byte sector
            // (two 128-bit stores queued twice the requests, each half a sector)
            asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(o), "r"(w8[0]),
                         "r"(w8[1]), "r"(w8[2]), "r"(w8[3]), "r"(w8[4]), "r"(w8[5]), "r"(w8[6]), "r"(w8[7])
                         : "memory");
          }
        }
        if (cnt) {
          __threadfence();
          __syncwarp();
          if (lane == 0) atomicAdd(cnt, 1);
        }
      };
      drain(acc * kOzBN, tm);
      if (!WIDE || t1 < 0) {
        release();
        store(t0, tm);
      } else {  // the second accumulator (row tile tm + 1) after the first is stored
        store(t0, tm);
        drain(kOzBN, tm + 1);
        release();
        store(t1, tm + 1);
      }
      if (WIDE) {
        acc_phase ^= 1u;
      } else if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ------------------------------------------------------------ 4. CRT
// Explicit CRT as a fraction.  With M = prod p_i and residues X = c_i r_i
// (mod p_i) for representatives |r_i| <= p_i - 1 and unit constants c_i (1/2
// for Re = (phi1 + phi2)/2, 1/(2 j_i) for Im = (phi1 - phi2)/(2 j_i)),
//     X / M = sum_i r_i u_i / p_i  (mod 1),   u_i = c_i (M/p_i)^-1 mod p_i,
// and |X| <= M/4 (the host's choice of b), so X / M is the representative of
// that sum in [-1/4, 1/4].  Each weight u_i / p_i is held as two 40-bit
// fixed-point limbs w_i1 = c_i1 2^-40, w_i2 = c_i2 2^-80 (rounded at 2^-80):
//     s1 = sum_i r_i w_i1   exact (every term a multiple of 2^-40, |s1| 2^40 <
//                           20 * 240 * 2^40 < 2^53),
//     s2 = sum_i r_i w_i2   (|s2| < 2^-27, rounded at 2^-106),
//     f  = (s1 - rn(s1)) + s2,   X = f * M.
// s1 - rn(s1) is exact, rn(s1) is the right integer because X / M is within
// 1/4 + 2^-27 of it, and the truncated weights err by < 20 * 240 * 2^-80: f
// carries X / M to ~2^-53 relative, so X = f * fl(M) is within ~2 ulp.  The
// limb count does not grow with n_mod (the former integer-limb form needed
// 4 limbs above 13 moduli) and no quotient sum is needed.
struct OzCrtConst {
  double w[2][kOzMaxMod][2];  // [Re, Im][modulus] fixed-point limbs of u_i / p_i
  double m;                   // fl(M)
};
__constant__ OzCrtConst c_oz_crt[kOzMaxMod - kOzMinMod + 1];  // one table per n_mod = 11 .. 20

// exact int -> double through the mantissa (no I2F): a double with high
// word 0x43300000 and low word w is 2^52 + w
__device__ __forceinline__ double i2d_exact(int v) {
  return __hiloint2double(0x43300000, static_cast<int>(static_cast<unsigned>(v) ^ 0x80000000u)) -
         4503601774854144.0;  // 2^52 + 2^31
}

// v - 2^31 for a biased word v = x + 2^31 (|x| < 2^31), exactly
__device__ __forceinline__ double i2d_biased(unsigned v) {
  return __hiloint2double(0x43300000, static_cast<int>(v)) - 4503601774854144.0;  // 2^52 + 2^31
}

// X / M for the 2 Re / 2j Im residue sums of one element (PART 0 / 1)
template <int NM, int PART>
__device__ __forceinline__ double crt_frac(const int (&r)[NM]) {
  const OzCrtConst& C = c_oz_crt[NM - kOzMinMod];
  double s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int i = 0; i < NM; ++i) {
    const double ri = i2d_exact(r[i]);
    s1 = fma(ri, C.w[PART][i][0], s1);
    s2 = fma(ri, C.w[PART][i][1], s2);
  }
  return (s1 - rint(s1)) + s2;
}

// 2^sh in two exact power-of-two factors (|sh| <= 2044)
__device__ __forceinline__ double scale2(double x, int sh) { return (x * pow2i(sh / 2)) * pow2i(sh - sh / 2); }

// sign-extended byte e of w (one PRMT / SGXT)
__device__ __forceinline__ int sbyte(uint32_t w, int e) { return static_cast<int8_t>(w >> (8 * e)); }

// Finish one element from its X / M fractions (Re, Im): scale by
// 2^(e_m + e_n - 2b), alpha / beta, Im(diag) = 0
template <bool PLAIN>
__device__ __forceinline__ double2 crt_finish(const OzCrtParams& p, double fr, double fi, double mm, int sh, int m,
                                              int n) {
  const double xr = scale2(fr * mm, sh);
  const double xi = scale2(fi * mm, sh);
  if (PLAIN) return make_double2(xr, (m == n && (p.flags & (kMirror | kZeroImagDiag))) ? 0.0 : xi);
  double vr = p.alpha_re * xr - p.alpha_im * xi;
  double vi = p.alpha_re * xi + p.alpha_im * xr;
  if (p.beta_re != 0.0 || p.beta_im != 0.0) {
    const double2 o = reinterpret_cast<const double2*>(p.c)[m + static_cast<int64_t>(n) * p.ldc];
    vr += p.beta_re * o.x - p.beta_im * o.y;
    vi += p.beta_re * o.y + p.beta_im * o.x;
  }
  if (m == n && ((p.flags & kMirror) || (p.flags & kZeroImagDiag))) vi = 0.0;
  return make_double2(vr, vi);
}

// destination of element (m, n): C, or the owner's receive slot (peer output)
__device__ __forceinline__ double2* crt_dst(const OzCrtParams& p, int m, int n) {
  if (p.peer) {
    const int q = static_cast<int>(n / p.cpr);
    return p.peer[q] + ((p.rank * p.cpr + (n - q * p.cpr)) * p.pld + m);
  }
  return reinterpret_cast<double2*>(p.c) + (m + static_cast<int64_t>(n) * p.ldc);
}

// Lower-triangle elements (m >= n).  A block owns 8 output columns (one per
// warp) x one 128-row chunk (aligned to 128, so it lies in one 256 x 256
// residue tile).  The block's residues -- 2 products x NM moduli x 8 columns x
// 128 rows, 1 KB per (product, modulus) -- are fetched with 16-byte cp.async
// into shared memory (no registers held, every byte in flight at once: the
// register-load form was load-latency bound); lane l then reads rows
// 4l .. 4l+3 of its warp's column (conflict-free 32-bit words) and C[m, n] is
// stored from registers (a warp's four stores cover 2 KB contiguously).  The
// mirror C[n, m] = conj(C[m, n]) (matcore.hermitian_mirror, matcore.py:89-105)
// is transposed through the same shared memory so that each warp store writes
// four full 128-byte lines (8 consecutive rows n of 4 columns m).  Block row y
// handles the column-block pair (y, ncb - 1 - y), whose chunk counts add up to
// about the same for every y.
constexpr int kCrtCols = 8;      // columns per block (= warps)
constexpr int kCrtRows = 128;    // rows per block (= 32 lanes x 4)
__device__ __forceinline__ int crt_chunks(int n, int cs) { return (n - 1) / kCrtRows - cs / kCrtRows + 1; }
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// PLAIN: alpha = 1, beta = 0 (every build call): no scaling, no read of C
// 4 blocks per SM (64 registers) up to 18 moduli; 19-20 would spill at 64, so keep 3
template <int NM, bool PLAIN>
__global__ void __launch_bounds__(256, NM <= 18 ? 4 : 3) ozaki_crt_kernel(const OzCrtParams p, int ncols) {
  // residues [product][modulus][column][128 rows], then (reused) the mirror stage
  constexpr int kResBytes = 2 * NM * kCrtCols * kCrtRows;
  constexpr int kStageBytes = kCrtCols * (kCrtRows + 1) * 16;
  __shared__ __align__(16) uint8_t smem[kResBytes > kStageBytes ? kResBytes : kStageBytes];
  auto stage = reinterpret_cast<double2 (*)[kCrtRows + 1]>(smem);  // [n][position], +1: conflict-free reads
  const int ncb = (ncols + kCrtCols - 1) / kCrtCols;
  const int cba = static_cast<int>(blockIdx.y), cbb = ncb - 1 - cba;
  const int csa = p.n0 + cba * kCrtCols, csb = p.n0 + cbb * kCrtCols;  // first column = first useful row
  int chunk = static_cast<int>(blockIdx.x), cs;
  const int cha = crt_chunks(p.n, csa);
  if (chunk < cha) {
    cs = csa;
  } else {
    chunk -= cha;
    if (cbb == cba || chunk >= crt_chunks(p.n, csb)) return;
    cs = csb;
  }
  const int r0 = (cs / kCrtRows + chunk) * kCrtRows;  // first row of the block
  const int nend = min(p.n0 + ncols, p.n);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = cs + warp;                            // this warp's column
  const int m0 = r0 + 4 * lane;
  const bool mirror = (p.flags & kMirror) != 0;

  // 1. every residue byte of the block in flight at once
  {
    const int t = p.tile_index[(r0 >> 8) * p.T + (cs >> 8)];
    const uint8_t* base = reinterpret_cast<const uint8_t*>(p.res) + static_cast<int64_t>(t) * kOzTileBytes +
                          (cs & 255) * 256 + (r0 & 255);
    // plane q = (product, modulus) sits q * mod_stride further (prod_stride =
    // n_mod * mod_stride); thread = (16-byte piece, column, first plane)
    const int part = threadIdx.x & 7, col = (threadIdx.x >> 3) & 7, q0 = threadIdx.x >> 6;
    const uint8_t* src = base + q0 * p.mod_stride + col * 256 + part * 16;
    uint32_t dst = smem_u32(smem) + q0 * 1024 + col * 128 + part * 16;
    for (int q = q0; q < 2 * NM; q += 4, src += 4 * p.mod_stride, dst += 4096) cp_async16(dst, src);
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  const bool active = n < nend && m0 < p.n && m0 + 3 >= n;
  uint32_t w1[NM], w2[NM];
#pragma unroll
  for (int i = 0; i < NM; ++i) {
    w1[i] = *reinterpret_cast<const uint32_t*>(smem + i * 1024 + warp * 128 + 4 * lane);
    w2[i] = *reinterpret_cast<const uint32_t*>(smem + (NM + i) * 1024 + warp * 128 + 4 * lane);
  }
  __syncthreads();  // the residue area becomes the mirror stage
  if (active) {
    // the four rows' limb sums: modulus outer, so each weight (uniform, from
    // the constant bank) serves four elements
    const OzCrtConst& C = c_oz_crt[NM - kOzMinMod];
    double r1[4], r2[4], i1[4], i2[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) r1[e] = r2[e] = i1[e] = i2[e] = 0.0;
#pragma unroll
    for (int i = 0; i < NM; ++i) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        // f1 + f2 = 2 Re C, f1 - f2 = 2 j Im C (mod p_i), read through the mantissa
        const int f1 = sbyte(w1[i], e), f2 = sbyte(w2[i], e);
        const double re = i2d_biased(static_cast<unsigned>(f1 + f2) + 0x80000000u);
        const double im = i2d_biased(static_cast<unsigned>(f1 - f2) + 0x80000000u);
        r1[e] = fma(re, C.w[0][i][0], r1[e]);
        r2[e] = fma(re, C.w[0][i][1], r2[e]);
        i1[e] = fma(im, C.w[1][i][0], i1[e]);
        i2[e] = fma(im, C.w[1][i][1], i2[e]);
      }
    }
    const double mm = C.m;
    const int ern = __ldg(p.er + n) - 2 * p.b;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int m = m0 + e;
      if (m < n || m >= p.n) continue;
      const double fr = (r1[e] - rint(r1[e])) + r2[e], fi = (i1[e] - rint(i1[e])) + i2[e];
      const double2 v = crt_finish<PLAIN>(p, fr, fi, mm, __ldg(p.el + m) + ern, m, n);
      *crt_dst(p, m, n) = v;
      stage[warp][e * 32 + lane] = v;
    }
  }
  if (!mirror) return;
  __syncthreads();
  // transposed: thread (c = tid & 7, j = tid >> 3) writes C[cs + c, r0 + j + 32 q]
  const int c = threadIdx.x & 7, nn = cs + c;
  if (nn >= nend) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int jr = (threadIdx.x >> 3) + 32 * q, m = r0 + jr;  // row of the staged element
    if (m <= nn || m >= p.n) continue;
    const double2 v = stage[c][(jr & 3) * 32 + (jr >> 2)];
    *crt_dst(p, nn, m) = make_double2(v.x, -v.y);
  }
}

// ------------------------------------------------------------ 5. V products
// L1_a = [T_AA | T_AB], L2_a = [T_AB^H | T_BB], column-major 256 x 256 per atom:
// the nl rows sit at rows d_a .. d_a + nl - 1 with d_a = (nl a) mod 16 -- the
// TMA k coordinate of the right operand (the atom's rows of the stack) must be
// 16-byte aligned, so its box starts d_a rows early -- the rest is zero, as
// are columns 2 nl .. 255
__global__ void ozaki_vblocks_kernel(const double2* __restrict__ taa, const double2* __restrict__ tab,
                                     const double2* __restrict__ tbb, int nl, int64_t na, double2* __restrict__ l1,
                                     double2* __restrict__ l2) {
  const int64_t nn = static_cast<int64_t>(nl) * nl, per = 256 * 256;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < na * per;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t a = idx / per;
    const int rem = static_cast<int>(idx - a * per);
    const int k = (rem & 255) - static_cast<int>((a * nl) & 15), c = rem >> 8;
    const double2* AA = taa + a * nn;
    const double2* AB = tab + a * nn;
    const double2* BB = tbb + a * nn;
    auto herm = [&](const double2* T, int i, int j) {  // (i, j) of the Hermitian completion of the lower triangle
      if (i > j) return T[i + static_cast<int64_t>(j) * nl];
      if (i < j) {
        const double2 w = T[j + static_cast<int64_t>(i) * nl];
        return make_double2(w.x, -w.y);
      }
      return make_double2(T[i + static_cast<int64_t>(i) * nl].x, 0.0);
    };
    double2 v1 = make_double2(0.0, 0.0), v2 = v1;
    if (k < 0 || k >= nl) {
      // padding rows
    } else if (c < nl) {
      v1 = herm(AA, k, c);
      const double2 w = AB[c + static_cast<int64_t>(k) * nl];  // (T_AB^H)[k, c]
      v2 = make_double2(w.x, -w.y);
    } else if (c < 2 * nl) {
      v1 = AB[k + static_cast<int64_t>(c - nl) * nl];
      v2 = herm(BB, k, c - nl);
    }
    l1[idx] = v1;
    l2[idx] = v2;
  }
}

// [V1; V2] from the residues of one batch of (atom, column tile) products:
// block = 256 rows r of one tile x 32 of its columns; per column the block's
// max |Re| + |Im| goes into er (the right-hand exponents of H = A^H V1 + B^H V2)
template <int NM>
__global__ void __launch_bounds__(256) ozaki_vcrt_kernel(const OzVcrtParams p) {
  const int al = static_cast<int>(blockIdx.y), a = p.atom0 + al;
  const int gt = static_cast<int>(blockIdx.x) >> 3, gsub = static_cast<int>(blockIdx.x) & 7;
  const int t = al * p.gtiles + gt;
  const int r = static_cast<int>(threadIdx.x);
  const bool valid = r < 2 * p.nl;
  const int st = valid ? __ldg(p.et + static_cast<int64_t>(a) * 256 + r) : 0;
  const uint8_t* base = reinterpret_cast<const uint8_t*>(p.res) + static_cast<int64_t>(t) * kOzTileBytes + r;
  double2* dst = reinterpret_cast<double2*>(r < p.nl ? p.v1 : p.v2) +
                 (static_cast<int64_t>(p.nl) * a + (r < p.nl ? r : r - p.nl));
  __shared__ double wmax[8];
  for (int j = 0; j < 32; ++j) {
    const int gl = gsub * 32 + j, g = gt * 256 + gl;
    if (g >= p.ng) break;  // uniform across the block
    double m = 0.0;
    if (valid) {
      int F1[NM], F2[NM];
      const uint8_t* r0 = base + gl * 256;
#pragma unroll
      for (int i = 0; i < NM; ++i) {
        F1[i] = static_cast<int8_t>(__ldg(r0 + i * p.mod_stride));
        F2[i] = static_cast<int8_t>(__ldg(r0 + p.prod_stride + i * p.mod_stride));
      }
      int re[NM], im[NM];
#pragma unroll
      for (int i = 0; i < NM; ++i) {
        re[i] = F1[i] + F2[i];
        im[i] = F1[i] - F2[i];
      }
      const int sh = st + __ldg(p.el + g) - p.bsum;
      const double mm = c_oz_crt[NM - kOzMinMod].m;
      const double xr = scale2(crt_frac<NM, 0>(re) * mm, sh);
      const double xi = scale2(crt_frac<NM, 1>(im) * mm, sh);
      dst[static_cast<int64_t>(g) * p.ldv] = make_double2(xr, xi);
      m = fabs(xr) + fabs(xi);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((r & 31) == 0) wmax[r >> 5] = m;
    __syncthreads();
    if (r == 0) {
      double mm = wmax[0];
#pragma unroll
      for (int w = 1; w < 8; ++w) mm = fmax(mm, wmax[w]);
      int ex = 0;
      frexp(mm, &ex);
      atomicMax(p.er + g, ex);
    }
    __syncthreads();
  }
}

// CRT tables for every n_mod (ozaki_crt_kernel's fraction form): the weights
// u_i / p_i as two 40-bit fixed-point limbs, rounded to nearest at 2^-80, from
// exact integer arithmetic (u_i < 2^8, so u_i 2^80 fits 128 bits); fl(M) from
// the exact product in 32-bit digits.
static OzCrtConst oz_crt_table(int n_mod) {
  using u128 = unsigned __int128;
  OzCrtConst c;
  std::memset(&c, 0, sizeof(c));
  auto inverse = [](int a, int p) {
    a = ((a % p) + p) % p;
    for (int x = 1; x < p; ++x)
      if ((a * x) % p == 1) return x;
    return 0;
  };
  for (int i = 0; i < n_mod; ++i) {
    const int pi = oz_mod(i);
    int mi = 1;  // (M / p_i) mod p_i
    for (int j = 0; j < n_mod; ++j)
      if (j != i) mi = (mi * (oz_mod(j) % pi)) % pi;
    const int mi_inv = inverse(mi, pi);
    // Re: c = 1/2 ; Im: c = 1/(2 j)
    const int cpart[2] = {inverse(2, pi), inverse(2 * oz_sqrtm1(i), pi)};
    for (int part = 0; part < 2; ++part) {
      const u128 u = static_cast<u128>((cpart[part] * mi_inv) % pi);
      const u128 q = ((u << 80) + static_cast<u128>(pi / 2)) / static_cast<u128>(pi);  // rn(2^80 u / p)
      const u128 mask = (static_cast<u128>(1) << 40) - 1;
      c.w[part][i][0] = std::ldexp(static_cast<double>(static_cast<uint64_t>(q >> 40)), -40);
      c.w[part][i][1] = std::ldexp(static_cast<double>(static_cast<uint64_t>(q & mask)), -80);
    }
  }
  // M in base-2^32 digits, then rounded once: the top 64 bits (exact in a u64)
  // plus a sticky bit for the rest
  uint32_t dg[8] = {1, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < n_mod; ++i) {
    uint64_t carry = 0;
    for (int j = 0; j < 8; ++j) {
      const uint64_t v = static_cast<uint64_t>(dg[j]) * static_cast<uint64_t>(oz_mod(i)) + carry;
      dg[j] = static_cast<uint32_t>(v);
      carry = v >> 32;
    }
  }
  // bit length, then the top 64 significant bits and a sticky bit
  int nbits = 0;
  for (int j = 7; j >= 0; --j)
    if (dg[j]) {
      nbits = 32 * j + 32 - __builtin_clz(dg[j]);
      break;
    }
  auto bit = [&](int k) { return k >= 0 ? (dg[k >> 5] >> (k & 31)) & 1u : 0u; };
  const int lo = nbits > 64 ? nbits - 64 : 0;
  uint64_t hi = 0;
  for (int k = nbits - 1; k >= lo; --k) hi = (hi << 1) | bit(k);
  bool sticky = false;
  for (int k = 0; k < lo; ++k) sticky = sticky || bit(k);
  if (sticky) hi |= 1;  // below the 11 bits the conversion drops: only breaks exact ties
  c.m = std::ldexp(static_cast<double>(hi), lo);
  return c;
}

// host copy of the reconstruction table (diagnostic export, hsb_oz_crt_table)
int oz_crt_table_host(int n_mod, double* w, double* m) {
  if (n_mod < kOzMinMod || n_mod > kOzMaxMod) return 1;
  const OzCrtConst c = oz_crt_table(n_mod);
  for (int part = 0; part < 2; ++part)
    for (int i = 0; i < n_mod; ++i)
      for (int l = 0; l < 2; ++l) w[(part * n_mod + i) * 2 + l] = c.w[part][i][l];
  *m = c.m;
  return 0;
}

// Constants and kernel attributes are per device: upload / set them the first
// time each device is used (a process may drive several GPUs, _lib.context).
static cudaError_t oz_init_once() {
  static PerDeviceOnce once;
  return per_device_once(once, [] {
    static OzCrtConst t[kOzMaxMod - kOzMinMod + 1];
    static std::once_flag built;
    std::call_once(built, [] {
      for (int nm = kOzMinMod; nm <= kOzMaxMod; ++nm) t[nm - kOzMinMod] = oz_crt_table(nm);
    });
    cudaError_t status = cudaMemcpyToSymbol(c_oz_crt, t, sizeof(t));
    if (status == cudaSuccess)
      status = cudaFuncSetAttribute(ozaki_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    OzG<false>::smem);
    if (status == cudaSuccess)
      status = cudaFuncSetAttribute(ozaki_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    OzG<true>::smem);
    return status;
  });
}

// ------------------------------------------------------------ launchers
static int grid_cap(int64_t want, int cap) { return static_cast<int>(want < cap ? (want > 0 ? want : 1) : cap); }

cudaError_t launch_ozaki_init_exp(int32_t* e, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ozaki_init_exp_kernel<<<grid_cap((n + 255) / 256, 1024), 256, 0, st>>>(e, n);
  return cudaGetLastError();
}

cudaError_t launch_ozaki_colexp(const double* x, int64_t ldx, int64_t k, int64_t cols, int32_t* exp_out,
                                cudaStream_t st, const double* rscale) {
  if (cols <= 0 || k <= 0) return cudaSuccess;
  ozaki_colexp_kernel<<<grid_cap((cols + 7) / 8, 148 * 16), 256, 0, st>>>(reinterpret_cast<const double2*>(x), ldx,
                                                                          k, cols, exp_out, rscale);
  return cudaGetLastError();
}

cudaError_t launch_ozaki_colexp_ab(const double* a, const double* b, int64_t ld, int64_t k, int64_t cols,
                                   const double* u, int32_t* exp_out, cudaStream_t st, bool with_b) {
  if (cols <= 0 || k <= 0) return cudaSuccess;
  ozaki_colexp_ab_kernel<<<grid_cap((cols + 7) / 8, 148 * 16), 256, 0, st>>>(
      reinterpret_cast<const double2*>(a), reinterpret_cast<const double2*>(b), ld, k, cols, u, exp_out,
      with_b ? 1 : 0);
  return cudaGetLastError();
}

int64_t oz_kpad(int64_t k) {
  static const int64_t align = [] {
    const char* e = std::getenv("HSB_OZ_KPAD");
    const int64_t v = e ? std::atoll(e) : 128;
    return v >= 16 && v % 16 == 0 ? v : int64_t{128};
  }();
  return (k + align - 1) / align * align;
}

// the driver's cuTensorMapEncodeTiled (through the runtime: no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 oz_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

cudaError_t launch_ozaki_residues_batch(const OzResSrc* srcs, int nsrc, int64_t cols, int b, int n_mod,
                                        cudaStream_t st) {
  if (nsrc <= 0 || cols <= 0) return cudaSuccess;
  if (nsrc > kOzResMaxSrc || (cols + kOzResCols - 1) / kOzResCols > 65535) return cudaErrorInvalidValue;
  const PFN_cuTensorMapEncodeTiled_v12000 encode = oz_encode_fn();
  if (!encode) return cudaErrorNotSupported;
  OzResBatch p;
  std::memset(&p, 0, sizeof(p));
  p.cols = cols;
  p.b = b;
  int64_t kmax = 0;
  for (int i = 0; i < nsrc; ++i) {
    const int64_t kpad = srcs[i].kpad;
    if (kpad <= 0 || kpad % 16 != 0) return cudaErrorInvalidValue;
    // out[plane][modulus][col][kpad] as a 4-D uint8 tensor; box = one block's tile
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(kpad), static_cast<cuuint64_t>(cols),
                                static_cast<cuuint64_t>(n_mod), 2};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(kpad), static_cast<cuuint64_t>(kpad * cols),
                                   static_cast<cuuint64_t>(kpad * cols * n_mod)};
    const cuuint32_t box[4] = {kOzResKBlk, kOzResCols, static_cast<cuuint32_t>(n_mod), 2}, es[4] = {1, 1, 1, 1};
    if (encode(&p.map[i], CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, srcs[i].out, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
    p.src[i] = srcs[i];
    p.kpad[i] = kpad;
    kmax = std::max(kmax, kpad);
  }
  const dim3 grid(static_cast<unsigned>((kmax + kOzResKBlk * kOzResTiles - 1) / (kOzResKBlk * kOzResTiles)),
                  static_cast<unsigned>((cols + kOzResCols - 1) / kOzResCols), static_cast<unsigned>(nsrc));
  switch (n_mod) {
#define HSB_OZ_RES(NM) \
  case NM:             \
    ozaki_residue_kernel<NM><<<grid, 256, 0, st>>>(p); \
    break;
    HSB_OZ_RES(11) HSB_OZ_RES(12) HSB_OZ_RES(13) HSB_OZ_RES(14) HSB_OZ_RES(15) HSB_OZ_RES(16)
    HSB_OZ_RES(17) HSB_OZ_RES(18) HSB_OZ_RES(19) HSB_OZ_RES(20)
#undef HSB_OZ_RES
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_ozaki_residues(const double* x, int64_t ldx, int64_t k, int64_t cols, const int32_t* col_exp,
                                  int b, int n_mod, int8_t* out, int64_t kpad, cudaStream_t st, const double* rscale) {
  if (cols <= 0 || kpad <= 0) return cudaSuccess;
  const OzResSrc src{x, ldx, k, col_exp, rscale, out, kpad};
  return launch_ozaki_residues_batch(&src, 1, cols, b, n_mod, st);
}

cudaError_t launch_ozaki_gemm(const OzGemmParams& p, cudaStream_t st) {
  cudaError_t e = oz_init_once();
  if (e != cudaSuccess) return e;
  int dev = 0, n_sm = 0;
  cudaGetDevice(&dev);
  e = cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  const int64_t nwork = static_cast<int64_t>(kOzProds) * p.nslab * p.n_mod * p.ntiles;
  if (nwork <= 0) return cudaSuccess;
  if (nwork > 0x7fffffff) return cudaErrorInvalidConfiguration;
  const int pairs = static_cast<int>(nwork < n_sm / 2 ? nwork : n_sm / 2);
  const int grid = 2 * pairs;
  e = launch_fill_i32(p.counter, 1, 0, st);  // a kernel, not a copy-engine memset
  if (e != cudaSuccess) return e;
  if (p.wide_list)
    ozaki_gemm_kernel<true><<<grid, kOzThreads, OzG<true>::smem, st>>>(p);
  else
    ozaki_gemm_kernel<false><<<grid, kOzThreads, OzG<false>::smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_ozaki_vblocks(const double* taa, const double* tab, const double* tbb, int nl, int64_t na,
                                 double* l1, double* l2, cudaStream_t st) {
  const int64_t total = na * 256 * 256;
  if (total <= 0) return cudaSuccess;
  ozaki_vblocks_kernel<<<grid_cap((total + 255) / 256, 148 * 16), 256, 0, st>>>(
      reinterpret_cast<const double2*>(taa), reinterpret_cast<const double2*>(tab),
      reinterpret_cast<const double2*>(tbb), nl, na, reinterpret_cast<double2*>(l1), reinterpret_cast<double2*>(l2));
  return cudaGetLastError();
}

cudaError_t launch_ozaki_vcrt(const OzVcrtParams& p, cudaStream_t st) {
  if (p.natoms <= 0 || p.ng <= 0) return cudaSuccess;
  cudaError_t ce = oz_init_once();
  if (ce != cudaSuccess) return ce;
  const dim3 grid(static_cast<unsigned>(p.gtiles * 8), static_cast<unsigned>(p.natoms)), block(256);
  switch (p.n_mod) {
#define HSB_OZ_VCRT(NMV)                                  \
  case NMV:                                             \
    ozaki_vcrt_kernel<NMV><<<grid, block, 0, st>>>(p);  \
    break;
    HSB_OZ_VCRT(11) HSB_OZ_VCRT(12) HSB_OZ_VCRT(13) HSB_OZ_VCRT(14) HSB_OZ_VCRT(15) HSB_OZ_VCRT(16)
    HSB_OZ_VCRT(17) HSB_OZ_VCRT(18) HSB_OZ_VCRT(19) HSB_OZ_VCRT(20)
#undef HSB_OZ_VCRT
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_ozaki_crt(const OzCrtParams& p, cudaStream_t st) {
  if (p.n <= 0) return cudaSuccess;
  cudaError_t ce = oz_init_once();
  if (ce != cudaSuccess) return ce;
  const int64_t ncols = p.n - p.n0;  // columns n0 .. n-1 unless the caller shrinks gridDim.y
  return launch_ozaki_crt_cols(p, ncols, st);
}

// 4 blocks of 35 KB per SM need the largest shared-memory carveout (the
// default the driver picks for this kernel holds 3)
template <int NM, bool PLAIN>
static cudaError_t crt_launch(dim3 grid, dim3 block, cudaStream_t st, const OzCrtParams& p, int nc) {
  static PerDeviceOnce attr;
  const cudaError_t e = per_device_once(attr, [] {
    return cudaFuncSetAttribute(ozaki_crt_kernel<NM, PLAIN>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                cudaSharedmemCarveoutMaxShared);
  });
  if (e != cudaSuccess) return e;
  ozaki_crt_kernel<NM, PLAIN><<<grid, block, 0, st>>>(p, nc);
  return cudaSuccess;
}

cudaError_t launch_ozaki_crt_cols(const OzCrtParams& p, int64_t ncols, cudaStream_t st) {
  if (ncols <= 0) return cudaSuccess;
  cudaError_t ce = oz_init_once();
  if (ce != cudaSuccess) return ce;
  if (p.n0 % kCrtCols != 0) return cudaErrorInvalidValue;  // column blocks stay inside a tile
  if (p.prod_stride != p.mod_stride * p.n_mod) return cudaErrorInvalidValue;  // planes evenly spaced
  // column-block pairs (y, ncb - 1 - y): 128-aligned row chunks from each
  // block's diagonal down to row n
  const int64_t ncb = (ncols + kCrtCols - 1) / kCrtCols;
  if ((ncb + 1) / 2 > 65535) return cudaErrorInvalidConfiguration;
  auto chunks = [&](int64_t cb) {
    const int64_t cs = p.n0 + cb * kCrtCols;
    return (p.n - 1) / kCrtRows - cs / kCrtRows + 1;
  };
  int64_t most = 0;
  for (int64_t y = 0; y < (ncb + 1) / 2; ++y) {
    const int64_t yb = ncb - 1 - y;
    most = std::max(most, chunks(y) + (yb == y ? 0 : chunks(yb)));
  }
  const dim3 grid(static_cast<unsigned>(most), static_cast<unsigned>((ncb + 1) / 2)), block(256);
  const int nc = static_cast<int>(ncols);
  const bool plain = p.alpha_re == 1.0 && p.alpha_im == 0.0 && p.beta_re == 0.0 && p.beta_im == 0.0;
#define HSB_OZ_CRT(NMV)                                                   \
  case NMV: {                                                           \
    const cudaError_t e = plain ? crt_launch<NMV, true>(grid, block, st, p, nc) \
                                : crt_launch<NMV, false>(grid, block, st, p, nc); \
    if (e != cudaSuccess) return e;                                     \
    break;                                                              \
  }
  switch (p.n_mod) {
    HSB_OZ_CRT(11)
    HSB_OZ_CRT(12)
    HSB_OZ_CRT(13)
    HSB_OZ_CRT(14)
    HSB_OZ_CRT(15)
    HSB_OZ_CRT(16)
    HSB_OZ_CRT(17)
    HSB_OZ_CRT(18)
    HSB_OZ_CRT(19)
    HSB_OZ_CRT(20)
    default: return cudaErrorInvalidValue;
  }
#undef HSB_OZ_CRT
  return cudaGetLastError();
}

}  // namespace hsb
