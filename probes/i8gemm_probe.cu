// i8gemm_probe.cu — standalone check of a tcgen05 kind::i8 GEMM on sm_100a:
// C (int32, M x N) = L^T R with L (K x M) and R (K x N) int8, K contiguous.
// Persistent, 1 CTA per SM: warp 0 TMA, warp 1 MMA issuer (+ TMEM owner),
// warps 2-5 epilogue (TMEM -> registers -> global).  Validates against a
// naive GPU kernel and times a large case.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -o probes/i8gemm_probe probes/i8gemm_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e = (x);                                                                \
    if (e != cudaSuccess) {                                                             \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      std::exit(1);                                                                     \
    }                                                                                   \
  } while (0)

constexpr int BM = 128, BN = 256, BK = 128, STAGES = 4;
constexpr int A_BYTES = BM * BK, B_BYTES = BN * BK, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
constexpr int THREADS = 192;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
// K-major, 128B-swizzled operand tile: 8-row atoms of 1024 B (SBO), LBO unused
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}
constexpr uint32_t kIdesc = (2u << 4)          // D: s32
                            | (1u << 7)        // A: signed int8
                            | (1u << 10)       // B: signed int8
                            | ((BN >> 3) << 17)  // N
                            | ((BM >> 4) << 24);  // M
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(THREADS, 1)
    i8gemm_kernel(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, int32_t* C,
                  int64_t ldc, int M, int N, int K) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bars = base + STAGES * STAGE_BYTES;
  auto full = [&](int s) { return bars + 8u * s; };
  auto empty = [&](int s) { return bars + 8u * (STAGES + s); };
  auto tfull = [&](int s) { return bars + 8u * (2 * STAGES + s); };
  auto tempty = [&](int s) { return bars + 8u * (2 * STAGES + 2 + s); };
  const uint32_t tmem_slot = bars + 8u * (2 * STAGES + 4);
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(smem_raw + (tmem_slot - raw));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN, ntiles = tiles_m * tiles_n;
  const int kchunks = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tfull(s), 1);
      mbar_init(tempty(s), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot_ptr;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 1;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int tm = t % tiles_m, tn = t / tiles_m;
        for (int kc = 0; kc < kchunks; ++kc) {
          mbar_wait(empty(stage), phase);
          mbar_expect_tx(full(stage), STAGE_BYTES);
          const uint32_t dst = base + stage * STAGE_BYTES;
          tma_load_2d(dst, &ma, kc * BK, tm * BM, full(stage));
          tma_load_2d(dst + A_BYTES, &mb, kc * BK, tn * BN, full(stage));
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 1;  // fresh tmem_empty barriers read as released
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        mbar_wait(tempty(acc), acc_phase);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + acc * BN;
        for (int kc = 0; kc < kchunks; ++kc) {
          mbar_wait(full(stage), phase);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a0 = base + stage * STAGE_BYTES, b0 = a0 + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 32; ++kk)
            mma_i8(d, sw128_desc(a0 + kk * 32), sw128_desc(b0 + kk * 32), (kc | kk) ? 1u : 0u);
          mma_commit(empty(stage));
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
        mma_commit(tfull(acc));
        if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
      }
    }
  } else {
    // epilogue: warp w reads TMEM lanes 32*(w%4) .. +31
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int tm = t % tiles_m, tn = t / tiles_m;
      mbar_wait(tfull(acc), acc_phase);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = tm * BM + q * 32 + lane;
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + ((q * 32) << 16) + acc * BN + c * 32, v);
        if (row < M) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int col = tn * BN + c * 32 + j;
            if (col < N) C[row + col * ldc] = static_cast<int32_t>(v[j]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty(acc));
      if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

__global__ void ref_kernel(const int8_t* L, const int8_t* R, int64_t ld, int32_t* C, int64_t ldc, int M, int N, int K) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x, n = blockIdx.y;
  if (m >= M) return;
  int32_t s = 0;
  for (int k = 0; k < K; ++k) s += int32_t(L[k + m * ld]) * int32_t(R[k + n * ld]);
  C[m + n * ldc] = s;
}

__global__ void fill_kernel(int8_t* p, int64_t n, uint32_t seed) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    uint32_t x = uint32_t(i) * 2654435761u ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = static_cast<int8_t>(x & 0xff);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode;
static CUtensorMap make_map(const void* base, int64_t k, int64_t rows, int64_t ld, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cuuint64_t(k), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld)};
  cuuint32_t box[2] = {BK, cuuint32_t(box_rows)}, es[2] = {1, 1};
  CUresult r = g_encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { std::fprintf(stderr, "encode failed %d\n", int(r)); std::exit(1); }
  return m;
}

static double run(int M, int N, int K, bool check, int reps) {
  const int64_t ld = (K + 15) / 16 * 16;
  int8_t *L, *R;
  int32_t *C, *C2;
  CK(cudaMalloc(&L, ld * M));
  CK(cudaMalloc(&R, ld * N));
  CK(cudaMalloc(&C, int64_t(M) * N * 4));
  fill_kernel<<<1024, 256>>>(L, ld * M, 1234u);
  fill_kernel<<<1024, 256>>>(R, ld * N, 777u);
  CK(cudaMemset(C, 0, int64_t(M) * N * 4));
  CUtensorMap ma = make_map(L, K, M, ld, BM), mb = make_map(R, K, N, ld, BN);
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int ntiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int grid = ntiles < nsm ? ntiles : nsm;
  CK(cudaFuncSetAttribute(i8gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  i8gemm_kernel<<<grid, THREADS, SMEM>>>(ma, mb, C, M, M, N, K);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  double ms_best = 0;
  if (check) {
    CK(cudaMalloc(&C2, int64_t(M) * N * 4));
    ref_kernel<<<dim3((M + 127) / 128, N), 128>>>(L, R, ld, C2, M, M, N, K);
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> h1(int64_t(M) * N), h2(int64_t(M) * N);
    CK(cudaMemcpy(h1.data(), C, h1.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2.data(), C2, h2.size() * 4, cudaMemcpyDeviceToHost));
    int64_t bad = 0, first = -1;
    for (size_t i = 0; i < h1.size(); ++i)
      if (h1[i] != h2[i]) { if (first < 0) first = i; ++bad; }
    std::printf("check M=%d N=%d K=%d: %lld mismatches", M, N, K, (long long)bad);
    if (first >= 0) std::printf(" (first at row %lld col %lld: got %d want %d)", first % M, first / M, h1[first], h2[first]);
    std::printf("\n");
    CK(cudaFree(C2));
  }
  if (reps > 0) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int r = 0; r < reps; ++r) {
      cudaEventRecord(e0);
      i8gemm_kernel<<<grid, THREADS, SMEM>>>(ma, mb, C, M, M, N, K);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r == 0 || ms < ms_best) ms_best = ms;
    }
    const double ops = 2.0 * M * N * double(K);
    std::printf("time M=%d N=%d K=%d: %.3f ms  %.1f TOPS\n", M, N, K, ms_best, ops / ms_best / 1e9);
  }
  CK(cudaFree(L));
  CK(cudaFree(R));
  CK(cudaFree(C));
  return ms_best;
}

int main() {
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q));
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  run(128, 256, 128, true, 0);
  run(256, 512, 384, true, 0);
  run(1000, 700, 1000, true, 0);
  run(2048, 2048, 4096, true, 0);
  run(8192, 8192, 11616, false, 5);
  run(16384, 16384, 11616, false, 3);
  return 0;
}
