// staging.cu — pinned-slot transfer engine (see staging.cuh).
#include <omp.h>
#include <string.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <deque>

#include "staging.cuh"

namespace hsb {

bool host_is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Leave a couple of cores to the driver / interpreter threads: a copy thread
// that gets descheduled stalls the whole chunk at the barrier.
static int copy_threads() { return std::max(1, std::min(12, omp_get_max_threads() - 2)); }

void parallel_memcpy(void* dst, const void* src, size_t bytes) {
  const size_t min_piece = size_t(1) << 20;
  int nt = static_cast<int>(std::min<size_t>(copy_threads(), std::max<size_t>(1, bytes / min_piece)));
  if (nt <= 1) {
    memcpy(dst, src, bytes);
    return;
  }
  const size_t piece = (bytes + nt - 1) / nt;
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int i = 0; i < nt; ++i) {
    const size_t off = static_cast<size_t>(i) * piece;
    if (off < bytes) memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, std::min(piece, bytes - off));
  }
}

void parallel_memcpy_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows) {
  if (dpitch == width && spitch == width) {
    parallel_memcpy(dst, src, width * rows);
    return;
  }
  const int nt = (width * rows >= (size_t(4) << 20)) ? copy_threads() : 1;
#pragma omp parallel for num_threads(nt) schedule(static)
  for (long long r = 0; r < static_cast<long long>(rows); ++r)
    memcpy(static_cast<char*>(dst) + r * dpitch, static_cast<const char*>(src) + r * spitch, width);
}

Stager::~Stager() {
  for (int i = 0; i < kSlots; ++i) {
    if (ev_[i]) cudaEventDestroy(ev_[i]);
    if (slot_[i]) cudaFreeHost(slot_[i]);
  }
}

cudaError_t Stager::ensure() {
  if (ready_) return cudaSuccess;
  for (int i = 0; i < kSlots; ++i) {
    cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&slot_[i]), kSlotBytes);
    if (e != cudaSuccess) return e;
    e = cudaEventCreateWithFlags(&ev_[i], cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  ready_ = true;
  return cudaSuccess;
}

namespace {
struct Chunk {
  const Copy2D* job;
  size_t row0, rows;
};
std::vector<Chunk> chunk_jobs(const std::vector<Copy2D>& jobs, size_t slot_bytes) {
  std::vector<Chunk> out;
  for (const Copy2D& j : jobs) {
    if (j.width == 0 || j.height == 0) continue;
    const size_t per = std::max<size_t>(1, slot_bytes / j.width);
    for (size_t r = 0; r < j.height; r += per) out.push_back({&j, r, std::min(per, j.height - r)});
  }
  return out;
}
}  // namespace

cudaError_t Stager::h2d(const std::vector<Copy2D>& jobs, cudaStream_t st) {
  std::vector<Copy2D> staged;
  for (const Copy2D& j : jobs) {
    if (j.width == 0 || j.height == 0) continue;
    if (host_is_pinned(j.src)) {
      cudaError_t e = cudaMemcpy2DAsync(j.dst, j.dpitch, j.src, j.spitch, j.width, j.height, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return e;
    } else {
      staged.push_back(j);
    }
  }
  if (staged.empty()) return cudaSuccess;
  cudaError_t e = ensure();
  if (e != cudaSuccess) return e;
  for (int i = 0; i < kSlots; ++i) {  // slots may still feed a previous call's DMA
    e = cudaEventSynchronize(ev_[i]);
    if (e != cudaSuccess) return e;
  }
  int slot = 0;
  int used = 0;
  for (const Chunk& c : chunk_jobs(staged, kSlotBytes)) {
    if (used >= kSlots) {
      e = cudaEventSynchronize(ev_[slot]);
      if (e != cudaSuccess) return e;
    }
    const Copy2D& j = *c.job;
    parallel_memcpy_2d(slot_[slot], j.width, static_cast<const char*>(j.src) + c.row0 * j.spitch, j.spitch, j.width,
                       c.rows);
    e = cudaMemcpy2DAsync(static_cast<char*>(j.dst) + c.row0 * j.dpitch, j.dpitch, slot_[slot], j.width, j.width,
                          c.rows, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    e = cudaEventRecord(ev_[slot], st);
    if (e != cudaSuccess) return e;
    slot = (slot + 1) % kSlots;
    ++used;
  }
  return cudaSuccess;
}

cudaError_t Stager::d2h(const std::vector<Copy2D>& jobs, cudaStream_t st) {
  std::vector<Copy2D> staged;
  for (const Copy2D& j : jobs) {
    if (j.width == 0 || j.height == 0) continue;
    if (host_is_pinned(j.dst)) {
      cudaError_t e = cudaMemcpy2DAsync(j.dst, j.dpitch, j.src, j.spitch, j.width, j.height, cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return e;
    } else {
      staged.push_back(j);
    }
  }
  if (staged.empty()) return cudaSuccess;
  cudaError_t e = ensure();
  if (e != cudaSuccess) return e;
  for (int i = 0; i < kSlots; ++i) {
    e = cudaEventSynchronize(ev_[i]);
    if (e != cudaSuccess) return e;
  }
  std::deque<std::pair<Chunk, int>> inflight;
  auto drain_one = [&]() -> cudaError_t {
    auto [c, s] = inflight.front();
    inflight.pop_front();
    cudaError_t err = cudaEventSynchronize(ev_[s]);
    if (err != cudaSuccess) return err;
    const Copy2D& j = *c.job;
    parallel_memcpy_2d(static_cast<char*>(j.dst) + c.row0 * j.dpitch, j.dpitch, slot_[s], j.width, j.width, c.rows);
    return cudaSuccess;
  };
  int slot = 0;
  for (const Chunk& c : chunk_jobs(staged, kSlotBytes)) {
    if (static_cast<int>(inflight.size()) == kSlots) {
      e = drain_one();
      if (e != cudaSuccess) return e;
    }
    const Copy2D& j = *c.job;
    e = cudaMemcpy2DAsync(slot_[slot], j.width, static_cast<const char*>(j.src) + c.row0 * j.spitch, j.spitch, j.width,
                          c.rows, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return e;
    e = cudaEventRecord(ev_[slot], st);
    if (e != cudaSuccess) return e;
    inflight.push_back({c, slot});
    slot = (slot + 1) % kSlots;
  }
  while (!inflight.empty()) {
    e = drain_one();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// true if any of the n doubles is NaN or +-Inf (exponent field all ones)
static inline bool any_nonfinite(const double* v, size_t n) {
  const uint64_t* b = reinterpret_cast<const uint64_t*>(v);
  uint64_t acc = 0;
  for (size_t i = 0; i < n; ++i) acc |= ((b[i] & 0x7ff0000000000000ull) == 0x7ff0000000000000ull);
  return acc != 0;
}

cudaError_t Stager::h2d_stack(double* dst, const double* const* blocks, int64_t n_atoms, int64_t rows,
                              int64_t cols, cudaStream_t st, int64_t* bad_block) {
  *bad_block = -1;
  if (n_atoms <= 0 || rows <= 0 || cols <= 0) return cudaSuccess;
  cudaError_t e = ensure();
  if (e != cudaSuccess) return e;
  for (int i = 0; i < kSlots; ++i) {
    e = cudaEventSynchronize(ev_[i]);
    if (e != cudaSuccess) return e;
  }
  const size_t col_bytes = static_cast<size_t>(n_atoms) * rows * 16;  // one stacked column
  if (col_bytes > kSlotBytes) {  // very tall stacks: per-atom 2-D copies, host-side finiteness scan
    std::vector<Copy2D> jobs;
    for (int64_t a = 0; a < n_atoms; ++a) {
      if (*bad_block < 0 && any_nonfinite(blocks[a], static_cast<size_t>(2 * rows * cols))) *bad_block = a;
      jobs.push_back({dst + 2 * a * rows, col_bytes, blocks[a], static_cast<size_t>(rows) * 16,
                      static_cast<size_t>(rows) * 16, static_cast<size_t>(cols)});
    }
    return h2d(jobs, st);
  }
  const int64_t per = std::max<int64_t>(1, static_cast<int64_t>(kSlotBytes / col_bytes));
  const size_t piece = static_cast<size_t>(rows) * 16;
  int64_t bad = INT64_MAX;
  int slot = 0, used = 0;
  const int nt = copy_threads();
  for (int64_t g0 = 0; g0 < cols; g0 += per) {
    const int64_t nc = std::min(per, cols - g0);
    if (used >= kSlots) {
      e = cudaEventSynchronize(ev_[slot]);
      if (e != cudaSuccess) return e;
    }
    char* base = slot_[slot];
    int64_t chunk_bad = INT64_MAX;
    // (column, atom) pieces of `rows` complex values each
#pragma omp parallel for num_threads(nt) schedule(dynamic, 16) reduction(min : chunk_bad)
    for (int64_t idx = 0; idx < nc * n_atoms; ++idx) {
      const int64_t g = idx / n_atoms, a = idx % n_atoms;
      const double* src = blocks[a] + 2 * (g0 + g) * rows;
      memcpy(base + g * col_bytes + a * piece, src, piece);
      if (any_nonfinite(src, 2 * rows) && a < chunk_bad) chunk_bad = a;
    }
    bad = std::min(bad, chunk_bad);
    e = cudaMemcpyAsync(reinterpret_cast<char*>(dst) + g0 * col_bytes, base, nc * col_bytes,
                        cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    e = cudaEventRecord(ev_[slot], st);
    if (e != cudaSuccess) return e;
    slot = (slot + 1) % kSlots;
    ++used;
  }
  if (bad != INT64_MAX) *bad_block = bad;
  return cudaSuccess;
}

}  // namespace hsb
