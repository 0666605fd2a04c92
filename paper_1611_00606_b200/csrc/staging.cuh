// staging.cuh — host <-> device transfer engine of the drop-in (host-buffer) path.
//
// The reference's inputs and outputs are ordinary (pageable) numpy arrays
// (probgen.py:78-92, builder.py:221-224).  DMA from pageable memory is slow
// and synchronous, so transfers go through a ring of pinned slots: host
// threads (OpenMP) copy a chunk into a slot while the copy engine moves the
// previous slot, and pinned user buffers skip the bounce entirely.  This is
// the B200 counterpart of the paper's "memory must be pinned" advice for
// cuBLAS-XT.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <vector>

namespace hsb {

struct Copy2D {
  void* dst;        // device (h2d) or host (d2h)
  size_t dpitch;    // bytes between rows of dst
  const void* src;  // host (h2d) or device (d2h)
  size_t spitch;
  size_t width;     // bytes per row
  size_t height;    // rows
};

bool host_is_pinned(const void* p);

class Stager {
 public:
  Stager() = default;
  ~Stager();
  Stager(const Stager&) = delete;
  Stager& operator=(const Stager&) = delete;

  // Enqueue host -> device copies on `st`.  Returns once every pageable
  // source byte has been copied into pinned slots (the DMAs may still be in
  // flight); pinned sources are DMA'd directly.
  cudaError_t h2d(const std::vector<Copy2D>& jobs, cudaStream_t st);
  // Device -> host copies ordered after prior work on `st`.  Pinned
  // destinations: enqueued only (caller synchronises `st`).  Pageable
  // destinations: staged through the slots; returns when the bytes are in place.
  cudaError_t d2h(const std::vector<Copy2D>& jobs, cudaStream_t st);
  // Upload n_atoms per-atom column-major blocks (rows x cols complex128 each,
  // contiguous) into the stacked (n_atoms*rows) x cols device matrix
  // (matcore.stack, matcore.py:68-86): host threads gather whole stacked
  // columns into a pinned slot, one contiguous DMA per slot.  While copying
  // they test every value for finiteness; *bad_block receives the first
  // block index holding a NaN/Inf, or -1.
  cudaError_t h2d_stack(double* dst, const double* const* blocks, int64_t n_atoms, int64_t rows, int64_t cols,
                        cudaStream_t st, int64_t* bad_block);

  static constexpr int kSlots = 4;
  static constexpr size_t kSlotBytes = size_t(32) << 20;

 private:
  cudaError_t ensure();
  char* slot_[kSlots] = {};
  cudaEvent_t ev_[kSlots] = {};
  bool ready_ = false;
};

// memcpy split over host threads (OpenMP), for multi-MB copies.
void parallel_memcpy(void* dst, const void* src, size_t bytes);
void parallel_memcpy_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows);

}  // namespace hsb
