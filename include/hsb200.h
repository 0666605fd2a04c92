/*
 * hsb200.h — C ABI of the B200-native H/S generator (libhsb200.so).
 *
 * This is the drop-in boundary for the reference package `hsgen`
 * (/root/reference/pkg/src/hsgen).  Every entry point below replaces one
 * reference interface; the citation next to each declaration names it.
 * Plain C types only: complex128 matrices are passed as `double*` pointing at
 * interleaved (re, im) pairs, column-major, leading dimension in complex
 * elements — the memory layout of a numpy complex128 Fortran-order array
 * (matcore.py:1-6).  Device pointers are CUDA global-memory pointers; the
 * `stream` argument is a `cudaStream_t` passed as `void*` (NULL = legacy
 * default stream).  No function throws across the ABI; every function returns
 * an hsb_status and stores a message retrievable with hsb_last_error().
 *
 * Status codes map onto the reference's exception classes
 * (matcore.py:16-25): DIMENSION -> DimensionError, INPUT -> InputError,
 * INVARIANT -> InvariantError.  CUDA/UNSUPPORTED/NOMEM have no reference
 * counterpart and surface as RuntimeError in the Python host layer.
 */
#ifndef HSB200_H
#define HSB200_H

#include <stdint.h>

#if defined(__GNUC__)
#define HSB_API __attribute__((visibility("default")))
#else
#define HSB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HSB_OK = 0,
  HSB_ERR_DIMENSION = 1,   /* matcore.DimensionError */
  HSB_ERR_INPUT = 2,       /* matcore.InputError */
  HSB_ERR_INVARIANT = 3,   /* matcore.InvariantError */
  HSB_ERR_CUDA = 4,        /* CUDA runtime / driver failure */
  HSB_ERR_UNSUPPORTED = 5, /* request outside what the sm_100a kernels implement */
  HSB_ERR_NOMEM = 6        /* device or pinned allocation failed */
} hsb_status;

typedef struct hsb_ctx hsb_ctx;

/* Version of the ABI (bumped on any signature change). */
HSB_API int32_t hsb_abi_version(void);

/* Context = one CUDA device + cached device workspace + TMA encoder.
 * Replaces the implicit process-wide state of the reference executor
 * (executor.py:25-39 ExecPolicy is per call; the context is per device). */
HSB_API hsb_status hsb_ctx_create(int32_t device, hsb_ctx** out);
HSB_API void hsb_ctx_destroy(hsb_ctx* ctx);
/* Message of the last failing call on this context (thread-unsafe, like the
 * reference's single-entrant build_hs).  ctx may be NULL for
 * errors raised by hsb_ctx_create. */
HSB_API const char* hsb_last_error(const hsb_ctx* ctx);
/* Release cached device workspace (the next call re-allocates). */
HSB_API hsb_status hsb_ctx_trim(hsb_ctx* ctx);

/* Real-arithmetic form of the complex products in every dense contraction.
 * HSB_CPLX_3M (default): Gauss/Karatsuba, 3 real DMMA products per complex
 *   product (P = Lr^T Rr, Q = Li^T Ri, W = (Lr -/+ Li)^T (Rr + Ri)), 25 % fewer
 *   tensor-core cycles than the reference's 8-flop complex MAC
 *   (kernels.py:66-85); results agree to ~1e-15 relative Frobenius.
 * HSB_CPLX_4M: 4 real products per complex product (the conventional form).
 * The ledger always charges the reference's model flops. */
#define HSB_CPLX_4M 0
#define HSB_CPLX_3M 1
HSB_API hsb_status hsb_ctx_set_complex_mult(hsb_ctx* ctx, int32_t algo);

/* Engine of the lower-triangle contractions (S, H, herk, her2k, gemmt).
 * HSB_ENGINE_AUTO (default): hsb_build_hs runs the INT8 engine at FP64 width
 *   (below); the kernel-level calls (hsb_zherk / hsb_zher2k / hsb_zgemm) run
 *   FP64 DMMA, whose rounding is elementwise like the reference kernels'.
 * HSB_ENGINE_DMMA: FP64 DMMA tensor cores (complex form above), ~1e-15.
 * HSB_ENGINE_INT8: FP64-accurate emulation on the INT8 tensor cores
 *   (tcgen05.mma kind::i8) by the Chinese-remainder / Ozaki-II scheme:
 *   operands rounded to b-bit integers per column, b >= min_bits (the
 *   fewest moduli that allow it, up to 20), then exact modular INT8 products
 *   and CRT reconstruction.  min_bits = 0 selects the default 53: every
 *   operand keeps a full FP64 mantissa relative to its column's max (the
 *   largest entries are exact), ~1e-16 relative Frobenius on S and H -- the
 *   DMMA engine's level.  min_bits in [30, 55]; fewer bits trade accuracy
 *   (~2^-min_bits of each column's max) for moduli.  Batched per-atom
 *   products (Loop 1 / Loop 2) and rectangular GEMMs always use DMMA.
 * Settings are per context; every entry point holds the context's lock, so
 * calls on one context serialise (use one context per thread to overlap). */
#define HSB_ENGINE_DMMA 0
#define HSB_ENGINE_INT8 1
#define HSB_ENGINE_AUTO 2
HSB_API hsb_status hsb_ctx_set_engine(hsb_ctx* ctx, int32_t engine, int32_t min_bits);

/* Diagnostic: the INT8 engine's reconstruction table for n_mod moduli
 * (11..20), as the device uses it -- weights[(part * n_mod + i) * 2 + limb]
 * (part 0: Re, 1: Im; two 40-bit fixed-point limbs of u_i / p_i) and fl(M).
 * Host-only (no device call); lets CPU tests check the table against the
 * Python restatement (engine.crt_weights). */
HSB_API hsb_status hsb_oz_crt_table(int32_t n_mod, double* weights, double* m);

/* ------------------------------------------------------------------------ */
/* Kernel level: the five large updates.  Device pointers, caller's stream.  */
/* These replace run_partitioned(kind, operands, policy) for kind in         */
/* {HERK, HER2K, GEMM} (executor.py:185-225) and the serial kernels herk     */
/* (kernels.py:256-264), her2k (kernels.py:267-281), gemm (kernels.py:195).  */
/* ------------------------------------------------------------------------ */

/* flags */
#define HSB_LOWER_ONLY   0x1u  /* gemm: write only the lower triangle (GEMMT) */
#define HSB_MIRROR       0x2u  /* also write the strict upper triangle as the
                                  conjugate of the lower one and a real
                                  diagonal (= matcore.hermitian_mirror,
                                  matcore.py:89-105, fused in the epilogue) */

/* Lower triangle of C <- alpha * A^H A + beta * C, Im(diag C) := 0.
 * A is k x n (lda >= k), C is n x n (ldc >= n).  kernels.herk / _update_lower
 * (kernels.py:234-264). */
HSB_API hsb_status hsb_zherk(hsb_ctx* ctx, void* stream, int64_t n, int64_t k,
                     double alpha, const double* a, int64_t lda,
                     double beta, double* c, int64_t ldc, uint32_t flags);

/* Lower triangle of C <- alpha Z^H B + conj(alpha) B^H Z + beta C, Im(diag C) := 0.
 * Z, B are k x n.  kernels.her2k (kernels.py:267-281). */
HSB_API hsb_status hsb_zher2k(hsb_ctx* ctx, void* stream, int64_t n, int64_t k,
                      double alpha_re, double alpha_im,
                      const double* z, int64_t ldz, const double* b, int64_t ldb,
                      double beta, double* c, int64_t ldc, uint32_t flags);

/* C <- alpha op(A) op(B) + beta C, op in {'N','T','C'} (kernels.gemm,
 * kernels.py:195-220).  With HSB_LOWER_ONLY only the lower triangle of the
 * (square) C is written.  op(A) is m x k, op(B) is k x n. */
HSB_API hsb_status hsb_zgemm(hsb_ctx* ctx, void* stream, char opa, char opb,
                     int64_t m, int64_t n, int64_t k,
                     double alpha_re, double alpha_im,
                     const double* a, int64_t lda, const double* b, int64_t ldb,
                     double beta_re, double beta_im, double* c, int64_t ldc,
                     uint32_t flags);

/* In place: upper triangle := conj(lower), Im(diag) := 0
 * (matcore.hermitian_mirror, matcore.py:89-105). */
HSB_API hsb_status hsb_hermitian_mirror(hsb_ctx* ctx, void* stream, int64_t n,
                                double* c, int64_t ldc);

/* ------------------------------------------------------------------------ */
/* Pipeline level: builder.build_hs (builder.py:211-224).                   */
/* ------------------------------------------------------------------------ */

#define HSB_LOC_HOST   0  /* per-atom host blocks (the reference's ProblemInstance
                             lists, probgen.py:78-92) */
#define HSB_LOC_DEVICE 1  /* stacked device arrays (see hsb_problem) */

typedef struct {
  int64_t n_atoms, n_l, n_g;  /* matcore.Dims (matcore.py:28-44) */
  int32_t location;           /* HSB_LOC_HOST or HSB_LOC_DEVICE */
  int32_t reserved;
  /* HSB_LOC_HOST: arrays of n_atoms pointers, one per atom, each to a
   * column-major complex128 block: a/b n_l x n_g, t_* n_l x n_l; u_norms n_l
   * float64 values.  (ProblemInstance.a_blocks ... u_norms.) */
  const double* const* a_blocks;
  const double* const* b_blocks;
  const double* const* t_aa;
  const double* const* t_ab;
  const double* const* t_bb;
  const double* const* u_norms;
  /* HSB_LOC_DEVICE: stacked device arrays.  a_stack/b_stack are
   * (n_atoms*n_l) x n_g column-major complex128 (ld = n_atoms*n_l), i.e.
   * matcore.stack(p.a_blocks) (matcore.py:68-86); t_* are n_atoms contiguous
   * n_l x n_l column-major blocks; u is n_atoms*n_l float64. */
  const double* a_stack;
  const double* b_stack;
  const double* t_aa_dev;
  const double* t_ab_dev;
  const double* t_bb_dev;
  const double* u_dev;
} hsb_problem;

#define HSB_OPT_FORCE_NONHPD 0x1u  /* builder.build_phase2 force_nonhpd hook
                                      (builder.py:138,146-147) */
#define HSB_OPT_UNFUSED      0x2u  /* one launch per reference section
                                      (S1, U norm, S2, H1, H2, H3 separately,
                                      mirror last) instead of the fused
                                      H and S launches */
#define HSB_OPT_VALIDATE     0x4u  /* host inputs: check the T blocks and u
                                      (finite, T_AA / T_BB Hermitian within
                                      1e-14 (1 + ||T||_F), u > 0) in the order
                                      of probgen.validate_instance
                                      (probgen.py:140-168) before any transfer;
                                      A / B finiteness is always checked while
                                      they are staged */
#define HSB_OPT_FULL_D2H     0x8u  /* pinned host outputs: download both
                                      triangles of H and S instead of the lower
                                      triangles + host-side conjugate mirror
                                      (the default on the streamed INT8 path;
                                      same bytes in the result) */
#define HSB_OPT_LOWER_ONLY   0x10u /* device outputs, fused path: write H and
                                      S as lower triangles with a real
                                      diagonal and no mirror (the strict upper
                                      triangles are left untouched) -- the
                                      partial sums of the triangle-packed
                                      reduce-scatter (distributed.py) */

/* Receive slots of an atom-sharded build across n_ranks GPUs (north star (3);
 * SURVEY 8f row 2).  Rank q owns columns [q * cols_per_rank, (q + 1) *
 * cols_per_rank) of H and S and a receive buffer of n_ranks slots, each
 * cols_per_rank columns x ld rows of complex128 (column-major): slot r holds
 * rank r's partial sum for q's columns.  h_slots / s_slots are DEVICE arrays
 * of n_ranks device pointers (peer pointers from hsb_ipc_open, or local ones
 * when the "ranks" share a device). */
typedef struct hsb_peer_out {
  int32_t n_ranks;
  int32_t rank;
  int64_t cols_per_rank;
  int64_t ld;
  double* const* h_slots;
  double* const* s_slots;
} hsb_peer_out;

/* The owner's reduction of the fused scatter: out[i] = sum over the n_slots
 * receive slots (slot r at slots + 2 * r * slot_stride doubles) of slot_r[i],
 * i < count complex128 elements, summed in rank order (deterministic).  Replaces
 * the reduction inside ncclReduceScatter of the north star's atom-sharded
 * build (the reference has no multi-GPU code).  Device pointers;
 * asynchronous on `stream`. (ABI 8) */
HSB_API hsb_status hsb_sum_slots(hsb_ctx* ctx, void* stream, const double* slots, int32_t n_slots,
                                 int64_t slot_stride, int64_t count, double* out);

/* CUDA IPC for the receive slots: a 64-byte handle of a device allocation,
 * and its mapping in another process (cudaIpcGetMemHandle / OpenMemHandle). */
HSB_API hsb_status hsb_ipc_handle(hsb_ctx* ctx, void* dev_ptr, uint8_t handle[64]);
HSB_API hsb_status hsb_ipc_open(hsb_ctx* ctx, const uint8_t handle[64], void** dev_ptr);
HSB_API hsb_status hsb_ipc_close(hsb_ctx* ctx, void* dev_ptr);

typedef struct {
  /* Output location: HSB_LOC_HOST -> h/s are host pointers,
   * HSB_LOC_DEVICE -> device pointers.  Both n_g x n_g column-major complex128,
   * leading dimension ld (>= n_g), FULL Hermitian (Fill.FULL). */
  int32_t location;
  int32_t reserved;
  int64_t ld;
  double* h;
  double* s;
  /* Optional (INT8 engine, fused, device outputs): scatter this rank's partial
   * H and S straight into the owners' receive slots (hsb_peer_out) from the
   * reconstruction epilogue, instead of writing h / s.  The reduce-scatter of
   * an atom-sharded build then only sums each owner's slots. */
  const struct hsb_peer_out* peer;
  /* Optional cudaEvent_t, recorded on the stream as soon as S is final (before
   * the H contraction), so a caller can start consuming S -- e.g. its
   * reduce-scatter -- while H computes.  With device inputs, device outputs
   * and timings == NULL, hsb_build_hs returns without waiting for the device
   * (the work completes in stream order). */
  void* s_ready;
  /* Optional cudaEvent_t ordering of pipelined host-path calls (k-point lanes,
   * each on its own context and stream): this call's host->device copies
   * start after h2d_after, and h2d_done is recorded once they have landed;
   * its kernels start after compute_after, and compute_done is recorded after
   * the last one (H final).  Chaining call i+1's *_after to call i's *_done
   * keeps the upload engine and the SMs each working on one k-point at a
   * time, in order, while other calls' downloads run concurrently (ABI 6).
   * An event is only waited on once the previous call has recorded it:
   * order_in points at the previous call's order_out, which this library
   * sets to 1 after recording h2d_done and to 2 after compute_done (or on any
   * early return); host threads of consecutive calls synchronise on it. */
  void* h2d_after;
  void* h2d_done;
  void* compute_after;
  void* compute_done;
  const int32_t* order_in;
  int32_t* order_out;
} hsb_output;

/* Section timings (seconds, from CUDA events) in the reference's section
 * vocabulary (kernels.py:38 SECTIONS).  For fused launches the launch time is
 * split across the sections it covers in proportion to model flops. */
typedef struct {
  double loop1, loop2, unorm, s1, s2, h1, h2, h3;
  double h2d, d2h, total;   /* transfers (host path only) and end-to-end */
  double s_core, h_core;    /* the fused S / H contraction kernel alone (DMMA zrk
                               or INT8 modular GEMM), included in the sections */
  int32_t n_hpd, n_nonhpd;  /* builder.SplitCounts (builder.py:51-54) */
  int32_t launches;         /* kernels launched by this call */
  int32_t reserved;
  double h2d_bytes, d2h_bytes;  /* PCIe bytes moved by this call (host inputs /
                                   outputs; lower-triangle downloads count once) */
} hsb_timings;

/* Build H and S.  `atom_info` (optional, n_atoms int32) receives the
 * potrf_lower info per atom: 0 = Cholesky succeeded (HPD path), j>0 = first
 * non-positive leading minor (kernels.py:296-325), -1 = forced non-HPD.
 * Shapes are the caller's (host layer's) to validate; values of T and u with
 * HSB_OPT_VALIDATE; A and B non-finite values are always reported
 * (HSB_ERR_INVARIANT). */
HSB_API hsb_status hsb_build_hs(hsb_ctx* ctx, void* stream, const hsb_problem* p,
                        uint32_t opts, const hsb_output* out,
                        hsb_timings* timings, int32_t* atom_info);

/* ------------------------------------------------------------------------ */
/* Matching coefficients (north star part 1; no reference implementation:   */
/* A, B are random inputs in probgen.py:131-132).  PAPER.md:226-241.        */
/* ------------------------------------------------------------------------ */

typedef struct {
  int64_t n_atoms, n_g;
  int32_t lmax, n_types;
  const int32_t* gvec;     /* host, n_g x 3 integer G in reciprocal-lattice coordinates */
  const double* tau;       /* host, n_atoms x 3 Cartesian positions (bohr) */
  const int32_t* type_of;  /* host, n_atoms, in [0, n_types) */
  const double* rmt;       /* host, n_types muffin-tin radii (bohr) */
  const double* radial;    /* host, n_types x (lmax+1) x 4: u_l(R), u_l'(R), udot_l(R), udot_l'(R) */
  double kpt[3];           /* k in reciprocal-lattice coordinates */
  double recip[9];         /* reciprocal lattice vectors b1, b2, b3 as rows (1/bohr) */
  double omega;            /* cell volume (bohr^3) */
} hsb_phys;

/* Device A, B stacks (n_atoms*(lmax+1)^2) x n_g, column-major complex128,
 * leading dimension ld (complex elements), rows (atom, L = l^2+l+m):
 *   A = c [j_l(KR) udot' - K j_l'(KR) udot]/D,  B = c [K j_l'(KR) u - j_l(KR) u']/D,
 *   c = 4 pi / sqrt(Omega) i^l exp(i K.tau) conj(Y_lm(K^)),  D = u udot' - udot u'. */
HSB_API hsb_status hsb_match_coeffs(hsb_ctx* ctx, void* stream, const hsb_phys* phys,
                                    double* a_stack, double* b_stack, int64_t ld);

/* North-star entry point in one call: the matching coefficients of `ph` into
 * the device stacks p->a_stack / p->b_stack (ld = n_atoms * N_L), then the
 * H/S build of hsb_build_hs on them (p: device location, T blocks and u on
 * the device; same opts / out / timings / atom_info).  With the INT8 engine
 * on the fused path the matching kernel also writes S's and H's left operands
 * -- the column exponents and the residue planes of A and of diag(u) B -- as
 * it generates each G column, so the build skips those
 * passes over the stacks.  Replaces the pair match_coeffs + build_hs. */
HSB_API hsb_status hsb_build_hs_physical(hsb_ctx* ctx, void* stream, const hsb_phys* ph, const hsb_problem* p,
                                         uint32_t opts, const hsb_output* out, hsb_timings* tm,
                                         int32_t* atom_info);

#ifdef __cplusplus
}
#endif
#endif /* HSB200_H */
