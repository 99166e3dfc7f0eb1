/*
 * fastilu.h -- C ABI of the B200-native FastILU library (libfastilu_b200.so).
 *
 * What it computes: the FastILU preconditioner of arXiv 2506.05793 (ShyLU-node),
 * Section 5.
 *   - create   : symbolic ILU(k) pattern S of A (level-of-fill, sum rule)
 *                and the device layouts.  One-time setup ("symbolic factorization",
 *                PAPER.md:100-107, 128).
 *   - compute  : diagonal scaling, initial guess from A, then `nsweeps` synchronous
 *                fixed-point sweeps updating every l_ij, u_ij of S from the sparse dot of
 *                row i of L and column j of U (Fig. algo:fastILU_comp).
 *   - apply    : x = s o U^-1 L^-1 (s o b), each inverse replaced by `ntrisweeps` Jacobi
 *                sweeps x <- D^-1 (b - (T - D) x) from x0 = 0 (FastSpTRSV, Fig. algo:fastILU
 *                b, out of place per PAPER.md:717).
 * Readings of the paper where it is silent or garbled are listed in DESIGN.md ("Readings",
 * R1-R8); the same readings define the CPU oracle the tests compare against.
 *
 * Conventions
 *   - Matrices are square CSR: row_ptr int64[n+1] (row_ptr[0] = 0, non-decreasing), col_idx
 *     int32[nnz] strictly increasing within each row, values double[nnz].  Explicit zeros are
 *     kept and are part of the pattern.  Every row must store its diagonal.
 *   - Ownership: every call copies what it needs from the caller's arrays before returning,
 *     except fastilu_apply / fastilu_set_values_device, which read caller-owned DEVICE arrays
 *     in stream order.  The handle owns all device memory; fastilu_destroy frees it.
 *   - Streams: compute and apply are enqueued on the handle's stream (options.stream, or a
 *     library-owned stream).  compute synchronises the stream at its end so that zero pivots
 *     can be returned; apply does not synchronise.
 *   - Errors: every call returns a fastilu_status; nothing is thrown across the ABI.  The
 *     offending row (global index) of the last error is fastilu_error_index(h).
 *   - Threads: a handle is not thread-safe; distinct handles are independent.
 *   - Precision: fp64 throughout (PAPER.md:95 leaves it open; reading G13).
 *   - Multi-GPU (nranks > 1): every rank calls every function collectively; rank r owns
 *     the contiguous global rows [row_begin, row_begin + n), ranks ordered by row_begin.
 */
#ifndef FASTILU_B200_H
#define FASTILU_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fastilu_handle_s *fastilu_handle; /* opaque */

typedef enum {
  FASTILU_OK = 0,
  FASTILU_ERR_INVALID_ARG = 1,  /* null pointer, negative size, k < 0, bad option     */
  FASTILU_ERR_BAD_MATRIX = 2,   /* row_ptr not monotone, column out of range,         */
                                /* unsorted or duplicate columns (index = row)        */
  FASTILU_ERR_MISSING_DIAG = 3, /* structurally missing diagonal (index = row)        */
  FASTILU_ERR_ZERO_DIAG = 4,    /* a_ii == 0: cannot scale (index = row)              */
  FASTILU_ERR_ZERO_PIVOT = 5,   /* some iterate 0..nsweeps has u_ii == 0 or non-finite */
                                /* (index = smallest such row)                        */
  FASTILU_ERR_STATE = 6,        /* e.g. apply before a successful compute             */
  FASTILU_ERR_CUDA = 7,
  FASTILU_ERR_NCCL = 8,
  FASTILU_ERR_OOM = 9,
  FASTILU_ERR_UNSUPPORTED = 10  /* e.g. a row of S longer than the kernels support    */
} fastilu_status;

typedef enum {
  FASTILU_COMM_NONE = 0,    /* single GPU                                              */
  FASTILU_COMM_NCCL = 1,    /* one process per GPU, NCCL send/recv halos               */
  FASTILU_COMM_LOCAL = 2    /* ranks are threads of one process (fastilu_group)        */
} fastilu_comm_kind;

typedef struct fastilu_group_s *fastilu_group; /* in-process rank group (tests/tools) */

typedef struct {
  double omega;          /* factor damping factor w in (0,1]; default 1.0   */
  double omega_tri;      /* trisolve damping factor; default 1.0                            */
  int device;            /* CUDA device ordinal; -1 = the calling thread's current device   */
  void *stream;          /* cudaStream_t to enqueue on; NULL = library-owned stream          */
  int num_threads;       /* host threads for the symbolic setup; 0 = hardware concurrency   */
  /* ---- multi-GPU row-block partition (ignored when nranks == 1) ---- */
  int rank, nranks;
  int comm_kind;              /* fastilu_comm_kind                                          */
  const void *nccl_unique_id; /* FASTILU_COMM_NCCL: the 128-byte ncclUniqueId of rank 0     */
  fastilu_group group;        /* FASTILU_COMM_LOCAL: group from fastilu_group_create        */
  int64_t global_n;           /* total number of rows over all ranks                        */
  int64_t row_begin;          /* first global row owned by this rank                        */
  int64_t n_lead;             /* rows of A supplied BEFORE row_begin (see create)           */
  /* ---- options the paper evaluates ---- */
  double shift;               /* Manteuffel shift alpha >= 0: the factors are computed for     */
                              /* A' = A + alpha diag(|a_ii|); default 0           */
} fastilu_options;

/* Fills *opts with the defaults above (single GPU, omega = omega_tri = 1). */
void fastilu_default_options(fastilu_options *opts);

/*
 * fastilu_create: validate A, compute the ILU(level_k) pattern S, build the device layouts.
 *   n         rows owned by this rank (single GPU: the matrix order).
 *   row_ptr   host int64[n_lead + n + 1]; col_idx host int32[row_ptr[n_lead+n]] holding GLOBAL
 *             column indices; values host double[...] (may be NULL: pattern only, then
 *             fastilu_set_values must be called before compute).
 *             Single GPU: n_lead = 0 and these are just A.  Multi-GPU: the first n_lead rows
 *             are global rows [row_begin - n_lead, row_begin) of A (needed to reproduce the
 *             exact pattern of the rows this rank reads from its lower neighbour); pass
 *             n_lead = min(row_begin, fastilu_required_lead_rows(bandwidth, level_k)).
 *   level_k   fill level k >= 0.
 * Returns BAD_MATRIX / MISSING_DIAG with the offending row in fastilu_error_index(*out).
 * On error *out is still a valid handle (for the error index) and must be destroyed.
 */
fastilu_status fastilu_create(fastilu_handle *out, int64_t n, const int64_t *row_ptr,
                              const int32_t *col_idx, const double *values, int level_k,
                              const fastilu_options *opts);

/* Rows of A needed before row_begin for a matrix of half-bandwidth `bandwidth`
 * (max |i - j| over stored entries): 2 (k+1) bandwidth. */
int64_t fastilu_required_lead_rows(int64_t bandwidth, int level_k);

/* New values on the same pattern as create (numeric phase re-run).
 * Host array of the create call's nnz (lead rows included).  */
fastilu_status fastilu_set_values(fastilu_handle h, const double *values);
/* Same, DEVICE array (stream-ordered read, no host round trip). */
fastilu_status fastilu_set_values_device(fastilu_handle h, const double *values_dev);

/* Scale, initialise and run nsweeps >= 0 synchronous sweeps; synchronises the stream.
 * Returns ZERO_DIAG / ZERO_PIVOT with the row in fastilu_error_index. */
fastilu_status fastilu_compute(fastilu_handle h, int nsweeps);

/* fastilu_set_values(values) followed by fastilu_compute(nsweeps), with the upload of the new
 * values (HOST array, same layout as for fastilu_set_values; pin it for overlap) pipelined with
 * the numeric phase: row chunks of at least A's bandwidth are uploaded on a second stream while
 * earlier chunks are scaled and swept (PAPER.md:121-125 numeric phase).  Factors,
 * pattern of errors and every per-entry value are those of set_values + compute; the residual
 * history is summed per chunk (equal up to rounding).  Falls back to the two calls when the
 * pipeline does not apply (multi-GPU, CSR or block path, omega != 1, fewer than 2 chunks).
 * Synchronises at the end like fastilu_compute; errors as fastilu_compute. */
fastilu_status fastilu_compute_host(fastilu_handle h, const double *values, int nsweeps);
/* fastilu_compute_host(values, nsweeps) followed by fastilu_apply_host(b, x, ntrisweeps): the
 * one-call host-to-host solve step (e2e); b's upload is queued behind the values so it lands
 * during the compute.  b, x: HOST arrays of n (pinned for overlap).  Synchronises. */
fastilu_status fastilu_solve_host(fastilu_handle h, const double *values, int nsweeps,
                                  const double *b, double *x, int ntrisweeps);

/* The paper's asynchronous in-place sweeps: every thread updates its entries in
 * place, reading whatever mix of old and already-updated values it finds (Gauss-Seidel-like,
 * non-deterministic; same fixed point).  The residual history is the by-product of those
 * mixed reads.  Template-SELL or block (3-dof) layout, single GPU (FASTILU_ERR_UNSUPPORTED
 * otherwise).  Default block size: half a row's targets (template) / one 3x3 block (block). */
fastilu_status fastilu_compute_async(fastilu_handle h, int nsweeps);
/* The same with the paper's option "Block Size (or number of nonzeroes per thread)"
 * (PAPER.md:722): every thread updates about nnz_per_thread consecutive entries of the factor,
 * in order and in place, so the later ones use its own new values.  Template layout: a
 * contiguous block of ceil(W / parts) targets of one row, parts = the power of two (<= 8) that
 * brings the block to <= nnz_per_thread; block layout: max(1, nnz_per_thread / bs^2)
 * consecutive bs x bs target blocks.  nnz_per_thread = 0: the default.  INVALID_ARG if < 0. */
fastilu_status fastilu_compute_async_block(fastilu_handle h, int nsweeps, int nnz_per_thread);

/* Option "Warm up": FastILU(0), FastILU(1), ..., FastILU(k), each with nsweeps
 * sweeps, the factors of level L-1 initialising the entries of S_{L-1} inside S_L (new fill
 * entries start at +0.0; level 0 starts from the usual initial guess).  The residual history
 * has nsweeps (k+1) entries.  Template-SELL layout only (FASTILU_ERR_UNSUPPORTED otherwise
 * when k > 0). */
fastilu_status fastilu_compute_warmup(fastilu_handle h, int nsweeps);

/* "Sweeps to convergence" (BASELINE config 3; reading G15): like fastilu_compute but
 * stops after the first sweep s whose by-product residual of iterate s-1 satisfies
 * r(s-1) = ||(Ahat - L U)|_S||_F <= rtol ||Ahat|_S||_F, or after max_sweeps.  The factors are
 * iterate s; *sweeps_done = s.  One host synchronisation per sweep.  rtol > 0. */
fastilu_status fastilu_compute_tol(fastilu_handle h, double rtol, int max_sweeps,
                                   int *sweeps_done);

/* x = s o U^-1 L^-1 (s o b) with ntrisweeps >= 1 Jacobi sweeps for each factor.
 * b, x: caller-owned DEVICE arrays of length n on the handle's device (x may alias b).
 * Enqueued on the handle's stream; does not synchronise. */
fastilu_status fastilu_apply(fastilu_handle h, const double *b, double *x, int ntrisweeps);

/* Same with HOST arrays (pinned or pageable): H2D copy of b, apply, D2H copy of x,
 * synchronises.  This is the end-to-end entry point. */
fastilu_status fastilu_apply_host(fastilu_handle h, const double *b, double *x, int ntrisweeps);

/* FastILU-preconditioned restarted GMRES(restart) on A x = b (BASELINE config 5; the consumer of
 * apply in the paper's experiments): right preconditioning with
 * M^-1 = fastilu_apply(., ntrisweeps), x0 = 0, classical Gram-Schmidt with the
 * reorthogonalisation delayed by one iteration (DCGS2: per iteration one pass of dot products and
 * one update pass over the Krylov basis, one synchronisation / one allreduce over ranks; every
 * finished column is projected twice -- fastilu_get_info reports gmres_reorth, and gmres_retry
 * for the explicit re-projections taken after a severe cancellation); stop when
 * ||b - A x|| / ||b|| <= rtol (true residual at restarts) or after max_iters inner iterations.
 * restart in [1, 120].  b, x: DEVICE arrays of the owned rows.  Needs a successful compute.
 * *iters = inner iterations, *relres = final relative residual.  Synchronises. */
fastilu_status fastilu_gmres(fastilu_handle h, const double *b, double *x, int restart,
                             double rtol, int max_iters, int ntrisweeps, int *iters,
                             double *relres);

/* Loads EXTERNAL factors instead of computing them (config 5 arm B: e.g. the exact ILU(k) of Ahat,
 * to isolate the factor-sweep error from the trisolve's; BASELINE.json configs[4], SURVEY.md
 * Sec. 8(d) "Config 5 comparison arms").  vals: HOST array of the owned rows' S entries in S row
 * order (the layout fastilu_get_factors returns: l_ij below the diagonal, u_ij on and above it);
 * s: HOST array of the n scaling factors (apply returns x = s o U^-1 L^-1 (s o b), reading R5).
 * The pattern is the handle's (create); the caller keeps ownership of both arrays.  Afterwards
 * apply / gmres use these factors until the next compute.  Errors: INVALID_ARG (NULL arrays),
 * ZERO_PIVOT (a u_ii that is 0 or non-finite; index = first such global row).  Synchronises. */
fastilu_status fastilu_set_factors(fastilu_handle h, const double *vals, const double *s);

/* Frees everything; fastilu_destroy(NULL) is a no-op. */
fastilu_status fastilu_destroy(fastilu_handle h);

/* ---------------- introspection (tests, bench) ---------------- */
/* Owned rows and nnz(S) over the owned rows. */
fastilu_status fastilu_get_sizes(fastilu_handle h, int64_t *n, int64_t *nnz_S, int64_t *nnz_A);
/* CUDA device ordinal the handle runs on (opts.device, or the caller's current device at create
 * time when opts.device < 0): device arrays passed to apply / gmres must live there. */
fastilu_status fastilu_get_device(fastilu_handle h, int *device);
/* Pattern of the owned rows (host arrays; row_ptr[n+1] rebased to 0, global columns,
 * level[nnz_S]); any pointer may be NULL. */
fastilu_status fastilu_get_pattern(fastilu_handle h, int64_t *row_ptr, int32_t *col_idx,
                                   int8_t *level);
/* Factor values of the owned rows in S row order (strict-lower entries are l_ij, the rest
 * u_ij; unit diagonal of L implied), and the scaling vector s (n). Host copies; synchronises. */
fastilu_status fastilu_get_factors(fastilu_handle h, double *vals, double *s);
/* r(s-1) = ||(Ahat - L U)|_S||_F of iterate s-1 for the sweeps of the last compute
 * (global over ranks).  *count = min(cap, nsweeps). */
fastilu_status fastilu_get_residual_history(fastilu_handle h, double *hist, int cap, int *count);
/* Device-time breakdown of the last compute/apply in milliseconds (CUDA events):
 * t[0] = scale+init, t[1] = all sweeps, t[2] = apply (last call).  */
fastilu_status fastilu_get_timings(fastilu_handle h, double *t3);
/* Split of t[1] of fastilu_get_timings (milliseconds, CUDA events on the handle's stream):
 * t2[0] = sweep 1 (for the template path: the kernel with the initial guess fused in, plus its
 * residual reduction), t2[1] = sweeps 2..nsweeps (0 if nsweeps < 2).  Host-only; no sync. */
fastilu_status fastilu_get_sweep_split(fastilu_handle h, double *t2);
/* One-line description of the handle's kernel configuration (path "tsell" = template-SELL
 * with the JIT-specialised sweep, "csr-classes" / "csr-hash" / "csr-bsearch" = CSR kernels),
 * written NUL-terminated into buf (at most cap bytes). */
fastilu_status fastilu_get_info(fastilu_handle h, char *buf, int cap);
const char *fastilu_status_string(fastilu_status s);
int64_t fastilu_error_index(fastilu_handle h);

/* Host-only symbolic ILU(k) (no GPU needed): S of a full (single-rank) CSR matrix.
 * Two-phase: returns nnz(S) in *nnz_out when col_idx_out == NULL; otherwise fills the
 * caller-allocated row_ptr_out[n+1], col_idx_out[nnz], level_out[nnz] (level may be NULL).
 * num_threads = 0 uses all hardware threads.  *bad_row receives the offending row on error. */
fastilu_status fastilu_symbolic(int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                                int level_k, int num_threads, int64_t *nnz_out,
                                int64_t *row_ptr_out, int32_t *col_idx_out, int8_t *level_out,
                                int64_t *bad_row);

/* Host-only symbolic ILU(k) of a ROW WINDOW (the multi-GPU setup's building block): the caller
 * supplies rows [row0, row0 + nrows) of a global matrix (global column indices; entries with a
 * column < row0 are ignored) and receives the exact pattern of global rows [out_begin,
 * out_end), which is exact when out_begin - row0 >= fastilu_required_lead_rows(bandwidth, k)
 * or row0 == 0.  Two-phase like fastilu_symbolic; row_ptr_out has out_end - out_begin + 1
 * entries (rebased to 0). */
fastilu_status fastilu_symbolic_window(int64_t nrows, const int64_t *row_ptr,
                                       const int32_t *col_idx, int64_t row0, int64_t ncols,
                                       int64_t out_begin, int64_t out_end, int level_k,
                                       int num_threads, int64_t *nnz_out, int64_t *row_ptr_out,
                                       int32_t *col_idx_out, int8_t *level_out, int64_t *bad_row);

/* In-process rank group for FASTILU_COMM_LOCAL (ranks = threads of one process, halos by
 * device-to-device copies).  Destroy after all member handles are destroyed. */
fastilu_status fastilu_group_create(fastilu_group *out, int nranks);
fastilu_status fastilu_group_destroy(fastilu_group g);

/* NCCL bootstrap helper: writes a fresh 128-byte ncclUniqueId (rank 0 only). */
fastilu_status fastilu_nccl_unique_id(void *id128);

#ifdef __cplusplus
}
#endif
#endif /* FASTILU_B200_H */
