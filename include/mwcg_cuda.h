/*
 * mwcg_cuda.h -- C ABI of libmwcg_cuda.so, the B200 (sm_100a) multi-word CG.
 *
 * This is the drop-in boundary for the reference package `mwcg`
 * (/root/reference/pkg/src/mwcg).  The reference has no FFI of its own: its
 * only native boundary is the Python -> numba call of the operator table
 * `_fast.KERNELS[mode][op]` (_fast.py:592-633, dispatched from
 * kernels.py:174-296) plus the solver entry `cg_solve` (cg.py:78-183).  Each
 * entry point below names the reference interface it replaces.
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch types.  Vector arguments are
 *    DEVICE pointers to structure-of-arrays word planes: word k of element i
 *    at v[k*ld + i] (the reference stores AoS records, kernels.py:39-40, 69-74;
 *    the values per word are identical).
 *  - mode: 0 fp64, 1 dw, 2 qdw, 3 tw, 4 qtw (kernels.py:35 MODES order).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Every call
 *    is stream-ordered; only the *_state / *_metrics / mwcg_cg_solve calls
 *    synchronize.
 *  - Return value 0 = success; otherwise a cudaError_t (< 1000) or
 *    MWCG_ERR_VALUE (1001, the reference's ValueError cases) /
 *    MWCG_ERR_STATE (1002).  mwcg_last_error() gives the message
 *    (thread-local).
 *  - There is no CPU fallback: without a CUDA device every compute entry
 *    point returns a cudaError_t.
 */
#ifndef MWCG_CUDA_H
#define MWCG_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MWCG_ABI_VERSION 1

enum { MWCG_FP64 = 0, MWCG_DW = 1, MWCG_QDW = 2, MWCG_TW = 3, MWCG_QTW = 4 };
/* Normalization (cg.py:27-32) */
enum { MWCG_NORM_NONE = 0, MWCG_NORM_AFTER_AXPY = 1, MWCG_NORM_EVERY_OP = 2 };
/* Dot-product reduction shape: the canonical device tile tree (fast), or
 * the reference's P-partition sequential shape (bitwise equal to the
 * reference's cg_solve(partitions=P); kernels.py:158-162, _fast.py:342-356). */
enum { MWCG_RED_TILE = 0, MWCG_RED_PARTITIONS = 1 };
/* SolverResult.reason (cg.py:69) */
enum { MWCG_RUNNING = 0, MWCG_CONVERGED = 1, MWCG_MAX_ITERATIONS = 2, MWCG_BREAKDOWN = 3 };

typedef struct mwcg_matrix mwcg_matrix;
typedef struct mwcg_solver mwcg_solver;

/* SolverConfig (cg.py:35-55) minus the per-solve scalars */
typedef struct {
    int mode;
    int normalization;
    int reduction;
    int reserved;
    int64_t partitions;
} mwcg_solver_config;

typedef struct {
    int64_t k;           /* completed iterations */
    int64_t iterations;  /* SolverResult.iterations once stopped */
    int status;          /* MWCG_RUNNING / CONVERGED / MAX_ITERATIONS / BREAKDOWN */
    int reserved;
    double rel;          /* recurrence residual ||r||/||b||, FP64 collapse */
    double rho[3], alpha[3], beta[3];
} mwcg_state;

typedef struct {
    int64_t iterations;
    int64_t n_hist;
    int status;
    int reserved;
    double final_rel;
    double loop_ms;      /* device time of the iteration loop (CUDA events) */
    double history_ms;   /* device time spent in history metrics */
    double stage_ms[3];  /* profile=1 only: K1 spmv+p.q, K2 update+r.r, K3 xpay */
    int64_t launches;    /* kernels launched by the solve (graph nodes included) */
} mwcg_solve_result;

/* ---- library ---- */
int mwcg_abi_version(void);
const char *mwcg_last_error(void);
int mwcg_words(int mode);                         /* kernels.py:43-46 mode_words */
int mwcg_device_check(void);                      /* 0 if an sm_100 device is usable */

/* ---- matrix: CsrMatrix (sparse.py:36-87) -> device SELL-32 ----
 * row_ptr/col_idx: device pointers, int64 (index_bytes=8, the reference's
 * dtype, sparse.py:47-48) or int32 (index_bytes=4). values: device f64. */
int mwcg_matrix_create(mwcg_matrix **out, int64_t n_rows, int64_t n_cols, int64_t nnz,
                       const void *row_ptr, const void *col_idx, const double *values,
                       int index_bytes, void *stream);
/* row_base: global index of local row 0 (a rank's rows of a partitioned
 * matrix with global columns; 0 otherwise).  col_format: -1 auto (slice-shared
 * column offsets when the 32 rows of each slice share them -- stencils, bands
 * -- else int16 column deltas when every |col - row| < 2^15, else int32),
 * 0 int32, 1 int16, 2 slice-shared offsets (error if a slice needs more than
 * its longest row + 2 slots).  The SELL layouts (0, 1, auto) sort the rows of
 * each 1024-row tile by length (SELL-sigma, sigma = 1024) when that cuts the
 * slice padding by >= 5 %; OR-ing MWCG_SELL_SIGMA forces the sort,
 * MWCG_SELL_NO_SIGMA disables it (with a flag, "auto" is written 15).  Row
 * results are unchanged (each row is still summed left to right).
 *
 * Slice-shared layout, value-uniform slices: when every slot of a 32-row
 * slice holds the same value bits in all the rows that have it (constant-
 * coefficient stencils), the value is kept once per slot in the slice's
 * pattern record and the slice streams no matrix bytes; slices that are not
 * uniform stream their values as before.  MWCG_DIA_STREAM_VALUES turns the
 * detection off (every slice streams its values).  Bitwise-identical
 * results either way. */
#define MWCG_SELL_SIGMA 16
#define MWCG_SELL_NO_SIGMA 32
#define MWCG_DIA_STREAM_VALUES 64
int mwcg_matrix_create_ex(mwcg_matrix **out, int64_t n_rows, int64_t n_cols, int64_t nnz,
                          const void *row_ptr, const void *col_idx, const double *values,
                          int index_bytes, int64_t row_base, int col_format, void *stream);
int mwcg_matrix_col_bytes(const mwcg_matrix *A);   /* 2 (int16 deltas), 4 (int32), 0 (slice-shared) */
int mwcg_matrix_sigma_sorted(const mwcg_matrix *A); /* 1 if the rows of each tile are length-sorted */
/* Column blocks: an irregular (int32-SELL) matrix with >= 2^22 columns, at
 * least 10 % of whose entries lie 2^21 or more columns away from their row,
 * also keeps its entries cut into column ranges of 2^21 (MWCG_COLBLOCK=<columns>
 * overrides, 0 = off); the solver's SpMV walks the ranges in turn, each
 * row's running sum carried in q, so one pass gathers only a range of p that
 * fits the L2.  Same additions in the same order: bitwise-identical q. */
int mwcg_matrix_col_blocks(const mwcg_matrix *A);   /* number of column blocks (0: not blocked) */
int64_t mwcg_matrix_block_columns(const mwcg_matrix *A); /* columns per block (0: not blocked) */
/* mwcg_matrix_create_ex with the caller's block width: cols_per_block > 0 cuts
 * an int32-SELL matrix into ranges of that many columns, 0 builds none, < 0
 * is the automatic choice.  The multi-GPU driver aligns the ranges with the
 * ranks' slices of p (dist.py, pipelined exchange). */
int mwcg_matrix_create_blocked(mwcg_matrix **out, int64_t n_rows, int64_t n_cols, int64_t nnz,
                               const void *row_ptr, const void *col_idx, const double *values,
                               int index_bytes, int64_t row_base, int col_format,
                               int64_t cols_per_block, void *stream);
int mwcg_matrix_destroy(mwcg_matrix *A);
int mwcg_matrix_info(const mwcg_matrix *A, int64_t *n_rows, int64_t *n_cols, int64_t *nnz,
                     int64_t *padded_entries);
/* value entries the layout stores (and streams per SpMV): padded_entries,
 * minus the entries of value-uniform slices (slice-shared layout) */
int64_t mwcg_matrix_stored_values(const mwcg_matrix *A);

/* ---- operator table: replaces _fast.KERNELS[mode][op] (_fast.py:592-633) ---- */
/* spmv_<mode> (_fast.py:284-290, 329-339, 383-393, 443-455, 501-513) */
int mwcg_spmv(int mode, const mwcg_matrix *A, const double *x, int64_t ldx, double *y,
              int64_t ldy, void *stream);
/* dot_<mode> (_fast.py:293-304, 342-356, 396-410, 458-474, 516-532).
 * partitions >= 1: the reference shape; partitions == 0: the device tile
 * tree.  out: device, 3 doubles.  work: device scratch of
 * mwcg_dot_work_bytes() bytes, ZERO-initialised before first use. */
int64_t mwcg_dot_work_bytes(int64_t n, int64_t partitions);
int mwcg_dot(int mode, int64_t n, const double *x, int64_t ldx, const double *y, int64_t ldy,
             int64_t partitions, double *out, void *work, void *stream);
/* axpy_<mode> (_fast.py:307-310, 359-363, 413-417, 477-481, 535-539);
 * alpha: HOST pointer to w words */
int mwcg_axpy(int mode, int64_t n, const double *alpha, const double *x, int64_t ldx, double *y,
              int64_t ldy, void *stream);
/* scal_add_<mode> (_fast.py:313-316, 366-370, ...): p <- r + beta p */
int mwcg_scal_add(int mode, int64_t n, const double *beta, double *p, int64_t ldp,
                  const double *r, int64_t ldr, void *stream);
/* residual_<mode> (_fast.py:319-322, ...): r = b - q, b FP64 */
int mwcg_residual(int mode, int64_t n, const double *b, const double *q, int64_t ldq, double *r,
                  int64_t ldr, void *stream);
/* normalize_arr_q{dw,tw} (_fast.py:433-436, 555-558); no-op for other modes */
int mwcg_normalize(int mode, int64_t n, double *v, int64_t ld, void *stream);
/* scalar ops on device pointers (3 doubles each), codes:
 * 0 add 1 mul 2 dxmul 3 dxadd 4 normalize 5 div 6 neg 7 two_sum
 * 8 quick_two_sum 9 two_prod 10 collapse 11 fma (a[0]*b[0]+a[1], one rounding)
 * (multiword.py / eft.py) */
int mwcg_scalar_op(int op, int mode, const double *a, const double *b, double *out, void *stream);
/* norm2_fp64 (kernels.py:290-296, sumsq_collapsed_1 _fast.py:565-571):
 * sequential unfused sum of squares of a HOST vector, then sqrt. */
int mwcg_norm2_host(const double *b, int64_t n, double *out);

/* ---- solver: replaces cg_solve (cg.py:78-183) ---- */
/* x: device buffer of w*n doubles for the solution words (NULL: internal) */
int mwcg_solver_create(mwcg_solver **out, const mwcg_matrix *A, const mwcg_solver_config *cfg,
                       double *x, void *stream);
int mwcg_solver_destroy(mwcg_solver *s);
/* b, x0 (nullable, FP64 initial guess), x_star (nullable): device f64[n].
 * b_norm: norm2_fp64(b) (0 is replaced by 1, cg.py:121-123). */
int mwcg_solver_start(mwcg_solver *s, const double *b, double b_norm, const double *x0,
                      const double *x_star, double epsilon, int64_t max_iterations);
/* enqueue iterations until stop or k == k_stop (one graph launch) */
int mwcg_solver_run(mwcg_solver *s, int64_t k_stop);
/* same, kernel-by-kernel with CUDA events; ms[0..2] += per-stage device ms */
int mwcg_solver_run_profiled(mwcg_solver *s, int64_t k_stop, double *ms);
/* Device µs of one SpMV+p.q launch (K1), averaged over `reps` back-to-back
 * launches on a started solver (bench.py's roofline.launch_us). */
int mwcg_solver_time_k1(mwcg_solver *s, int reps, double *us);
int mwcg_solver_state(mwcg_solver *s, mwcg_state *out);
/* Kernel configuration the solver chose (introspection for tests / bench):
 * out[0..3] grid of K1 / K2 / K3 / init, [4] TMA-staged K2, [5] TMA-staged
 * K3, [6] SELL-sigma row order, [7] column blocks K1 walks (0: none).
 * n: capacity of out. */
int mwcg_solver_describe(const mwcg_solver *s, int64_t *out, int n);
/* norm_metrics_tw (kernels.py:305-328) of the current iterate */
int mwcg_solver_metrics(mwcg_solver *s, double *err, double *true_res);
/* whole solve with history (ConvergenceRecord, cg.py:58-63, 129-136) */
int mwcg_cg_solve(mwcg_solver *s, const double *b, double b_norm, const double *x0,
                  const double *x_star, double epsilon, int64_t max_iterations,
                  int64_t history_stride, int profile, mwcg_solve_result *res,
                  int64_t hist_cap, int64_t *h_k, double *h_rel, double *h_true, double *h_err);

/* ---- row-partitioned multi-GPU rank (driven by dist.py) ----
 * A: this rank's rows, GLOBAL column indices.  p_full (ldp records of w
 * interleaved words) and part are caller-owned; the caller all-gathers
 * p_full after XPAY (or exchanges the neighbour halos) and the tile partials
 * before each FINAL stage.  part is RANK-BLOCKED: rank r's tiles occupy one
 * contiguous block of w * part_tb doubles at r * w * part_tb (word k of its
 * tile j at + k * part_tb + j), so the partials gather is ONE all-gather.
 * x0 for mwcg_solver_start is the full (ldp) initial guess.  Results are
 * bitwise identical to the 1-GPU tile-order solve.
 *
 * Overlap of the halo exchange with the SpMV: SPMV_INTERIOR runs the local
 * tiles [ilo, ihi) set by mwcg_solver_set_interior (tiles whose rows read
 * only this rank's slice of p -- they need no halo), SPMV_BOUNDARY the rest;
 * together they are exactly SPMV.  Every row is computed whole in one of
 * them, so each row's left-to-right sum (kernels.py:175-180) is unchanged. */
enum {
    MWCG_STAGE_INIT = 0,        /* r = b - q, p = r, r.r partials (after start's SpMV) */
    MWCG_STAGE_FINAL_INIT = 1,  /* canonical reduce of all partials: rho, rel, stop-at-0 */
    MWCG_STAGE_SPMV = 2,        /* q = A p, p.q partials */
    MWCG_STAGE_FINAL_ALPHA = 3, /* reduce, breakdown test, alpha */
    MWCG_STAGE_UPDATE = 4,      /* x, r update, r.r partials */
    MWCG_STAGE_FINAL_BETA = 5,  /* reduce, rel, stop / breakdown, beta, k++ */
    MWCG_STAGE_XPAY = 6,        /* p slice = r + beta p */
    MWCG_STAGE_SPMV_INTERIOR = 7, /* SPMV on the interior tiles only */
    MWCG_STAGE_SPMV_BOUNDARY = 8  /* SPMV on the remaining tiles */
};
int mwcg_solver_create_dist(mwcg_solver **out, const mwcg_matrix *A, const mwcg_solver_config *cfg,
                            double *x, double *p_full, int64_t ldp, int64_t p_off, double *part,
                            int64_t part_tb, int64_t tile_off, int64_t ntiles_glob, void *stream);
/* local tile range [ilo, ihi) of SPMV_INTERIOR (0 <= ilo <= ihi <= local tiles) */
int mwcg_solver_set_interior(mwcg_solver *s, int64_t ilo, int64_t ihi);
/* stream: NULL = the solver's stream (graph capture passes the capture stream) */
int mwcg_solver_dist_stage(mwcg_solver *s, int stage, void *stream);
/* SPMV restricted to the column blocks [b0, b1) of a blocked matrix (launch
 * b starts from the running sums block b-1 left in q; the last block adds the
 * p.q partials).  Calling it for [0, k1), [k1, k2) ... [kn, nblocks) in order is
 * exactly SPMV -- and each call needs only the columns of its blocks, so the
 * driver can run block b as soon as the rank owning those rows of p has
 * delivered its slice (dist.py: pipelined exchange). */
int mwcg_solver_dist_spmv_blocks(mwcg_solver *s, int b0, int b1, void *stream);

/* ---- ingestion: Matrix Market coordinate text (sparse.py:115-196) ----
 * Two calls: with rows == NULL it parses the banner and size line into info;
 * then with rows/cols/vals of info->nnz entries it parses the entries (0-based
 * indices, file order; the caller builds the CSR, summing duplicates).
 * Returns 0, MWCG_MM_ERROR (malformed input: mwcg_last_error() holds the
 * reference's message, info->error_line its line number, -1 if none), or
 * MWCG_MM_FALLBACK (input outside the native grammar -- non-ASCII bytes, lone
 * CR, '_' separators, hex floats, int64 overflow -- parse it the Python way). */
enum { MWCG_MM_ERROR = 1101, MWCG_MM_FALLBACK = 1102 };
typedef struct {
    int64_t n_rows, n_cols, nnz;
    int symmetric;
    int reserved;
    int64_t error_line;
} mwcg_mm_info;
int mwcg_mm_parse(const char *data, int64_t len, mwcg_mm_info *info, int64_t *rows, int64_t *cols,
                  double *vals);

/* ---- exact problem generation (problemgen.py:47-108, `generate`) ----
 * Replaces the reference's pure-Python ExactValue row sums (oracle.py:35-128)
 * for the all-ones solution: b_i = the exact row sum rounded to nearest FP64,
 * the rounding gap absorbed into the diagonal, b_i nudged by up to 4 ulps until
 * the perturbed diagonal is an FP64 number (problemgen.py:37-44).  Host code;
 * `threads` host threads over rows (<= 0: all).  CSR is int64, columns sorted
 * inside each row.  new_values (nnz) may alias values; b and deltas have n
 * entries (deltas[i] = FP64 new_diag - old_diag, 0 where unchanged).  Returns
 * 0 or MWCG_ERR_VALUE with the reference's message for the first failing row. */
int mwcg_problem_generate(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                          const double *values, double *new_values, double *b, double *deltas,
                          int64_t *max_ulp_adjustment, int threads);

/* ---- measurement helpers (bench.py) ---- */
/* FP64 pipe microbenchmark: DFMA chains on all SMs; returns FP64 ops/s
 * (FMA = 1 op, the SURVEY §8(d) convention) and the elapsed ms. */
int mwcg_fp64_peak(double *ops_per_s, double *ms, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MWCG_CUDA_H */
