// mwcg_internal.h -- declarations shared by the translation units of
// libmwcg_cuda.so (not part of the public C ABI; see include/mwcg_cuda.h).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>
#include "common.cuh"

// library error codes (cudaError_t values are returned as-is, all < 1000)
#define MWCG_ERR_VALUE 1001
#define MWCG_ERR_STATE 1002

namespace mwcg {

struct SellMatrixOwned {
    SellMatrix view{};
    int64_t *slice_ptr = nullptr;
    void *cols = nullptr;
    double *vals = nullptr;
    ulonglong2 *pat = nullptr;  // slice-shared-offset pattern table (dia layout)
    uint16_t *perm = nullptr;  // SELL-sigma row permutation (common.cuh: sell_row)
    int64_t n_patterns_words = 0;
    int64_t col0 = 0, col1 = 0;  // column range when this is one block of a column-blocked matrix
};

// the dia descriptor table is padded with this many empty slices
constexpr int DESC_PAD = 2;

// col_format: -1 auto (slice-shared offsets when they pay, else int16 deltas
// when they fit, else int32), 0 force int32, 1 force int16, 2 force slice-shared
int sell_create(SellMatrixOwned **out, int64_t n_rows, int64_t n_cols, int64_t nnz,
                const void *row_ptr, const void *col_idx, const double *values, int index_bytes,
                int64_t row_base, int col_format, cudaStream_t st);
void sell_destroy(SellMatrixOwned *M);
// Column blocks of an int32-SELL matrix (sell.cu): `out` stays empty when the
// layout is banded (slice-shared / int16 deltas), cols_per_block <= 0, the
// matrix has at most cols_per_block columns, or (automatic) fewer than 10 % of
// its entries lie cols_per_block or more columns away from their row.
int sell_colblocks(std::vector<SellMatrixOwned *> &out, const SellMatrixOwned *M, const void *row_ptr,
                   const void *col_idx, const double *values, int index_bytes, int64_t cols_per_block,
                   bool automatic, cudaStream_t st);

// operator-level launches (ops.cu); all stream-ordered
int launch_spmv(int mode, const SellMatrix &A, const double *x, int64_t ldx, double *y, int64_t ldy,
                cudaStream_t st);
int launch_dot_tile(int mode, int64_t n, const double *x, int64_t ldx, const double *y, int64_t ldy,
                    double *out, double *work, unsigned int *ticket, cudaStream_t st);
int launch_dot_partitions(int mode, int64_t n, const double *x, int64_t ldx, const double *y,
                          int64_t ldy, int64_t parts, double *out, double *work, cudaStream_t st);
int launch_axpy(int mode, int64_t n, const double *alpha, const double *x, int64_t ldx, double *y,
                int64_t ldy, cudaStream_t st);
int launch_scal_add(int mode, int64_t n, const double *beta, double *p, int64_t ldp, const double *r,
                    int64_t ldr, cudaStream_t st);
int launch_residual(int mode, int64_t n, const double *b, const double *q, int64_t ldq, double *r,
                    int64_t ldr, cudaStream_t st);
int launch_normalize(int mode, int64_t n, double *v, int64_t ld, cudaStream_t st);
int launch_scalar_op(int op, int mode, const double *a, const double *b, double *out, cudaStream_t st);

inline bool valid_mode(int m) { return m >= 0 && m <= 4; }

// Device memory comes from the stream-ordered pool (cudaMallocAsync) with the
// release threshold raised, so repeated solves / matrix rebuilds reuse memory
// instead of paying cudaMalloc/cudaFree (capi.cu).
cudaError_t pool_alloc(void **p, size_t bytes, cudaStream_t st);
void pool_free(void *p, cudaStream_t st);

}  // namespace mwcg
