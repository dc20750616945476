// sell.cu -- CsrMatrix (sparse.py:36-87, int64 or int32 indices, FP64 values)
// -> device SELL-32 layout (common.cuh: SellMatrix).
//
// The reference keeps CSR and walks rows with one scalar thread.  On B200 the
// SpMV is HBM-bound, so the layout is chosen for coalescing: slices of 32 rows
// (one warp), entries column-major inside a slice.  Row order of entries is
// preserved, so the per-row left-to-right accumulation (and hence every bit of
// the result) is unchanged.
#include <cub/cub.cuh>
#include "common.cuh"
#include "mwcg_internal.h"

namespace mwcg {

template <typename I>
__global__ void sell_row_len_kernel(const I *__restrict__ rp, int64_t n_rows, int64_t n_pad,
                                    int32_t *__restrict__ row_len, int64_t *__restrict__ slice_sz) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int len = 0;
    if (r < n_rows) len = (int)(rp[r + 1] - rp[r]);
    if (r < n_pad) row_len[r] = len;
    // slice max via warp reduction (blockDim multiple of 32, slices warp-aligned)
    int m = len;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0 && r < n_pad) slice_sz[r >> 5] = (int64_t)m * SLICE;
}

template <typename I>
__global__ void sell_fill_kernel(const I *__restrict__ rp, const I *__restrict__ ci,
                                 const double *__restrict__ va, int64_t n_rows,
                                 const int64_t *__restrict__ slice_ptr, int32_t *__restrict__ cols,
                                 double *__restrict__ vals) {
    // one warp per row: coalesced reads of the CSR row, strided SELL writes
    int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (gw >= n_rows) return;
    int64_t r = gw;
    int64_t base = slice_ptr[r >> 5] + (r & 31);
    int64_t lo = rp[r], hi = rp[r + 1];
    for (int64_t k = lo + lane; k < hi; k += 32) {
        int64_t kk = k - lo;
        cols[base + kk * SLICE] = (int32_t)ci[k];
        vals[base + kk * SLICE] = va[k];
    }
}

template <typename I>
static int build_sell(SellMatrixOwned *M, const I *rp, const I *ci, const double *va,
                      cudaStream_t st) {
    SellMatrix &A = M->view;
    int64_t n_pad = A.n_slices * SLICE;
    int64_t *slice_sz = nullptr;
    MWCG_CUDA(pool_alloc((void **)&M->row_len, sizeof(int32_t) * (n_pad > 0 ? n_pad : 1), st));
    MWCG_CUDA(pool_alloc((void **)&M->slice_ptr, sizeof(int64_t) * (A.n_slices + 1), st));
    MWCG_CUDA(pool_alloc((void **)&slice_sz, sizeof(int64_t) * (A.n_slices + 1), st));
    MWCG_CUDA(cudaMemsetAsync(slice_sz, 0, sizeof(int64_t) * (A.n_slices + 1), st));
    if (n_pad > 0) {
        int threads = 256;
        int64_t blocks = (n_pad + threads - 1) / threads;
        sell_row_len_kernel<I><<<(unsigned)blocks, threads, 0, st>>>(rp, A.n_rows, n_pad, M->row_len,
                                                                     slice_sz);
        MWCG_CHECK_LAUNCH();
    }
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, slice_sz, M->slice_ptr, A.n_slices + 1, st);
    void *tmp = nullptr;
    MWCG_CUDA(pool_alloc(&tmp, tmp_bytes, st));
    MWCG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, slice_sz, M->slice_ptr, A.n_slices + 1, st));
    int64_t total = 0;
    MWCG_CUDA(cudaMemcpyAsync(&total, M->slice_ptr + A.n_slices, sizeof(int64_t),
                              cudaMemcpyDeviceToHost, st));
    MWCG_CUDA(cudaStreamSynchronize(st));
    pool_free(tmp, st);
    pool_free(slice_sz, st);
    A.total = total;
    MWCG_CUDA(pool_alloc((void **)&M->cols, sizeof(int32_t) * (total > 0 ? total : 1), st));
    MWCG_CUDA(pool_alloc((void **)&M->vals, sizeof(double) * (total > 0 ? total : 1), st));
    // padding slots: column 0 / value 0, so chunked readers may load them safely
    MWCG_CUDA(cudaMemsetAsync(M->cols, 0, sizeof(int32_t) * (total > 0 ? total : 1), st));
    MWCG_CUDA(cudaMemsetAsync(M->vals, 0, sizeof(double) * (total > 0 ? total : 1), st));
    if (A.n_rows > 0) {
        int threads = 256;
        int64_t blocks = (A.n_rows * 32 + threads - 1) / threads;
        sell_fill_kernel<I><<<(unsigned)blocks, threads, 0, st>>>(rp, ci, va, A.n_rows, M->slice_ptr,
                                                                  M->cols, M->vals);
        MWCG_CHECK_LAUNCH();
    }
    A.slice_ptr = M->slice_ptr;
    A.row_len = M->row_len;
    A.cols = M->cols;
    A.vals = M->vals;
    MWCG_CUDA(cudaStreamSynchronize(st));
    return 0;
}

int sell_create(SellMatrixOwned **out, int64_t n_rows, int64_t n_cols, int64_t nnz,
                const void *row_ptr, const void *col_idx, const double *values, int index_bytes,
                cudaStream_t st) {
    if (n_rows < 0 || n_cols < 0 || nnz < 0) {
        set_error("negative dimensions");
        return MWCG_ERR_VALUE;
    }
    if (n_cols > INT32_MAX || n_rows > INT32_MAX) {
        set_error("dimensions above 2^31-1 are not supported by the int32 SELL layout");
        return MWCG_ERR_VALUE;
    }
    if (index_bytes != 4 && index_bytes != 8) {
        set_error("index_bytes must be 4 or 8");
        return MWCG_ERR_VALUE;
    }
    auto *M = new SellMatrixOwned();
    M->view.n_rows = n_rows;
    M->view.n_cols = n_cols;
    M->view.nnz = nnz;
    M->view.n_slices = (n_rows + SLICE - 1) / SLICE;
    int rc = (index_bytes == 8)
                 ? build_sell<int64_t>(M, (const int64_t *)row_ptr, (const int64_t *)col_idx, values, st)
                 : build_sell<int32_t>(M, (const int32_t *)row_ptr, (const int32_t *)col_idx, values, st);
    if (rc != 0) {
        sell_destroy(M);
        return rc;
    }
    *out = M;
    return 0;
}

void sell_destroy(SellMatrixOwned *M) {
    if (!M) return;
    pool_free(M->row_len, 0);
    pool_free(M->slice_ptr, 0);
    pool_free(M->cols, 0);
    pool_free(M->vals, 0);
    delete M;
}

}  // namespace mwcg
