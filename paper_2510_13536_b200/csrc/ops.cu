// ops.cu -- operator-level kernels: the device replacement of the reference's
// operator table _fast.KERNELS[mode][op] (_fast.py:592-633) over SoA word
// planes.  The CG solver uses the fused kernels in cg.cu; these exist for the
// drop-in operator API (kernels.py:174-296) and for per-kernel parity tests.
#include "ops.cuh"
#include "mwcg_internal.h"

namespace mwcg {

using namespace mw;

template <int M, typename CT>
__global__ void __launch_bounds__(TILE_THREADS) spmv_kernel(SellMatrix A, const double *__restrict__ x,
                                                            int64_t ldx, double *__restrict__ y,
                                                            int64_t ldy) {
    constexpr int W = Arith<M>::W;
    const int64_t base = (int64_t)blockIdx.x * TILE + threadIdx.x;
#pragma unroll 1
    for (int j = 0; j < TILE_ELEMS; j++) {
        int64_t pos = base + j * TILE_THREADS;  // storage position; output at its natural row
        if (pos < A.n_rows) store<W>(y, ldy, sell_row(A, pos), spmv_row<M, 8, CT>(A, x, ldx, pos));
    }
}

// Tile-tree dot (canonical order, common.cuh).  work: W*ntiles partials.
template <int M>
__global__ void __launch_bounds__(TILE_THREADS) dot_tile_kernel(int64_t n, const double *__restrict__ x,
                                                                int64_t ldx, const double *__restrict__ y,
                                                                int64_t ldy, double *__restrict__ part,
                                                                int64_t ntiles, unsigned int *ticket,
                                                                double *__restrict__ out) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    __shared__ double smem[tree_smem<W>()];
    __shared__ int s_last;
    V<W> acc = zero<W>();
    const int64_t base = (int64_t)blockIdx.x * TILE + threadIdx.x;
#pragma unroll
    for (int j = 0; j < TILE_ELEMS; j++) {
        int64_t i = base + j * TILE_THREADS;
        if (i < n) acc = Ar::add(acc, Ar::mul(load_ro<W>(x, ldx, i), load_ro<W>(y, ldy, i)));
    }
    acc = block_tree<M, TILE_THREADS>(acc, smem);
    if (threadIdx.x == 0) store_part<W>(part, ntiles, blockIdx.x, acc);
    if (!last_block_done(ticket, &s_last)) return;
    V<W> r = reduce_partials_block<M>(part, ntiles, ntiles, smem);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < 3; k++) out[k] = k < W ? r.w[k] : 0.0;
        *ticket = 0u;
    }
}

// Reference-shape dot (kernels.py:158-162, _fast.py:342-356): partition p is
// one sequential chain; the P results are combined left to right.
template <int M>
__global__ void dot_part_kernel(int64_t n, const double *__restrict__ x, int64_t ldx,
                                const double *__restrict__ y, int64_t ldy, int64_t parts,
                                double *__restrict__ part) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= parts) return;
    int64_t lo = (int64_t)(((__int128)n * p) / parts);
    int64_t hi = (int64_t)(((__int128)n * (p + 1)) / parts);
    V<W> t = zero<W>();
    for (int64_t i = lo; i < hi; i++) t = Ar::add(t, Ar::mul(load<W>(x, ldx, i), load<W>(y, ldy, i)));
    store<W>(part, parts, p, t);
}

template <int M>
__global__ void dot_part_combine_kernel(const double *__restrict__ part, int64_t parts,
                                        double *__restrict__ out) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    V<W> s = load<W>(part, parts, 0);
    for (int64_t p = 1; p < parts; p++) s = Ar::add(s, load<W>(part, parts, p));
#pragma unroll
    for (int k = 0; k < 3; k++) out[k] = k < W ? s.w[k] : 0.0;
}

template <int M>
struct ScalarArg {
    double w[3];
};

// axpy_<mode>: y <- add(y, mul(alpha, x)) (_fast.py:307-310, 359-363, ...)
template <int M>
__global__ void axpy_kernel(int64_t n, ScalarArg<M> alpha, const double *__restrict__ x, int64_t ldx,
                            double *__restrict__ y, int64_t ldy) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    V<W> a;
#pragma unroll
    for (int k = 0; k < W; k++) a.w[k] = alpha.w[k];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        store<W>(y, ldy, i, Ar::add(load<W>(y, ldy, i), Ar::mul(a, load<W>(x, ldx, i))));
}

// scal_add_<mode>: p <- add(r, mul(beta, p)) (_fast.py:313-316, 366-370, ...)
template <int M>
__global__ void scal_add_kernel(int64_t n, ScalarArg<M> beta, double *__restrict__ p, int64_t ldp,
                                const double *__restrict__ r, int64_t ldr) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    V<W> b;
#pragma unroll
    for (int k = 0; k < W; k++) b.w[k] = beta.w[k];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        store<W>(p, ldp, i, Ar::add(load<W>(r, ldr, i), Ar::mul(b, load<W>(p, ldp, i))));
}

// residual_<mode>: r = dxadd(b, -q) (_fast.py:319-322, 373-376, ...)
template <int M>
__global__ void residual_kernel(int64_t n, const double *__restrict__ b, const double *__restrict__ q,
                                int64_t ldq, double *__restrict__ r, int64_t ldr) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        store<W>(r, ldr, i, Ar::dxadd(b[i], neg<W>(load<W>(q, ldq, i))));
}

// normalize_arr_q{dw,tw} (_fast.py:433-436, 555-558)
template <int M>
__global__ void normalize_kernel(int64_t n, double *__restrict__ v, int64_t ld) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        store<W>(v, ld, i, Ar::norm(load<W>(v, ld, i)));
}

// scalar ops for unit parity (op codes as oracle orc_scalar_op)
template <int M>
__global__ void scalar_op_kernel(int op, const double *a, const double *b, double *out) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    V<W> A, B;
#pragma unroll
    for (int k = 0; k < W; k++) {
        A.w[k] = a[k];
        B.w[k] = b[k];
    }
    V<W> R = zero<W>();
    double r0 = 0, r1 = 0;
    switch (op) {
    case 0: R = Ar::add(A, B); break;
    case 1: R = Ar::mul(A, B); break;
    case 2: R = Ar::dxmul(a[0], B); break;
    case 3: R = Ar::dxadd(a[0], B); break;
    case 4: R = Ar::norm(A); break;
    case 5: R = Ar::div(A, B); break;
    case 6: R = neg<W>(A); break;
    case 7: two_sum(a[0], b[0], r0, r1); break;
    case 8: quick_two_sum(a[0], b[0], r0, r1); break;
    case 9: two_prod(a[0], b[0], r0, r1); break;
    case 10: R.w[0] = Ar::collapse(A); break;
    case 11: R.w[0] = __fma_rn(a[0], b[0], a[1]); break;  // eft.fma: c rides in a[1]
    }
    if (op >= 7 && op <= 9) {
        out[0] = r0;
        out[1] = r1;
        out[2] = 0.0;
        return;
    }
#pragma unroll
    for (int k = 0; k < 3; k++) out[k] = k < W ? R.w[k] : 0.0;
}

// --------------------------------------------------------------- dispatch
#define MWCG_DISPATCH(mode, F)                 \
    switch (mode) {                            \
    case FP64: F(FP64); break;                 \
    case DW: F(DW); break;                     \
    case QDW: F(QDW); break;                   \
    case TW: F(TW); break;                     \
    case QTW: F(QTW); break;                   \
    default: set_error("bad mode %d", mode); return MWCG_ERR_VALUE; \
    }

static unsigned elementwise_blocks(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    return (unsigned)(b < 1 ? 1 : b);
}

int launch_spmv(int mode, const SellMatrix &A, const double *x, int64_t ldx, double *y, int64_t ldy,
                cudaStream_t st) {
    int64_t tiles = num_tiles(A.n_rows);
    if (tiles == 0) return 0;
#define L(Mx)                                                                                          \
    do {                                                                                               \
        if (A.dia) spmv_kernel<Mx, DiaTag><<<(unsigned)tiles, TILE_THREADS, 0, st>>>(A, x, ldx, y, ldy);   \
        else if (A.col16) spmv_kernel<Mx, int16_t><<<(unsigned)tiles, TILE_THREADS, 0, st>>>(A, x, ldx, y, ldy); \
        else spmv_kernel<Mx, int32_t><<<(unsigned)tiles, TILE_THREADS, 0, st>>>(A, x, ldx, y, ldy);         \
    } while (0)
    MWCG_DISPATCH(mode, L);
#undef L
    MWCG_CHECK_LAUNCH();
    return 0;
}

int launch_dot_tile(int mode, int64_t n, const double *x, int64_t ldx, const double *y, int64_t ldy,
                    double *out, double *work, unsigned int *ticket, cudaStream_t st) {
    int64_t tiles = num_tiles(n);
    if (tiles == 0) {
        MWCG_CUDA(cudaMemsetAsync(out, 0, 3 * sizeof(double), st));
        return 0;
    }
#define L(Mx)                                                                                  \
    dot_tile_kernel<Mx><<<(unsigned)tiles, TILE_THREADS, 0, st>>>(n, x, ldx, y, ldy, work, tiles, \
                                                                   ticket, out)
    MWCG_DISPATCH(mode, L);
#undef L
    MWCG_CHECK_LAUNCH();
    return 0;
}

int launch_dot_partitions(int mode, int64_t n, const double *x, int64_t ldx, const double *y,
                          int64_t ldy, int64_t parts, double *out, double *work, cudaStream_t st) {
    if (parts < 1) {
        set_error("partition count must be >= 1");
        return MWCG_ERR_VALUE;
    }
    unsigned blocks = (unsigned)((parts + 127) / 128);
#define L(Mx)                                                                             \
    do {                                                                                  \
        dot_part_kernel<Mx><<<blocks, 128, 0, st>>>(n, x, ldx, y, ldy, parts, work);      \
        dot_part_combine_kernel<Mx><<<1, 1, 0, st>>>(work, parts, out);                   \
    } while (0)
    MWCG_DISPATCH(mode, L);
#undef L
    MWCG_CHECK_LAUNCH();
    return 0;
}

int launch_axpy(int mode, int64_t n, const double *alpha, const double *x, int64_t ldx, double *y,
                int64_t ldy, cudaStream_t st) {
    if (n == 0) return 0;
    unsigned blocks = elementwise_blocks(n);
#define L(Mx)                                                                     \
    do {                                                                          \
        ScalarArg<Mx> a{};                                                        \
        for (int k = 0; k < words_of(Mx); k++) a.w[k] = alpha[k];                 \
        axpy_kernel<Mx><<<blocks, 256, 0, st>>>(n, a, x, ldx, y, ldy);            \
    } while (0)
    MWCG_DISPATCH(mode, L);
#undef L
    MWCG_CHECK_LAUNCH();
    return 0;
}

int launch_scal_add(int mode, int64_t n, const double *beta, double *p, int64_t ldp, const double *r,
                    int64_t ldr, cudaStream_t st) {
    if (n == 0) return 0;
    unsigned blocks = elementwise_blocks(n);
#define L(Mx)                                                                     \
    do {                                                                          \
        ScalarArg<Mx> b{};                                                        \
        for (int k = 0; k < words_of(Mx); k++) b.w[k] = beta[k];                  \
        scal_add_kernel<Mx><<<blocks, 256, 0, st>>>(n, b, p, ldp, r, ldr);        \
    } while (0)
    MWCG_DISPATCH(mode, L);
#undef L
    MWCG_CHECK_LAUNCH();
    return 0;
}

int launch_residual(int mode, int64_t n, const double *b, const double *q, int64_t ldq, double *r,
                    int64_t ldr, cudaStream_t st) {
    if (n == 0) return 0;
    unsigned blocks = elementwise_blocks(n);
#define L(Mx) residual_kernel<Mx><<<blocks, 256, 0, st>>>(n, b, q, ldq, r, ldr)
    MWCG_DISPATCH(mode, L);
#undef L
    MWCG_CHECK_LAUNCH();
    return 0;
}

int launch_normalize(int mode, int64_t n, double *v, int64_t ld, cudaStream_t st) {
    if (n == 0 || (mode != QDW && mode != QTW)) return 0;
    unsigned blocks = elementwise_blocks(n);
#define L(Mx) normalize_kernel<Mx><<<blocks, 256, 0, st>>>(n, v, ld)
    MWCG_DISPATCH(mode, L);
#undef L
    MWCG_CHECK_LAUNCH();
    return 0;
}

int launch_scalar_op(int op, int mode, const double *a, const double *b, double *out, cudaStream_t st) {
#define L(Mx) scalar_op_kernel<Mx><<<1, 1, 0, st>>>(op, a, b, out)
    MWCG_DISPATCH(mode, L);
#undef L
    MWCG_CHECK_LAUNCH();
    return 0;
}

}  // namespace mwcg
