// capi.cu -- library-level C ABI: errors, version, operator wrappers,
// the host norm, and the FP64-pipe microbenchmark used for the roofline.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include "mwcg_internal.h"
#include "../../include/mwcg_cuda.h"

namespace mwcg {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

// FP64 pipe: each thread runs 8 independent DFMA chains (ILP hides the
// latency); 148 SMs x 2048 threads.
__global__ void fp64_peak_kernel(double *out, int iters, double a, double b) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = threadIdx.x * 1e-9 + k;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 8; k++) v[k] = __fma_rn(v[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s += v[k];
    if (s == 12345.678) out[0] = s;  // keep the chains live
}

cudaError_t pool_alloc(void **p, size_t bytes, cudaStream_t st) {
    static unsigned configured = 0;  // bit per device
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 32 && !(configured & (1u << dev))) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        configured |= 1u << dev;
    }
    return cudaMallocAsync(p, bytes > 0 ? bytes : 16, st);
}

void pool_free(void *p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}

}  // namespace mwcg

using namespace mwcg;

extern "C" {

int mwcg_abi_version(void) { return MWCG_ABI_VERSION; }

const char *mwcg_last_error(void) { return g_err; }

int mwcg_words(int mode) { return valid_mode(mode) ? mw::words_of(mode) : -1; }

int mwcg_device_check(void) {
    int dev = 0, count = 0;
    MWCG_CUDA(cudaGetDeviceCount(&count));
    if (count < 1) {
        set_error("no CUDA device");
        return MWCG_ERR_STATE;
    }
    MWCG_CUDA(cudaGetDevice(&dev));
    cudaDeviceProp p;
    MWCG_CUDA(cudaGetDeviceProperties(&p, dev));
    if (p.major != 10) {
        set_error("device %s is sm_%d%d; this library is built for sm_100a", p.name, p.major, p.minor);
        return MWCG_ERR_STATE;
    }
    return 0;
}

int64_t mwcg_dot_work_bytes(int64_t n, int64_t partitions) {
    int64_t slots = partitions >= 1 ? partitions : num_tiles(n);
    if (slots < 1) slots = 1;
    return 16 + (int64_t)sizeof(double) * 3 * slots;
}

int mwcg_dot(int mode, int64_t n, const double *x, int64_t ldx, const double *y, int64_t ldy,
             int64_t partitions, double *out, void *work, void *stream) {
    if (!valid_mode(mode) || n < 0 || partitions < 0) {
        set_error("bad mode / length / partitions");
        return MWCG_ERR_VALUE;
    }
    unsigned int *ticket = (unsigned int *)work;
    double *part = (double *)((char *)work + 16);
    if (partitions >= 1)
        return launch_dot_partitions(mode, n, x, ldx, y, ldy, partitions, out, part, (cudaStream_t)stream);
    return launch_dot_tile(mode, n, x, ldx, y, ldy, out, part, ticket, (cudaStream_t)stream);
}

int mwcg_axpy(int mode, int64_t n, const double *alpha, const double *x, int64_t ldx, double *y,
              int64_t ldy, void *stream) {
    if (!valid_mode(mode) || !alpha) {
        set_error("bad mode or alpha");
        return MWCG_ERR_VALUE;
    }
    return launch_axpy(mode, n, alpha, x, ldx, y, ldy, (cudaStream_t)stream);
}

int mwcg_scal_add(int mode, int64_t n, const double *beta, double *p, int64_t ldp, const double *r,
                  int64_t ldr, void *stream) {
    if (!valid_mode(mode) || !beta) {
        set_error("bad mode or beta");
        return MWCG_ERR_VALUE;
    }
    return launch_scal_add(mode, n, beta, p, ldp, r, ldr, (cudaStream_t)stream);
}

int mwcg_residual(int mode, int64_t n, const double *b, const double *q, int64_t ldq, double *r,
                  int64_t ldr, void *stream) {
    if (!valid_mode(mode)) {
        set_error("bad mode");
        return MWCG_ERR_VALUE;
    }
    return launch_residual(mode, n, b, q, ldq, r, ldr, (cudaStream_t)stream);
}

int mwcg_normalize(int mode, int64_t n, double *v, int64_t ld, void *stream) {
    if (!valid_mode(mode)) {
        set_error("bad mode");
        return MWCG_ERR_VALUE;
    }
    return launch_normalize(mode, n, v, ld, (cudaStream_t)stream);
}

int mwcg_scalar_op(int op, int mode, const double *a, const double *b, double *out, void *stream) {
    if (!valid_mode(mode) || op < 0 || op > 11) {
        set_error("bad mode or op");
        return MWCG_ERR_VALUE;
    }
    return launch_scalar_op(op, mode, a, b, out, (cudaStream_t)stream);
}

// Host code compiled with -fmad=false semantics: plain sequential loop; the
// translation unit is built with -Xcompiler -ffp-contract=off.
int mwcg_norm2_host(const double *b, int64_t n, double *out) {
    if (!out || (n > 0 && !b)) {
        set_error("null argument");
        return MWCG_ERR_VALUE;
    }
    volatile double s = 0.0;  // volatile: forbid reassociation / vectorisation
    for (int64_t i = 0; i < n; i++) {
        double c = b[i];
        double sq = c * c;
        s = s + sq;
    }
    *out = __builtin_sqrt(s);
    return 0;
}

int mwcg_fp64_peak(double *ops_per_s, double *ms, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, sms = 0;
    MWCG_CUDA(cudaGetDevice(&dev));
    MWCG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    double *d = nullptr;
    MWCG_CUDA(cudaMalloc(&d, sizeof(double)));
    const int threads = 512, blocks = sms * 4, iters = 4096;
    fp64_peak_kernel<<<blocks, threads, 0, st>>>(d, 64, 0.999999, 1e-7);  // warm-up
    cudaEvent_t e0, e1;
    MWCG_CUDA(cudaEventCreate(&e0));
    MWCG_CUDA(cudaEventCreate(&e1));
    MWCG_CUDA(cudaEventRecord(e0, st));
    fp64_peak_kernel<<<blocks, threads, 0, st>>>(d, iters, 0.999999, 1e-7);
    MWCG_CUDA(cudaEventRecord(e1, st));
    MWCG_CUDA(cudaEventSynchronize(e1));
    float t = 0;
    cudaEventElapsedTime(&t, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    double ops = (double)blocks * threads * iters * 8.0;
    if (ms) *ms = t;
    if (ops_per_s) *ops_per_s = ops / (t * 1e-3);
    return 0;
}

}  // extern "C"
