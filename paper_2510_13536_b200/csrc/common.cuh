// common.cuh -- shared device structures: SELL-32 matrix, CG state, the
// canonical tile-tree reduction, error plumbing.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "mw.cuh"

namespace mwcg {

// ---------------------------------------------------------------------------
// Canonical tile shape.  A tile is TILE_THREADS
// threads x TILE_ELEMS elements; thread t of tile b owns elements
// b*TILE + j*TILE_THREADS + t, j = 0..TILE_ELEMS-1 (coalesced).  Every fused
// dot follows this order, and oracle/mwcg_oracle.c:tile_tree_dot_impl
// reproduces it bit-for-bit on the CPU.
// ---------------------------------------------------------------------------
constexpr int TILE_THREADS = 256;
constexpr int TILE_ELEMS = 4;
constexpr int TILE = TILE_THREADS * TILE_ELEMS;
constexpr int SLICE = 32;  // SELL slice height = one warp

inline int64_t num_tiles(int64_t n) { return (n + TILE - 1) / TILE; }

// SELL-32 matrix (built on device from CSR, sell.cu).  Entry k of row r sits
// at slice_ptr[r/32] + k*32 + r%32 (column-major inside a slice), so a warp
// walking its 32 rows in lock-step issues coalesced loads while each thread
// keeps the reference's strict left-to-right order inside its row
// (kernels.py:175-180).  Padding slots (after a row's last entry) hold a
// SENTINEL column, so no per-row length array is stored or loaded.
//
// Column storage: when every |col - (row_base + row)| < 2^15 (stencils,
// banded matrices) the columns are int16 deltas (2 B/entry instead of 4;
// sentinel INT16_MIN), otherwise absolute int32 (sentinel -1).
//
// Slice-shared offsets ("DIA" slices, chosen at build time when the rows of
// each slice use (almost) the same column offsets -- stencils, bands): slot k
// of slice j holds, for all 32 rows, the entry at column offset om_k (one
// uint64 per slot: int32 offset | 32-lane presence mask << 32).  A row's
// present slots are its CSR entries in ascending column order, so the
// left-to-right sum is unchanged; no column array is streamed, and a row's
// gathers depend only on the (L1-resident, warp-uniform) offset word, not on
// a column load from HBM.
//
// Slice-uniform values: when, in every slot of a slice, all present lanes hold
// the SAME value bits (constant-coefficient stencils: every row of the slice
// carries the same coefficient at a given offset), the slot's value is stored
// once, next to its offset word, in the pattern record -- such a slice streams
// no matrix bytes at all (its whole description is an L1-resident pattern).
// The arithmetic and its order are unchanged: dxmul(a, x) sees the same a.
constexpr int16_t COL16_SENT = -32768;
constexpr int32_t COL32_SENT = -1;

struct SellMatrix {
    int64_t n_rows;
    int64_t n_cols;
    int64_t nnz;
    int64_t n_slices;
    int64_t total;          // padded entry count (slots * 32, all slices)
    int64_t stored;         // value entries actually stored (dia: non-uniform slices only)
    int64_t row_base;       // global index of local row 0 (row-partitioned ranks)
    int col16;              // 1: int16 deltas, 0: int32 absolute
    int dia;                // 1: slice-shared offsets (om; no column array)
    const int64_t *slice_ptr;
    const void *cols;
    const double *vals;
    const ulonglong2 *pat;  // dia: pattern table of slot records {lane mask << 32 | uint32 offset,
                            // uniform value bits}; slice_ptr then holds two descriptor words
                            // per slice: {start/32 | L << 40 | uniform << 48, pattern base}
    const uint16_t *perm;   // SELL-sigma: storage position -> row within its 1024-row tile
                            // (rows of a tile sorted by length; nullptr: identity)
    int64_t pat_len;        // dia: records in the pattern table (bounds checks)
};

// Debug build (-DMWCG_BOUNDS, libmwcg_cuda_bounds.so): every index the matrix
// walks form -- pattern record, value slot, gathered column -- is checked on the
// device and a violation traps (compute-sanitizer is not available on every
// pool; tests/test_gpu_bounds.py runs the layouts through this build).
#ifdef MWCG_BOUNDS
#define MWCG_ASSERT(cond)                                                           \
    do {                                                                            \
        if (!(cond)) {                                                              \
            printf("MWCG_BOUNDS %s:%d: %s\n", __FILE__, __LINE__, #cond);           \
            __trap();                                                               \
        }                                                                           \
    } while (0)
#else
#define MWCG_ASSERT(cond) ((void)0)
#endif

// Natural row of storage position `pos` (SELL-sigma permutes rows inside
// their tile only, so tiles and the canonical tile order are unchanged).
__device__ __forceinline__ int64_t sell_row(const SellMatrix &A, int64_t pos) {
    return A.perm ? ((pos & ~(int64_t)1023) + __ldg(A.perm + pos)) : pos;
}

// Format tag of the slice-shared-offset layout (the column-type template
// parameter of the walks, next to int16_t / int32_t).
struct DiaTag {};

// Solver status (cg.py:138-183 reasons)
enum Status : int { RUNNING = 0, CONVERGED = 1, MAX_ITERS = 2, BREAKDOWN = 3 };

// Device-resident CG scalar state.  All scalars live in the mode's
// arithmetic (rho, alpha, beta: cg.py:118-181), padded to 3 words.
struct CgState {
    double rho[3];
    double rho_new[3];
    double pq[3];
    double alpha[3];
    double neg_alpha[3];
    double beta[3];
    double rel;          // ||r||/||b|| FP64 collapse (cg.py:125-127)
    double b_norm;       // norm2_fp64(b), 0 -> 1 (cg.py:121-123)
    double eps;
    long long k;         // completed iterations
    long long k_stop;    // pause point (history records)
    long long max_iters;
    long long iterations;  // reported count when status != RUNNING
    int status;
    int norm_r;          // normalize r (quasi & policy != none)
    int norm_all;        // every-op normalization
    int pause;           // K1 reached k_stop inside an unrolled graph body:
                         // the rest of the body is skipped (cleared by the host)
    int x_pending;       // K2 ran this iteration: K3 owes x += alpha p
    unsigned int ticket[4];  // last-block-done counters
    double metrics[4];   // err^2 sum, res^2 sum (collapsed), bnorm_sq, xs_sq
};

// ---------------------------------------------------------------------------
// Tree helpers.  Warp: lane l <- add(lane l, lane l+off), off = 16..1.  Block:
// the same over the TILE_THREADS/32 warp results.  Result valid in thread 0.
// ---------------------------------------------------------------------------
template <int M>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> warp_tree(mw::V<mw::Arith<M>::W> v) {
    using A = mw::Arith<M>;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        auto o = mw::shfl_down<A::W>(v, off);
        v = A::add(v, o);
    }
    return v;
}

// The SAME tree with every addition executed once: the 256 leaves go through
// shared memory, level 1 (128 additions) runs on 4 warps, level 2 (64) on 2,
// and warp 0 finishes levels 3-5 and the three cross-warp levels with
// shuffles -- 12 warp-level additions per tile instead of 43 (each of the 8
// warps running the 5-level shuffle tree, then warp 0's 3 levels).  Pairings
// and operand order are those of warp_tree + the cross-warp stage above, so
// every bit of the result is unchanged; what changes is the issue and
// FP64-pipe load of the tile reductions (a third of K2's instruction stream).
// smem: tree_smem<W>() doubles.  Every thread of the block must call it; the
// first TILE_THREADS threads hold the leaves.  Result valid in thread 0.
template <int W>
__host__ __device__ constexpr int tree_smem() {
    return W * (TILE_THREADS + TILE_THREADS / 2 + TILE_THREADS / 4);
}

// COLD: the copy that runs ONCE per kernel, in the last CTA's reduction of the
// tile partials.  That serial tail executes each instruction once, so its time
// is instruction fetch, and for TW -- 204 instructions per addition -- the fully
// inlined tail was ~4000 straight-line instructions during which every other SM
// sat idle (ncu, C2 TW: 41 % of K2's and ~20 % of K1's elapsed cycles had no
// resident warp outside that one CTA; profiles/r2v_ncu_k23_tw.json).  The cold
// copy calls ONE out-of-line tw_add (mw::add_cold) instead: TW 451 -> 391 us/it.
// The cheap additions of the other modes stay inline (calls and rolled loops
// cost them 4-6 us/it: profiles/r2w_*.json).
template <int M, bool COLD>
struct TailAdd {
    static __device__ __forceinline__ mw::V<mw::Arith<M>::W> add(mw::V<mw::Arith<M>::W> a,
                                                                 mw::V<mw::Arith<M>::W> b) {
        if constexpr (COLD && M == mw::TW) return mw::add_cold<M>(a, b);
        else return mw::Arith<M>::add(a, b);
    }
};

template <int M, bool COLD = false>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> dense_tree(mw::V<mw::Arith<M>::W> v, double *smem) {
    using A = TailAdd<M, COLD>;
    constexpr int W = mw::Arith<M>::W;
    static_assert(TILE_THREADS == 256, "the level split below is written for 8 warps");
    double *s0 = smem, *s1 = smem + W * 256, *s2 = s1 + W * 128;
    const int t = threadIdx.x;
    if (t < 256) {
#pragma unroll
        for (int k = 0; k < W; k++) s0[k * 256 + t] = v.w[k];
    }
    __syncthreads();
    if (t < 128) {  // level 1: leaf (w, l) + leaf (w, l + 16), l < 16; result index w*16 + l == t
        const int i = (t >> 4) * 32 + (t & 15);
        mw::V<W> a, b;
#pragma unroll
        for (int k = 0; k < W; k++) {
            a.w[k] = s0[k * 256 + i];
            b.w[k] = s0[k * 256 + i + 16];
        }
        a = A::add(a, b);
#pragma unroll
        for (int k = 0; k < W; k++) s1[k * 128 + t] = a.w[k];
    }
    __syncthreads();
    if (t < 64) {  // level 2: (w, l) + (w, l + 8), l < 8; result index w*8 + l == t
        const int i = (t >> 3) * 16 + (t & 7);
        mw::V<W> a, b;
#pragma unroll
        for (int k = 0; k < W; k++) {
            a.w[k] = s1[k * 128 + i];
            b.w[k] = s1[k * 128 + i + 8];
        }
        a = A::add(a, b);
#pragma unroll
        for (int k = 0; k < W; k++) s2[k * 64 + t] = a.w[k];
    }
    __syncthreads();
    if (t < 32) {  // lane = w*4 + l
        const int i = (t >> 2) * 8 + (t & 3);
        mw::V<W> a, b;
#pragma unroll
        for (int k = 0; k < W; k++) {
            a.w[k] = s2[k * 64 + i];
            b.w[k] = s2[k * 64 + i + 4];
        }
        a = A::add(a, b);                            // level 3: (w, l) + (w, l + 4), l < 4
        a = A::add(a, mw::shfl_down<W>(a, 2));       // level 4: l < 2
        a = A::add(a, mw::shfl_down<W>(a, 1));       // level 5: warp w's sum at lane 4w
        a = A::add(a, mw::shfl_down<W>(a, 16));      // cross-warp: w + (w + 4)
        a = A::add(a, mw::shfl_down<W>(a, 8));       //             w + (w + 2)
        a = A::add(a, mw::shfl_down<W>(a, 4));       //             w + (w + 1)
        v = a;
    }
    __syncthreads();
    return v;
}

#ifndef MWCG_TREE_SHUFFLE
template <int M, int NT>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> block_tree(mw::V<mw::Arith<M>::W> v, double *smem) {
    static_assert(NT == TILE_THREADS, "tile tree");
    return dense_tree<M>(v, smem);
}
template <int M, int NT>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> block_tree_first(mw::V<mw::Arith<M>::W> v, double *smem) {
    static_assert(NT == TILE_THREADS, "tile tree");
    return dense_tree<M>(v, smem);
}
#else
template <int M, int NT>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> block_tree(mw::V<mw::Arith<M>::W> v,
                                                             double *smem /* W*NT/32 */) {
    using A = mw::Arith<M>;
    constexpr int W = A::W;
    constexpr int NW = NT / 32;
    v = warp_tree<M>(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < W; k++) smem[k * NW + wid] = v.w[k];
    }
    __syncthreads();
    if (wid == 0) {
        mw::V<W> u = mw::zero<W>();
        if (lane < NW) {
#pragma unroll
            for (int k = 0; k < W; k++) u.w[k] = smem[k * NW + lane];
        }
#pragma unroll
        for (int off = NW / 2; off >= 1; off >>= 1) {
            auto o = mw::shfl_down<W>(u, off);
            u = A::add(u, o);
        }
        v = u;
    }
    __syncthreads();
    return v;
}

// Same tree, but only the first NT threads of a (possibly larger) block hold
// the values; every thread of the block must call it (it synchronises).
template <int M, int NT>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> block_tree_first(mw::V<mw::Arith<M>::W> v,
                                                                   double *smem /* W*NT/32 */) {
    using A = mw::Arith<M>;
    constexpr int W = A::W;
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (wid < NW) {
        v = warp_tree<M>(v);
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < W; k++) smem[k * NW + wid] = v.w[k];
        }
    }
    __syncthreads();
    if (wid == 0) {
        mw::V<W> u = mw::zero<W>();
        if (lane < NW) {
#pragma unroll
            for (int k = 0; k < W; k++) u.w[k] = smem[k * NW + lane];
        }
#pragma unroll
        for (int off = NW / 2; off >= 1; off >>= 1) {
            auto o = mw::shfl_down<W>(u, off);
            u = A::add(u, o);
        }
        v = u;
    }
    __syncthreads();
    return v;
}

#endif  // MWCG_TREE_SHUFFLE

// Tile-partial layout: rank-blocked word planes.  Word k of global tile t
// lives at part[(t / tb) * (W * tb) + k * tb + t % tb]: the tiles of one rank
// of a row partition (tb = tiles per rank) form ONE contiguous block of W*tb
// doubles, so a multi-GPU gather of the partials is a single all-gather; on
// one GPU tb covers every tile and the layout is plain word planes of
// leading dimension tb.
__device__ __forceinline__ int64_t part_index(int64_t tb, int W, int k, int64_t t) {
    // (a `t < tb ? 0 : t / tb` short cut was measured: it costs the TW / QTW kernels
    // 2-6 % per iteration -- the store of a tile's partial sits in the hot loop)
    const int64_t blk = t / tb;
    return blk * (W * tb) + (int64_t)k * tb + (t - blk * tb);
}
template <int W>
__device__ __forceinline__ void store_part(double *part, int64_t tb, int64_t t, mw::V<W> v) {
#pragma unroll
    for (int k = 0; k < W; k++) part[part_index(tb, W, k, t)] = v.w[k];
}

// Thread t of the reducing block accumulates partials t, t+256, t+512, ...
// in increasing order (the canonical order).  The loads are issued PF at a
// time before the dependent additions, so the serial tail of the last block
// pays one L2 round trip per PF partials instead of one per partial.
template <int M>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> accumulate_partials(const double *part, int64_t ld,
                                                                      int64_t ntiles) {
    using A = TailAdd<M, true>;
    constexpr int W = mw::Arith<M>::W;
    constexpr int PF = 8;
    mw::V<W> acc = mw::zero<W>();
    for (int64_t b = threadIdx.x; b < ntiles; b += (int64_t)PF * TILE_THREADS) {
        mw::V<W> t[PF];
#pragma unroll
        for (int j = 0; j < PF; j++) {
            const int64_t idx = b + (int64_t)j * TILE_THREADS;
#pragma unroll
            for (int k = 0; k < W; k++) t[j].w[k] = idx < ntiles ? __ldcg(part + part_index(ld, W, k, idx)) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < PF; j++)
            if (b + (int64_t)j * TILE_THREADS < ntiles) acc = A::add(acc, t[j]);
    }
    return acc;
}

template <int M>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> reduce_partials_first(const double *part, int64_t ld,
                                                                         int64_t ntiles, double *smem) {
    using A = mw::Arith<M>;
    constexpr int W = A::W;
    mw::V<W> acc = mw::zero<W>();
    if (threadIdx.x < TILE_THREADS) acc = accumulate_partials<M>(part, ld, ntiles);
    return dense_tree<M, true>(acc, smem);
}

// Second pass over ntiles partials (layout above, tile block ld) by one block of
// TILE_THREADS threads; identical procedure to a tile with E=ceil(ntiles/TB).
// Partials written by other CTAs in this grid are read with ld.cg (L2) loads.
template <int M>
__device__ __forceinline__ mw::V<mw::Arith<M>::W> reduce_partials_block(const double *part, int64_t ld,
                                                                         int64_t ntiles, double *smem) {
    return dense_tree<M, true>(accumulate_partials<M>(part, ld, ntiles), smem);
}

// Last-block-done election: returns true in every thread of the block that
// finished last.  The caller must have stored its partial before calling.
__device__ __forceinline__ bool last_block_done(unsigned int *ticket, int *s_flag) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned int t = atomicAdd(ticket, 1u);
        *s_flag = (t == gridDim.x - 1) ? 1 : 0;
    }
    __syncthreads();
    bool last = *s_flag != 0;
    if (last) __threadfence();
    return last;
}

}  // namespace mwcg

// ---------------------------------------------------------------------------
// error plumbing for the C ABI
// ---------------------------------------------------------------------------
namespace mwcg {
void set_error(const char *fmt, ...);
}
#define MWCG_CUDA(call)                                                             \
    do {                                                                            \
        cudaError_t e_ = (call);                                                    \
        if (e_ != cudaSuccess) {                                                    \
            ::mwcg::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,            \
                              cudaGetErrorString(e_));                              \
            return (int)e_;                                                         \
        }                                                                           \
    } while (0)
#define MWCG_CHECK_LAUNCH() MWCG_CUDA(cudaGetLastError())
