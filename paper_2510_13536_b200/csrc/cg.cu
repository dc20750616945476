// cg.cu -- the fused CG iteration (Algorithm 1, cg.py:78-183) on device.
//
// One iteration = three kernels, captured once into a CUDA graph whose body
// sits inside a conditional WHILE node, so a whole segment of iterations runs
// with no host round-trip:
//
//   K1 cg_spmv_pq   q = A p (SELL-32, per-row left-to-right), [every-op: norm q],
//                   p.q tile partials; the last CTA reduces them in the
//                   canonical order and runs the scalar step
//                   (pq breakdown test cg.py:156-158, alpha = rho/pq cg.py:159).
//   K2 cg_update    x += alpha p [norm x], r += (-alpha) q [norm r], r.r tile
//                   partials; last CTA: rho_new, rel (cg.py:167-169), stop /
//                   breakdown tests (cg.py:172-176), beta (cg.py:177), k++,
//                   and the WHILE condition.
//   K3 cg_xpay      p = r + beta p [norm p]   (cg.py:178-180)
//
// Reference-order mode (reduction=partitions, bitwise equal to the reference
// cg_solve(partitions=P)) replaces the fused tile-tree dots by the reference's
// P-partition sequential dots (two extra kernels per dot).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <vector>
#include "ops.cuh"
#include "tma.cuh"
#include "mwcg_internal.h"
#include "../../include/mwcg_cuda.h"

namespace mwcg {

using namespace mw;

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void set_cond(cudaGraphConditionalHandle h, int use_cond, unsigned v) {
    if (use_cond) cudaGraphSetConditional(h, v);
}

// ---------------------------------------------------------------- scalar steps
// The scalar inputs of a step (rho, k, the stop parameters) are loaded by the
// last CTA's thread 0 BEFORE it joins the reduction of the partials, so their
// L2 round trip runs under the reduction instead of after it (the serial
// tail of K1 / K2 is pure latency: DESIGN.md §3).
struct ScalarIn {
    double rho[3];
    long long k, k_stop, max_iters;
    double b_norm, eps;
};
__device__ __forceinline__ ScalarIn scalar_inputs(const CgState *st) {
    ScalarIn in;
    for (int i = 0; i < 3; i++) in.rho[i] = st->rho[i];
    in.k = st->k;
    in.k_stop = st->k_stop;
    in.max_iters = st->max_iters;
    in.b_norm = st->b_norm;
    in.eps = st->eps;
    return in;
}

template <int M>
__device__ void scalar_alpha(CgState *st, V<Arith<M>::W> pq, cudaGraphConditionalHandle h, int use_cond,
                             const ScalarIn *pre = nullptr) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    ScalarIn in = pre ? *pre : scalar_inputs(st);
    for (int k = 0; k < W; k++) st->pq[k] = pq.w[k];
    double pq_f = Ar::collapse(pq);
    if (pq_f == 0.0 || !isfinite(pq_f)) {
        st->status = BREAKDOWN;
        st->iterations = in.k;  // finish(False, "breakdown", k - 1): cg.py:157-158
        set_cond(h, use_cond, 0u);
        return;
    }
    V<W> rho;
    for (int k = 0; k < W; k++) rho.w[k] = in.rho[k];
    V<W> a = Ar::div(rho, pq);
    for (int k = 0; k < W; k++) {
        st->alpha[k] = a.w[k];
        st->neg_alpha[k] = -a.w[k];
    }
}

template <int M>
__device__ void scalar_beta(CgState *st, V<Arith<M>::W> rho_new, cudaGraphConditionalHandle h,
                            int use_cond, const ScalarIn *pre = nullptr) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    ScalarIn in = pre ? *pre : scalar_inputs(st);
    long long k = in.k + 1;
    st->k = k;
    st->x_pending = 1;  // K3 applies x += alpha p (cg.py:162) for this iteration
    for (int i = 0; i < W; i++) st->rho_new[i] = rho_new.w[i];
    double rf = Ar::collapse(rho_new);
    double rel = sqrt(fabs(rf)) / in.b_norm;  // rel_residual: cg.py:125-127
    st->rel = rel;
    if (rel < in.eps) {
        st->status = CONVERGED;
        st->iterations = k;
    } else if (rf == 0.0 || !isfinite(rf)) {
        st->status = BREAKDOWN;
        st->iterations = k;
    } else {
        V<W> rho;
        for (int i = 0; i < W; i++) rho.w[i] = in.rho[i];
        V<W> b = Ar::div(rho_new, rho);
        for (int i = 0; i < W; i++) {
            st->beta[i] = b.w[i];
            st->rho[i] = rho_new.w[i];
        }
        if (k >= in.max_iters) {
            st->status = MAX_ITERS;
            st->iterations = k;
        }
    }
    set_cond(h, use_cond, (st->status == RUNNING && k < in.k_stop) ? 1u : 0u);
}

template <int M>
__device__ void scalar_init(CgState *st, V<Arith<M>::W> rho) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    for (int i = 0; i < W; i++) st->rho[i] = rho.w[i];
    double rel = sqrt(fabs(Ar::collapse(rho))) / st->b_norm;
    st->rel = rel;
    st->k = 0;
    if (rel < st->eps) {  // cg.py:147-148
        st->status = CONVERGED;
        st->iterations = 0;
    } else if (st->max_iters <= 0) {
        st->status = MAX_ITERS;
        st->iterations = st->max_iters;  // finish(False, "max_iterations", max_iters): cg.py:183
    } else {
        st->status = RUNNING;
    }
}

__device__ __forceinline__ bool halted(const CgState *st) { return st->status != RUNNING || st->pause; }

__device__ __forceinline__ bool stopped(const CgState *st, cudaGraphConditionalHandle h, int use_cond) {
    if (halted(st)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(h, use_cond, 0u);
        return true;
    }
    return false;
}

// K1 starts an iteration: it also stops at the pause point k_stop (history
// records), which an unrolled graph body reaches mid-body.
__device__ __forceinline__ bool stopped_k1(CgState *st, cudaGraphConditionalHandle h, int use_cond) {
    if (halted(st)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(h, use_cond, 0u);
        return true;
    }
    if (st->k >= st->k_stop) {  // every block sees the same k, k_stop
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            st->pause = 1;  // read by the body's later kernels only
            set_cond(h, use_cond, 0u);
        }
        return true;
    }
    return false;
}

// Snake order: each kernel walks the tiles in the direction opposite to the
// kernel before it, so its first reads hit the lines the previous kernel
// touched last (still in L2).  Iteration k: SpMV dir = k&1, update = !(k&1),
// xpay (after k++) = !(k'&1) = k&1.  Reduction order is unaffected (partials
// are indexed by tile).
__device__ __forceinline__ int64_t snake(int64_t t, int64_t ntiles, int dir) {
    return dir ? (ntiles - 1 - t) : t;
}

// Geometry of one solver's rows.  Single GPU: n = ld = ldp = n_rows, p_off =
// tile_off = 0, part_ld = ntiles = ntiles_glob, final_ = 1.  Rank r of a row
// partition: local rows / tiles, p a full replica (ldp =
// padded global length) with the local slice at p_off, partials written at
// global tile indices, final_ = 0 (reduced by cg_finalize after the gather).
// The search direction p is stored INTERLEAVED (AoS, record = W words): it is
// the gathered vector, and one record per gather halves (DW) / thirds (TW)
// the sectors a random column costs; x, r, q stay in SoA word planes.
struct Geo {
    int64_t n, ld, ldp, p_off;
    int64_t ntiles, tile_off, part_ld, ntiles_glob;  // part_ld: tile block of the partials (common.cuh)
    int final_;
    // tiles K1 processes: [a0, a1) then [b0, b1) (local indices); all tiles
    // by default, the interior or the boundary set for the overlapped
    // multi-GPU SpMV (mwcg_solver_set_interior)
    int64_t a0, a1, b0, b1;
    // column-blocked K1 (sell.cu): this launch starts every row from the
    // running sum left in q by the previous block (acc_in) and / or leaves
    // its running sum there for the next one (acc_out: no p.q, no scalar step)
    int acc_in, acc_out;
};
__device__ __forceinline__ int64_t k1_count(const Geo &g) { return (g.a1 - g.a0) + (g.b1 - g.b0); }
__device__ __forceinline__ int64_t k1_tile(const Geo &g, int64_t t) {
    return t < g.a1 - g.a0 ? g.a0 + t : g.b0 + (t - (g.a1 - g.a0));
}

// Persistent tile loop: every fused kernel runs grid = min(ntiles, resident
// CTAs) blocks, block b handling tiles b, b+grid, ...  Partials are indexed by
// tile, so the reduction order is independent of the grid size.
//
// ---------------------------------------------------------------- K1
// K1: one tile (1024 rows) per CTA of SP_THREADS(M) threads, each thread
// walking 1024/SP_THREADS rows of the tile (row = tile*1024 + tid + k*THREADS).
// High occupancy is what keeps enough loads in flight (Little's law; see
// DESIGN.md "SpMV").  The p.q terms of the tile are staged in shared memory
// and the canonical tile order (thread t: terms t, t+256, t+512, t+768, then
// the 256-thread tree) is replayed by the first 256 threads, so the thread
// mapping of the SpMV is free while the reduction order stays canonical.
template <int M>
struct SpTraits {
#ifdef MWCG_SP_THREADS_OVERRIDE
    static constexpr int THREADS = MWCG_SP_THREADS_OVERRIDE;
#else
    static constexpr int THREADS = (M == FP64) ? 512 : 256;
#endif
#ifdef MWCG_SP_MINB_OVERRIDE
    static constexpr int MINB = MWCG_SP_MINB_OVERRIDE;
#else
    // 4 CTAs of 256 threads (64 registers): the row walk holds a chunk of
    // records and gathers plus the running sums without spilling (DW C2 K1
    // 49.5 us at 5 CTAs / 48 registers, 43.4 us at 4 / 64)
    static constexpr int MINB = (M == FP64) ? 3 : 4;
#endif
    static constexpr int RPT = TILE / THREADS;
#ifdef MWCG_SP_U_OVERRIDE
    static constexpr int U = MWCG_SP_U_OVERRIDE;
#else
    static constexpr int U = (M == FP64) ? 8 : ((M == TW) ? 3 : 4);  // measured per mode (C2)
#endif
    // rows of a thread walked in pairs when they share a uniform pattern
    // (ops.cuh: spmv_pair_dia); UP: slots per chunk of a pair (<= 4), 0: off
#ifdef MWCG_SP_PAIR_OVERRIDE
    static constexpr int UP = MWCG_SP_PAIR_OVERRIDE;
#else
    static constexpr int UP = 0;
#endif
    // chunk of a value-uniform slice (no value registers: ops.cuh)
#ifdef MWCG_SP_UU_OVERRIDE
    static constexpr int UU = MWCG_SP_UU_OVERRIDE;
#else
    static constexpr int UU = U;
#endif
};

template <int M, bool FUSED, typename CT>
__global__ void __launch_bounds__(SpTraits<M>::THREADS, SpTraits<M>::MINB)
    cg_spmv_pq(SellMatrix A, const double *__restrict__ p, double *__restrict__ q, Geo g,
               double *__restrict__ part, CgState *st, cudaGraphConditionalHandle h, int use_cond) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    constexpr int NT = SpTraits<M>::THREADS;
    // 256 threads: thread t owns rows t + 256 j, which IS the canonical tile
    // mapping, so its p.q terms accumulate in registers in canonical order;
    // 512 threads (FP64) and the SELL layouts (whose rows may be sorted by
    // length inside the tile: SELL-sigma) stage the terms in shared memory by
    // natural row, and the first 256 threads replay the canonical order
    constexpr bool STAGE = FUSED && (NT != TILE_THREADS || !std::is_same<CT, DiaTag>::value);
    constexpr bool BLK = std::is_same<CT, int32_t>::value;  // the layout column blocks use
    __shared__ double terms[STAGE ? W * TILE : 1];
    __shared__ double smem[tree_smem<W>()];
    __shared__ int s_last;
    if (stopped_k1(st, h, use_cond)) return;
    const bool norm_all = st->norm_all != 0;
    // rows < 2^31 (sell_create): tile and row indices are 32-bit, so the
    // per-row address arithmetic is one wide multiply-add per access
    const int n = (int)g.n;
    const int dir = (int)(st->k & 1);
    const int cnt = (int)k1_count(g), cnt_a = (int)(g.a1 - g.a0);
    const double *__restrict__ pl = p + g.p_off * W;  // the local slice of p (AoS)
    for (int t = blockIdx.x; t < cnt; t += gridDim.x) {
        const int ts = dir ? cnt - 1 - t : t;  // snake order
        const int tile = ts < cnt_a ? (int)g.a0 + ts : (int)g.b0 + (ts - cnt_a);
        // storage position of the thread's current row; the tile and the row
        // count are read back from it (tile = pos >> 10, last row when
        // pos + NT leaves the tile), so the row loop carries one index
        int pos = tile * TILE + (int)threadIdx.x;
        SliceWords sw = slice_words<CT>(A, pos);
        V<W> acc = zero<W>();
        constexpr int UP = SpTraits<M>::UP;
        if constexpr (UP > 0 && std::is_same<CT, DiaTag>::value && !STAGE && FUSED && (TILE / NT) % 2 == 0) {
            // pairs (pos, pos + NT): canonical p.q order kept (A's term, then B's)
#pragma unroll 1
            for (int k = 0; k < TILE / NT; k += 2, pos += 2 * NT) {
                const int pb = pos + NT;
                const SliceWords swa = k ? slice_words<CT>(A, pos) : sw;
                const SliceWords swb = slice_words<CT>(A, pb);
                V<W> sa = zero<W>(), sb = zero<W>();
                bool done = false;
                if (pb < n) done = spmv_pair_dia<M, UP, true>(A, p, 0, pos, pb, swa, swb, sa, sb);
                if (!done) {
                    if (pos < n) sa = spmv_row<M, SpTraits<M>::U, CT, true, SpTraits<M>::UU>(A, p, 0, pos, swa);
                    if (pb < n) sb = spmv_row<M, SpTraits<M>::U, CT, true, SpTraits<M>::UU>(A, p, 0, pb, swb);
                }
                if (pos < n) {
                    if (norm_all) sa = Ar::norm(sa);
                    acc = Ar::add(acc, Ar::mul(load_aos_ro<W>(pl + (int64_t)pos * W, 0), sa));
                    store<W>(q + pos, g.ld, 0, sa);
                }
                if (pb < n) {
                    if (norm_all) sb = Ar::norm(sb);
                    acc = Ar::add(acc, Ar::mul(load_aos_ro<W>(pl + (int64_t)pb * W, 0), sb));
                    store<W>(q + pb, g.ld, 0, sb);
                }
            }
            pos -= NT;  // the tile is read back from pos below
        } else
#pragma unroll 1
        for (;;) {
            const bool more = ((pos + NT) >> 10) == (pos >> 10);
            V<W> term = zero<W>();
            const int row = std::is_same<CT, DiaTag>::value ? pos : (int)sell_row(A, pos);
            if (pos < n) {
                // columns are global: p is the full (replicated) vector
                V<W> sv;
                if constexpr (BLK) {
                    V<W> s0 = zero<W>();
                    if (g.acc_in) s0 = load<W>(q + row, g.ld, 0);
                    sv = spmv_row_sell<M, SpTraits<M>::U, CT, true>(A, p, 0, pos, sw, s0);
                } else {
                    sv = spmv_row<M, SpTraits<M>::U, CT, true, SpTraits<M>::UU>(A, p, 0, pos, sw);
                }
                // the next row's slice words head its dependency chain: their
                // load is issued here, under this row's p.q term
                if (more) sw = slice_words<CT>(A, pos + NT);
                MWCG_ASSERT(row >= 0 && row < n && (row >> 10) == (pos >> 10));
                if (!BLK || !g.acc_out) {
                    if (norm_all) sv = Ar::norm(sv);
                    if (FUSED) term = Ar::mul(load_aos_ro<W>(pl + (int64_t)row * W, 0), sv);
                    if (FUSED && !STAGE) acc = Ar::add(acc, term);
                }
                store<W>(q + row, g.ld, 0, sv);
            } else if (more) {
                sw = slice_words<CT>(A, pos + NT);
            }
            if (STAGE && !(BLK && g.acc_out)) {
#pragma unroll
                for (int w = 0; w < W; w++) terms[w * TILE + (row & (TILE - 1))] = term.w[w];
            }
            if (!more) break;
            pos += NT;
        }
        const int tile2 = pos >> 10;
        if (BLK && g.acc_out) continue;  // grid-uniform: this block only carries the sums
        if (STAGE) {
            __syncthreads();
            if (threadIdx.x < TILE_THREADS) {
                const int base = tile2 * TILE + (int)threadIdx.x;
#pragma unroll
                for (int j = 0; j < TILE_ELEMS; j++) {
                    if (base + j * TILE_THREADS < n) {
                        V<W> t;
#pragma unroll
                        for (int w = 0; w < W; w++) t.w[w] = terms[w * TILE + threadIdx.x + j * TILE_THREADS];
                        acc = Ar::add(acc, t);
                    }
                }
            }
        }
        if (FUSED) {
            acc = block_tree_first<M, TILE_THREADS>(acc, smem);
            if (threadIdx.x == 0) store_part<W>(part, g.part_ld, g.tile_off + tile2, acc);
        }
    }
    if (!FUSED || !g.final_ || (BLK && g.acc_out)) return;
    if (!last_block_done(&st->ticket[0], &s_last)) return;
    ScalarIn in{};
    if (threadIdx.x == 0) in = scalar_inputs(st);
    V<W> pq = reduce_partials_first<M>(part, g.part_ld, g.ntiles_glob, smem);
    if (threadIdx.x == 0) {
        st->ticket[0] = 0u;
        scalar_alpha<M>(st, pq, h, use_cond, &in);
    }
}

// ---------------------------------------------------------------- K2
// r += (-alpha) q [norm r], r.r tile partials; last CTA: beta and the stop
// tests.  The x update (cg.py:162) needs only alpha and the OLD p, so it is
// deferred to K3, which reads p anyway: K2 streams 3 vector passes (r, q in;
// r out) instead of 6, and K3 5 instead of 3 -- one p pass fewer per
// iteration.  Elementwise operations and their inputs are unchanged, so
// every bit of x is too.
//
// Loads are hoisted HOIST elements at a time (all loads of a group issue
// before any arithmetic).  TW is FP64-bound: no hoisting, registers go to
// occupancy instead.
template <int M>
struct Hoist {
#ifdef MWCG_UP_HOIST_OVERRIDE
    static constexpr int value = (M == TW) ? 1 : MWCG_UP_HOIST_OVERRIDE;
#else
    static constexpr int value = (M == TW) ? 1 : TILE_ELEMS;
#endif
#ifdef MWCG_UP_MINB_OVERRIDE
    static constexpr int MINB = MWCG_UP_MINB_OVERRIDE;
#else
    // an explicit minimum is needed: with (256, 1) ptxas spends up to 255
    // registers and halves occupancy
    static constexpr int MINB = (M == TW) ? 3 : 2;
#endif
};

template <int M, bool FUSED>
__global__ void __launch_bounds__(TILE_THREADS, Hoist<M>::MINB)
    cg_update(double *__restrict__ r, const double *__restrict__ q, Geo g, double *__restrict__ part,
              CgState *st, cudaGraphConditionalHandle h, int use_cond) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    constexpr int H = Hoist<M>::value;
    __shared__ double smem[tree_smem<W>()];
    __shared__ int s_last;
    if (stopped(st, h, use_cond)) return;
    const bool norm_r = st->norm_r != 0;
    V<W> nalpha;
#pragma unroll
    for (int k = 0; k < W; k++) nalpha.w[k] = st->neg_alpha[k];
    const int64_t n = g.n, ld = g.ld;
    const int dir = (int)((st->k & 1) ^ 1);
    for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
        const int64_t tile = snake(t, g.ntiles, dir);
        const int64_t base = tile * TILE + threadIdx.x;
        V<W> acc = zero<W>();
#pragma unroll
        for (int j0 = 0; j0 < TILE_ELEMS; j0 += H) {
            V<W> rv[H], qv[H];
#pragma unroll
            for (int h2 = 0; h2 < H; h2++) {
                int64_t i = base + (j0 + h2) * TILE_THREADS;
                if (i < n) {
                    rv[h2] = load<W>(r, ld, i);
                    qv[h2] = load_ro<W>(q, ld, i);
                }
            }
#pragma unroll
            for (int h2 = 0; h2 < H; h2++) {
                int64_t i = base + (j0 + h2) * TILE_THREADS;
                if (i < n) {
                    V<W> ri = Ar::add(rv[h2], Ar::mul(nalpha, qv[h2]));
                    if (norm_r) ri = Ar::norm(ri);
                    store<W>(r, ld, i, ri);
                    if (FUSED) acc = Ar::add(acc, Ar::mul(ri, ri));
                }
            }
        }
        if (FUSED) {
            acc = block_tree<M, TILE_THREADS>(acc, smem);
            if (threadIdx.x == 0) store_part<W>(part, g.part_ld, g.tile_off + tile, acc);
        }
    }
    if (!FUSED || !g.final_) return;
    if (!last_block_done(&st->ticket[1], &s_last)) return;
    ScalarIn in{};
    if (threadIdx.x == 0) in = scalar_inputs(st);
    V<W> rn = reduce_partials_block<M>(part, g.part_ld, g.ntiles_glob, smem);
    if (threadIdx.x == 0) {
        st->ticket[1] = 0u;
        scalar_beta<M>(st, rn, h, use_cond, &in);
    }
}

// ---------------------------------------------------------------- K3
// x += alpha p_old [norm x] (cg.py:162-164, deferred from K2) whenever K2 ran
// this iteration (x_pending, set by scalar_beta) -- also on the iteration
// that converges or breaks down after the x update, as the reference does --
// and p = r + beta p [norm p] (cg.py:178-180) while the solve is running.
// The last CTA clears x_pending.
__device__ __forceinline__ bool k3_begin(CgState *st, cudaGraphConditionalHandle h, int use_cond, bool &do_p) {
    if (!st->x_pending) {
        if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(h, use_cond, 0u);
        return false;
    }
    do_p = !halted(st);
    if (!do_p && blockIdx.x == 0 && threadIdx.x == 0) set_cond(h, use_cond, 0u);
    return true;
}

__device__ __forceinline__ void k3_end(CgState *st, int *s_last) {
    if (last_block_done(&st->ticket[3], s_last) && threadIdx.x == 0) {
        st->ticket[3] = 0u;
        st->x_pending = 0;
    }
}

template <int M, bool DO_P>
__device__ __forceinline__ void k3_element(double *__restrict__ x, double *__restrict__ pl, int64_t ld, int64_t i,
                                           V<Arith<M>::W> rv, V<Arith<M>::W> pv, V<Arith<M>::W> xv,
                                           const V<Arith<M>::W> &alpha, const V<Arith<M>::W> &beta,
                                           bool norm_all) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    V<W> xi = Ar::add(xv, Ar::mul(alpha, pv));
    if (norm_all) xi = Ar::norm(xi);
    store<W>(x, ld, i, xi);
    if (DO_P) {
        V<W> pi = Ar::add(rv, Ar::mul(beta, pv));
        if (norm_all) pi = Ar::norm(pi);
        store_aos<W>(pl, i, pi);
    }
}

template <int M>
struct XpHoist {
#ifdef MWCG_XP_HOIST_OVERRIDE
    static constexpr int value = MWCG_XP_HOIST_OVERRIDE;
#else
    static constexpr int value = (M == TW) ? 1 : TILE_ELEMS;  // TW: FP64-bound, occupancy first
#endif
#ifdef MWCG_XP_MINB_OVERRIDE
    static constexpr int MINB = MWCG_XP_MINB_OVERRIDE;
#else
    static constexpr int MINB = (M == TW) ? 3 : ((M == QTW) ? 2 : 1);
#endif
};

template <int M>
__global__ void __launch_bounds__(TILE_THREADS, XpHoist<M>::MINB)
    cg_xpay(double *__restrict__ x, double *__restrict__ p, const double *__restrict__ r, Geo g, CgState *st,
            cudaGraphConditionalHandle h, int use_cond) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    constexpr int H = XpHoist<M>::value;
    __shared__ int s_last;
    bool do_p = false;
    if (!k3_begin(st, h, use_cond, do_p)) return;
    const bool norm_all = st->norm_all != 0;
    V<W> alpha, beta;
#pragma unroll
    for (int k = 0; k < W; k++) {
        alpha.w[k] = st->alpha[k];
        beta.w[k] = st->beta[k];
    }
    const int64_t n = g.n, ld = g.ld;
    double *__restrict__ pl = p + g.p_off * W;
    const int dir = (int)((st->k & 1) ^ 1);
    for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
        const int64_t tile = snake(t, g.ntiles, dir);
        const int64_t base = tile * TILE + threadIdx.x;
#pragma unroll
        for (int j0 = 0; j0 < TILE_ELEMS; j0 += H) {
            V<W> rv[H], pv[H], xv[H];
#pragma unroll
            for (int j = 0; j < H; j++) {
                int64_t i = base + (j0 + j) * TILE_THREADS;
                if (i < n) {
                    if (do_p) rv[j] = load_ro<W>(r, ld, i);
                    pv[j] = load_aos<W>(pl, i);
                    xv[j] = load<W>(x, ld, i);
                }
            }
#pragma unroll
            for (int j = 0; j < H; j++) {
                int64_t i = base + (j0 + j) * TILE_THREADS;
                if (i < n) {
                    if (do_p) k3_element<M, true>(x, pl, ld, i, rv[j], pv[j], xv[j], alpha, beta, norm_all);
                    else k3_element<M, false>(x, pl, ld, i, rv[j], pv[j], xv[j], alpha, beta, norm_all);
                }
            }
        }
    }
    k3_end(st, &s_last);
}

// ---------------------------------------------------------------- TMA-staged K2 / K3
// The vector passes are pure streams: each tile's operands (word planes, the
// AoS slice of p) are contiguous 8-KB runs, so one thread issues them as 1-D
// bulk copies (cp.async.bulk) into a shared-memory ring of NS stages and the
// copy engine, not registers, holds the bytes in flight.  One CTA of
// TILE_THREADS threads per SM; the canonical tile mapping (thread t: elements
// t + j*256) and the canonical r.r tree are unchanged, so results are bitwise
// those of cg_update / cg_xpay.  A partial last tile is read with plain loads
// (its stage is completed by a plain arrive, so the ring's phase bits stay in
// step).  Requires 16-B aligned planes (ld even).
template <int M>
struct UpTma {
    static constexpr int W = Arith<M>::W;
    static constexpr int STAGE = 2 * W * TILE;  // doubles: r, q planes
#ifdef MWCG_UP_NS
    static constexpr int NS = MWCG_UP_NS;
#else
    // 2 stages: 2-3 CTAs per SM (measured better than a deeper ring in one CTA:
    // the per-tile r.r tree needs the extra warps)
    static constexpr int NS = 2;
#endif
    static constexpr size_t SMEM = sizeof(double) * STAGE * NS;
#ifdef MWCG_UP_TMA_MINB
    static constexpr int MINB = MWCG_UP_TMA_MINB;
#else
    // keeps the 2-word modes at 3 CTAs per SM (<= 85 registers) and the 3-word
    // ones at 2: left to itself ptxas takes 94 registers for DW and drops a CTA
    // (C3 / C4 DW +7-9 % per iteration)
    static constexpr int MINB = (W <= 2) ? 3 : 2;
#endif
};
template <int M>
struct XpTma {
    static constexpr int W = Arith<M>::W;
    static constexpr int STAGE = 3 * W * TILE;  // r, x planes + p AoS
#ifdef MWCG_XP_NS
    static constexpr int NS = MWCG_XP_NS;
#else
    static constexpr int NS = (M == FP64) ? 4 : (W == 2 ? 3 : 2);
#endif
    static constexpr size_t SMEM = sizeof(double) * STAGE * NS;
};

// issue the bulk copies of one tile: NP word-plane groups of W planes
// (srcs[0..NP-1]) then, if pl, the AoS slice of p; a partial tile arrives
// without transactions
template <int W, int NP>
__device__ __forceinline__ void tile_issue(double *stage, uint64_t *bar, const double *const (&srcs)[NP],
                                           const double *pl, int64_t ld, int64_t tile, bool full) {
    if (!full) {
        mbar_arrive(bar);
        return;
    }
    constexpr uint32_t PB = TILE * sizeof(double);
    mbar_arrive_expect_tx(bar, (uint32_t)(NP * W + (pl ? W : 0)) * PB);
    const int64_t e0 = tile * TILE;
#pragma unroll
    for (int v = 0; v < NP; v++)
#pragma unroll
        for (int k = 0; k < W; k++) bulk_g2s(stage + (v * W + k) * TILE, srcs[v] + k * ld + e0, PB, bar);
    if (pl) bulk_g2s(stage + NP * W * TILE, pl + e0 * W, W * PB, bar);
}

template <int M, bool FUSED>
__global__ void __launch_bounds__(TILE_THREADS, UpTma<M>::MINB)
    cg_update_tma(double *__restrict__ r, const double *__restrict__ q, Geo g, double *__restrict__ part,
                  CgState *st, cudaGraphConditionalHandle h, int use_cond) {
    using Ar = Arith<M>;
    using T = UpTma<M>;
    constexpr int W = Ar::W;
    extern __shared__ __align__(128) double ring[];
    __shared__ uint64_t bar[T::NS];
    __shared__ double smem[tree_smem<W>()];
    __shared__ int s_last;
    if (stopped(st, h, use_cond)) return;
    const bool norm_r = st->norm_r != 0;
    V<W> nalpha;
#pragma unroll
    for (int k = 0; k < W; k++) nalpha.w[k] = st->neg_alpha[k];
    const int64_t n = g.n, ld = g.ld;
    const int dir = (int)((st->k & 1) ^ 1);
    const int64_t nmine = g.ntiles > blockIdx.x ? (g.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const double *const srcs[2] = {r, q};
    if (threadIdx.x == 0) {
        for (int i = 0; i < T::NS; i++) mbar_init(&bar[i], 1);
        mbar_init_fence();
        for (int64_t i = 0; i < T::NS && i < nmine; i++) {
            const int64_t tile = snake(blockIdx.x + i * gridDim.x, g.ntiles, dir);
            tile_issue<W, 2>(ring + i * T::STAGE, &bar[i], srcs, nullptr, ld, tile, (tile + 1) * TILE <= n);
        }
    }
    __syncthreads();
    for (int64_t i = 0; i < nmine; i++) {
        const int64_t tile = snake(blockIdx.x + i * gridDim.x, g.ntiles, dir);
        const int sidx = (int)(i % T::NS);
        const double *sg = ring + sidx * T::STAGE;
        const bool full = (tile + 1) * TILE <= n;
        mbar_wait(&bar[sidx], (uint32_t)((i / T::NS) & 1));
        const int64_t base = tile * TILE + threadIdx.x;
        V<W> acc = zero<W>();
#pragma unroll
        for (int j = 0; j < TILE_ELEMS; j++) {
            const int li = threadIdx.x + j * TILE_THREADS;
            const int64_t e = base + j * TILE_THREADS;
            V<W> rv, qv;
            if (full) {
#pragma unroll
                for (int k = 0; k < W; k++) {
                    rv.w[k] = sg[(0 * W + k) * TILE + li];
                    qv.w[k] = sg[(1 * W + k) * TILE + li];
                }
            } else if (e < n) {
                rv = load<W>(r, ld, e);
                qv = load_ro<W>(q, ld, e);
            }
            if (e < n) {
                V<W> ri = Ar::add(rv, Ar::mul(nalpha, qv));
                if (norm_r) ri = Ar::norm(ri);
                store<W>(r, ld, e, ri);
                if (FUSED) acc = Ar::add(acc, Ar::mul(ri, ri));
            }
        }
        __syncthreads();  // every thread is done reading stage sidx
        if (threadIdx.x == 0 && i + T::NS < nmine) {
            fence_proxy_async_smem();
            const int64_t nt = snake(blockIdx.x + (i + T::NS) * gridDim.x, g.ntiles, dir);
            tile_issue<W, 2>(ring + sidx * T::STAGE, &bar[sidx], srcs, nullptr, ld, nt, (nt + 1) * TILE <= n);
        }
        if (FUSED) {
            acc = block_tree<M, TILE_THREADS>(acc, smem);
            if (threadIdx.x == 0) store_part<W>(part, g.part_ld, g.tile_off + tile, acc);
        }
    }
    if (!FUSED || !g.final_) return;
    if (!last_block_done(&st->ticket[1], &s_last)) return;
    ScalarIn in{};
    if (threadIdx.x == 0) in = scalar_inputs(st);
    V<W> rn = reduce_partials_block<M>(part, g.part_ld, g.ntiles_glob, smem);
    if (threadIdx.x == 0) {
        st->ticket[1] = 0u;
        scalar_beta<M>(st, rn, h, use_cond, &in);
    }
}

template <int M>
__global__ void __launch_bounds__(TILE_THREADS, 1)
    cg_xpay_tma(double *__restrict__ x, double *__restrict__ p, const double *__restrict__ r, Geo g, CgState *st,
                cudaGraphConditionalHandle h, int use_cond) {
    using Ar = Arith<M>;
    using T = XpTma<M>;
    constexpr int W = Ar::W;
    extern __shared__ __align__(128) double ring[];
    __shared__ uint64_t bar[T::NS];
    __shared__ int s_last;
    bool do_p = false;
    if (!k3_begin(st, h, use_cond, do_p)) return;
    const bool norm_all = st->norm_all != 0;
    V<W> alpha, beta;
#pragma unroll
    for (int k = 0; k < W; k++) {
        alpha.w[k] = st->alpha[k];
        beta.w[k] = st->beta[k];
    }
    const int64_t n = g.n, ld = g.ld;
    double *__restrict__ pl = p + g.p_off * W;
    const int dir = (int)((st->k & 1) ^ 1);
    const int64_t nmine = g.ntiles > blockIdx.x ? (g.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const double *const srcs[2] = {r, x};
    if (threadIdx.x == 0) {
        for (int i = 0; i < T::NS; i++) mbar_init(&bar[i], 1);
        mbar_init_fence();
        for (int64_t i = 0; i < T::NS && i < nmine; i++) {
            const int64_t tile = snake(blockIdx.x + i * gridDim.x, g.ntiles, dir);
            tile_issue<W, 2>(ring + i * T::STAGE, &bar[i], srcs, pl, ld, tile, (tile + 1) * TILE <= n);
        }
    }
    __syncthreads();
    for (int64_t i = 0; i < nmine; i++) {
        const int64_t tile = snake(blockIdx.x + i * gridDim.x, g.ntiles, dir);
        const int sidx = (int)(i % T::NS);
        const double *sg = ring + sidx * T::STAGE;
        const bool full = (tile + 1) * TILE <= n;
        mbar_wait(&bar[sidx], (uint32_t)((i / T::NS) & 1));
        const int64_t base = tile * TILE + threadIdx.x;
#pragma unroll
        for (int j = 0; j < TILE_ELEMS; j++) {
            const int li = threadIdx.x + j * TILE_THREADS;
            const int64_t e = base + j * TILE_THREADS;
            V<W> rv, xv, pv;
            if (full) {
#pragma unroll
                for (int k = 0; k < W; k++) {
                    rv.w[k] = sg[(0 * W + k) * TILE + li];
                    xv.w[k] = sg[(1 * W + k) * TILE + li];
                    pv.w[k] = sg[2 * W * TILE + li * W + k];
                }
            } else if (e < n) {
                rv = load_ro<W>(r, ld, e);
                xv = load<W>(x, ld, e);
                pv = load_aos<W>(pl, e);
            }
            if (e < n) {
                if (do_p) k3_element<M, true>(x, pl, ld, e, rv, pv, xv, alpha, beta, norm_all);
                else k3_element<M, false>(x, pl, ld, e, rv, pv, xv, alpha, beta, norm_all);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && i + T::NS < nmine) {
            fence_proxy_async_smem();
            const int64_t nt = snake(blockIdx.x + (i + T::NS) * gridDim.x, g.ntiles, dir);
            tile_issue<W, 2>(ring + sidx * T::STAGE, &bar[sidx], srcs, pl, ld, nt, (nt + 1) * TILE <= n);
        }
    }
    k3_end(st, &s_last);
}

// ---------------------------------------------------------------- init
// r = b - q (residual, cg.py:114), [norm r] (cg.py:115-116), p = r (117),
// rho = r.r (118), rel, converged-at-0 test (147-148).
template <int M, bool FUSED>
__global__ void __launch_bounds__(TILE_THREADS)
    cg_init(const double *__restrict__ b, const double *__restrict__ q, double *__restrict__ r,
            double *__restrict__ p, Geo g, double *__restrict__ part, CgState *st) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    __shared__ double smem[tree_smem<W>()];
    __shared__ int s_last;
    const bool norm_r = st->norm_r != 0;
    const int64_t n = g.n, ld = g.ld;
    double *__restrict__ pl = p + g.p_off * W;
    for (int64_t tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x) {
        const int64_t base = tile * TILE + threadIdx.x;
        V<W> acc = zero<W>();
#pragma unroll
        for (int j = 0; j < TILE_ELEMS; j++) {
            int64_t i = base + j * TILE_THREADS;
            if (i < n) {
                V<W> ri = Ar::dxadd(b[i], neg<W>(load<W>(q, ld, i)));
                if (norm_r) ri = Ar::norm(ri);
                store<W>(r, ld, i, ri);
                store_aos<W>(pl, i, ri);
                if (FUSED) acc = Ar::add(acc, Ar::mul(ri, ri));
            }
        }
        if (FUSED) {
            acc = block_tree<M, TILE_THREADS>(acc, smem);
            if (threadIdx.x == 0) store_part<W>(part, g.part_ld, g.tile_off + tile, acc);
        }
    }
    if (!FUSED || !g.final_) return;
    if (!last_block_done(&st->ticket[2], &s_last)) return;
    V<W> rho = reduce_partials_block<M>(part, g.part_ld, g.ntiles_glob, smem);
    if (threadIdx.x == 0) {
        st->ticket[2] = 0u;
        scalar_init<M>(st, rho);
    }
}

// ---------------------------------------------------------------- dist start
// p (AoS, full replica) <- x0 word 0; q = A p for the local rows (no
// normalisation: cg.py:113 applies none to the initial q)
template <int W>
__global__ void spread_x0_kernel(int64_t n, const double *__restrict__ x0, double *__restrict__ p) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        V<W> v = zero<W>();
        v.w[0] = x0 ? x0[i] : 0.0;
        store_aos<W>(p, i, v);
    }
}

template <int M, typename CT>
__global__ void __launch_bounds__(TILE_THREADS)
    spmv_aos_kernel(SellMatrix A, const double *__restrict__ p, double *__restrict__ q, int64_t ldq) {
    constexpr int W = Arith<M>::W;
    for (int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < A.n_rows;
         pos += (int64_t)gridDim.x * blockDim.x)
        store<W>(q, ldq, sell_row(A, pos), spmv_row<M, 8, CT, true>(A, p, 0, pos));
}

// ---------------------------------------------------------------- finalize (multi-rank)
// After the tile partials of every rank have been gathered, one block reduces
// all global tiles in the canonical order and runs the scalar step -- the
// same procedure as the fused last-block path, so R ranks reproduce the
// 1-GPU result bit for bit.  phase 0: init (rho), 1: alpha (p.q), 2: beta.
template <int M>
__global__ void __launch_bounds__(TILE_THREADS)
    cg_finalize(const double *__restrict__ part, Geo g, CgState *st, int phase) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    __shared__ double smem[tree_smem<W>()];
    if (phase != 0 && halted(st)) return;
    V<W> v = reduce_partials_block<M>(part, g.part_ld, g.ntiles_glob, smem);
    if (threadIdx.x == 0) {
        cudaGraphConditionalHandle h{};
        if (phase == 0) scalar_init<M>(st, v);
        else if (phase == 1) scalar_alpha<M>(st, v, h, 0);
        else scalar_beta<M>(st, v, h, 0);
    }
}

// ---------------------------------------------------------------- reference-order dots
template <int M, bool XAOS>
__global__ void cg_dot_part(int64_t n, const double *__restrict__ x, const double *__restrict__ y,
                            int64_t ld, int64_t parts, double *__restrict__ part, const CgState *st,
                            int check_status) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    if (check_status && halted(st)) return;
    int64_t pidx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pidx >= parts) return;
    int64_t lo = (int64_t)(((__int128)n * pidx) / parts);
    int64_t hi = (int64_t)(((__int128)n * (pidx + 1)) / parts);
    V<W> t = zero<W>();
    for (int64_t i = lo; i < hi; i++)
        t = Ar::add(t, Ar::mul(XAOS ? load_aos<W>(x, i) : load<W>(x, ld, i), load<W>(y, ld, i)));
    store<W>(part, parts, pidx, t);
}

// phase 0: init (rho), 1: alpha (pq), 2: beta (rho_new)
template <int M>
__global__ void cg_ref_combine(const double *__restrict__ part, int64_t parts, CgState *st, int phase,
                               cudaGraphConditionalHandle h, int use_cond) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    if (phase != 0 && halted(st)) {
        set_cond(h, use_cond, 0u);
        return;
    }
    V<W> s = load<W>(part, parts, 0);
    for (int64_t pi = 1; pi < parts; pi++) s = Ar::add(s, load<W>(part, parts, pi));
    if (phase == 0) scalar_init<M>(st, s);
    else if (phase == 1) scalar_alpha<M>(st, s, h, use_cond);
    else scalar_beta<M>(st, s, h, use_cond);
}

// ---------------------------------------------------------------- history metrics
// norm_metrics_tw (kernels.py:305-328): x promoted to TW (107-112), TW SpMV,
// TW residual b - Ax, and x* - x; the TW sums of squares use the solver's
// reduction shape (tile tree, or partitions=1 in reference-order mode,
// matching _tw_norm_sq kernels.py:299-302).
template <int M>
__global__ void promote_kernel(int64_t n, const double *__restrict__ x, int64_t ldx,
                               double *__restrict__ xt) {
    constexpr int W = Arith<M>::W;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int k = 0; k < 3; k++) xt[k * n + i] = k < W ? x[k * ldx + i] : 0.0;
    }
}

__global__ void promote_fp64_kernel(int64_t n, const double *__restrict__ v, double *__restrict__ vt) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        vt[i] = v[i];
        vt[n + i] = 0.0;
        vt[2 * n + i] = 0.0;
    }
}

template <typename CT>
__global__ void __launch_bounds__(TILE_THREADS)
    metrics_vec_kernel(SellMatrix A, const double *__restrict__ xt, const double *__restrict__ b,
                       const double *__restrict__ xs, double *__restrict__ res, double *__restrict__ diff) {
    const int64_t n = A.n_rows;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = sell_row(A, i);  // i: storage position of a row
        V<3> qi = spmv_row<TW, 8, CT>(A, xt, n, i);
        store<3>(res, n, r, dxtw_add(b[r], neg<3>(qi)));
        if (xs) store<3>(diff, n, i, dxtw_add(xs[i], neg<3>(load<3>(xt, n, i))));
    }
}

}  // namespace mwcg

// =====================================================================
// Host runtime
// =====================================================================
using namespace mwcg;

struct mwcg_matrix {
    SellMatrixOwned *M;
    std::vector<SellMatrixOwned *> blocks;  // column blocks for K1 (sell.cu); empty: none
};

struct mwcg_solver {
    SellMatrix A{};
    std::vector<SellMatrix> blocks;      // column blocks of A (K1 walks them in turn); empty: none
    std::vector<int64_t> block_col0;     // first column of each block (+ n_cols at the end)
    int mode = 0, W = 1;
    mwcg_solver_config cfg{};
    int64_t n = 0, ntiles = 0, parts = 1;
    bool fused = true;
    int unroll = 8;  // CG iterations per WHILE-body run (MWCG_UNROLL)
    cudaStream_t stream = nullptr;       // caller's stream (all work ordered on it)
    cudaStream_t cap = nullptr;          // private stream for graph capture
    double *x = nullptr, *r = nullptr, *p = nullptr, *q = nullptr;
    bool own_x = false;
    double *part = nullptr;
    CgState *st = nullptr;
    CgState *st_host = nullptr;          // pinned mirror
    long long *kstop_host = nullptr;     // pinned
    const double *b = nullptr, *x_star = nullptr;
    // metrics scratch
    double *xt = nullptr, *res = nullptr, *diff = nullptr, *bt = nullptr;
    double *mpart = nullptr, *mout = nullptr, *mout_host = nullptr;
    unsigned int *mticket = nullptr;
    double bnorm_sq = 1.0, xs_sq = 1.0;
    bool norms_ready = false;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphConditionalHandle cond{};
    cudaEvent_t ev[8] = {};
    unsigned grid[4] = {1, 1, 1, 1};  // spmv_pq, update, xpay, init
    Geo geo{};
    bool dist = false;                   // rank of a row partition (no graph; see dist.py)
    bool tma = false;                    // TMA-staged K3 (aligned planes; MWCG_TMA=0/1 overrides)
    bool tma2 = false;                   // TMA-staged K2 (MWCG_TMA2=0/1 overrides)
    cudaAccessPolicyWindow l2win{};      // K1's persisting-L2 window over p (num_bytes 0: none)
    size_t l2_aside = 0;                 // the device's persisting set-aside (bytes)
    int blk_lo = 0, blk_hi = -1;         // column blocks the next K1 launch walks ([lo, hi); hi < 0: all)
    int64_t ilo = 0, ihi = 0;            // interior tiles of a rank (SPMV_INTERIOR)
};

namespace {

void copy_blocks(mwcg_solver *s, const mwcg_matrix *A) {
    s->blocks.clear();
    s->block_col0.clear();
    for (auto *b : A->blocks) {
        s->blocks.push_back(b->view);
        s->block_col0.push_back(b->col0);
    }
    if (!A->blocks.empty()) s->block_col0.push_back(A->blocks.back()->col1);
}

// Stage launchers shared by the graph body, the profiled (kernel-by-kernel)
// loop and the multi-rank driver.  fused: tile-tree dots inside K1/K2;
// otherwise the reference-order dots (cg_dot_part + cg_ref_combine).
inline int64_t k1_count_host(const Geo &g) { return (g.a1 - g.a0) + (g.b1 - g.b0); }

template <int M, bool FUSED>
void launch_k1(mwcg_solver *s, cudaStream_t st, cudaGraphConditionalHandle h, int use_cond) {
    const Geo &g = s->geo;
    const unsigned g0 = (unsigned)std::max<int64_t>(1, std::min<int64_t>(s->grid[0], k1_count_host(g)));
    // K1 carries an L2 access-policy window over p (the gathered vector):
    // a share of p's lines persists in L2 against the matrix stream and the
    // random gathers of irregular matrices (C5: p is twice the L2)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g0);
    cfg.blockDim = dim3(SpTraits<M>::THREADS);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeAccessPolicyWindow;
    at[0].val.accessPolicyWindow = s->l2win;
    cfg.attrs = at;
    cfg.numAttrs = s->l2win.num_bytes > 0 ? 1 : 0;
    const double *pc = s->p;
#define K1_LAUNCH(CT) \
    cudaLaunchKernelEx(&cfg, cg_spmv_pq<M, FUSED, CT>, s->A, pc, s->q, g, s->part, s->st, h, use_cond)
    if (!s->blocks.empty()) {  // (any tile subset: the running sums in q are per row)
        // column blocks: one launch per block, the row sums carried in q; each
        // launch pins ITS range of p in L2 (the block is sized to fit)
        const size_t nblk = s->blocks.size();
        const size_t b_lo = s->blk_hi < 0 ? 0 : (size_t)s->blk_lo;
        const size_t b_hi = s->blk_hi < 0 ? nblk : std::min(nblk, (size_t)s->blk_hi);
        for (size_t b = b_lo; b < b_hi; b++) {
            Geo gb = g;
            gb.acc_in = b > 0;
            gb.acc_out = b + 1 < nblk;
            cudaAccessPolicyWindow w = s->l2win;
            if (w.num_bytes > 0) {
                const size_t rec = sizeof(double) * (size_t)s->W;
                w.base_ptr = (void *)(s->p + s->block_col0[b] * s->W);
                w.num_bytes = (size_t)(s->block_col0[b + 1] - s->block_col0[b]) * rec;
                w.hitRatio = (float)std::min(1.0, (double)s->l2_aside / (double)w.num_bytes);
                at[0].val.accessPolicyWindow = w;
            }
            cudaLaunchKernelEx(&cfg, cg_spmv_pq<M, FUSED, int32_t>, s->blocks[b], pc, s->q, gb, s->part, s->st, h,
                               use_cond);
        }
        return;
    }
    if (s->A.dia) K1_LAUNCH(DiaTag);
    else if (s->A.col16) K1_LAUNCH(int16_t);
    else K1_LAUNCH(int32_t);
#undef K1_LAUNCH
}

template <int M, bool FUSED>
void launch_k2(mwcg_solver *s, cudaStream_t st, cudaGraphConditionalHandle h, int use_cond) {
    const Geo &g = s->geo;
    if (s->tma2)
        cg_update_tma<M, FUSED><<<s->grid[1], TILE_THREADS, UpTma<M>::SMEM, st>>>(s->r, s->q, g,
                                                                                  s->part, s->st, h, use_cond);
    else
        cg_update<M, FUSED><<<s->grid[1], TILE_THREADS, 0, st>>>(s->r, s->q, g, s->part, s->st, h,
                                                                 use_cond);
}

template <int M>
void launch_k3(mwcg_solver *s, cudaStream_t st, cudaGraphConditionalHandle h, int use_cond) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(s->grid[2]);
    cfg.blockDim = dim3(TILE_THREADS);
    cfg.dynamicSmemBytes = s->tma ? XpTma<M>::SMEM : 0;
    cfg.stream = st;
    const double *rc = s->r;
    if (s->tma) cudaLaunchKernelEx(&cfg, cg_xpay_tma<M>, s->x, s->p, rc, s->geo, s->st, h, use_cond);
    else cudaLaunchKernelEx(&cfg, cg_xpay<M>, s->x, s->p, rc, s->geo, s->st, h, use_cond);
}

// stage 0: K1 [+ reference p.q], 1: K2 [+ reference r.r], 2: K3
template <int M>
int enqueue_stage(mwcg_solver *s, int stage, cudaStream_t st, cudaGraphConditionalHandle h, int use_cond) {
    const unsigned pb = (unsigned)((s->parts + 127) / 128);
    if (stage == 0) {
        if (s->fused) {
            launch_k1<M, true>(s, st, h, use_cond);
        } else {
            launch_k1<M, false>(s, st, h, use_cond);
            cg_dot_part<M, true><<<pb, 128, 0, st>>>(s->n, s->p, s->q, s->n, s->parts, s->part, s->st, 1);
            cg_ref_combine<M><<<1, 1, 0, st>>>(s->part, s->parts, s->st, 1, h, use_cond);
        }
    } else if (stage == 1) {
        if (s->fused) {
            launch_k2<M, true>(s, st, h, use_cond);
        } else {
            launch_k2<M, false>(s, st, h, use_cond);
            cg_dot_part<M, false><<<pb, 128, 0, st>>>(s->n, s->r, s->r, s->n, s->parts, s->part, s->st, 1);
            cg_ref_combine<M><<<1, 1, 0, st>>>(s->part, s->parts, s->st, 2, h, use_cond);
        }
    } else {
        launch_k3<M>(s, st, h, use_cond);
    }
    MWCG_CHECK_LAUNCH();
    return 0;
}

int enqueue_stage_mode(mwcg_solver *s, int stage, cudaStream_t st, cudaGraphConditionalHandle h, int use_cond) {
    switch (s->mode) {
    case FP64: return enqueue_stage<FP64>(s, stage, st, h, use_cond);
    case DW: return enqueue_stage<DW>(s, stage, st, h, use_cond);
    case QDW: return enqueue_stage<QDW>(s, stage, st, h, use_cond);
    case TW: return enqueue_stage<TW>(s, stage, st, h, use_cond);
    default: return enqueue_stage<QTW>(s, stage, st, h, use_cond);
    }
}

int enqueue_iteration_mode(mwcg_solver *s, cudaStream_t st, cudaGraphConditionalHandle h, int use_cond) {
    for (int k = 0; k < 3; k++)
        if (int rc = enqueue_stage_mode(s, k, st, h, use_cond)) return rc;
    return 0;
}

template <int M>
int enqueue_init(mwcg_solver *s) {
    cudaStream_t st = s->stream;
    const unsigned tiles = s->grid[3];
    const Geo &g = s->geo;
    if (s->fused) {
        cg_init<M, true><<<tiles, TILE_THREADS, 0, st>>>(s->b, s->q, s->r, s->p, g, s->part, s->st);
    } else {
        const unsigned pb = (unsigned)((s->parts + 127) / 128);
        cg_init<M, false><<<tiles, TILE_THREADS, 0, st>>>(s->b, s->q, s->r, s->p, g, s->part, s->st);
        cg_dot_part<M, false><<<pb, 128, 0, st>>>(s->n, s->r, s->r, s->n, s->parts, s->part, s->st, 0);
        cg_ref_combine<M><<<1, 1, 0, st>>>(s->part, s->parts, s->st, 0, cudaGraphConditionalHandle{}, 0);
    }
    MWCG_CHECK_LAUNCH();
    return 0;
}

// one stage of a multi-rank iteration (dist.py drives the exchanges between them)
template <int M>
int enqueue_dist_stage(mwcg_solver *s, int stage) {
    cudaStream_t st = s->stream;
    const Geo &g = s->geo;
    cudaGraphConditionalHandle h{};
    switch (stage) {
    case MWCG_STAGE_INIT:
        cg_init<M, true><<<s->grid[3], TILE_THREADS, 0, st>>>(s->b, s->q, s->r, s->p, g, s->part, s->st);
        break;
    case MWCG_STAGE_FINAL_INIT: cg_finalize<M><<<1, TILE_THREADS, 0, st>>>(s->part, g, s->st, 0); break;
    case MWCG_STAGE_SPMV: launch_k1<M, true>(s, st, h, 0); break;
    case MWCG_STAGE_SPMV_INTERIOR:
    case MWCG_STAGE_SPMV_BOUNDARY: {
        // launch_k1 reads s->geo: swap in the tile subset for this launch
        const Geo keep = s->geo;
        if (stage == MWCG_STAGE_SPMV_INTERIOR) {
            s->geo.a0 = s->ilo;
            s->geo.a1 = s->ihi;
            s->geo.b0 = s->geo.b1 = 0;
        } else {
            s->geo.a0 = 0;
            s->geo.a1 = s->ilo;
            s->geo.b0 = s->ihi;
            s->geo.b1 = s->ntiles;
        }
        if (k1_count_host(s->geo) > 0) launch_k1<M, true>(s, st, h, 0);
        s->geo = keep;
        break;
    }
    case MWCG_STAGE_FINAL_ALPHA: cg_finalize<M><<<1, TILE_THREADS, 0, st>>>(s->part, g, s->st, 1); break;
    case MWCG_STAGE_UPDATE: launch_k2<M, true>(s, st, h, 0); break;
    case MWCG_STAGE_FINAL_BETA: cg_finalize<M><<<1, TILE_THREADS, 0, st>>>(s->part, g, s->st, 2); break;
    case MWCG_STAGE_XPAY: launch_k3<M>(s, st, h, 0); break;
    default: set_error("unknown stage %d", stage); return MWCG_ERR_VALUE;
    }
    MWCG_CHECK_LAUNCH();
    return 0;
}

// Process-wide persisting-L2 set-aside: set under a lock and only ever grown
// (32 MB for 2-word, 40 MB for 3-word records), so solvers of different
// arithmetics alternating in one process do not reconfigure the L2 on every
// switch; each solver's window hit ratio follows the size actually in force.
size_t configure_l2_aside(size_t aside) {
    static std::mutex mu;
    static size_t configured = 0;
    std::lock_guard<std::mutex> lock(mu);
    if (aside > configured) {
        if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, aside) == cudaSuccess) configured = aside;
    }
    size_t cur = 0;
    if (cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize) != cudaSuccess) cur = 0;
    cudaGetLastError();  // both calls are advisory
    return cur;
}

template <int M>
int compute_grids_t(mwcg_solver *s) {
    int dev = 0, sms = 0;
    MWCG_CUDA(cudaGetDevice(&dev));
    MWCG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    {
        // persisting-L2 window over p for K1: a 32-MB set-aside (measured on
        // C2: DW 99.4 -> 94.1 us/it, QDW 92.5 -> 87.8, QTW 148.2 -> 140.9; the
        // persisting lines of p also serve K3's read of p; larger set-asides
        // starve the other vectors: 64 MB -> DW 139 us/it; neutral for FP64,
        // C4 and C5).  MWCG_L2PIN=0 disables, =<MB> sets the set-aside.
        const char *t = std::getenv("MWCG_L2PIN");
        int max_persist = 0, max_win = 0;
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
        cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        const size_t pbytes = sizeof(double) * (size_t)Arith<M>::W * (size_t)s->geo.ldp;
        // set-aside by record width: 32 MB for DW/QDW (p = 33.5 MB at C2), 40 MB
        // for TW/QTW (p = 50 MB; C2 QTW: 32 MB 140.9, 40 MB 138.9, 48 MB 139.9 us/it)
        size_t aside = std::min((size_t)max_persist, (size_t)(Arith<M>::W >= 3 ? 40 : 32) << 20);
        if (t && atoi(t) > 0) aside = std::min((size_t)max_persist, (size_t)atoi(t) << 20);
        const bool on = t ? t[0] != '0' : (Arith<M>::W >= 2);
        s->l2win = cudaAccessPolicyWindow{};
        if (on && aside > 0 && max_win > 0 && pbytes > 0) {
            // the device-wide set-aside is configured once per process and size
            // (re-setting it per solver reconfigures the L2: seen as a 2x slower
            // create-solve-destroy loop)
            const size_t cur = configure_l2_aside(aside);
            const size_t win = std::min(pbytes, (size_t)max_win);
            s->l2_aside = cur;
            s->l2win.base_ptr = s->p;
            s->l2win.num_bytes = win;
            s->l2win.hitRatio = (float)std::min(1.0, (double)cur / (double)win);
            s->l2win.hitProp = cudaAccessPropertyPersisting;
            s->l2win.missProp = cudaAccessPropertyStreaming;
        }
        cudaGetLastError();  // the limit calls are advisory
    }
    int nb[4] = {1, 1, 1, 1};
    {
        // TMA-staged vector passes: measured faster for QTW (C2: K2 62.6 ->
        // 58.1 us, K3 28.5 -> 26.6 us), neutral for DW/QDW, slower for FP64
        // and TW; MWCG_TMA=0/1 overrides
        const char *t = std::getenv("MWCG_TMA");
        s->tma = t ? t[0] != '0' : (M == QTW);
        const char *t2 = std::getenv("MWCG_TMA2");
        s->tma2 = t2 ? t2[0] != '0' : (M != FP64 && M != TW);
    }
    if (s->fused) {
        MWCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb[0], cg_spmv_pq<M, true, int32_t>,
                                                                SpTraits<M>::THREADS, 0));
        MWCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb[1], cg_update<M, true>, TILE_THREADS, 0));
        MWCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb[3], cg_init<M, true>, TILE_THREADS, 0));
    } else {
        MWCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb[0], cg_spmv_pq<M, false, int32_t>,
                                                                SpTraits<M>::THREADS, 0));
        MWCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb[1], cg_update<M, false>, TILE_THREADS, 0));
        MWCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb[3], cg_init<M, false>, TILE_THREADS, 0));
    }
    MWCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb[2], cg_xpay<M>, TILE_THREADS, 0));
    {
        // alignment of every plane the bulk copies touch (16 B)
        const int W = Arith<M>::W;
        auto al = [](const void *ptr) { return ((uintptr_t)ptr & 15u) == 0; };
        const bool ok = al(s->x) && al(s->r) && al(s->q) && al(s->p) && (s->geo.ld % 2 == 0) &&
                        ((s->geo.p_off * W) % 2 == 0);
        s->tma = s->tma && ok;
        s->tma2 = s->tma2 && ok;
    }
    if (s->tma2) {
        MWCG_CUDA(cudaFuncSetAttribute(cg_update_tma<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)UpTma<M>::SMEM));
        MWCG_CUDA(cudaFuncSetAttribute(cg_update_tma<M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)UpTma<M>::SMEM));
        MWCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb[1], cg_update_tma<M, true>, TILE_THREADS,
                                                                UpTma<M>::SMEM));
    }
    if (s->tma) {
        MWCG_CUDA(cudaFuncSetAttribute(cg_xpay_tma<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)XpTma<M>::SMEM));
        MWCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb[2], cg_xpay_tma<M>, TILE_THREADS,
                                                                XpTma<M>::SMEM));
    }
    // bit i of `full` -> kernel i (K1, K2, K3, init) gets one CTA per tile
    // (hardware-balanced) instead of a persistent grid: measured faster for
    // the compute-heavy TW kernels (C2: 495 -> 466 us/it) and for QTW's K1,
    // slower for the streaming ones; MWCG_GRID_FULL=<mask> overrides
    unsigned full = (M == TW) ? 7u : ((M == QTW) ? 1u : 0u);
    if (const char *t = std::getenv("MWCG_GRID_FULL")) full = (unsigned)std::atoi(t);
    for (int i = 0; i < 4; i++) {
        int64_t g = (int64_t)(nb[i] > 0 ? nb[i] : 1) * sms;
        if (g > s->geo.ntiles || ((full >> i) & 1u)) g = s->geo.ntiles;
        s->grid[i] = (unsigned)(g > 0 ? g : 1);
    }
    return 0;
}

int compute_grids(mwcg_solver *s) {
    switch (s->mode) {
    case FP64: return compute_grids_t<FP64>(s);
    case DW: return compute_grids_t<DW>(s);
    case QDW: return compute_grids_t<QDW>(s);
    case TW: return compute_grids_t<TW>(s);
    default: return compute_grids_t<QTW>(s);
    }
}

int build_graph(mwcg_solver *s) {
    MWCG_CUDA(cudaGraphCreate(&s->graph, 0));
    MWCG_CUDA(cudaGraphConditionalHandleCreate(&s->cond, s->graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = s->cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    MWCG_CUDA(cudaGraphAddNode(&node, s->graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    MWCG_CUDA(cudaStreamBeginCaptureToGraph(s->cap, body, nullptr, nullptr, 0,
                                            cudaStreamCaptureModeThreadLocal));
    // U iterations per body run: one conditional evaluation per U
    // iterations; an iteration after a stop (or the k_stop pause) launches
    // kernels that return at once
    int rc = 0;
    for (int u = 0; u < s->unroll && !rc; u++) rc = enqueue_iteration_mode(s, s->cap, s->cond, 1);
    cudaGraph_t out_graph;
    cudaError_t e = cudaStreamEndCapture(s->cap, &out_graph);
    if (rc) return rc;
    MWCG_CUDA(e);
    MWCG_CUDA(cudaGraphInstantiate(&s->exec, s->graph, 0));
    return 0;
}

void free_solver(mwcg_solver *s) {
    if (!s) return;
    if (s->exec) cudaGraphExecDestroy(s->exec);
    if (s->graph) cudaGraphDestroy(s->graph);
    cudaStream_t st = s->stream;
    if (s->own_x) pool_free(s->x, st);
    pool_free(s->r, st);
    pool_free(s->q, st);
    if (!s->dist) {  // caller-owned in the distributed solver
        pool_free(s->p, st);
        pool_free(s->part, st);
    }
    pool_free(s->st, st);
    pool_free(s->xt, st);
    pool_free(s->res, st);
    pool_free(s->diff, st);
    pool_free(s->bt, st);
    pool_free(s->mpart, st);
    pool_free(s->mout, st);
    pool_free(s->mticket, st);
    delete[] reinterpret_cast<double *>(s->st_host);
    for (auto &e : s->ev)
        if (e) cudaEventDestroy(e);
    if (s->cap) cudaStreamDestroy(s->cap);
    delete s;
}

// TW sum of squares of a 3-plane vector into mout[slot*3 .. +3] (device)
int tw_sumsq(mwcg_solver *s, const double *v, int slot) {
    double *out = s->mout + 3 * slot;
    if (s->fused) return launch_dot_tile(TW, s->n, v, s->n, v, s->n, out, s->mpart, s->mticket, s->stream);
    return launch_dot_partitions(TW, s->n, v, s->n, v, s->n, 1, out, s->mpart, s->stream);
}

}  // namespace

extern "C" {

int mwcg_matrix_create(mwcg_matrix **out, int64_t n_rows, int64_t n_cols, int64_t nnz, const void *row_ptr,
                       const void *col_idx, const double *values, int index_bytes, void *stream) {
    if (!out) {
        set_error("null output handle");
        return MWCG_ERR_VALUE;
    }
    return mwcg_matrix_create_ex(out, n_rows, n_cols, nnz, row_ptr, col_idx, values, index_bytes, 0, -1,
                                 stream);
}

int mwcg_matrix_create_ex(mwcg_matrix **out, int64_t n_rows, int64_t n_cols, int64_t nnz, const void *row_ptr,
                          const void *col_idx, const double *values, int index_bytes, int64_t row_base,
                          int col_format, void *stream) {
    return mwcg_matrix_create_blocked(out, n_rows, n_cols, nnz, row_ptr, col_idx, values, index_bytes, row_base,
                                      col_format, -1, stream);
}

int mwcg_matrix_create_blocked(mwcg_matrix **out, int64_t n_rows, int64_t n_cols, int64_t nnz,
                               const void *row_ptr, const void *col_idx, const double *values, int index_bytes,
                               int64_t row_base, int col_format, int64_t cols_per_block, void *stream) {
    if (!out) {
        set_error("null output handle");
        return MWCG_ERR_VALUE;
    }
    SellMatrixOwned *M = nullptr;
    int rc = sell_create(&M, n_rows, n_cols, nnz, row_ptr, col_idx, values, index_bytes, row_base, col_format,
                         (cudaStream_t)stream);
    if (rc) return rc;
    auto *A = new mwcg_matrix{M, {}};
    // column blocks for K1 (sell.cu): irregular (int32-SELL) matrices whose
    // gathered vector outgrows the L2.  MWCG_COLBLOCK=<columns per block>
    // overrides (0: off); default 2^21 columns (a 32-MB range of a DW p) once
    // the matrix has at least twice as many.
    int64_t cpb = (n_cols >= ((int64_t)1 << 22)) ? ((int64_t)1 << 21) : 0;
    bool automatic = true;
    if (const char *e = std::getenv("MWCG_COLBLOCK")) {
        cpb = std::atoll(e);
        automatic = false;
    }
    if (cols_per_block >= 0) {  // the caller's choice (0: none)
        cpb = cols_per_block;
        automatic = false;
    }
    rc = sell_colblocks(A->blocks, M, row_ptr, col_idx, values, index_bytes, cpb, automatic,
                        (cudaStream_t)stream);
    if (rc) {
        sell_destroy(M);
        delete A;
        return rc;
    }
    *out = A;
    return 0;
}

int mwcg_matrix_col_blocks(const mwcg_matrix *A) { return A ? (int)A->blocks.size() : -1; }

int64_t mwcg_matrix_block_columns(const mwcg_matrix *A) {
    return (A && !A->blocks.empty()) ? A->blocks[0]->col1 - A->blocks[0]->col0 : 0;
}

int mwcg_matrix_sigma_sorted(const mwcg_matrix *A) { return A && A->M->view.perm ? 1 : 0; }

int mwcg_matrix_col_bytes(const mwcg_matrix *A) {
    return A ? (A->M->view.dia ? 0 : (A->M->view.col16 ? 2 : 4)) : -1;
}

int64_t mwcg_matrix_stored_values(const mwcg_matrix *A) { return A ? A->M->view.stored : -1; }

int mwcg_matrix_destroy(mwcg_matrix *A) {
    if (A) {
        sell_destroy(A->M);
        for (auto *b : A->blocks) sell_destroy(b);
        delete A;
    }
    return 0;
}

int mwcg_matrix_info(const mwcg_matrix *A, int64_t *n_rows, int64_t *n_cols, int64_t *nnz,
                     int64_t *padded) {
    if (!A) {
        set_error("null matrix");
        return MWCG_ERR_VALUE;
    }
    if (n_rows) *n_rows = A->M->view.n_rows;
    if (n_cols) *n_cols = A->M->view.n_cols;
    if (nnz) *nnz = A->M->view.nnz;
    if (padded) *padded = A->M->view.total;
    return 0;
}

int mwcg_spmv(int mode, const mwcg_matrix *A, const double *x, int64_t ldx, double *y, int64_t ldy,
              void *stream) {
    if (!A || !valid_mode(mode)) {
        set_error("bad matrix or mode");
        return MWCG_ERR_VALUE;
    }
    return launch_spmv(mode, A->M->view, x, ldx, y, ldy, (cudaStream_t)stream);
}

int mwcg_solver_create(mwcg_solver **out, const mwcg_matrix *A, const mwcg_solver_config *cfg, double *x,
                       void *stream) {
    if (!out || !A || !cfg) {
        set_error("null argument");
        return MWCG_ERR_VALUE;
    }
    if (!valid_mode(cfg->mode)) {
        set_error("unknown arithmetic mode %d", cfg->mode);
        return MWCG_ERR_VALUE;
    }
    if (A->M->view.n_rows != A->M->view.n_cols) {
        set_error("matrix must be square");
        return MWCG_ERR_VALUE;
    }
    if (cfg->reduction == MWCG_RED_PARTITIONS && cfg->partitions < 1) {
        set_error("partitions must be >= 1");
        return MWCG_ERR_VALUE;
    }
    auto *s = new mwcg_solver();
    s->A = A->M->view;
    copy_blocks(s, A);
    s->mode = cfg->mode;
    s->W = words_of(cfg->mode);
    s->cfg = *cfg;
    s->n = s->A.n_rows;
    s->ntiles = num_tiles(s->n);
    s->fused = cfg->reduction != MWCG_RED_PARTITIONS;
    if (const char *u = std::getenv("MWCG_UNROLL")) s->unroll = std::max(1, std::min(16, std::atoi(u)));
    s->parts = s->fused ? 1 : cfg->partitions;
    s->stream = (cudaStream_t)stream;
    s->geo = Geo{s->n, s->n, s->n, 0, s->ntiles, 0, s->ntiles, s->ntiles, 1, 0, s->ntiles, 0, 0};
    const size_t vbytes = sizeof(double) * (size_t)s->W * (size_t)(s->n > 0 ? s->n : 1);
    int rc = 0;
#define TRY(call)                                  \
    do {                                           \
        cudaError_t e_ = (call);                   \
        if (e_ != cudaSuccess) {                   \
            set_error("%s: %s", #call, cudaGetErrorString(e_)); \
            free_solver(s);                        \
            return (int)e_;                        \
        }                                          \
    } while (0)
    if (x) {
        s->x = x;
    } else {
        TRY(pool_alloc((void **)&s->x, vbytes, s->stream));
        s->own_x = true;
    }
    TRY(pool_alloc((void **)&s->r, vbytes, s->stream));
    TRY(pool_alloc((void **)&s->p, vbytes, s->stream));
    TRY(pool_alloc((void **)&s->q, vbytes, s->stream));
    int64_t np = s->fused ? (s->ntiles > 0 ? s->ntiles : 1) : s->parts;
    TRY(pool_alloc((void **)&s->part, sizeof(double) * 3 * (size_t)np, s->stream));
    TRY(pool_alloc((void **)&s->st, sizeof(CgState), s->stream));
    TRY(cudaMemsetAsync(s->st, 0, sizeof(CgState), s->stream));
    // one pinned block for the host mirrors: state, k_stop, metric sums
    // host mirrors in pageable memory: every D2H of the state is followed by a
    // stream sync anyway, and pinned alloc/free (cudaFreeHost synchronizes the
    // device) would dominate short solves that create and drop solvers
    s->st_host = (CgState *)new double[(sizeof(CgState) + 16 * sizeof(double) + 7) / 8];
    s->kstop_host = (long long *)((char *)s->st_host + sizeof(CgState));
    s->mout_host = (double *)((char *)s->st_host + sizeof(CgState) + 2 * sizeof(double));
    TRY(cudaStreamCreateWithFlags(&s->cap, cudaStreamNonBlocking));
    for (auto &e : s->ev) TRY(cudaEventCreate(&e));
#undef TRY
    if (s->n > 0) {
        rc = compute_grids(s);
        if (rc) {
            free_solver(s);
            return rc;
        }
        rc = build_graph(s);
        if (rc) {
            free_solver(s);
            return rc;
        }
    }
    *out = s;
    return 0;
}

// Rank of a row partition.  A: the rank's rows with GLOBAL
// column indices.  p_full: caller-owned replica of p (ldp AoS records);
// part: caller-owned rank-blocked tile partials of all ranks (part_tb tiles
// per rank block, common.cuh part_index).  The caller gathers them between
// stages (dist.py).
int mwcg_solver_create_dist(mwcg_solver **out, const mwcg_matrix *A, const mwcg_solver_config *cfg,
                            double *x, double *p_full, int64_t ldp, int64_t p_off, double *part,
                            int64_t part_tb, int64_t tile_off, int64_t ntiles_glob, void *stream) {
    if (!out || !A || !cfg || !x || !p_full || !part) {
        set_error("null argument");
        return MWCG_ERR_VALUE;
    }
    if (!valid_mode(cfg->mode) || cfg->reduction != MWCG_RED_TILE) {
        set_error("distributed solver: bad mode or reduction (tile order only)");
        return MWCG_ERR_VALUE;
    }
    const int64_t n = A->M->view.n_rows;
    if (p_off < 0 || p_off + n > ldp || tile_off < 0 || part_tb < 1 || num_tiles(n) > part_tb ||
        tile_off % part_tb != 0 || A->M->view.n_cols > ldp) {
        set_error("distributed solver: inconsistent geometry");
        return MWCG_ERR_VALUE;
    }
    auto *s = new mwcg_solver();
    s->A = A->M->view;
    copy_blocks(s, A);
    s->mode = cfg->mode;
    s->W = words_of(cfg->mode);
    s->cfg = *cfg;
    s->n = n;
    s->ntiles = num_tiles(n);
    s->fused = true;
    s->dist = true;
    s->stream = (cudaStream_t)stream;
    s->x = x;
    s->p = p_full;
    s->part = part;
    s->geo = Geo{n, n, ldp, p_off, s->ntiles, tile_off, part_tb, ntiles_glob, 0, 0, s->ntiles, 0, 0};
    const size_t vbytes = sizeof(double) * (size_t)s->W * (size_t)(n > 0 ? n : 1);
#define TRY(call)                                                \
    do {                                                         \
        cudaError_t e_ = (call);                                 \
        if (e_ != cudaSuccess) {                                 \
            set_error("%s: %s", #call, cudaGetErrorString(e_));  \
            s->p = nullptr;                                      \
            s->part = nullptr;                                   \
            free_solver(s);                                      \
            return (int)e_;                                      \
        }                                                        \
    } while (0)
    TRY(pool_alloc((void **)&s->r, vbytes, s->stream));
    TRY(pool_alloc((void **)&s->q, vbytes, s->stream));
    TRY(pool_alloc((void **)&s->st, sizeof(CgState), s->stream));
    TRY(cudaMemsetAsync(s->st, 0, sizeof(CgState), s->stream));
    // host mirrors in pageable memory: every D2H of the state is followed by a
    // stream sync anyway, and pinned alloc/free (cudaFreeHost synchronizes the
    // device) would dominate short solves that create and drop solvers
    s->st_host = (CgState *)new double[(sizeof(CgState) + 16 * sizeof(double) + 7) / 8];
    s->kstop_host = (long long *)((char *)s->st_host + sizeof(CgState));
    s->mout_host = (double *)((char *)s->st_host + sizeof(CgState) + 2 * sizeof(double));
    for (auto &e : s->ev) TRY(cudaEventCreate(&e));
#undef TRY
    if (n > 0) {
        int rc = compute_grids(s);
        if (rc) {
            s->p = nullptr;
            s->part = nullptr;
            free_solver(s);
            return rc;
        }
    }
    *out = s;
    return 0;
}

int mwcg_solver_set_interior(mwcg_solver *s, int64_t ilo, int64_t ihi) {
    if (!s || !s->dist) {
        set_error("not a distributed solver");
        return MWCG_ERR_STATE;
    }
    if (ilo < 0 || ihi < ilo || ihi > s->ntiles) {
        set_error("interior tiles [%lld, %lld) outside [0, %lld)", (long long)ilo, (long long)ihi,
                  (long long)s->ntiles);
        return MWCG_ERR_VALUE;
    }
    s->ilo = ilo;
    s->ihi = ihi;
    return 0;
}

int mwcg_solver_dist_stage(mwcg_solver *s, int stage, void *stream) {
    if (!s || !s->dist) {
        set_error("not a distributed solver");
        return MWCG_ERR_STATE;
    }
    // launch on the caller's current stream (lets dist.py capture a segment
    // into a CUDA graph); NULL keeps the solver's stream
    struct StreamGuard {
        mwcg_solver *s;
        cudaStream_t old;
        ~StreamGuard() { s->stream = old; }
    } guard{s, s->stream};
    if (stream) s->stream = (cudaStream_t)stream;
    if (s->n == 0 && (stage == MWCG_STAGE_INIT || stage == MWCG_STAGE_SPMV || stage == MWCG_STAGE_UPDATE ||
                      stage == MWCG_STAGE_XPAY || stage == MWCG_STAGE_SPMV_INTERIOR ||
                      stage == MWCG_STAGE_SPMV_BOUNDARY))
        return 0;  // a rank without rows still takes part in the finalize stages
    switch (s->mode) {
    case FP64: return enqueue_dist_stage<FP64>(s, stage);
    case DW: return enqueue_dist_stage<DW>(s, stage);
    case QDW: return enqueue_dist_stage<QDW>(s, stage);
    case TW: return enqueue_dist_stage<TW>(s, stage);
    default: return enqueue_dist_stage<QTW>(s, stage);
    }
}

int mwcg_solver_dist_spmv_blocks(mwcg_solver *s, int b0, int b1, void *stream) {
    if (!s || !s->dist) {
        set_error("not a distributed solver");
        return MWCG_ERR_STATE;
    }
    if (s->blocks.empty() || b0 < 0 || b1 < b0 || b1 > (int)s->blocks.size()) {
        set_error("bad column-block range [%d, %d) of %d", b0, b1, (int)s->blocks.size());
        return MWCG_ERR_VALUE;
    }
    if (b0 == b1) return 0;
    s->blk_lo = b0;
    s->blk_hi = b1;
    const int rc = mwcg_solver_dist_stage(s, MWCG_STAGE_SPMV, stream);
    s->blk_lo = 0;
    s->blk_hi = -1;
    return rc;
}

int mwcg_solver_describe(const mwcg_solver *s, int64_t *out, int n) {
    if (!s || !out) {
        set_error("null argument");
        return MWCG_ERR_VALUE;
    }
    const int64_t v[8] = {s->grid[0], s->grid[1], s->grid[2], s->grid[3], s->tma2 ? 1 : 0, s->tma ? 1 : 0,
                          s->A.perm ? 1 : 0, (int64_t)s->blocks.size()};
    for (int i = 0; i < n && i < 8; i++) out[i] = v[i];
    return 0;
}

int mwcg_solver_destroy(mwcg_solver *s) {
    free_solver(s);
    return 0;
}

// x0 (FP64, nullable) -> x word 0 (kernels.py:62-67); q = A x; init.
int mwcg_solver_start(mwcg_solver *s, const double *b, double b_norm, const double *x0,
                      const double *x_star, double epsilon, int64_t max_iterations) {
    if (!s) {
        set_error("null solver");
        return MWCG_ERR_VALUE;
    }
    cudaStream_t st = s->stream;
    s->b = b;
    s->x_star = x_star;
    s->norms_ready = false;
    const size_t vbytes = sizeof(double) * (size_t)s->W * (size_t)s->n;
    CgState init{};
    init.b_norm = (b_norm == 0.0) ? 1.0 : b_norm;
    init.eps = epsilon;
    init.max_iters = max_iterations;
    init.k_stop = LLONG_MAX;  // no pause point until mwcg_solver_run sets one
    const bool quasi = (s->mode == QDW || s->mode == QTW);
    init.norm_r = quasi && s->cfg.normalization != MWCG_NORM_NONE;
    init.norm_all = quasi && s->cfg.normalization == MWCG_NORM_EVERY_OP;
    init.status = RUNNING;
    *s->st_host = init;
    MWCG_CUDA(cudaMemcpyAsync(s->st, s->st_host, sizeof(CgState), cudaMemcpyHostToDevice, st));
    if (s->n == 0 && !s->dist) {
        // empty system: rho = 0 -> rel = 0 < eps -> converged at 0
        s->st_host->status = CONVERGED;
        s->st_host->rel = 0.0;
        MWCG_CUDA(cudaMemcpyAsync(s->st, s->st_host, sizeof(CgState), cudaMemcpyHostToDevice, st));
        return 0;
    }
    MWCG_CUDA(cudaMemsetAsync(s->x, 0, vbytes, st));
    int rc = 0;
    if (!s->dist) {
        if (x0) MWCG_CUDA(cudaMemcpyAsync(s->x, x0, sizeof(double) * (size_t)s->n, cudaMemcpyDeviceToDevice, st));
        rc = launch_spmv(s->mode, s->A, s->x, s->n, s->q, s->n, st);
    } else {
        // x0 is the FULL (global, padded) initial guess on every rank: the
        // local slice seeds x; the SpMV reads it through p's buffer (AoS),
        // which the init stage overwrites right after.
        const int64_t ldp = s->geo.ldp;
        if (x0) MWCG_CUDA(cudaMemcpyAsync(s->x, x0 + s->geo.p_off, sizeof(double) * (size_t)s->n,
                                          cudaMemcpyDeviceToDevice, st));
        const unsigned eb = (unsigned)std::max<int64_t>(1, std::min<int64_t>((ldp + 255) / 256, 148 * 16));
        const unsigned sb = (unsigned)std::max<int64_t>(1, std::min<int64_t>((s->n + 255) / 256, 148 * 16));
#define START(Mx)                                                                                    \
    do {                                                                                             \
        spread_x0_kernel<words_of(Mx)><<<eb, 256, 0, st>>>(ldp, x0, s->p);                          \
        if (s->A.dia) spmv_aos_kernel<Mx, DiaTag><<<sb, TILE_THREADS, 0, st>>>(s->A, s->p, s->q, s->n);  \
        else if (s->A.col16) spmv_aos_kernel<Mx, int16_t><<<sb, TILE_THREADS, 0, st>>>(s->A, s->p, s->q, s->n); \
        else spmv_aos_kernel<Mx, int32_t><<<sb, TILE_THREADS, 0, st>>>(s->A, s->p, s->q, s->n);          \
    } while (0)
        switch (s->mode) {
        case FP64: START(FP64); break;
        case DW: START(DW); break;
        case QDW: START(QDW); break;
        case TW: START(TW); break;
        default: START(QTW); break;
        }
#undef START
        MWCG_CHECK_LAUNCH();
        switch (s->mode) {  // local init stage only; dist.py gathers + finalizes
        case FP64: return enqueue_dist_stage<FP64>(s, MWCG_STAGE_INIT);
        case DW: return enqueue_dist_stage<DW>(s, MWCG_STAGE_INIT);
        case QDW: return enqueue_dist_stage<QDW>(s, MWCG_STAGE_INIT);
        case TW: return enqueue_dist_stage<TW>(s, MWCG_STAGE_INIT);
        default: return enqueue_dist_stage<QTW>(s, MWCG_STAGE_INIT);
        }
    }
    if (rc) return rc;
    switch (s->mode) {
    case FP64: rc = enqueue_init<FP64>(s); break;
    case DW: rc = enqueue_init<DW>(s); break;
    case QDW: rc = enqueue_init<QDW>(s); break;
    case TW: rc = enqueue_init<TW>(s); break;
    default: rc = enqueue_init<QTW>(s); break;
    }
    return rc;
}

// Run iterations until the solve stops or k == k_stop (async on the stream).
int mwcg_solver_run(mwcg_solver *s, int64_t k_stop) {
    if (!s) {
        set_error("null solver");
        return MWCG_ERR_VALUE;
    }
    if (s->n == 0) return 0;
    cudaStream_t st = s->stream;
    // k_stop lives in device state; written from pinned memory (stream-ordered)
    MWCG_CUDA(cudaStreamSynchronize(st));
    *s->kstop_host = (long long)k_stop;
    MWCG_CUDA(cudaMemcpyAsync(&s->st->k_stop, s->kstop_host, sizeof(long long), cudaMemcpyHostToDevice, st));
    MWCG_CUDA(cudaMemsetAsync(&s->st->pause, 0, sizeof(int), st));
    MWCG_CUDA(cudaGraphLaunch(s->exec, st));
    return 0;
}

// Device duration of the SpMV kernel (K1) alone: `reps` back-to-back
// launches between two events on the solver's stream (no host gaps).  K1 is
// idempotent on a running state (q = A p, the p.q partials and alpha are
// recomputed from the same p and rho), so this is valid after
// mwcg_solver_start; the state's pause point is lifted for the measurement.
int mwcg_solver_time_k1(mwcg_solver *s, int reps, double *us) {
    if (!s || !us || reps < 1) {
        set_error("bad argument");
        return MWCG_ERR_VALUE;
    }
    if (s->n == 0) {
        *us = 0.0;
        return 0;
    }
    cudaStream_t st = s->stream;
    MWCG_CUDA(cudaStreamSynchronize(st));
    *s->kstop_host = LLONG_MAX;
    MWCG_CUDA(cudaMemcpyAsync(&s->st->k_stop, s->kstop_host, sizeof(long long), cudaMemcpyHostToDevice, st));
    MWCG_CUDA(cudaMemsetAsync(&s->st->pause, 0, sizeof(int), st));
    cudaGraphConditionalHandle h{};
    // MWCG_NOTAIL=1 (tools/): time K1 without its serial tail (the last CTA's
    // reduction of the partials and the scalar step) -- a diagnostic, results unused
    const int final_saved = s->geo.final_;
    if (const char *e = std::getenv("MWCG_NOTAIL")) {
        if (std::atoi(e) != 0) s->geo.final_ = 0;
    }
    for (int pass = 0; pass < 2; pass++) {  // pass 0 warms up
        MWCG_CUDA(cudaEventRecord(s->ev[6], st));
        for (int r = 0; r < reps; r++) {
            switch (s->mode) {
            case FP64: s->fused ? launch_k1<FP64, true>(s, st, h, 0) : launch_k1<FP64, false>(s, st, h, 0); break;
            case DW: s->fused ? launch_k1<DW, true>(s, st, h, 0) : launch_k1<DW, false>(s, st, h, 0); break;
            case QDW: s->fused ? launch_k1<QDW, true>(s, st, h, 0) : launch_k1<QDW, false>(s, st, h, 0); break;
            case TW: s->fused ? launch_k1<TW, true>(s, st, h, 0) : launch_k1<TW, false>(s, st, h, 0); break;
            default: s->fused ? launch_k1<QTW, true>(s, st, h, 0) : launch_k1<QTW, false>(s, st, h, 0); break;
            }
        }
        MWCG_CHECK_LAUNCH();
        MWCG_CUDA(cudaEventRecord(s->ev[7], st));
        MWCG_CUDA(cudaEventSynchronize(s->ev[7]));
    }
    s->geo.final_ = final_saved;
    float ms = 0.f;
    MWCG_CUDA(cudaEventElapsedTime(&ms, s->ev[6], s->ev[7]));
    *us = 1e3 * (double)ms / reps;
    return 0;
}

// Same as run, but one kernel launch at a time with CUDA events around each
// stage; accumulates device milliseconds into ms[0..2] = K1, K2, K3 (fused)
// or K1, K2, K3 incl. the reference dots (partitions mode).
int mwcg_solver_run_profiled(mwcg_solver *s, int64_t k_stop, double *ms) {
    if (!s) {
        set_error("null solver");
        return MWCG_ERR_VALUE;
    }
    if (s->n == 0) return 0;
    cudaStream_t st = s->stream;
    MWCG_CUDA(cudaStreamSynchronize(st));
    *s->kstop_host = (long long)k_stop;
    MWCG_CUDA(cudaMemcpyAsync(&s->st->k_stop, s->kstop_host, sizeof(long long), cudaMemcpyHostToDevice, st));
    MWCG_CUDA(cudaMemsetAsync(&s->st->pause, 0, sizeof(int), st));
    MWCG_CUDA(cudaMemcpyAsync(s->st_host, s->st, sizeof(CgState), cudaMemcpyDeviceToHost, st));
    MWCG_CUDA(cudaStreamSynchronize(st));
    cudaGraphConditionalHandle h{};
    while (s->st_host->status == RUNNING && s->st_host->k < k_stop) {
        MWCG_CUDA(cudaEventRecord(s->ev[0], st));
        for (int k = 0; k < 3; k++) {
            if (int rc = enqueue_stage_mode(s, k, st, h, 0)) return rc;
            if (k < 2) MWCG_CUDA(cudaEventRecord(s->ev[1 + k], st));
        }
        MWCG_CHECK_LAUNCH();
        MWCG_CUDA(cudaEventRecord(s->ev[3], st));
        MWCG_CUDA(cudaMemcpyAsync(s->st_host, s->st, sizeof(CgState), cudaMemcpyDeviceToHost, st));
        MWCG_CUDA(cudaStreamSynchronize(st));
        float a = 0, b = 0, c = 0;
        cudaEventElapsedTime(&a, s->ev[0], s->ev[1]);
        cudaEventElapsedTime(&b, s->ev[1], s->ev[2]);
        cudaEventElapsedTime(&c, s->ev[2], s->ev[3]);
        if (ms) {
            ms[0] += a;
            ms[1] += b;
            ms[2] += c;
        }
    }
    return 0;
}

int mwcg_solver_state(mwcg_solver *s, mwcg_state *out) {
    if (!s || !out) {
        set_error("null argument");
        return MWCG_ERR_VALUE;
    }
    MWCG_CUDA(cudaMemcpyAsync(s->st_host, s->st, sizeof(CgState), cudaMemcpyDeviceToHost, s->stream));
    MWCG_CUDA(cudaStreamSynchronize(s->stream));
    const CgState &h = *s->st_host;
    out->k = h.k;
    out->status = h.status;
    out->iterations = h.status == RUNNING ? h.k : h.iterations;
    out->rel = h.rel;
    for (int i = 0; i < 3; i++) {
        out->rho[i] = h.rho[i];
        out->alpha[i] = h.alpha[i];
        out->beta[i] = h.beta[i];
    }
    return 0;
}

// TW-accurate error norm and true residual of the current x
// (norm_metrics_tw, kernels.py:305-328).  *err is NaN when x_star is null.
int mwcg_solver_metrics(mwcg_solver *s, double *err, double *true_res) {
    if (!s) {
        set_error("null solver");
        return MWCG_ERR_VALUE;
    }
    cudaStream_t st = s->stream;
    const int64_t n = s->n;
    if (s->dist) {  // TW metrics of a partitioned iterate: not implemented (NaN)
        if (err) *err = NAN;
        if (true_res) *true_res = NAN;
        return 0;
    }
    if (n == 0) {
        if (err) *err = s->x_star ? 0.0 : NAN;
        if (true_res) *true_res = 0.0;
        return 0;
    }
    const size_t b3 = sizeof(double) * 3 * (size_t)n;
    if (!s->xt) {
        MWCG_CUDA(pool_alloc((void **)&s->xt, b3, st));
        MWCG_CUDA(pool_alloc((void **)&s->res, b3, st));
        MWCG_CUDA(pool_alloc((void **)&s->diff, b3, st));
        MWCG_CUDA(pool_alloc((void **)&s->bt, b3, st));
        MWCG_CUDA(pool_alloc((void **)&s->mpart, sizeof(double) * 3 * (size_t)(s->ntiles > 0 ? s->ntiles : 1), st));
        MWCG_CUDA(pool_alloc((void **)&s->mout, sizeof(double) * 12, st));
        MWCG_CUDA(pool_alloc((void **)&s->mticket, sizeof(unsigned int), st));
        MWCG_CUDA(cudaMemsetAsync(s->mticket, 0, sizeof(unsigned int), st));
    }
    const unsigned eb = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
    int rc;
    if (!s->norms_ready) {
        promote_fp64_kernel<<<eb, 256, 0, st>>>(n, s->b, s->bt);
        if ((rc = tw_sumsq(s, s->bt, 2))) return rc;
        if (s->x_star) {
            promote_fp64_kernel<<<eb, 256, 0, st>>>(n, s->x_star, s->bt);
            if ((rc = tw_sumsq(s, s->bt, 3))) return rc;
        }
    }
    switch (s->mode) {
    case FP64: promote_kernel<FP64><<<eb, 256, 0, st>>>(n, s->x, n, s->xt); break;
    case DW: promote_kernel<DW><<<eb, 256, 0, st>>>(n, s->x, n, s->xt); break;
    case QDW: promote_kernel<QDW><<<eb, 256, 0, st>>>(n, s->x, n, s->xt); break;
    case TW: promote_kernel<TW><<<eb, 256, 0, st>>>(n, s->x, n, s->xt); break;
    default: promote_kernel<QTW><<<eb, 256, 0, st>>>(n, s->x, n, s->xt); break;
    }
    if (s->A.dia)
        metrics_vec_kernel<DiaTag><<<eb, TILE_THREADS, 0, st>>>(s->A, s->xt, s->b, s->x_star, s->res, s->diff);
    else if (s->A.col16)
        metrics_vec_kernel<int16_t><<<eb, TILE_THREADS, 0, st>>>(s->A, s->xt, s->b, s->x_star, s->res, s->diff);
    else
        metrics_vec_kernel<int32_t><<<eb, TILE_THREADS, 0, st>>>(s->A, s->xt, s->b, s->x_star, s->res, s->diff);
    MWCG_CHECK_LAUNCH();
    if ((rc = tw_sumsq(s, s->res, 0))) return rc;
    if (s->x_star && (rc = tw_sumsq(s, s->diff, 1))) return rc;
    MWCG_CUDA(cudaMemcpyAsync(s->mout_host, s->mout, sizeof(double) * 12, cudaMemcpyDeviceToHost, st));
    MWCG_CUDA(cudaStreamSynchronize(st));
    auto coll = [](const double *v) { return (v[0] + v[1]) + v[2]; };
    if (!s->norms_ready) {
        s->bnorm_sq = coll(s->mout_host + 6);
        if (s->bnorm_sq == 0.0) s->bnorm_sq = 1.0;
        s->xs_sq = s->x_star ? coll(s->mout_host + 9) : 1.0;
        if (s->xs_sq == 0.0) s->xs_sq = 1.0;
        s->norms_ready = true;
    }
    if (true_res) *true_res = std::sqrt(coll(s->mout_host) / s->bnorm_sq);
    if (err) *err = s->x_star ? std::sqrt(coll(s->mout_host + 3) / s->xs_sq) : NAN;
    return 0;
}

// The whole cg_solve loop (cg.py:78-183) with history records every
// `history_stride` iterations plus the start / end records.  History arrays
// are host memory of capacity hist_cap; *n_hist receives the record count
// (may exceed hist_cap: extra records are counted but not stored).
int mwcg_cg_solve(mwcg_solver *s, const double *b, double b_norm, const double *x0, const double *x_star,
                  double epsilon, int64_t max_iterations, int64_t history_stride, int profile,
                  mwcg_solve_result *res, int64_t hist_cap, int64_t *h_k, double *h_rel,
                  double *h_true, double *h_err) {
    if (!s || !res) {
        set_error("null argument");
        return MWCG_ERR_VALUE;
    }
    if (history_stride < 1) {
        set_error("history_stride must be >= 1");
        return MWCG_ERR_VALUE;
    }
    if (s->l2win.num_bytes > 0) {
        // persisting lines left by earlier solvers (other p buffers, possibly
        // freed) would hold the set-aside: return them to normal first
        MWCG_CUDA(cudaStreamSynchronize(s->stream));
        cudaCtxResetPersistingL2Cache();
    }
    int rc = mwcg_solver_start(s, b, b_norm, x0, x_star, epsilon, max_iterations);
    if (rc) return rc;
    mwcg_state stt{};
    if ((rc = mwcg_solver_state(s, &stt))) return rc;
    int64_t nh = 0, last_rec = -1, metric_launches = 0;
    double loop_ms = 0.0, hist_ms = 0.0;
    double stage_ms[3] = {0, 0, 0};
    auto record = [&](int64_t k, double rel) -> int {
        double e = NAN, t = NAN;
        cudaEventRecord(s->ev[4], s->stream);
        const bool first = !s->norms_ready;
        int r2 = mwcg_solver_metrics(s, &e, &t);
        if (r2) return r2;
        // promote x, metrics rows, 1-2 dots (2 kernels each in partitions mode)
        const int dk = s->fused ? 1 : 2;
        metric_launches += 2 + dk * (s->x_star ? 2 : 1);
        if (first) metric_launches += (1 + dk) * (s->x_star ? 2 : 1);
        cudaEventRecord(s->ev[5], s->stream);
        cudaEventSynchronize(s->ev[5]);
        float ms = 0;
        cudaEventElapsedTime(&ms, s->ev[4], s->ev[5]);
        hist_ms += ms;
        if (nh < hist_cap) {
            h_k[nh] = k;
            h_rel[nh] = rel;
            h_true[nh] = t;
            h_err[nh] = e;
        }
        nh++;
        last_rec = k;
        return 0;
    };
    if ((rc = record(0, stt.rel))) return rc;
    int64_t body_kernels = 0;  // kernels launched by the iteration loop
    // column blocks: K1 is one launch per block
    const int per_it = (s->fused ? 3 : 7) + (s->blocks.empty() ? 0 : (int)s->blocks.size() - 1);
    while (stt.status == RUNNING) {
        const int64_t k_before = stt.k;
        int64_t next = (stt.k / history_stride + 1) * history_stride;
        if (next > max_iterations) next = max_iterations;
        if (profile) {
            if ((rc = mwcg_solver_run_profiled(s, next, stage_ms))) return rc;
        } else {
            MWCG_CUDA(cudaEventRecord(s->ev[6], s->stream));
            if ((rc = mwcg_solver_run(s, next))) return rc;
            MWCG_CUDA(cudaEventRecord(s->ev[7], s->stream));
        }
        if ((rc = mwcg_solver_state(s, &stt))) return rc;
        {
            // iterations this run executed (a breakdown is counted as one
            // more: exact for a K1 breakdown, which does not advance k)
            const int64_t d = stt.k - k_before + (stt.status == BREAKDOWN ? 1 : 0);
            // graph: whole bodies of `unroll` iterations (the tail returns at once)
            body_kernels += profile ? per_it * d
                                    : (int64_t)per_it * s->unroll * std::max<int64_t>(1, (d + s->unroll - 1) / s->unroll);
        }
        if (!profile) {
            float ms = 0;
            cudaEventElapsedTime(&ms, s->ev[6], s->ev[7]);
            loop_ms += ms;
        }
        if (stt.k % history_stride == 0 && stt.k != last_rec && stt.k > 0 &&
            (stt.status == RUNNING || stt.iterations == stt.k)) {
            if ((rc = record(stt.k, stt.rel))) return rc;
        }
    }
    if (last_rec != stt.iterations) {
        if ((rc = record(stt.iterations, stt.rel))) return rc;
    }
    res->iterations = stt.iterations;
    res->status = stt.status;
    res->final_rel = stt.rel;
    res->n_hist = nh;
    res->loop_ms = profile ? (stage_ms[0] + stage_ms[1] + stage_ms[2]) : loop_ms;
    res->history_ms = hist_ms;
    // kernels launched by this solve: SpMV + init, the iteration loop, metrics
    res->launches = 2 + body_kernels + metric_launches;
    res->stage_ms[0] = stage_ms[0];
    res->stage_ms[1] = stage_ms[1];
    res->stage_ms[2] = stage_ms[2];
    return 0;
}

}  // extern "C"
