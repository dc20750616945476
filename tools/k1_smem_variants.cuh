// tools/k1_smem_variants.cuh -- NOT BUILT.  Two alternative SpMV (K1) kernels
// for the slice-shared-offset layout, kept out of the product after they
// measured slower than the classic walk (cg.cu: cg_spmv_pq) on every mode of
// C2 and C4 (round 2; DESIGN.md §3 "measured and rejected",
// profiles/r2_k1_variants.json).  Both were bitwise equal to the classic
// kernel on the parity set (tests were in tests/test_gpu_k1w.py, git history).
//
//   K1P  values of a thread's next row prefetched into shared memory by
//        per-thread cp.async (L2 evict-first) -- C2 DW K1 55.8 -> 65.4 us
//   K1W  p windows (+ values when they fit) of whole tiles staged by
//        cp.async.bulk in a 2-slot ring, 1024 threads (one per row) --
//        C2 DW K1 55.8 -> 81.3 us; a 512-consumer + producer-warp version
//        with 512-row stages: 67.8 us ("wait" + barrier stalls, 17 warps/SM)
//
// To try one again, paste the kernels back into cg.cu before the K2 section
// and restore the selection / launch code below.

// ---------------------------------------------------------------- K1P
// K1 for the slice-shared-offset layout with the matrix values of a thread's
// NEXT row prefetched into shared memory by per-thread async copies
// (cp.async, evict-first L2 policy) while the current row computes.  The
// classic walk pays one HBM round trip per chunk of values; here the values
// arrive a whole row ahead (a row of a few entries takes several
// microseconds of chain latency under load, far more than the HBM
// latency), so a row's chain is slice words -> pattern word (L1) -> gathers
// of p (L2) -> FP64 chain, with no dependent HBM access.  Up to PF slots of a
// row are prefetched (double-buffered: 2 * PF * THREADS doubles of dynamic
// shared memory); longer rows load the rest directly.  Thread / row mapping,
// per-row order and the p.q reduction are K1's: results are bitwise K1's.
constexpr int K1P_PF = 8;

__device__ __forceinline__ void cp_async8(double *dst_smem, const double *src, uint64_t policy) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(smem_u32(dst_smem)), "l"(src),
                 "l"(policy)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// issue the copies of up to PF value slots of `row` (sw: its slice words)
template <int NT>
__device__ __forceinline__ void k1p_prefetch(const SellMatrix &A, int64_t row, int64_t n, SliceWords sw,
                                             double *vb, uint64_t pol) {
    constexpr uint64_t LO = (1ull << 36) - 1;
    if (row < n) {
        const int L = (int)(((uint64_t)sw.w1 & LO) - ((uint64_t)sw.w0 & LO));
        const double *vp = A.vals + ((int64_t)((uint64_t)sw.w0 & LO) << 5) + (row & 31);
#pragma unroll
        for (int k = 0; k < K1P_PF; k++)
            if (k < L) cp_async8(vb + k * NT, vp + k * SLICE, pol);
    }
    cp_async_commit();  // one group per row (empty past the end): counts stay in step
}

template <int M, int U, int NT>
__device__ __forceinline__ V<Arith<M>::W> k1p_row(const SellMatrix &A, const double *__restrict__ x, int64_t row,
                                                  SliceWords sw, const double *vb) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    constexpr uint64_t LO = (1ull << 36) - 1;
    const uint64_t d0 = (uint64_t)sw.w0, d1 = (uint64_t)sw.w1;
    const int L = (int)((d1 & LO) - (d0 & LO));
    const int lane = (int)(row & 31);
    const int grow = (int)(A.row_base + row);
    const uint64_t *__restrict__ op = A.om + (d0 >> 36);
    const double *__restrict__ vp = A.vals + ((int64_t)(d0 & LO) << 5) + lane;
    V<W> s = zero<W>();
    for (int k0 = 0; k0 < L; k0 += U) {
        uint64_t om[U];
        double a[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            om[u] = __ldg(op + k0 + u);
            a[u] = (k0 + u < K1P_PF) ? vb[(k0 + u) * NT] : ld_stream(vp + (k0 + u) * SLICE);
        }
        bool ok[U];
        V<W> xv[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            ok[u] = (uint32_t)(om[u] >> 32) & (1u << lane);
            const int c = grow + (ok[u] ? (int)(uint32_t)om[u] : 0);
            xv[u] = load_aos_ro<W>(x, c);
        }
#pragma unroll
        for (int u = 0; u < U; u++)
            if (ok[u]) s = Ar::add(s, Ar::dxmul(a[u], xv[u]));
    }
    return s;
}

template <int M, bool FUSED>
__global__ void __launch_bounds__(SpTraits<M>::THREADS, SpTraits<M>::MINB)
    cg_spmv_pq_pf(SellMatrix A, const double *__restrict__ p, double *__restrict__ q, Geo g,
                  double *__restrict__ part, CgState *st, cudaGraphConditionalHandle h, int use_cond) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    constexpr int NT = SpTraits<M>::THREADS;
    constexpr int RPT = SpTraits<M>::RPT;
    constexpr bool STAGE = FUSED && NT != TILE_THREADS;
    extern __shared__ __align__(16) double vbuf[];  // [2][K1P_PF][NT]
    __shared__ double terms[STAGE ? W * TILE : 1];
    __shared__ double smem[W * TILE_THREADS / 32];
    __shared__ int s_last;
    if (stopped_k1(st, h, use_cond)) return;
    const bool norm_all = st->norm_all != 0;
    const int64_t n = g.n;
    const int dir = (int)(st->k & 1);
    const int64_t cnt = k1_count(g);
    const int64_t nmine = cnt > blockIdx.x ? (cnt - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint64_t pol = l2_policy_evict_first();
    auto tile_at = [&](int64_t t) { return k1_tile(g, snake(blockIdx.x + t * gridDim.x, cnt, dir)); };
    double *myb = vbuf + threadIdx.x;
    int64_t tile = nmine ? tile_at(0) : 0;
    SliceWords sw = slice_words(A, tile * TILE + threadIdx.x);
    if (nmine) k1p_prefetch<NT>(A, tile * TILE + threadIdx.x, n, sw, myb, pol);
#pragma unroll 1
    for (int64_t t = 0; t < nmine; t++) {
        const int64_t tile_next = (t + 1 < nmine) ? tile_at(t + 1) : -1;
        V<W> acc = zero<W>();
#pragma unroll 1
        for (int k = 0; k < RPT; k++) {
            const int li = threadIdx.x + k * NT;
            const int64_t row = tile * TILE + li;
            // next row (the next tile's first after the last): slice words,
            // then its values into the other buffer (RPT is even: the buffer
            // parity is k's)
            const int64_t nrow = (k + 1 < RPT) ? row + NT : (tile_next >= 0 ? tile_next * TILE + threadIdx.x : -1);
            SliceWords nsw = sw;
            if (nrow >= 0) {
                nsw = slice_words(A, nrow);
                k1p_prefetch<NT>(A, nrow, n, nsw, myb + ((k + 1) & 1) * K1P_PF * NT, pol);
            } else {
                cp_async_commit();
            }
            cp_async_wait1();  // this row's values have landed (this thread's own copies)
            V<W> term = zero<W>();
            if (row < n) {
                V<W> sv = k1p_row<M, SpTraits<M>::U, NT>(A, p, row, sw, myb + (k & 1) * K1P_PF * NT);
                if (norm_all) sv = Ar::norm(sv);
                store<W>(q, g.ld, row, sv);
                if (FUSED) term = Ar::mul(load_aos_ro<W>(p, g.p_off + row), sv);
                if (FUSED && !STAGE) acc = Ar::add(acc, term);
            }
            if (STAGE) {
#pragma unroll
                for (int w = 0; w < W; w++) terms[w * TILE + li] = term.w[w];
            }
            sw = nsw;
        }
        if (STAGE) {
            __syncthreads();
            if (threadIdx.x < TILE_THREADS) {
                const int64_t base = tile * TILE + threadIdx.x;
#pragma unroll
                for (int e = 0; e < TILE_ELEMS; e++) {
                    if (base + e * TILE_THREADS < n) {
                        V<W> tv;
#pragma unroll
                        for (int w = 0; w < W; w++) tv.w[w] = terms[w * TILE + threadIdx.x + e * TILE_THREADS];
                        acc = Ar::add(acc, tv);
                    }
                }
            }
        }
        if (FUSED) {
            acc = block_tree_first<M, TILE_THREADS>(acc, smem);
            if (threadIdx.x == 0) store_part<W>(part, g.part_ld, g.tile_off + tile, acc);
        }
        tile = tile_next;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (!FUSED || !g.final_) return;
    if (!last_block_done(&st->ticket[0], &s_last)) return;
    V<W> pq = reduce_partials_first<M>(part, g.part_ld, g.ntiles_glob, smem);
    if (threadIdx.x == 0) {
        st->ticket[0] = 0u;
        scalar_alpha<M>(st, pq, h, use_cond);
    }
}

// ---------------------------------------------------------------- K1W
// Windowed K1 for the slice-shared-offset layout (stencils, bands: C1-C4).
// The tile's rows are processed in stages of R rows (R = 256, 512 or 1024).
// A producer warp brings everything a stage reads into a shared-memory ring
// with 1-D bulk copies (cp.async.bulk, mbarrier per stage):
//   * the stage's slice descriptors and its matrix values (contiguous),
//   * the windows of p the stage gathers from: the distinct column offsets
//     of the matrix, clustered (offsets closer than R + 4 share a cluster),
//     give one contiguous window per cluster, [g0 + omin_j, g0 + R - 1 +
//     omax_j] for a stage starting at global row g0.
// The consumer threads (256 or 512) then walk their rows with every operand in shared
// memory: a row's dependency chain is the L1-resident slot word -> a shared
// load -> the FP64 chain, instead of descriptor (L2) -> pattern (L1) ->
// gather of p (L2) with HBM values in between (round 1: K1 was latency-bound
// on that chain, DESIGN.md §3 item 1).  The p.q terms are reduced in the
// canonical tile order and each row's left-to-right sum is unchanged --
// results are bitwise K1's.
constexpr int K1W_MAXCLU = 16;
constexpr int K1W_MAXNS = 8;

struct WinPlan {
    int NS, nclu, vs;                // ring slots (whole tiles), p windows, values staged
    int stage_doubles;               // one ring stage
    int val_off, win_off, desc_off;  // section offsets (doubles) in a stage
    int sd0;                         // shared index delta of the diagonal record
    int omin[K1W_MAXCLU], pre[K1W_MAXCLU], span[K1W_MAXCLU];
    const uint2 *tab;                // per pattern slot: {lane mask, shared index delta}
};

// named barriers of K1W (0 is __syncthreads)
__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// block tree over the first NT threads, synchronised with named barrier 1
// (the producer warp and any further consumers do not take part)
template <int M, int NT>
__device__ __forceinline__ V<Arith<M>::W> block_tree_bar(V<Arith<M>::W> v, double *smem) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    constexpr int NW = NT / 32;
    v = warp_tree<M>(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < W; k++) smem[k * NW + wid] = v.w[k];
    }
    named_bar(1, NT);
    if (wid == 0) {
        V<W> u = zero<W>();
        if (lane < NW) {
#pragma unroll
            for (int k = 0; k < W; k++) u.w[k] = smem[k * NW + lane];
        }
#pragma unroll
        for (int off = NW / 2; off >= 1; off >>= 1) u = Ar::add(u, shfl_down<W>(u, off));
        v = u;
    }
    named_bar(1, NT);
    return v;
}

template <int W>
__device__ __forceinline__ V<W> ld_rec(const double *base, int idx) {
    V<W> r;
    if (W == 2) {
        const double2 t = *reinterpret_cast<const double2 *>(base + 2 * idx);
        r.w[0] = t.x;
        r.w[W - 1] = t.y;
    } else {
#pragma unroll
        for (int k = 0; k < W; k++) r.w[k] = base[W * idx + k];
    }
    return r;
}

// One thread per row of the tile: 1024 threads (32 warps), row c of every
// tile the CTA walks is thread c's.  A ring of NS whole-tile slots; thread 0
// refills a slot with the CTA's tile NS ahead once every thread is done with
// it (two CTA barriers per tile), so NS - 1 tiles of operands are in flight
// while one is computed.  A slot holds the tile's slice descriptors, the p
// windows and -- when they fit (VS: values staged; stencils with few slots)
// -- the tile's matrix values; otherwise the values stream straight from HBM
// (ld.global.cs, all U loads of a chunk in flight per thread).  The p.q
// terms are replayed by the first 256 threads in the canonical order from
// the q just written (global, this CTA's own stores) and p (the window).
constexpr int K1W_THREADS = TILE;

template <int M, bool VS>
struct K1wTraits {
    static constexpr int U = VS ? 4 : 8;
};

template <int M, bool FUSED, bool VS>
__global__ void __launch_bounds__(K1W_THREADS, 1)
    cg_spmv_pq_win(SellMatrix A, const double *__restrict__ p, double *__restrict__ q, Geo g,
                   double *__restrict__ part, CgState *st, WinPlan wp, cudaGraphConditionalHandle h,
                   int use_cond) {
    using Ar = Arith<M>;
    constexpr int W = Ar::W;
    constexpr int U = K1wTraits<M, VS>::U;
    constexpr uint64_t LO = (1ull << 36) - 1;
    extern __shared__ __align__(128) double ring[];
    __shared__ uint64_t full[K1W_MAXNS];
    __shared__ double smem[W * TILE_THREADS / 32];
    __shared__ int s_last;
    if (stopped_k1(st, h, use_cond)) return;
    const bool norm_all = st->norm_all != 0;
    const int64_t n = g.n;
    const int dir = (int)(st->k & 1);
    const int NS = wp.NS;
    const int64_t cnt = k1_count(g);
    const int64_t nmine = cnt > blockIdx.x ? (cnt - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int c = threadIdx.x, lane = c & 31;
    const int64_t ldp_even = (g.ldp + 1) & ~(int64_t)1;
    constexpr int ND = TILE / SLICE + 2;  // descriptors per slot (even count)
    // slot refill (thread 0): descriptors, [values], p windows of tile tix
    auto issue = [&](int64_t tix) {
        const int sidx = (int)(tix % NS);
        double *stg = ring + (size_t)sidx * wp.stage_doubles;
        const int64_t tile = k1_tile(g, snake(blockIdx.x + tix * gridDim.x, cnt, dir));
        const int64_t r0 = tile * TILE;
        const int64_t sl0 = r0 >> 5;
        const int64_t sl1 = min(sl0 + TILE / SLICE, A.n_slices);
        const int64_t v0 = (int64_t)(__ldg((const unsigned long long *)A.slice_ptr + sl0) & LO) << 5;
        const int64_t v1 = (int64_t)(__ldg((const unsigned long long *)A.slice_ptr + sl1) & LO) << 5;
        const int64_t g0 = A.row_base + r0;
        // window j: global records [lo, hi) clipped to [0, ldp), widened to
        // even records (16-B aligned copies; pre[j] keeps the shared
        // position's parity equal to the global one)
        auto win = [&](int j, int64_t &lo, int64_t &clo, int64_t &chi) {
            lo = g0 + wp.omin[j];
            const int64_t hi = g0 + TILE + wp.omin[j] + wp.span[j];
            clo = max(lo, (int64_t)0) & ~(int64_t)1;
            chi = min((min(hi, g.ldp) + 1) & ~(int64_t)1, ldp_even);
        };
        uint32_t bytes = (uint32_t)(ND * 8) + (VS ? (uint32_t)((v1 - v0) * 8) : 0u);
        for (int j = 0; j < wp.nclu; j++) {
            int64_t lo, clo, chi;
            win(j, lo, clo, chi);
            if (chi > clo) bytes += (uint32_t)((chi - clo) * 8 * W);
        }
        const uint64_t pol_stream = l2_policy_evict_first(), pol_keep = l2_policy_evict_last();
        mbar_arrive_expect_tx(&full[sidx], bytes);
        bulk_g2s(stg + wp.desc_off, A.slice_ptr + sl0, (uint32_t)(ND * 8), &full[sidx]);
        if (VS && v1 > v0)
            bulk_g2s_hint(stg + wp.val_off, A.vals + v0, (uint32_t)((v1 - v0) * 8), &full[sidx], pol_stream);
        for (int j = 0; j < wp.nclu; j++) {
            int64_t lo, clo, chi;
            win(j, lo, clo, chi);
            if (chi > clo)
                bulk_g2s_hint(stg + wp.win_off + (int64_t)(j * TILE + wp.pre[j] + (clo - lo)) * W, p + clo * W,
                              (uint32_t)((chi - clo) * 8 * W), &full[sidx], pol_keep);
        }
    };
    if (c == 0) {
        for (int i = 0; i < NS; i++) mbar_init(&full[i], 1);
        mbar_init_fence();
        for (int64_t i = 0; i < NS && i < nmine; i++) issue(i);
    }
    __syncthreads();
    for (int64_t tix = 0; tix < nmine; tix++) {
        const int sidx = (int)(tix % NS);
        const int64_t tile = k1_tile(g, snake(blockIdx.x + tix * gridDim.x, cnt, dir));
        const int64_t row = tile * TILE + c;
        mbar_wait(&full[sidx], (uint32_t)((tix / NS) & 1));
        const double *stg = ring + (size_t)sidx * wp.stage_doubles;
        const double *sw = stg + wp.win_off;
        if (row < n) {
            const uint64_t *dsc = reinterpret_cast<const uint64_t *>(stg + wp.desc_off);
            const uint64_t d0 = dsc[c >> 5], d1 = dsc[(c >> 5) + 1];
            const int L = (int)((d1 & LO) - (d0 & LO));
            const uint2 *tp = wp.tab + (d0 >> 36);
            const double *vp = VS ? stg + wp.val_off + (((d0 & LO) - (dsc[0] & LO)) << 5) + lane
                                  : A.vals + ((int64_t)(d0 & LO) << 5) + lane;
            V<W> sacc = zero<W>();
            for (int k0 = 0; k0 < L; k0 += U, tp += U, vp += U * SLICE) {
                uint2 tw[U];
                double a[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    tw[u] = __ldg(tp + u);
                    a[u] = VS ? vp[u * SLICE] : ld_stream(vp + u * SLICE);  // (padded past the end)
                }
                bool ok[U];
                V<W> xv[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    ok[u] = (tw[u].x >> lane) & 1u;
                    xv[u] = ld_rec<W>(sw, c + (ok[u] ? (int)tw[u].y : wp.sd0));
                }
#pragma unroll
                for (int u = 0; u < U; u++)
                    if (ok[u]) sacc = Ar::add(sacc, Ar::dxmul(a[u], xv[u]));
            }
            if (norm_all) sacc = Ar::norm(sacc);
            store<W>(q, g.ld, row, sacc);
        }
        __syncthreads();  // q of the whole tile is written (and visible to the CTA)
        if (FUSED && c < TILE_THREADS) {
            V<W> acc = zero<W>();
#pragma unroll
            for (int j = 0; j < TILE_ELEMS; j++) {
                const int cc = c + j * TILE_THREADS;
                const int64_t rr = tile * TILE + cc;
                if (rr < n) acc = Ar::add(acc, Ar::mul(ld_rec<W>(sw, cc + wp.sd0), load<W>(q, g.ld, rr)));
            }
            const V<W> tot = block_tree_bar<M, TILE_THREADS>(acc, smem);
            if (c == 0) store_part<W>(part, g.part_ld, g.tile_off + tile, tot);
        }
        __syncthreads();  // slot sidx is free
        if (c == 0 && tix + NS < nmine) {
            fence_proxy_async_smem();
            issue(tix + NS);
        }
    }
    if (!FUSED || !g.final_) return;
    if (!last_block_done(&st->ticket[0], &s_last)) return;
    V<W> pq = reduce_partials_first<M>(part, g.part_ld, g.ntiles_glob, smem);
    if (threadIdx.x == 0) {
        st->ticket[0] = 0u;
        scalar_alpha<M>(st, pq, h, use_cond);
    }
}


// ---- host plan (K1W)
// Plan the windowed K1 (cg_spmv_pq_win) for a dia-layout matrix: cluster
// the distinct column offsets (offsets closer than a tile share a window),
// size one whole-tile ring slot (descriptors + windows [+ values]), and take
// the values into the slot when >= 2 such slots fit `budget` (else they
// stream from HBM and only windows are staged, >= 2 slots).  Builds the
// per-slot table {lane mask, shared index delta}.  Returns false when no
// ring fits (the classic K1 is used).  MWCG_K1W_VS=0/1 forces the variant.
bool plan_windows(mwcg_solver *s, int W, size_t budget) {
    const SellMatrixOwned *M = s->Mown;
    if (!M || !s->A.dia || M->pat_host.empty() || (s->A.row_base & 1)) return false;
    const std::vector<uint64_t> &pat = M->pat_host;
    std::vector<int> offs{0};
    for (uint64_t w : pat)
        if (w >> 32) offs.push_back((int)(uint32_t)w);
    std::sort(offs.begin(), offs.end());
    offs.erase(std::unique(offs.begin(), offs.end()), offs.end());
    const int64_t ns = s->A.n_slices;
    auto align16 = [](int64_t d) { return (d + 15) & ~(int64_t)15; };  // doubles -> 128 B
    WinPlan wp{};
    std::vector<int> omin, omax;
    for (int o : offs) {
        if (omin.empty() || (int64_t)o - omax.back() > TILE + 4) {
            omin.push_back(o);
            omax.push_back(o);
        } else {
            omax.back() = o;
        }
    }
    if ((int)omin.size() > K1W_MAXCLU) return false;
    wp.nclu = (int)omin.size();
    int64_t pre = 1;
    for (int j = 0; j < wp.nclu; j++) {
        if (((pre - omin[j]) % 2 + 2) % 2) pre++;  // window j copies start 16-B aligned
        wp.omin[j] = omin[j];
        wp.span[j] = omax[j] - omin[j];
        wp.pre[j] = (int)pre;
        pre += wp.span[j] + 4;
    }
    const int64_t win_recs = (int64_t)wp.nclu * TILE + pre;
    int64_t vslots = 0;  // most value slots any tile holds
    for (int64_t sl = 0; sl < ns; sl += TILE / SLICE) {
        const int64_t e = std::min<int64_t>(sl + TILE / SLICE, ns);
        vslots = std::max<int64_t>(vslots, (int64_t)((M->desc_host[e] & ((1ull << 36) - 1)) -
                                                     (M->desc_host[sl] & ((1ull << 36) - 1))));
    }
    const char *fv = std::getenv("MWCG_K1W_VS");
    for (int vs : {1, 0}) {
        if (fv && std::atoi(fv) != vs) continue;
        wp.vs = vs;
        wp.val_off = 0;
        wp.win_off = vs ? (int)align16(vslots * SLICE + 8 * SLICE) : 0;  // + slack: chunks read past a slice
        wp.desc_off = (int)(wp.win_off + align16(win_recs * W));
        wp.stage_doubles = (int)(wp.desc_off + align16(TILE / SLICE + 2));
        const size_t slot_bytes = sizeof(double) * (size_t)wp.stage_doubles;
        const int NS = (int)std::min<size_t>(K1W_MAXNS, budget / slot_bytes);
        if (NS < 2) continue;
        wp.NS = NS;
        // shared index delta of every pattern slot (row c reads record c + delta)
        auto delta = [&](int off) {
            int j = 0;
            while (j + 1 < wp.nclu && off > omax[j]) j++;
            return j * TILE + wp.pre[j] + (off - wp.omin[j]);
        };
        wp.sd0 = delta(0);
        std::vector<uint2> tab(pat.size());
        for (size_t k = 0; k < pat.size(); k++) {
            const uint32_t mask = (uint32_t)(pat[k] >> 32);
            tab[k] = make_uint2(mask, (unsigned)(mask ? delta((int)(uint32_t)pat[k]) : wp.sd0));
        }
        if (s->wtab) pool_free(s->wtab, s->stream);
        s->wtab = nullptr;
        if (pool_alloc((void **)&s->wtab, sizeof(uint2) * tab.size(), s->stream) != cudaSuccess) return false;
        if (cudaMemcpyAsync(s->wtab, tab.data(), sizeof(uint2) * tab.size(), cudaMemcpyHostToDevice,
                            s->stream) != cudaSuccess ||
            cudaStreamSynchronize(s->stream) != cudaSuccess)
            return false;
        wp.tab = s->wtab;
        s->wp = wp;
        s->k1w_smem = slot_bytes * (size_t)NS;
        return true;
    }
    return false;
}


// ---- launch_k1 branches
#if 0
    if (s->k1p) {
        cfg.dynamicSmemBytes = sizeof(double) * 2 * K1P_PF * SpTraits<M>::THREADS;
        cudaLaunchKernelEx(&cfg, cg_spmv_pq_pf<M, FUSED>, s->A, pc, s->q, g, s->part, s->st, h, use_cond);
        return;
    }
    if (s->k1w) {
        cfg.blockDim = dim3(K1W_THREADS);
        cfg.dynamicSmemBytes = s->k1w_smem;
        if (s->wp.vs)
            cudaLaunchKernelEx(&cfg, cg_spmv_pq_win<M, FUSED, true>, s->A, pc, s->q, g, s->part, s->st, s->wp, h,
                               use_cond);
        else
            cudaLaunchKernelEx(&cfg, cg_spmv_pq_win<M, FUSED, false>, s->A, pc, s->q, g, s->part, s->st, s->wp, h,
                               use_cond);
        return;
    }
#endif
// ---- compute_grids_t selection
#if 0
    {
        // windowed K1 for the slice-shared-offset layout (MWCG_K1W=0/1 overrides)
        const char *t = std::getenv("MWCG_K1W");
        s->k1w = false;
        if (t && t[0] == '1') {
            int maxsm = 0;
            cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
            // dynamic budget: the opt-in maximum less the static shared memory
            const size_t budget = (size_t)std::max(0, maxsm - 1024);
            s->k1w = plan_windows(s, Arith<M>::W, budget);
            if (s->k1w) {
                // the attribute is per function (shared by every solver of this
                // mode): always the full budget, never one solver's ring size
                const int dyn = (int)budget;
                cudaFuncSetAttribute(cg_spmv_pq_win<M, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
                cudaFuncSetAttribute(cg_spmv_pq_win<M, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
                cudaFuncSetAttribute(cg_spmv_pq_win<M, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
                cudaFuncSetAttribute(cg_spmv_pq_win<M, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
                if (cudaGetLastError() != cudaSuccess) s->k1w = false;
            }
        }
        cudaGetLastError();
    }
    {
        // K1 with prefetched values for the slice-shared-offset layout
        const char *t = std::getenv("MWCG_K1P");
        s->k1p = !s->k1w && s->A.dia && (t ? t[0] != '0' : true);
        if (s->k1p) {
            const int dyn = (int)(sizeof(double) * 2 * K1P_PF * SpTraits<M>::THREADS);
            cudaFuncSetAttribute(cg_spmv_pq_pf<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
            cudaFuncSetAttribute(cg_spmv_pq_pf<M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
            if (cudaGetLastError() != cudaSuccess) s->k1p = false;
        }
    }
    if (s->k1w) {
        nb[0] = 1;             // one CTA (ring) per SM, persistent
        full &= ~1u;
    }
    if (s->k1p) {
        MWCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &nb[0], cg_spmv_pq_pf<M, true>, SpTraits<M>::THREADS, sizeof(double) * 2 * K1P_PF * SpTraits<M>::THREADS));
        full &= ~1u;           // persistent: the prefetch runs across the CTA's tiles
    }
#endif
