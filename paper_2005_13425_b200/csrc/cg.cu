// CG vector kernels (Nekbone add2s1 / add2s2 / glsc3) and the fused,
// device-resident CG iteration of sembench/cg.py:114-193.
//
// * add2s1 / add2s2 are bit-exact restatements of _scale_add / _axpy_into
//   (cg.py:95-104): multiply rounded, then add rounded (no FMA).
// * glsc3 is a deterministic fixed-tree reduction (reduce.cuh); on the box
//   the weight 1/multiplicity is recomputed from the lattice, so the three
//   weighted dots of an iteration read 2 streams instead of 3.
// * The CG driver keeps rtz / pap / alpha / beta in a device-side
//   sem_cg_state and never synchronises the host; early exits (rtz == 0,
//   tolerance, breakdown) set a device stop flag that turns the remaining
//   queued launches into no-ops.  Single GPU (sem_cg_run): two streaming
//   launches plus one single-block settle per iteration --
//     1. Ax with the iteration head fused in (ax_pencil.cuh, CGM = 2):
//        x += alpha_prev p_old (deferred from the previous iteration),
//        p = beta p + r, w = A_local p, per-CTA partials of <p, A p>;
//     1b. cg_settle_kernel: the partials in a fixed order -> alpha;
//     2. cg_update2_kernel: r += (-alpha) mask(dssum(w)) with the ordered
//        dssum gathered per row, and <r, r>_c -> rnorm, beta's numerator;
//   and sem_cg_finalize applies the last pending x update.  120 B per point
//   per iteration (Ax 96: p, x read+write, r, g, w; update 24: w, r r+w)
//   against the 240 B of the paper's model.  The multi-GPU slab solver runs
//   the same two kernels per rank (sem_cg_ax_slab, sem_cg_update_slab), each
//   leaving a partial sum that the ranks combine (sem_cg_finish).
#include <math.h>

#include <stdlib.h>

#include <algorithm>
#include <atomic>

#ifndef SEM_UPD_MINB
#define SEM_UPD_MINB 6
#endif

#include "box.cuh"
#include "reduce.cuh"
#include "flat.cuh"
#include "rows.cuh"
#include "ax_pencil.cuh"

namespace sem {

int ax_dispatch(const double* u, const double* g, const double* dx, double* w, int64_t E,
                int n, int variant, cudaStream_t stream, int pdl = -1);
int ax_cg_dispatch(const double* g, const double* dx, double* w, int64_t E, int n, CgpArgs a,
                   int mode, cudaStream_t stream);

constexpr int kVecThreads = 256;

static unsigned vec_grid(int64_t pairs)
{
    const int64_t per = (int64_t)kVecThreads;
    int64_t b = (pairs + per - 1) / per;
    const int64_t cap = 16LL * sm_count();
    if (b > cap) b = cap;
    return (unsigned)(b > 0 ? b : 1);
}

// ---------------------------------------------------------- add2s1/add2s2 --
__global__ void __launch_bounds__(kVecThreads)
add2s1_kernel(double* __restrict__ p, const double* __restrict__ z, double beta, int64_t m)
{
    const int64_t stride = (int64_t)gridDim.x * kVecThreads;
    for (int64_t q = (int64_t)blockIdx.x * kVecThreads + threadIdx.x; q < m; q += stride)
        p[q] = add_rn(mul_rn(beta, p[q]), __ldg(z + q));
}

__global__ void __launch_bounds__(kVecThreads)
add2s2_kernel(double* __restrict__ x, const double* __restrict__ y, double alpha, int64_t m)
{
    const int64_t stride = (int64_t)gridDim.x * kVecThreads;
    for (int64_t q = (int64_t)blockIdx.x * kVecThreads + threadIdx.x; q < m; q += stride)
        x[q] = add_rn(x[q], mul_rn(alpha, __ldg(y + q)));
}

// ------------------------------------------------------------- glsc3 -----
__global__ void __launch_bounds__(kReduceThreads)
glsc3_kernel(const double* __restrict__ a, const double* __restrict__ b,
             const double* __restrict__ wt, int64_t m, double* out, ReduceScratch* rs)
{
    double acc = 0.0;
    const int64_t stride = (int64_t)gridDim.x * kReduceThreads;
    for (int64_t q = (int64_t)blockIdx.x * kReduceThreads + threadIdx.x; q < m; q += stride)
        acc += mul_rn(mul_rn(__ldg(a + q), __ldg(b + q)), __ldg(wt + q));
    const double vals[1] = {acc};
    reduce_publish_and_finish<1, kReduceThreads>(vals, rs, [&](const double (&t)[1]) { *out = t[0]; });
}

// Box-weighted dot over flat point pairs (flat.cuh): w = 1/multiplicity from
// the lattice.  The loop nest (and so the summation order) is shared with the
// fused CG kernels below, so weighted_dot reproduces their reductions
// bit-for-bit.
#define SEM_PAIR_LOOP(E_)                                                              \
    constexpr int NP = PairCfg<N>::NP;                                                 \
    const int64_t units_ = (E_) * (int64_t)(N * N * N) / NP;                           \
    for (int64_t u_ = (int64_t)blockIdx.x * PairCfg<N>::THREADS + threadIdx.x; u_ < units_; \
         u_ += (int64_t)gridDim.x * PairCfg<N>::THREADS)

template <int N>
__global__ void __launch_bounds__(PairCfg<N>::THREADS)
glsc3_box_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t E,
                 BoxFlat bf, double* out, ReduceScratch* rs)
{
    double acc = 0.0;
    SEM_PAIR_LOOP(E) {
        const int64_t q0 = u_ * NP;
        ElemCoord c;
        int i, j, k;
        pair_point<N>(q0, bf, c, i, j, k);
        double va[NP], vb[NP];
        ld_pair<N>(a + q0, va);
        ld_pair<N>(b + q0, vb);
#pragma unroll
        for (int h = 0; h < NP; ++h)
            acc += mul_rn(mul_rn(va[h], vb[h]), inv_mult_of<N>(c, i + h, j, k, bf.b));
    }
    const double vals[1] = {acc};
    reduce_publish_and_finish<1, PairCfg<N>::THREADS>(vals, rs,
                                                      [&](const double (&tt)[1]) { *out = tt[0]; });
}

// ------------------------------------------------------------ CG kernels --
// Scalar bookkeeping of the three reductions of an iteration, shared by the
// single-GPU kernels (total = this GPU's sum) and the multi-GPU finish kernel
// (total = per-rank partials combined in rank order).
constexpr int kPhaseInit = 0, kPhasePap = 1;  // 2 = <r,r> (fin_rr)

__device__ __forceinline__ void fin_init(sem_cg_state* st, double rtz)
{
    st->rtz = rtz;
    st->rtz_old = 1.0;  // cg.py:146 (unused: beta = 0 on iteration 1)
    st->pap = 0.0;
    st->alpha = 0.0;
    st->beta = 0.0;
    st->it = 0;
    st->iterations_run = 0;
    st->stop = 0;
    st->breakdown_it = 0;
    st->x_pending = 0;
}

// pap_s: <p, A p> as the fused kernels accumulate it, scaled by
// 2^(2k), k = pap_scale_exp(rtz) (sem_common.cuh): alpha = (rtz 2^(2k)) / pap_s
// is the unscaled rtz / pap bit for bit in the normal range
// rtz, it0: st->rtz, st->it as the calling kernel loaded them at entry (no
// kernel changes them in between), so the finishing thread pays no further
// state round trip after its sum
__device__ __forceinline__ void fin_pap_v(sem_cg_state* st, double pap_s, double rtz, int it0)
{
    const int k = pap_scale_exp(rtz);
    st->pap = ldexp(pap_s, -2 * k);  // reported value (may underflow)
    st->x_pending = 0;  // the Ax prologues of this iteration applied it
    if (pap_s <= 0.0) {  // cg.py:164-169 breakdown
        st->stop = 2;
        st->breakdown_it = it0 + 1;
    } else {
        st->alpha = ldexp(rtz, 2 * k) / pap_s;
    }
}

__device__ __forceinline__ void fin_pap(sem_cg_state* st, double pap_s)
{
    fin_pap_v(st, pap_s, st->rtz, st->it);
}

// the state fields fin_rr reads, loaded ahead (reduce_publish_and_finish_pre)
struct RrCtx {
    int it0;
    double rtz0, tol;
};
__device__ __forceinline__ RrCtx rr_ctx(const sem_cg_state* st)
{
    return RrCtx{st->it, st->rtz, st->tolerance};
}

__device__ __forceinline__ void fin_rr_v(sem_cg_state* st, double rtr, double* history, const RrCtx& c)
{
    const int it = c.it0 + 1;
    const double rnorm = sqrt(rtr);
    history[it - 1] = rnorm;
    st->iterations_run = it;
    st->rtz_old = c.rtz0;
    st->rtz = rtr;  // equals <r,r>_c at the top of the next iteration
    st->it = it;
    st->x_pending = 1;  // x += alpha p of this iteration: next Ax prologue / finalize
    if (c.tol > 0.0 && rnorm < c.tol) st->stop = 3;
}

__device__ __forceinline__ void fin_rr(sem_cg_state* st, double rtr, double* history)
{
    fin_rr_v(st, rtr, history, rr_ctx(st));
}

__device__ __forceinline__ void fin_phase(sem_cg_state* st, int phase, double total,
                                          double* history)
{
    if (phase == kPhaseInit) fin_init(st, total);
    else if (phase == kPhasePap) fin_pap(st, total);
    else fin_rr(st, total, history);
}

// init: r = mask(f) (assembly.py:123-129), x = p = 0, rtz = <r,r>_c.
template <int N, bool DIST>
__global__ void __launch_bounds__(PairCfg<N>::THREADS)
cg_init_kernel(const double* __restrict__ f, double* __restrict__ x, double* __restrict__ r,
               double* __restrict__ p, int64_t E, BoxFlat bf, sem_cg_state* st,
               ReduceScratch* rs, int max_iterations, double tolerance)
{
    double acc = 0.0;
    SEM_PAIR_LOOP(E) {
        const int64_t q0 = u_ * NP;
        ElemCoord c;
        int i, j, k;
        pair_point<N>(q0, bf, c, i, j, k);
        double fv[NP], z[NP];
        ld_pair<N>(f + q0, fv);
#pragma unroll
        for (int h = 0; h < NP; ++h) {
            fv[h] = mul_rn(fv[h], mask_of<N>(c, i + h, j, k, bf.b));
            z[h] = 0.0;
            acc += mul_rn(mul_rn(fv[h], fv[h]), inv_mult_of<N>(c, i + h, j, k, bf.b));
        }
        st_pair<N>(r + q0, fv);
        st_pair<N>(x + q0, z);
        st_pair<N>(p + q0, z);
    }
    const double vals[1] = {acc};
    reduce_publish_and_finish<1, PairCfg<N>::THREADS>(vals, rs, [&](const double (&t)[1]) {
        st->max_iterations = max_iterations;
        st->tolerance = tolerance;
        if (DIST) {
            st->local_sum = t[0];
            fin_init(st, 0.0);  // rtz set by sem_cg_finish once ranks are combined
        } else {
            fin_init(st, t[0]);
        }
    });
}

// fixed-size grid for the row reductions (a function of E and n only, so
// the reduction tree -- and every result -- is reproducible)
// fixed grids for the reductions (functions of E and n only, so the
// reduction trees -- and every result -- are reproducible)
template <int N>
static unsigned red_grid(int64_t E)
{
    return flat_grid<N>(E, kReduceBlocks);
}

template <int N>
static unsigned row_grid(int64_t E)
{
    const int64_t blocks = (E * N * N + kRowThreads - 1) / kRowThreads;
    return (unsigned)(blocks < kReduceBlocks ? (blocks > 0 ? blocks : 1) : kReduceBlocks);
}

// update2 grid: ONE full wave of the row kernel -- 768 threads per SM
// (6 blocks of 128 threads, or 3 of 256) x 148 SMs -- each thread walking its
// rows grid-stride (tools/upd_minb2.sh: one wave beat 1.3-2 waves by 10-25%).
// 3 x 256 threads measured ~1% faster per CG iteration than 6 x 128 (tools/
// row_threads.sh, profiles/r01_cg_row_threads.txt); in round 1 its reduction
// tree sent the reference's own manufactured-solution property (verify.py:
// 457-476: 1331 iterations at tol 0, deep into FP64 underflow) into a
// <p, A p> = 0 breakdown, so 128 stayed.  With <p, A p> accumulated at an
// exact power-of-two scale (fin_pap) both trees pass (tests/
// test_gpu_parity.py pins both), so 256 is the default; SEM_CG_ROW_THREADS
// = 128 (read per solve) selects the other.  The grid is a function of E and
// n only, never of the device, so the tree is fixed.
constexpr int kUpdBlocks = SEM_UPD_MINB * 148;
static_assert(kUpdBlocks <= kReduceBlocksMax, "update grid exceeds the partial slots");

template <int N, int RT = kRowThreads>
static unsigned upd_grid(int64_t E)
{
    static const int cap = getenv("SEM_CG_UPD_BLOCKS") ? atoi(getenv("SEM_CG_UPD_BLOCKS")) : 0;
    const int64_t rows = E * N * N;
    constexpr int64_t kBlocks = (int64_t)kUpdBlocks * kRowThreads / RT;
    int64_t blocks = std::min<int64_t>(kBlocks, (rows + RT - 1) / RT);
    if (cap > 0 && cap <= kReduceBlocksMax) blocks = std::min<int64_t>(rows, cap);
    return (unsigned)(blocks > 0 ? blocks : 1);
}

// threads per update block (SEM_CG_ROW_THREADS: 256 default, or 128)
static int upd_row_threads()
{
    const char* env = getenv("SEM_CG_ROW_THREADS");
    return (env && atoi(env) == kRowThreads) ? kRowThreads : 256;
}

template <int N>
static int cg_init_n(const double* f, double* x, double* r, double* p, sem_cg_state* st,
                     int64_t E, Box bx, ReduceScratch* rs, int max_it, double tol,
                     cudaStream_t s)
{
    cg_init_kernel<N, false><<<red_grid<N>(E), PairCfg<N>::THREADS, 0, s>>>(f, x, r, p, E, make_box_flat(bx), st, rs,
                                                                     max_it, tol);
    SEM_CHECK_LAUNCH("sem_cg_init launch");
    return 0;
}

// Iteration tail (cg.py:170-186 minus the x update, which the next Ax
// prologue applies): r += (-alpha) mask(dssum(w)), with the ordered row
// gather of rows.cuh (faces shared with another rank from the halo planes),
// and <r, r>_c -> history, tolerance flag, beta's numerator (DIST: this
// rank's partial -> state->local_sum, combined by sem_cg_finish).
template <int N, bool DIST, int RT = kRowThreads>
__global__ void __launch_bounds__(RT, SEM_UPD_MINB * kRowThreads / RT)
cg_update2_kernel(const double* __restrict__ w, double* __restrict__ r, int64_t E, BoxFlat bf,
                  sem_cg_state* st, double* history, ReduceScratch* rs,
                  const double* __restrict__ bot, const double* __restrict__ top,
                  bool deferred = false, const double* __restrict__ gathered = nullptr,
                  int nranks = 0, int reverse = 0)
{
    constexpr int NN = N * N, NNN = N * N * N;
    SEM_TRACE_ENTRY(st);
    griddep_wait();
    SEM_TRACE_WAITED(st);
#ifdef SEM_UPD_EARLY_TRIGGER
    griddep_launch();  // tuning probe: the next Ax may take freed SM slots during the row loop
#endif
    // both state fields in one round trip; on the default path (alpha from
    // the settle launch) the stop flag is first tested after the first row's
    // loads are issued, so the state round trip overlaps them
    const int st_stop = st->stop;
    const double st_alpha = st->alpha;
    if (st_stop && gathered != nullptr) return;
    double alpha;
    if (DIST && gathered != nullptr) {
        // multi-GPU phase-1 finish folded in: every CTA combines the ranks'
        // <p, A p> partials in rank order (the same sum cg_finish_kernel
        // forms) and derives alpha itself; block 0 records the state
        double pap_s = 0.0;
        for (int q = 0; q < nranks; ++q) pap_s += __ldg(gathered + q);
        if (blockIdx.x == 0 && threadIdx.x == 0) fin_pap(st, pap_s);
        if (pap_s <= 0.0) return;  // breakdown (block 0 set stop = 2)
        alpha = ldexp(st->rtz, 2 * pap_scale_exp(st->rtz)) / pap_s;
    } else if (gathered != nullptr) {
        // single GPU, settle folded in: every CTA sums the Ax launch's
        // per-CTA <p, A p> partials in one fixed order (so every CTA derives
        // the same alpha bit for bit) -- no settle launch between the two
        // streaming kernels; block 0 records the state
        __shared__ double pap_sh;
        const double t = settle_sum<RT>(gathered, nranks);
        if (threadIdx.x == 0) pap_sh = t;
        __syncthreads();
        const double pap_s = pap_sh;
        if (blockIdx.x == 0 && threadIdx.x == 0) fin_pap(st, pap_s);
        if (pap_s <= 0.0) return;  // breakdown (block 0 set stop = 2)
        alpha = ldexp(st->rtz, 2 * pap_scale_exp(st->rtz)) / pap_s;
    } else {
        alpha = st_alpha;
    }
    const double nalpha = -alpha;
    double acc = 0.0;
    // reverse: walk the rows from the last element down, so the first rows
    // updated are those of the elements the Ax launch processed LAST (their
    // w and r still in L2) and the last rows written are the first elements
    // the next Ax launch reads (r still in L2)
    const int64_t nrows = E * NN;
    for (int64_t q = (int64_t)blockIdx.x * RT + threadIdx.x; q < nrows;
         q += (int64_t)gridDim.x * RT) {
        const int64_t row = reverse ? nrows - 1 - q : q;
        const Box& bx = bf.b;
        const Row<N> rw = make_row<N>(row, bf);
        const int64_t base = rw.e * NNN + rw.jk * N;
        double v[N], rv[N];
        // the r row first: its loads are independent of the ordered sum, so
        // they share the first round trip with the w copies instead of
        // following the sum's additions
        load_row_rw<N>(r + base, rv);
        dssum_row<N>(w, rw, bx, DIST ? bot : nullptr, DIST ? top : nullptr, v);
        if (st_stop) break;  // uniform: queued after a stop, nothing is written
#pragma unroll
        for (int i = 0; i < N; ++i) {
            rv[i] = add_rn(rv[i], mul_rn(nalpha, mul_rn(v[i], row_mask<N>(rw, i))));
            acc += mul_rn(mul_rn(rv[i], rv[i]), row_inv_mult<N>(rw, i));
        }
        store_row<N>(r + base, rv);
    }
    if (st_stop) return;
    if (!DIST) SEM_TRACE_EXIT(st, 2);
#ifndef SEM_UPD_EARLY_TRIGGER
    griddep_launch();
#endif
    const double vals[1] = {acc};
    if (deferred) {  // single GPU: cg_settle_kernel finishes <r, r>
        reduce_publish_only<1, RT>(vals, rs);
        return;
    }
    // the last block's thread 0 loads the state fields fin_rr needs together
    // with the partials (one round trip before the state is final)
    reduce_publish_and_finish_pre<1, RT>(
        vals, rs, [&] { return DIST ? RrCtx{} : rr_ctx(st); },
        [&](const double (&t)[1], const RrCtx& c) {
            if (DIST) st->local_sum = t[0];
            else fin_rr_v(st, t[0], history, c);
        });
}

// Element-granular form of the same iteration tail ("cube" update): each
// CTA holds SLOTS elements; for each, the element's own w and the copies its
// 26 neighbours hold of its boundary nodes are gathered into an extended
// (n+2)^3 cube in shared memory by asynchronous copies (cp.async: nothing
// is staged in registers, so every copy of the element is in flight at
// once), then one thread per (j, k) row sums its points' copies from the
// cube in ascending element order -- z, then y, then x, the order of
// dssum_row, so the assembled values are bit-identical -- and updates its r
// row.  The row kernel issues a row's loads only after the previous row's
// arithmetic (latency-bound at small E); here the fill of a whole element
// is one round trip.
__device__ __forceinline__ void cp_async8(double* dst, const double* src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(double* dst, const double* src)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all()
{
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// cube index (0 .. N+1) of the copies of local index l along y or z, in
// ascending element order (axis_copies)
template <int N>
__device__ __forceinline__ void cube_copies(int ec, int l, int ecount, int& cnt, int& h0, int& h1)
{
    if (l == 0 && ec > 0) {
        cnt = 2; h0 = 0; h1 = 1;
    } else if (l == N - 1 && ec < ecount - 1) {
        cnt = 2; h0 = N; h1 = N + 1;
    } else {
        cnt = 1; h0 = l + 1; h1 = l + 1;
    }
}

template <int N>
struct CubeCfg {
    static constexpr int NN = N * N, NNN = N * N * N;
    // per slot (doubles): W own w [n^3] | R r [n^3] | ZF z-face planes of the
    // z neighbours [2][n^2] | YF y-face rows of the y neighbours [2][n][n] |
    // ED edge rows of the yz-diagonal neighbours [4][n] | XS x-neighbour
    // copies of the end nodes of every cube row [2][n+2][n+2]
    static constexpr int OW = 0, OR = NNN, OZ = 2 * NNN, OY = OZ + 2 * NN, OE = OY + 2 * NN,
                         OX = OE + 4 * N, XSP = (N + 2) * (N + 2);
    static constexpr int SLOT_D = (OX + 2 * XSP + 1) / 2 * 2;
    static constexpr int SLOTS = 1;
    static constexpr int THREADS = ((SLOTS * NN + 31) / 32) * 32;
    static constexpr size_t SMEM = sizeof(double) * (size_t)SLOTS * SLOT_D + 16;  // + mbarrier
    static constexpr int BY_SMEM = (int)((228 * 1024) / (SMEM + 1024));
    static constexpr int BY_THREADS = 1024 / THREADS;
    static constexpr int MINB = BY_SMEM < BY_THREADS ? BY_SMEM : BY_THREADS;
};

// cube row (kk, jj) of a slot: its N values
template <int N>
__device__ __forceinline__ const double* cube_row(const double* S, int kk, int jj)
{
    using C = CubeCfg<N>;
    const bool zin = kk >= 1 && kk <= N, yin = jj >= 1 && jj <= N;
    if (zin && yin) return S + C::OW + (kk - 1) * C::NN + (jj - 1) * N;
    if (zin) return S + C::OY + (jj == 0 ? 0 : C::NN) + (kk - 1) * N;
    if (yin) return S + C::OZ + (kk == 0 ? 0 : C::NN) + (jj - 1) * N;
    return S + C::OE + ((kk == 0 ? 0 : 2) + (jj == 0 ? 0 : 1)) * N;
}

// x-neighbour copies (lo, hi) of the end nodes of cube row (kk, jj) whose
// source row is (j2, k2) of element e2
template <int N>
__device__ __forceinline__ void fill_row_ends(double* S, const double* __restrict__ w, int64_t e2,
                                              int j2, int k2, int kk, int jj, bool lo, bool hi)
{
    using C = CubeCfg<N>;
    const double* src = w + e2 * C::NNN + (k2 * N + j2) * N;
    if (lo) cp_async8(S + C::OX + kk * (N + 2) + jj, src - C::NNN + (N - 1));
    if (hi) cp_async8(S + C::OX + C::XSP + kk * (N + 2) + jj, src + C::NNN);
}

template <int N>
__global__ void __launch_bounds__(CubeCfg<N>::THREADS, CubeCfg<N>::MINB)
cg_update_cube_kernel(const double* __restrict__ w, double* __restrict__ r, int64_t E,
                      BoxFlat bf, sem_cg_state* st, double* history, ReduceScratch* rs)
{
    using C = CubeCfg<N>;
    static_assert(N % 2 == 0, "bulk copies of n-double rows need even n");
    constexpr int NN = C::NN, NNN = C::NNN;
    extern __shared__ __align__(16) double smem[];
    double* S = smem;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::SLOT_D);
    const int tid = threadIdx.x;
    if (tid == 0) mbar_init(bar, 1);
    __syncthreads();
    griddep_wait();
    if (st->stop) return;
    const double nalpha = -st->alpha;
    const Box& b = bf.b;
    const int q = tid, j = q % N, k = q / N;
    const bool lane_ok = q < NN;
    const int64_t ys = b.ex, zs = (int64_t)b.ex * b.ey;
    double acc = 0.0;
    unsigned phase = 0;
    for (int64_t e = blockIdx.x; e < E; e += gridDim.x, phase ^= 1u) {
        const ElemCoord c = elem_coord_fast((uint32_t)e, bf);
        const bool zlo = c.iz > 0, zhi = c.iz < b.ez - 1, ylo = c.iy > 0, yhi = c.iy < b.ey - 1;
        const bool lo = c.ix > 0, hi = c.ix < b.ex - 1;
        // warp 0: the bulk copies (TMA engine), one per lane
        if (tid < 32) {
            unsigned bytes = 2u * NNN * 8 + (zlo + zhi) * NN * 8 + (ylo + yhi) * NN * 8 +
                             ((zlo + zhi) * (ylo + yhi)) * N * 8;
            if (tid == 0) mbar_expect_tx(bar, bytes);
            __syncwarp();
            const double* we = w + e * NNN;
            // copy index: 0 W, 1 R, 2/3 z planes, 4..4+2N-1 y rows, then 4 edges
            for (int cidx = tid; cidx < 4 + 2 * N + 4; cidx += 32) {
                if (cidx == 0) bulk_g2s(S + C::OW, we, NNN * 8, bar);
                else if (cidx == 1) bulk_g2s(S + C::OR, r + e * NNN, NNN * 8, bar);
                else if (cidx == 2) { if (zlo) bulk_g2s(S + C::OZ, we - zs * NNN + (N - 1) * NN, NN * 8, bar); }
                else if (cidx == 3) { if (zhi) bulk_g2s(S + C::OZ + NN, we + zs * NNN, NN * 8, bar); }
                else if (cidx < 4 + 2 * N) {
                    const int side = (cidx - 4) / N, kr = (cidx - 4) % N;
                    if (side == 0 ? ylo : yhi)
                        bulk_g2s(S + C::OY + side * NN + kr * N,
                                 we + (side == 0 ? -ys : ys) * NNN + kr * NN + (side == 0 ? (N - 1) * N : 0),
                                 N * 8, bar);
                } else {
                    const int d = cidx - 4 - 2 * N, zsd = d >> 1, ysd = d & 1;
                    if ((zsd == 0 ? zlo : zhi) && (ysd == 0 ? ylo : yhi))
                        bulk_g2s(S + C::OE + d * N,
                                 we + ((zsd == 0 ? -zs : zs) + (ysd == 0 ? -ys : ys)) * NNN +
                                     (zsd == 0 ? (N - 1) * NN : 0) + (ysd == 0 ? (N - 1) * N : 0),
                                 N * 8, bar);
                }
            }
        }
        // every thread: the x-neighbour copies of its row's end nodes (and
        // of the y / z / yz neighbour rows it sums)
        int dy = 0, dz = 0;
        if (lane_ok) {
            dy = (j == 0 && ylo) ? -1 : ((j == N - 1 && yhi) ? 1 : 0);
            dz = (k == 0 && zlo) ? -1 : ((k == N - 1 && zhi) ? 1 : 0);
            const int jj = dy < 0 ? 0 : N + 1, kk = dz < 0 ? 0 : N + 1;
            const int j2 = dy < 0 ? N - 1 : 0, k2 = dz < 0 ? N - 1 : 0;
            fill_row_ends<N>(S, w, e, j, k, k + 1, j + 1, lo, hi);
            if (dy != 0) fill_row_ends<N>(S, w, e + dy * ys, j2, k, k + 1, jj, lo, hi);
            if (dz != 0) fill_row_ends<N>(S, w, e + dz * zs, j, k2, kk, j + 1, lo, hi);
            if (dy != 0 && dz != 0) fill_row_ends<N>(S, w, e + dy * ys + dz * zs, j2, k2, kk, jj, lo, hi);
        }
        cp_async_wait_all();
        if (tid == 0) mbar_wait(bar, phase);  // the others wait at the barrier
        __syncthreads();
        if (lane_ok) {
            Row<N> rw;
            rw.e = e;
            rw.jk = q;
            rw.j = j;
            rw.k = k;
            rw.c = c;
            const int gz = c.iz + b.gz0;
            rw.yz_inner = axis_interior<N>(c.iy, j, b.ey) && axis_interior<N>(gz, k, b.ez_global);
            const int m = axis_mult<N>(c.iy, j, b.ey) * axis_mult<N>(gz, k, b.ez_global);
            rw.inv_myz = m == 1 ? 1.0 : (m == 2 ? 0.5 : 0.25);
            rw.x_lo_in = lo;
            rw.x_hi_in = hi;
            int cy, y0, y1, cz, z0, z1;
            cube_copies<N>(c.iy, j, b.ey, cy, y0, y1);
            cube_copies<N>(c.iz, k, b.ez, cz, z0, z1);
            double v[N];
#pragma unroll
            for (int i = 0; i < N; ++i) v[i] = 0.0;
#pragma unroll
            for (int zc = 0; zc < 2; ++zc) {
                if (zc >= cz) break;
#pragma unroll
                for (int yc = 0; yc < 2; ++yc) {
                    if (yc >= cy) break;
                    const int kk = zc ? z1 : z0, jj = yc ? y1 : y0;
                    double s[N];
                    stack_row_ld<N>(cube_row<N>(S, kk, jj), s);
                    const double xl = lo ? S[C::OX + kk * (N + 2) + jj] : 0.0;
                    const double xh = hi ? S[C::OX + C::XSP + kk * (N + 2) + jj] : 0.0;
                    v[0] = lo ? add_rn(add_rn(v[0], xl), s[0]) : add_rn(v[0], s[0]);
#pragma unroll
                    for (int i = 1; i < N - 1; ++i) v[i] = add_rn(v[i], s[i]);
                    v[N - 1] = hi ? add_rn(add_rn(v[N - 1], s[N - 1]), xh) : add_rn(v[N - 1], s[N - 1]);
                }
            }
            double rv[N];
            stack_row_ld<N>(S + C::OR + q * N, rv);
#pragma unroll
            for (int i = 0; i < N; ++i) {
                rv[i] = add_rn(rv[i], mul_rn(nalpha, mul_rn(v[i], row_mask<N>(rw, i))));
                acc += mul_rn(mul_rn(rv[i], rv[i]), row_inv_mult<N>(rw, i));
            }
            store_row<N>(r + e * NNN + q * N, rv);
        }
        __syncthreads();  // the slot is refilled for the next element
    }
    griddep_launch();
    const double vals[1] = {acc};
    reduce_publish_and_finish<1, C::THREADS>(vals, rs,
                                             [&](const double (&t)[1]) { fin_rr(st, t[0], history); });
}

// cube-update grid: one resident wave of CTAs, a function of E and n only
// (so the reduction tree is fixed)
template <int N>
static unsigned upd_cube_grid(int64_t E)
{
    using C = CubeCfg<N>;
    static const int cap = getenv("SEM_CG_EUPD_BLOCKS") ? atoi(getenv("SEM_CG_EUPD_BLOCKS")) : 0;
    const int64_t nb = E;
    int64_t blocks = std::min<int64_t>(nb, (int64_t)C::MINB * 148);
    if (cap > 0 && cap <= kReduceBlocksMax) blocks = std::min<int64_t>(nb, cap);
    return (unsigned)(blocks > 0 ? blocks : 1);
}

// update form (SEM_CG_UPD_ELEM: 1 element kernel, 0 row kernel)
static int upd_elem()
{
    static const int k = getenv("SEM_CG_UPD_ELEM") ? atoi(getenv("SEM_CG_UPD_ELEM")) : 0;
    return k;
}

template <int N, bool DIST>
static void launch_update(const double* w, double* r, int64_t E, const Box& bx, sem_cg_state* st,
                          double* history, ReduceScratch* rs, const double* bot,
                          const double* top, cudaStream_t s, const double* gathered = nullptr,
                          int nranks = 0)
{
    cg_update2_kernel<N, DIST><<<upd_grid<N>(E), kRowThreads, 0, s>>>(
        w, r, E, make_box_flat(bx), st, history, rs, bot, top, false, gathered, nranks);
}

// Finish a deferred reduction of the single-GPU iteration: the fixed-order
// sum of the launch's block partials, then the phase bookkeeping
// (PH = kPhasePap: alpha / breakdown; PH = 2: rnorm history, beta's numerator).
constexpr int kSettleThreads = 1024;
// PH = kPhaseLocal (z-slab rank): add the sum to state->local_sum, or reset
// it first (accumulate == 0).
constexpr int kPhaseLocal = 3;
template <int PH>
__global__ void __launch_bounds__(kSettleThreads)
cg_settle_kernel(const double* __restrict__ partials, int count, sem_cg_state* st,
                 double* history, int accumulate = 0)
{
    SEM_TRACE_ENTRY(st);
    griddep_wait();
    SEM_TRACE_WAITED(st);
    griddep_launch();
    // the stop flag and the partials in one round trip (after a stop the
    // partials are stale and unused)
    const int stop = st->stop, st_it = st->it;
    const double st_rtz = st->rtz;
    const double tot = settle_sum<kSettleThreads>(partials, count);
    if (stop) return;
    SEM_TRACE_EXIT(st, 1);
    if (threadIdx.x != 0) return;
    if (PH == kPhaseLocal) st->local_sum = (accumulate ? st->local_sum : 0.0) + tot;
    else if (PH == kPhasePap) fin_pap_v(st, tot, st_rtz, st_it);
    else fin_phase(st, PH, tot, history);
}

// alternate the element walk direction every iteration (SEM_CG_ALT: 1
// default): even iterations run the Ax launch forward and the update
// backward, odd ones the Ax backward (it starts on the metric blocks and
// vectors the previous Ax ended on, which the update's ~100 MB left partly
// in L2) and the update forward.  tools/cg_ab.py, 8 idle-gapped solves per
// setting on one box (profiles/r02_cg_graph_pdl.txt): E = 4096 median
// 96.9 -> 94.2 us; E = 32768 unchanged.
static int cg_alt()
{
    static const int k = getenv("SEM_CG_ALT") ? atoi(getenv("SEM_CG_ALT")) : 1;
    return k;
}

// update row order (SEM_CG_UPD_REV: 1 (default) = last element first, 0 =
// first element first).  The Ax launch walks the elements forward, so the
// reversed update starts on the elements whose w and r are still in L2 and
// finishes on the ones the next Ax reads first (tools/cg_ab.py with idle
// gaps, profiles/r02_cg_graph_pdl.txt: E = 4096 94.3-96.1 -> 93.4-93.8 us,
// E = 32768 unchanged)
static int upd_rev()
{
    static const int k = getenv("SEM_CG_UPD_REV") ? atoi(getenv("SEM_CG_UPD_REV")) : 1;
    return k;
}

// <p, A p> settle: 1 (default) a one-block settle launch after the Ax
// launch, 0 folded into every update CTA (SEM_CG_SETTLE)
static int settle_launch()
{
    static const int k = getenv("SEM_CG_SETTLE") ? atoi(getenv("SEM_CG_SETTLE")) : 1;
    return k;
}

// tuning hook SEM_CG_FIN (0: fused reductions, 1: both deferred, 2: the Ax
// reduction deferred only)
static int fin_mode()
{
    static const int k = getenv("SEM_CG_FIN") ? atoi(getenv("SEM_CG_FIN")) : 2;
    return k;
}
// programmatic dependent launch of the iteration chain (SEM_CG_PDL: 0 off,
// 1 (default) every launch, 2 the settle and update launches only).  With
// several iterations captured per CUDA graph (cg.py GRAPH_ITERATIONS) the
// next iteration's Ax CTAs become resident as the update drains and issue
// their metric bulk copy before griddep_wait; a timeline trace (-DSEM_TRACE,
// tools/cg_trace.py) showed ~5-7 us between the update's end and the next
// Ax's first CTA when every iteration was its own graph launch.  Measured
// with idle gaps (tools/cg_ab.py, profiles/r02_cg_graph_pdl.txt): E = 4096
// 98.0-99.2 us (1 iteration per graph) -> 93.8-94.9 us (10 per graph, PDL
// on every launch); E = 32768 619-622 -> 605-614 us.
static int cg_pdl()
{
    static const int k = getenv("SEM_CG_PDL") ? atoi(getenv("SEM_CG_PDL")) : 1;
    return k;
}

// The owed x += alpha p of the last iteration (every exit except breakdown).
__global__ void __launch_bounds__(kVecThreads)
cg_finalize_kernel(double* __restrict__ x, const double* __restrict__ p, int64_t m,
                   const sem_cg_state* st)
{
    if (!st->x_pending || st->stop == 2) return;
    const double alpha = st->alpha;
    const int64_t stride = (int64_t)gridDim.x * kVecThreads;
    for (int64_t q = (int64_t)blockIdx.x * kVecThreads + threadIdx.x; q < m; q += stride)
        x[q] = add_rn(x[q], mul_rn(alpha, __ldg(p + q)));
}

__global__ void cg_clear_pending_kernel(sem_cg_state* st) { st->x_pending = 0; }

// launch of the cube update (even n only: n-double rows are bulk-copied)
template <int N>
static int launch_cube_update(const double* w, double* r, int64_t E, const Box& bx,
                              sem_cg_state* st, double* history, ReduceScratch* rs, cudaStream_t s,
                              bool pdl)
{
    if constexpr (N % 2 != 0) {
        set_error("cube update: odd n");
        return SEM_E_INVALID;
    } else {
        using UC = CubeCfg<N>;
        auto kern = cg_update_cube_kernel<N>;
        static std::atomic<uint64_t> configured{0};
        int dev = 0;
        if (cudaError_t e = cudaGetDevice(&dev)) return fail_cuda(e, "cube update: cudaGetDevice");
        const uint64_t bit = 1ull << (dev & 63);
        if (!(configured.load(std::memory_order_acquire) & bit)) {
            if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)UC::SMEM))
                return fail_cuda(e, "cube update: attribute");
            configured.fetch_or(bit, std::memory_order_release);
        }
        cudaError_t e = launch_k(kern, dim3(upd_cube_grid<N>(E)), dim3(UC::THREADS), UC::SMEM, s, pdl,
                                 w, r, E, make_box_flat(bx), st, history, rs);
        return e == cudaSuccess ? 0 : fail_cuda(e, "cg update (cube) kernel");
    }
}

template <int N>
static int cg_run_n(const double* g, const double* dx, double* x, double* r, double* p,
                    double* w, double* w2, sem_cg_state* st, double* history, int iters,
                    int64_t E, Box bx, ReduceScratch* rs, cudaStream_t s,
                    cudaEvent_t* marks = nullptr, int first_it = 1)
{
    // marks (optional, 3*iters+1 events): recorded before each iteration's
    // Ax, assemble and update launches and after the last one
    auto mark = [&](int q) { return marks ? cudaEventRecord(marks[q], s) : cudaSuccess; };
    // w2 (the second half of the w scratch) holds the Ax kernel's per-CTA
    // <p, A p> partials (one per element at most)
    const bool defer = fin_mode() == 1, defer_ax = fin_mode() >= 1;
    // PDL chain (no phase events in between): each kernel may launch while
    // its predecessor drains and waits on it in-kernel (griddep_wait)
    // (SEM_CG_PDL=1: every launch; 2: the settle and update launches only)
    const bool pdl = cg_pdl() != 0 && marks == nullptr;
    const bool rt256 = upd_row_threads() == 256;
    unsigned ax_grid = 0;
    const CgpArgs a{p, r, st, history, x, w2, &rs->counter, 0, defer_ax ? 1 : 0, &ax_grid,
                    (pdl && cg_pdl() == 1) ? 1 : 0};
    auto chk = [](cudaError_t e, const char* what) { return e == cudaSuccess ? 0 : fail_cuda(e, what); };
    for (int it = 0; it < iters; ++it) {
        if (cudaError_t e = mark(3 * it)) return fail_cuda(e, "sem_cg_run: event");
        // SEM_CG_ALT: odd iterations walk the elements backward (the Ax
        // launch starts on the metric the previous Ax left in L2) and their
        // update forward
        // (parity of the GLOBAL 1-based iteration number, so any split of a
        // solve into sem_cg_run_at calls -- eager, graph-replayed, one per
        // callback -- walks the same way and rounds identically)
        const bool back = ((first_it + it) % 2) == 0;
        CgpArgs ai = a;
        ai.reverse = (cg_alt() && back) ? 1 : 0;
        const int urev = cg_alt() ? (back ? 0 : 1) : upd_rev();
        if (int rc = ax_cg_dispatch(g, dx, w, E, N, ai, 2, s)) return rc;
        const bool fold = defer_ax && !defer && !settle_launch() && !upd_elem();
        if (defer_ax && !fold) {
            if (int rc = chk(launch_k(cg_settle_kernel<kPhasePap>, dim3(1), dim3(kSettleThreads), 0, s,
                                      pdl, (const double*)w2, (int)ax_grid, st, history, 0),
                             "cg settle (pap)"))
                return rc;
        }
        if (cudaError_t e = mark(3 * it + 1)) return fail_cuda(e, "sem_cg_run: event");
        if (N % 2 == 0 && upd_elem() && !defer) {
            if (int rc = launch_cube_update<N>(w, r, E, bx, st, history, rs, s, pdl)) return rc;
        } else if (defer) {
            const unsigned ug = rt256 ? upd_grid<N, 256>(E) : upd_grid<N>(E);
            if (int rc = chk(rt256 ? launch_k(cg_update2_kernel<N, false, 256>, dim3(ug), dim3(256), 0, s,
                                              pdl, (const double*)w, r, E, make_box_flat(bx), st,
                                              history, rs, (const double*)nullptr,
                                              (const double*)nullptr, true, (const double*)nullptr, 0,
                                              urev)
                                   : launch_k(cg_update2_kernel<N, false>, dim3(ug), dim3(kRowThreads), 0,
                                              s, pdl, (const double*)w, r, E, make_box_flat(bx), st,
                                              history, rs, (const double*)nullptr,
                                              (const double*)nullptr, true, (const double*)nullptr, 0,
                                              urev),
                             "cg update kernel"))
                return rc;
            if (int rc = chk(launch_k(cg_settle_kernel<2>, dim3(1), dim3(kSettleThreads), 0, s, pdl,
                                      (const double*)rs->partials[0], (int)ug, st, history, 0),
                             "cg settle (rr)"))
                return rc;
        } else {
            const double* gath = fold ? (const double*)w2 : (const double*)nullptr;
            const int ng = fold ? (int)ax_grid : 0;
            if (int rc = chk(rt256 ? launch_k(cg_update2_kernel<N, false, 256>, dim3(upd_grid<N, 256>(E)),
                                              dim3(256), 0, s, pdl, (const double*)w, r, E,
                                              make_box_flat(bx), st, history, rs,
                                              (const double*)nullptr, (const double*)nullptr, false, gath, ng,
                                              urev)
                                   : launch_k(cg_update2_kernel<N, false>, dim3(upd_grid<N>(E)),
                                              dim3(kRowThreads), 0, s, pdl, (const double*)w, r, E,
                                              make_box_flat(bx), st, history, rs,
                                              (const double*)nullptr, (const double*)nullptr, false, gath, ng,
                                              urev),
                             "cg update kernel"))
                return rc;
        }
        SEM_CHECK_LAUNCH("cg update kernel");
        if (cudaError_t e = mark(3 * it + 2)) return fail_cuda(e, "sem_cg_run: event");
    }
    if (cudaError_t e = mark(3 * iters)) return fail_cuda(e, "sem_cg_run: event");
    return 0;
}

}  // namespace sem

using namespace sem;

extern "C" int64_t sem_reduce_scratch_bytes(void) { return (int64_t)sizeof(ReduceScratch); }

extern "C" int sem_add2s1(double* p, const double* z, double beta, int64_t m, sem_stream_t stream)
{
    if (!p || !z || m < 0) { set_error("sem_add2s1: bad arguments"); return SEM_E_INVALID; }
    if (m == 0) return 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    add2s1_kernel<<<vec_grid(m), kVecThreads, 0, s>>>(p, z, beta, m);
    SEM_CHECK_LAUNCH("sem_add2s1 launch");
    return 0;
}

extern "C" int sem_add2s2(double* x, const double* y, double alpha, int64_t m, sem_stream_t stream)
{
    if (!x || !y || m < 0) { set_error("sem_add2s2: bad arguments"); return SEM_E_INVALID; }
    if (m == 0) return 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    add2s2_kernel<<<vec_grid(m), kVecThreads, 0, s>>>(x, y, alpha, m);
    SEM_CHECK_LAUNCH("sem_add2s2 launch");
    return 0;
}

extern "C" int sem_glsc3(const double* a, const double* b, const double* wt, int64_t m,
                         double* out_dev, void* scratch, sem_stream_t stream)
{
    if (!a || !b || !wt || !out_dev || !scratch || m < 0) {
        set_error("sem_glsc3: bad arguments");
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    const unsigned grid = (unsigned)std::min<int64_t>(
        kReduceBlocks, std::max<int64_t>(1, (m + kReduceThreads - 1) / kReduceThreads));
    glsc3_kernel<<<grid, kReduceThreads, 0, s>>>(a, b, wt, m, out_dev,
                                                 static_cast<ReduceScratch*>(scratch));
    SEM_CHECK_LAUNCH("sem_glsc3 launch");
    return 0;
}

extern "C" int sem_glsc3_box(const double* a, const double* b, int32_t ex, int32_t ey,
                             int32_t ez, int32_t n, double* out_dev, void* scratch,
                             sem_stream_t stream)
{
    if (int rc = check_box(ex, ey, ez, n, "sem_glsc3_box")) return rc;
    if (!a || !b || !out_dev || !scratch) { set_error("sem_glsc3_box: null pointer"); return SEM_E_INVALID; }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    const Box bx{ex, ey, ez, 0, ez};
    const int64_t E = (int64_t)ex * ey * ez;
    auto* rs = static_cast<ReduceScratch*>(scratch);
    SEM_SWITCH_N(n, {
        glsc3_box_kernel<NV><<<red_grid<NV>(E), PairCfg<NV>::THREADS, 0, s>>>(a, b, E, make_box_flat(bx), out_dev, rs);
        SEM_CHECK_LAUNCH("sem_glsc3_box launch");
        return 0;
    });
}

extern "C" int sem_cg_init(const double* f, double* x, double* r, double* p, sem_cg_state* state,
                           double* history, int32_t max_iterations, double tolerance,
                           int32_t ex, int32_t ey, int32_t ez, int32_t n, void* scratch,
                           sem_stream_t stream)
{
    if (int rc = check_box(ex, ey, ez, n, "sem_cg_init")) return rc;
    if (!f || !x || !r || !p || !state || !history || !scratch || max_iterations < 1 ||
        tolerance < 0.0) {
        set_error("sem_cg_init: bad arguments");
        return SEM_E_INVALID;
    }
    if (int rc = check_fields_aligned("sem_cg_init", n, nullptr, {f, x, r, p})) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    const Box bx{ex, ey, ez, 0, ez};
    const int64_t E = (int64_t)ex * ey * ez;
    auto* rs = static_cast<ReduceScratch*>(scratch);
    SEM_SWITCH_N(n, return cg_init_n<NV>(f, x, r, p, state, E, bx, rs, max_iterations,
                                         tolerance, s));
}

extern "C" int sem_cg_run_at(const double* g, const double* dx, const double* dxt, double* x,
                             double* r, double* p, double* w, sem_cg_state* state,
                             double* history, int32_t iterations, int32_t first_iteration,
                             int32_t ex, int32_t ey, int32_t ez, int32_t n, void* scratch,
                             sem_stream_t stream)
{
    (void)dxt;
    if (int rc = check_box(ex, ey, ez, n, "sem_cg_run")) return rc;
    if (first_iteration < 1) {
        set_error("sem_cg_run_at: first_iteration is 1-based");
        return SEM_E_INVALID;
    }
    if (!g || !dx || !x || !r || !p || !w || !state || !history || !scratch || iterations < 0) {
        set_error("sem_cg_run: bad arguments");
        return SEM_E_INVALID;
    }
    if (int rc = check_fields_aligned("sem_cg_run", n, g, {x, r, p, w})) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    const Box bx{ex, ey, ez, 0, ez};
    const int64_t E = (int64_t)ex * ey * ez;
    const int64_t m = E * n * n * n;
    auto* rs = static_cast<ReduceScratch*>(scratch);
    // w holds two E*n^3 vectors: the local Ax output, then the per-CTA
    // partial slots -- started on an even double so the settle's 16-byte
    // loads are aligned when E*n^3 is odd (odd E and odd n; the slots need
    // at most E < E*n^3 - 1 doubles, so the shift stays inside w)
    double* w_local = w;
    double* w_asm = w + m + (m & 1);
    SEM_SWITCH_N(n, return cg_run_n<NV>(g, dx, x, r, p, w_local, w_asm, state, history,
                                        iterations, E, bx, rs, s, nullptr, first_iteration));
}

extern "C" int sem_cg_run(const double* g, const double* dx, const double* dxt, double* x,
                          double* r, double* p, double* w, sem_cg_state* state, double* history,
                          int32_t iterations, int32_t ex, int32_t ey, int32_t ez, int32_t n,
                          void* scratch, sem_stream_t stream)
{
    return sem_cg_run_at(g, dx, dxt, x, r, p, w, state, history, iterations, 1, ex, ey, ez, n,
                         scratch, stream);
}

extern "C" int sem_cg_finalize(double* x, const double* p, sem_cg_state* state,
                               int64_t num_points, sem_stream_t stream)
{
    if (!x || !p || !state || num_points < 0) {
        set_error("sem_cg_finalize: bad arguments");
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    cg_finalize_kernel<<<vec_grid(num_points > 0 ? num_points : 1), kVecThreads, 0, s>>>(
        x, p, num_points, state);
    SEM_CHECK_LAUNCH("cg_finalize_kernel");
    cg_clear_pending_kernel<<<1, 1, 0, s>>>(state);
    SEM_CHECK_LAUNCH("cg_clear_pending_kernel");
    return 0;
}

// Instrumented form of sem_cg_run: the same launches, eagerly, with CUDA
// events between them; synchronises and adds each phase's device time (ms)
// to phase_ms[0] (Ax with the fused iteration head and <p, A p>), [1] (r
// update with the fused dssum + mask, <r,r>), [2] (unused, 0).  Measurement
// only (harness.py).
extern "C" int sem_cg_run_phases(const double* g, const double* dx, const double* dxt, double* x,
                                 double* r, double* p, double* w, sem_cg_state* state,
                                 double* history, int32_t iterations, int32_t ex, int32_t ey,
                                 int32_t ez, int32_t n, void* scratch, double* phase_ms,
                                 sem_stream_t stream)
{
    (void)dxt;
    if (int rc = check_box(ex, ey, ez, n, "sem_cg_run_phases")) return rc;
    if (!g || !dx || !x || !r || !p || !w || !state || !history || !scratch || !phase_ms ||
        iterations < 0 || iterations > 100000) {
        set_error("sem_cg_run_phases: bad arguments");
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    const Box bx{ex, ey, ez, 0, ez};
    const int64_t E = (int64_t)ex * ey * ez;
    const int64_t m = E * n * n * n;
    auto* rs = static_cast<ReduceScratch*>(scratch);
    const int nev = 3 * iterations + 1;
    cudaEvent_t* marks = new cudaEvent_t[nev];
    int made = 0, rc = 0;
    cudaError_t err = cudaSuccess;
    for (; made < nev && err == cudaSuccess; ++made) err = cudaEventCreate(&marks[made]);
    if (err != cudaSuccess) {
        --made;
        rc = fail_cuda(err, "sem_cg_run_phases: events");
    }
    if (rc == 0) {
        SEM_SWITCH_N(n, rc = cg_run_n<NV>(g, dx, x, r, p, w, w + m + (m & 1), state, history,
                                          iterations, E, bx, rs, s, marks); break);
    }
    if (rc == 0 && (err = cudaEventSynchronize(marks[nev - 1])) != cudaSuccess)
        rc = fail_cuda(err, "sem_cg_run_phases: sync");
    for (int q = 0; rc == 0 && q < nev - 1; ++q) {
        float ms = 0.f;
        if ((err = cudaEventElapsedTime(&ms, marks[q], marks[q + 1])) != cudaSuccess)
            rc = fail_cuda(err, "sem_cg_run_phases: elapsed");
        phase_ms[q % 3] += ms;
    }
    for (int q = 0; q < made; ++q) cudaEventDestroy(marks[q]);
    delete[] marks;
    return rc;
}

// ------------------------------------------------- multi-GPU (z-slab) CG --
// The same kernels with DIST=true: each reduction leaves this rank's partial
// in state->local_sum; the host gathers the partials of all ranks (NCCL
// all_gather, dist.py) and sem_cg_finish combines them in rank order and
// runs the phase's scalar bookkeeping -- identically on every rank.

namespace sem {

__global__ void cg_finish_kernel(sem_cg_state* st, const double* __restrict__ gathered,
                                 int nranks, int phase, double* history)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (phase != kPhaseInit && st->stop) return;
    double total = 0.0;
    for (int r = 0; r < nranks; ++r) total += gathered[r];
    fin_phase(st, phase, total, history);
}

static Box slab_box(int ex, int ey, int ez, int gz0, int ezg) { return Box{ex, ey, ez, gz0, ezg}; }

static int check_slab(int ex, int ey, int ez, int n, int gz0, int ezg, const char* who)
{
    if (int rc = check_box(ex, ey, ez, n, who)) return rc;
    if (gz0 < 0 || ezg < gz0 + ez) {
        set_error("%s: slab [%d, %d) outside the global %d element layers", who, gz0, gz0 + ez,
                  ezg);
        return SEM_E_INVALID;
    }
    return 0;
}

}  // namespace sem

extern "C" int sem_cg_init_slab(const double* f, double* x, double* r, double* p,
                                sem_cg_state* state, double* history, int32_t max_iterations,
                                double tolerance, int32_t ex, int32_t ey, int32_t ez, int32_t n,
                                int32_t gz0, int32_t ez_global, void* scratch,
                                sem_stream_t stream)
{
    if (int rc = check_slab(ex, ey, ez, n, gz0, ez_global, "sem_cg_init_slab")) return rc;
    if (!f || !x || !r || !p || !state || !history || !scratch || max_iterations < 1 ||
        tolerance < 0.0) {
        set_error("sem_cg_init_slab: bad arguments");
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    const Box bx = slab_box(ex, ey, ez, gz0, ez_global);
    const int64_t E = (int64_t)ex * ey * ez;
    auto* rs = static_cast<ReduceScratch*>(scratch);
    SEM_SWITCH_N(n, {
        cg_init_kernel<NV, true><<<red_grid<NV>(E), PairCfg<NV>::THREADS, 0, s>>>(
            f, x, r, p, E, make_box_flat(bx), state, rs, max_iterations, tolerance);
        SEM_CHECK_LAUNCH("sem_cg_init_slab launch");
        return 0;
    });
}

extern "C" int sem_cg_ax_slab(double* p, const double* r, double* x, const double* g,
                              const double* dx, const double* dxt, double* w,
                              int64_t num_elements, int32_t n, sem_cg_state* state,
                              double* history, double* partials, void* scratch,
                              int32_t accumulate, sem_stream_t stream)
{
    if (!p || !r || !x || !g || !dx || !dxt || !w || !state || !history || !partials ||
        !scratch || num_elements < 0 || n < 2 || n > 16) {
        set_error("sem_cg_ax_slab: bad arguments");
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    auto* rs = static_cast<ReduceScratch*>(scratch);
    // deferred <p, A p> partial: the CTAs only publish, one settle block sums
    unsigned grid = 0;
    const CgpArgs a{p, r, state, history, x, partials, &rs->counter, accumulate > 0 ? 1 : 0, 1,
                    &grid, 0};
    if (num_elements == 0) return 0;
    if (int rc = ax_cg_dispatch(g, dx, w, num_elements, n, a, 3, s)) return rc;
    if (accumulate < 0) {
        // the caller settles later (sem_cg_settle_slab) over one slot per
        // element: slots past this launch's grid (several elements per CTA)
        // are zeroed so the later sum sees exactly this range's partials
        if ((int64_t)grid < num_elements) {
            cudaError_t e = cudaMemsetAsync(partials + grid, 0,
                                            sizeof(double) * (size_t)(num_elements - grid), s);
            if (e != cudaSuccess) return fail_cuda(e, "sem_cg_ax_slab: pad partials");
        }
        return 0;
    }
    cg_settle_kernel<kPhaseLocal><<<1, kSettleThreads, 0, s>>>(partials, (int)grid, state, history,
                                                               accumulate ? 1 : 0);
    SEM_CHECK_LAUNCH("sem_cg_ax_slab settle");
    return 0;
}

extern "C" int sem_cg_settle_slab(const double* partials, int64_t count, sem_cg_state* state,
                                  int32_t accumulate, sem_stream_t stream)
{
    if (!partials || !state || count < 0 || count > 0x7fffffffLL) {
        set_error("sem_cg_settle_slab: bad arguments");
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    cg_settle_kernel<kPhaseLocal><<<1, kSettleThreads, 0, s>>>(partials, (int)count, state, nullptr,
                                                               accumulate ? 1 : 0);
    SEM_CHECK_LAUNCH("sem_cg_settle_slab");
    return 0;
}

extern "C" int sem_cg_update_slab(const double* w, double* r, const double* bottom_totals,
                                  const double* top_totals, sem_cg_state* state, int32_t ex,
                                  int32_t ey, int32_t ez, int32_t n, int32_t gz0,
                                  int32_t ez_global, void* scratch, sem_stream_t stream)
{
    if (int rc = check_slab(ex, ey, ez, n, gz0, ez_global, "sem_cg_update_slab")) return rc;
    if (!w || !r || !state || !scratch || w == r) {
        set_error("sem_cg_update_slab: bad arguments");
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    const Box bx = slab_box(ex, ey, ez, gz0, ez_global);
    const int64_t E = (int64_t)ex * ey * ez;
    auto* rs = static_cast<ReduceScratch*>(scratch);
    SEM_SWITCH_N(n, {
        launch_update<NV, true>(w, r, E, bx, state, nullptr, rs, bottom_totals, top_totals, s);
        SEM_CHECK_LAUNCH("sem_cg_update_slab launch");
        return 0;
    });
}

extern "C" int sem_cg_update_slab_alpha(const double* w, double* r, const double* bottom_totals,
                                        const double* top_totals, sem_cg_state* state,
                                        const double* gathered_pap, int32_t nranks, int32_t ex,
                                        int32_t ey, int32_t ez, int32_t n, int32_t gz0,
                                        int32_t ez_global, void* scratch, sem_stream_t stream)
{
    if (int rc = check_slab(ex, ey, ez, n, gz0, ez_global, "sem_cg_update_slab_alpha")) return rc;
    if (!w || !r || !state || !scratch || w == r || !gathered_pap || nranks < 1) {
        set_error("sem_cg_update_slab_alpha: bad arguments");
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    const Box bx = slab_box(ex, ey, ez, gz0, ez_global);
    const int64_t E = (int64_t)ex * ey * ez;
    auto* rs = static_cast<ReduceScratch*>(scratch);
    SEM_SWITCH_N(n, {
        launch_update<NV, true>(w, r, E, bx, state, nullptr, rs, bottom_totals, top_totals, s,
                                gathered_pap, nranks);
        SEM_CHECK_LAUNCH("sem_cg_update_slab_alpha launch");
        return 0;
    });
}

extern "C" int sem_cg_finish(sem_cg_state* state, const double* gathered, int32_t nranks,
                             int32_t phase, double* history, sem_stream_t stream)
{
    if (!state || !gathered || nranks < 1 || phase < 0 || phase > 2 || !history) {
        set_error("sem_cg_finish: bad arguments");
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    cg_finish_kernel<<<1, 32, 0, s>>>(state, gathered, nranks, phase, history);
    SEM_CHECK_LAUNCH("sem_cg_finish launch");
    return 0;
}

extern "C" int sem_glsc3_slab(const double* a, const double* b, int32_t ex, int32_t ey,
                              int32_t ez, int32_t n, int32_t gz0, int32_t ez_global,
                              double* out_dev, void* scratch, sem_stream_t stream)
{
    if (int rc = check_slab(ex, ey, ez, n, gz0, ez_global, "sem_glsc3_slab")) return rc;
    if (!a || !b || !out_dev || !scratch) {
        set_error("sem_glsc3_slab: null pointer");
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    const Box bx = slab_box(ex, ey, ez, gz0, ez_global);
    const int64_t E = (int64_t)ex * ey * ez;
    auto* rs = static_cast<ReduceScratch*>(scratch);
    SEM_SWITCH_N(n, {
        glsc3_box_kernel<NV><<<red_grid<NV>(E), PairCfg<NV>::THREADS, 0, s>>>(a, b, E, make_box_flat(bx), out_dev, rs);
        SEM_CHECK_LAUNCH("sem_glsc3_slab launch");
        return 0;
    });
}
