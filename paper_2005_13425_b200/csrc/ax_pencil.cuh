// "Pencil" Ax kernel: the layered algorithm restructured so that every
// contraction is a register-resident GEMV over a whole N-pencil whose D
// entries are compile-time constant-bank operands.
//
// Why (measured, profiles/r01_ax_layered_ncu.txt): in the per-point layered
// kernel each thread re-reads a u row / column (N values) from shared memory
// for every point it owns, and shared-memory wavefronts count REQUESTED
// bytes (a broadcast LDS.128 still costs 4 wavefronts), so the data path
// moved ~450 B/point and capped the kernel near 30% of the HBM roofline.
// Here a thread that loads an N-pencil produces N outputs from it (N^2
// FMAs), so each contraction costs one shared load + one store per point:
// ~17 shared accesses (~136 B) per point in total.
//
// Per element (one "slot" = N^2 threads), one CTA = SLOTS elements:
//   S3  k-pencil (i,j): u column from HBM (prefetched a batch ahead),
//       wt = D u_col (regs), column -> U (smem)                    | sync
//   S1  i-pencil (j,k): U row -> wr = D row -> A
//   S2  j-pencil (i,k): U col -> ws = D col -> B                    | sync
//   S4  k-pencil: per layer k, metric (g from HBM, prefetched one layer
//       ahead): ur -> A, us -> B, ut scattered into Wt = D^T ut    | sync
//   S5  i-pencil: A row -> D^T -> A ;  S6 j-pencil: B col -> D^T -> B | sync
//   S7  k-pencil: w = A + B + Wt -> HBM (coalesced)
// The three pencil families are the same threads with different index
// maps, chosen so consecutive threads touch consecutive addresses.  Layer
// strides of U/B are padded (stride == N mod 16 doubles) so the strided
// j-pencil accesses are bank-conflict free.
#pragma once
#include "sem_common.cuh"
#include "reduce.cuh"

namespace sem {

template <int N>
struct PencilCfg {
    static constexpr int NN = N * N;
    static constexpr int NNN = N * N * N;
    // layer strides in doubles
    // row stride RS (doubles): == 2 (mod 4) for even N so the i-pencil's
    // 128-bit row loads of consecutive threads hit distinct bank groups
    // (N = 4, 8, 12, 16 would otherwise put every row on the same banks);
    // odd N use scalar loads and RS = N (odd) is conflict-free (padding odd
    // rows to 128-bit accesses measured 6% slower at n = 13, 15:
    // profiles/r01_ax_row_stride.txt)
    static constexpr bool VECROW = (N % 2 == 0);
    static constexpr int RS = (N % 2 == 1 || N % 4 == 2) ? N : N + 2;
    static constexpr int LSA = N * RS;                              // row-friendly
    static constexpr int LSB = N * RS + (((N - N * RS) % 16) + 16) % 16;  // == N (mod 16)
    // U is read by 128-bit rows too: keep its layers 16-byte aligned
    static constexpr int LSU = (VECROW && LSB % 2) ? LSB + 1 : LSB;
    static constexpr int SLOT_DOUBLES = (N * (LSU + LSA + LSB) + 1) / 2 * 2;
    static constexpr int SLOTS = (N <= 4)  ? (512 / NN)
                               : (N <= 6)  ? (576 / NN)
                               : (N <= 8)  ? 8
                               : (N == 9)  ? 7
                               : (N == 10) ? 6
                               : (N <= 12) ? 4
                               : (N <= 14) ? 2
                               : 2;
    static constexpr int THREADS = ((SLOTS * NN + 31) / 32) * 32;
    static constexpr size_t SMEM = sizeof(double) * (size_t)SLOTS * SLOT_DOUBLES;
    static constexpr bool VEC = (N % 2) == 0;
};

// One stack row (N doubles at a 16-byte-aligned row start) to / from
// registers: 128-bit accesses when the row stride allows them (the pad
// double of an odd row is read and ignored / written as 0).
template <int N>
__device__ __forceinline__ void stack_row_ld(const double* src, double (&v)[N])
{
    if constexpr (PencilCfg<N>::VECROW) {
#pragma unroll
        for (int q = 0; q < (N + 1) / 2; ++q) {
            const double2 t = reinterpret_cast<const double2*>(src)[q];
            v[2 * q] = t.x;
            if (2 * q + 1 < N) v[2 * q + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int l = 0; l < N; ++l) v[l] = src[l];
    }
}
template <int N>
__device__ __forceinline__ void stack_row_st(double* dst, const double (&v)[N])
{
    if constexpr (PencilCfg<N>::VECROW) {
#pragma unroll
        for (int q = 0; q < (N + 1) / 2; ++q)
            reinterpret_cast<double2*>(dst)[q] =
                make_double2(v[2 * q], 2 * q + 1 < N ? v[2 * q + 1] : 0.0);
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) dst[i] = v[i];
    }
}

// One private copy of D per contraction stage: with a single copy the
// compiler common-subexpressions the constant loads across stages and keeps
// all N^2 values live in registers (spills); distinct copies keep each
// stage's uniform constant loads local to the stage.  6 x N^2 x 8 B fits the
// (CUDA >= 12.1) 32 KB kernel-parameter space.
constexpr int kStS3 = 0, kStS1 = 1, kStS2 = 2, kStS4 = 3, kStS5 = 4, kStS6 = 5;

template <int N>
struct DParamP {
    static constexpr int H = N / 2;
    double d[6][N * N];
    // even-odd ("fold") form of the stage matrix M (M = D for S3/S1/S2,
    // M = D^T for S4/S5/S6), valid when M is centro-antisymmetric
    // (M[n-1-i][n-1-l] = -M[i][l], true of every GLL derivative matrix):
    //   a[i][l] = (M[i][l] + M[i][n-1-l]) / 2,  b[i][l] = (M[i][l] - M[i][n-1-l]) / 2
    //   mc[i] = M[i][c], mr[l] = (M[c][l] - M[c][n-1-l]) / 2   (odd n, c = (n-1)/2)
    double a[6][H * H > 0 ? H * H : 1];
    double b[6][H * H > 0 ? H * H : 1];
    double mc[6][H > 0 ? H : 1];
    double mr[6][H > 0 ? H : 1];
};

// out = M in for one pencil.  FOLD uses the even-odd form: with e = in_l +
// in_{n-1-l}, o = in_l - in_{n-1-l}, S_i = a e (+ mc in_c), T_i = b o:
// out_i = S_i + T_i, out_{n-1-i} = T_i - S_i -- n^2/2 FMAs + 2n adds instead
// of n^2 FMAs (fewer FP64 and constant-load instructions per point).
template <int N, bool FOLD, bool TRANS>
__device__ __forceinline__ void pencil_gemv(const DParamP<N>& D, int st, const double (&in)[N],
                                            double (&out)[N])
{
    if constexpr (!FOLD) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
            double s = 0.0;
#pragma unroll
            for (int l = 0; l < N; ++l)
                s = fma(TRANS ? D.d[st][l * N + i] : D.d[st][i * N + l], in[l], s);
            out[i] = s;
        }
    } else {
        constexpr int H = N / 2;
        constexpr int c = (N - 1) / 2;
        double e[H > 0 ? H : 1], o[H > 0 ? H : 1];
#pragma unroll
        for (int l = 0; l < H; ++l) {
            e[l] = in[l] + in[N - 1 - l];
            o[l] = in[l] - in[N - 1 - l];
        }
#pragma unroll
        for (int i = 0; i < H; ++i) {
            double S = 0.0, T = 0.0;
#pragma unroll
            for (int l = 0; l < H; ++l) {
                S = fma(D.a[st][i * H + l], e[l], S);
                T = fma(D.b[st][i * H + l], o[l], T);
            }
            if constexpr (N % 2 == 1) S = fma(D.mc[st][i], in[c], S);
            out[i] = S + T;
            out[N - 1 - i] = T - S;
        }
        if constexpr (N % 2 == 1) {
            double T = 0.0;
#pragma unroll
            for (int l = 0; l < H; ++l) T = fma(D.mr[st][l], o[l], T);
            out[c] = T;
        }
    }
}

// Bulk L2 prefetch (sm_90+ cp.async.bulk.prefetch.L2): one instruction
// pulls a whole element's u or g block from HBM into L2, so the demand
// loads of a later CTA hit L2 instead of paying DRAM latency.  Sizes and
// addresses are rounded to the 16-byte granularity the instruction needs
// and clamped to the array.
__device__ __forceinline__ void prefetch_l2_bulk(const void* base, int64_t lo, int64_t hi,
                                                 int64_t limit)
{
    // 16-byte granularity on the ABSOLUTE address (a field may start at any
    // 8-byte boundary, e.g. a staged host buffer), kept inside [base, base+limit)
    const uint64_t b = reinterpret_cast<uint64_t>(base);
    uint64_t a0 = (b + (uint64_t)lo) & ~uint64_t(15);
    uint64_t a1 = (b + (uint64_t)(hi < limit ? hi : limit) + 15) & ~uint64_t(15);
    const uint64_t first = (b + 15) & ~uint64_t(15), last = (b + (uint64_t)limit) & ~uint64_t(15);
    if (a0 < first) a0 = first;
    if (a1 > last) a1 = last;
    if (a1 <= a0) return;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((unsigned)(a1 - a0))
                 : "memory");
}

// mbarrier + bulk-copy (TMA engine) helpers for the staged-metric mode
__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase)
{
    asm volatile(
        "{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        " @!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// GMODE 0: the metric of layers k+1..k+PD is held in a register ring.
// GMODE 1: the element's whole metric block (48 n^3 B, contiguous) is pulled
//          into shared memory by ONE bulk copy (TMA engine) at CTA start, so
//          every byte of g is in flight from the first cycle without costing
//          registers; S4 reads it with conflict-free LDS.  (SLOTS == 1.)
// GMODE 2: as 1, and u also arrives by bulk copies (one per k-layer, straight
//          into the padded U stack) on its own mbarrier, so S3 starts as soon
//          as u lands while g is still streaming.
// CG fusion (CGM >= 2): the top of a CG iteration (sembench/cg.py:149-160:
// exact-zero exit, beta = rtz/rtz_old, p = beta*p + r, unfused multiply-add)
// is folded into the Ax prologue: the kernel reads p_old and r, writes p_new
// back and applies the operator to it -- one pass over p fewer per iteration.
// It also folds in
//  * the PREVIOUS iteration's x += alpha p (cg.py:171), deferred so it reads
//    the p_old this prologue loads anyway (same operands, same rounding);
//  * <p, A p>_c (cg.py:163) as the LOCAL sum over element points of
//    p * (A_local p): p is continuous and masked, so
//    sum_c p . mask(dssum(w)) / mult == sum_local p . w exactly in real
//    arithmetic (rounding-level difference, element energies >= 0 so no
//    cancellation).  CGM == 2 (single GPU): the last CTA settles
//    alpha = rtz / pap.  CGM == 3 (z-slab rank): the last CTA adds this
//    launch's sum to state->local_sum (reset by the first launch of an
//    iteration), which the ranks then combine (dist.py).
struct CgpArgs {
    double* p;            // p (read old, write new)
    const double* r;
    sem_cg_state* st;
    double* history;
    double* x;            // x (read, write)
    double* partials;     // one double per CTA
    unsigned* counter;    // arrival counter (zero between launches)
    int accumulate;       // CGM == 3: add to (1) or reset (0) state->local_sum
    int deferred;         // only publish the CTA partial (no fence / arrival
                          // counter); cg_settle_kernel finishes the sum
    unsigned* grid_out;   // host side: the launch's grid size (may be null)
    int pdl;              // launched as a programmatic dependent (GMODE 4: the
                          // metric copy is issued before griddep_wait)
    int reverse = 0;      // CGM == 2: CTA b processes element E-1-b (the
                          // iteration walks the elements backward)
    // CTAs stagger_lo..stagger_hi-1 wait stagger_ns at entry (stagger_wait:
    // large-n plain Ax; CGM == 2 only under the SEM_CG_STAGGER probe)
    int stagger_ns = 0, stagger_lo = 0, stagger_hi = 0;
};

// Doubles of layer stacks per slot: U, A, B -- or U and A only when B
// aliases U (ALIAS: U is dead once S1/S2 have read it; one extra barrier).
template <int N, bool ALIAS>
constexpr int slot_doubles()
{
    using C = PencilCfg<N>;
    return ALIAS ? (N * (C::LSU + C::LSA) + 1) / 2 * 2 : C::SLOT_DOUBLES;
}

// bulk (TMA engine) store of a whole shared-memory block to global memory,
// tracked as a bulk group; wait_read returns once the source has been read
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int N, int SLOTS, int THREADS, int MINB, bool PERSIST, int PD = 1, int L2PF = 0,
          int GMODE = 0, bool FOLD = false, int CGM = 0, bool ALIAS = false, bool WBULK = false>
__global__ void __launch_bounds__(THREADS, MINB)
ax_pencil_kernel(const double* __restrict__ u, const double* __restrict__ g,
                 double* __restrict__ w, int64_t num_elements, const DParamP<N> D,
                 int64_t pf_elems, CgpArgs cgp)
{
    using C = PencilCfg<N>;
    constexpr int NN = C::NN, NNN = C::NNN, LSU = C::LSU, LSA = C::LSA, LSB = C::LSB, RS = C::RS;
    extern __shared__ __align__(16) double smem[];

    const int tid = threadIdx.x;
    const int slot = tid / NN;
    const int p = tid - slot * NN;
    const bool lane_ok = slot < SLOTS;
    const int sl = lane_ok ? slot : 0;
    static_assert(!ALIAS || (!PERSIST && CGM == 0 && GMODE < 2 && C::LSB == C::LSU),
                  "B aliases U: one batch per CTA, U not needed after S2");
    constexpr int SLOT_D = slot_doubles<N, ALIAS>();
    double* U = smem + (size_t)sl * SLOT_D;
    double* A = U + N * LSU;
    double* B = ALIAS ? U : A + N * LSA;
    // GMODE >= 1: per-slot staged metric blocks after the slot stacks, then
    // the two mbarriers (u, g) shared by the CTA
    double* Gbase = smem + ((size_t)SLOTS * SLOT_D + 1) / 2 * 2;  // 16-B aligned
    double* G = Gbase + (size_t)sl * 6 * NNN;
    uint64_t* gbar = reinterpret_cast<uint64_t*>(Gbase + (GMODE ? (size_t)SLOTS * 6 * NNN : 0));
    uint64_t* ubar = gbar + 1;
    static_assert(GMODE == 0 || !PERSIST, "staged metric: one batch per CTA");

    // index maps of the three pencil families (see header comment)
    const int kp_i = p % N, kp_j = p / N;          // k-pencil (i,j): p = j*N + i
    const int kp = kp_j * RS + kp_i;               // its offset within a stack layer
    const int ip_j = p % N, ip_k = p / N;          // i-pencil (j,k): p = k*N + j
    const int jp_i = p % N, jp_k = p / N;          // j-pencil (i,k): p = k*N + i

    const int64_t nbatches = (num_elements + SLOTS - 1) / SLOTS;
    int64_t batch = (CGM == 2 && !PERSIST && cgp.reverse) ? nbatches - 1 - (int64_t)blockIdx.x
                                                           : (int64_t)blockIdx.x;
    // PERSIST: grid-stride over batches with the next batch's u prefetched;
    // otherwise one batch per CTA (D constants are not loop-invariant, so
    // the compiler keeps them in uniform registers only around their use).

    if constexpr (CGM != 3) stagger_wait(cgp.stagger_ns, cgp.stagger_lo, cgp.stagger_hi);
    double beta = 0.0, alpha_prev = 0.0, pap_s = 1.0;
    bool xpend = false;
#ifdef SEM_TRACE
    unsigned long long _sem_t0 = sem_gtimer(), _sem_t1 = 0;
#endif
    // GMODE 4: every bulk copy of the CTA (p, r, x, g) is issued before the
    // CG scalars are read, so the state round trip overlaps the transfers;
    // x is staged unconditionally (unused on the first iteration)
    if constexpr (GMODE == 4) {
        if (tid == 0) {
            mbar_init(gbar, 1);
            mbar_init(ubar, 1);
        }
        __syncthreads();
        // the metric is never written during a solve: its copy may start
        // while the previous kernel of the iteration chain is still running
        if (tid == 0) {
            mbar_expect_tx(gbar, (unsigned)(6 * NNN * 8));
            bulk_g2s(Gbase, g + batch * (6 * NNN), 6 * NNN * 8, gbar);
        }
        griddep_wait();
#ifdef SEM_TRACE
        _sem_t1 = sem_gtimer();
#endif
        if (tid == 0) {
            const int64_t e0 = batch;
            mbar_expect_tx(ubar, (unsigned)(3 * NNN * 8));
            for (int k = 0; k < N; ++k)
                bulk_g2s(U + k * LSU, cgp.p + e0 * NNN + k * NN, NN * 8, ubar);
            bulk_g2s(A, cgp.r + e0 * NNN, NNN * 8, ubar);
            for (int k = 0; k < N; ++k)
                bulk_g2s(B + k * LSB, cgp.x + e0 * NNN + k * NN, NN * 8, ubar);
        }
    } else if constexpr (CGM != 0) {
        griddep_wait();
    } else {
        // plain Ax launched as a programmatic dependent: wait for the
        // predecessor to complete, then let our own dependent launch (its
        // CTAs take residency while this grid drains and wait the same way)
        if (cgp.pdl) {
            // before waiting: pull this CTA's u and g blocks into L2.  A bulk
            // L2 prefetch is only a hint (L2 is the coherence point; nothing
            // is read into the SM before the wait), so it is safe even if the
            // predecessor is still writing them -- and it overlaps this
            // grid's DRAM ramp with the predecessor's drain (pdl == 2)
            if (cgp.pdl >= 2 && tid == 0) {
                const int64_t e0 = batch * SLOTS;
                const int64_t e1 = (e0 + SLOTS < num_elements) ? e0 + SLOTS : num_elements;
                prefetch_l2_bulk(u, e0 * NNN * 8, e1 * NNN * 8, num_elements * NNN * 8);
                prefetch_l2_bulk(g, e0 * 6 * NNN * 8, e1 * 6 * NNN * 8, num_elements * 6 * NNN * 8);
            }
            griddep_wait();
            griddep_launch();
        }
    }
    // a CTA must not retire with bulk copies into its shared memory in flight
    auto drain = [&]() {
        if constexpr (GMODE == 4) {
            mbar_wait(ubar, 0);
            mbar_wait(gbar, 0);
        }
    };
    if constexpr (CGM != 0) {
        static_assert(!PERSIST && GMODE != 2, "CG fusion: one batch per CTA, p via registers or GMODE 4");
        sem_cg_state* st = cgp.st;
        // every state field this prologue uses is loaded up front, before
        // the first branch: one round trip instead of the stop flag's and
        // then the scalars'
        const int st_stop = st->stop, st_it = st->it, st_xp = st->x_pending;
        const double rtz = st->rtz, st_rtz_old = st->rtz_old, st_alpha = st->alpha;
        if (st_stop) {                              // uniform over the grid
            drain();
            return;
        }
        const int it = st_it + 1;
        if (rtz == 0.0) {                            // cg.py:151-158
            if (blockIdx.x == 0 && tid == 0) {
                cgp.history[it - 1] = 0.0;
                st->iterations_run = it;
                st->stop = 1;
            }
            drain();
            return;
        }
        beta = (it == 1) ? 0.0 : rtz / st_rtz_old;
        pap_s = ldexp(1.0, pap_scale_exp(rtz));  // exact power of two (fin_pap)
        xpend = st_xp != 0;
        alpha_prev = st_alpha;
        if (blockIdx.x == 0 && tid == 0) st->beta = beta;
    }
    double pap_acc = 0.0;
    double ucol[N];
    auto load_ucol = [&](int64_t b) {
        const int64_t e = b * SLOTS + slot;
        const bool ok = lane_ok && b < nbatches && e < num_elements;
        if constexpr (CGM != 0) {
            const int64_t off = (ok ? e : 0) * NNN + kp_j * N + kp_i;
            double* pp = cgp.p + off;
            const double* rp = cgp.r + off;
            if (xpend && ok) {  // x += alpha_prev * p_old (cg.py:171)
                // every load issued before any store (p, x, r may alias as far
                // as the compiler knows)
                double* xp = cgp.x + off;
                double xv[N], rv[N];
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    ucol[k] = pp[k * NN];
                    xv[k] = xp[k * NN];
                    rv[k] = __ldg(rp + k * NN);
                }
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    xv[k] = add_rn(xv[k], mul_rn(alpha_prev, ucol[k]));
                    ucol[k] = add_rn(mul_rn(beta, ucol[k]), rv[k]);
                }
#pragma unroll
                for (int k = 0; k < N; ++k) xp[k * NN] = xv[k];
            } else {
                double pv[N], rv[N];
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    pv[k] = ok ? pp[k * NN] : 0.0;
                    rv[k] = ok ? __ldg(rp + k * NN) : 0.0;
                }
#pragma unroll
                for (int k = 0; k < N; ++k) ucol[k] = ok ? add_rn(mul_rn(beta, pv[k]), rv[k]) : 0.0;
            }
            if (ok) {
#pragma unroll
                for (int k = 0; k < N; ++k) pp[k * NN] = ucol[k];
            }
        } else {
            const double* src = u + (ok ? e : 0) * NNN + kp_j * N + kp_i;
#pragma unroll
            for (int k = 0; k < N; ++k) ucol[k] = ok ? __ldg(src + k * NN) : 0.0;
        }
    };
    static_assert(GMODE < 2 || RS == N, "bulk copies into the stacks need unpadded rows");
    static_assert(GMODE != 3, "GMODE 3 (in-loop CG staging) was superseded by GMODE 4");
    static_assert(GMODE < 4 || (CGM != 0 && SLOTS == 1 && N % 2 == 0),
                  "GMODE 4: CG fusion, one element per CTA, 16-byte layer copies");
    if constexpr (GMODE < 2) load_ucol(batch);

    for (; batch < nbatches; batch += (PERSIST ? gridDim.x : nbatches)) {
        const int64_t e = batch * SLOTS + slot;
        const bool active = lane_ok && e < num_elements;
        const double* ge = g + (active ? e : 0) * (6 * NNN) + p;  // k-pencil point (i,j)
        // metric of layers 0..PD-1: issued first, in flight during S3/S1/S2
        double gq[GMODE ? 1 : PD][6];
        if constexpr (GMODE >= 1) {
            if (GMODE != 4 && tid == 0) {
                mbar_init(gbar, 1);
                if (GMODE >= 2) mbar_init(ubar, 1);
            }
            if constexpr (GMODE != 4) __syncthreads();
            if (GMODE != 4 && tid == 0) {
                const int64_t e0 = batch * SLOTS;
                const int nact = (int)((num_elements - e0) < SLOTS ? (num_elements - e0) : SLOTS);
                if constexpr (GMODE == 2) {
                    mbar_expect_tx(ubar, (unsigned)(nact * NNN * 8));
                    for (int s2 = 0; s2 < nact; ++s2)
                        for (int k = 0; k < N; ++k)
                            bulk_g2s(smem + (size_t)s2 * SLOT_D + k * LSU,
                                     u + (e0 + s2) * NNN + k * NN, NN * 8, ubar);
                }
                mbar_expect_tx(gbar, (unsigned)(nact * 6 * NNN * 8));
                for (int s2 = 0; s2 < nact; ++s2)
                    bulk_g2s(Gbase + (size_t)s2 * 6 * NNN, g + (e0 + s2) * (6 * NNN),
                             6 * NNN * 8, gbar);
            }
            if constexpr (GMODE == 4) {
                // iteration head from the staged operands (same arithmetic as
                // load_ucol): x += alpha_prev p_old, p = beta p_old + r
                mbar_wait(ubar, 0);
                if (active) {
                    const int64_t off = e * NNN + p;
#pragma unroll
                    for (int k = 0; k < N; ++k) {
                        const double po = U[k * LSU + kp];
                        if (xpend)
                            cgp.x[off + k * NN] = add_rn(B[k * LSB + kp], mul_rn(alpha_prev, po));
                        ucol[k] = add_rn(mul_rn(beta, po), A[k * LSA + kp]);
                        cgp.p[off + k * NN] = ucol[k];
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < N; ++k) ucol[k] = 0.0;
                }
            }
            if constexpr (GMODE == 2) {
                mbar_wait(ubar, 0);
#pragma unroll
                for (int k = 0; k < N; ++k) ucol[k] = active ? U[k * LSU + kp] : 0.0;
            }
        } else {
#pragma unroll
            for (int d = 0; d < PD; ++d)
#pragma unroll
                for (int m = 0; m < 6; ++m)
                    gq[d][m] = (active && d < N) ? __ldg(ge + m * NNN + d * NN) : 0.0;
        }
        // warm L2 with the element this slot will process pf_elems later
        // (L2PF 1: the one that replaces it a resident wave later; L2PF 2:
        // pf_elems = 0, its own element -- the whole block is requested at
        // once, so the register-ring loads that follow hit L2)
        // (L2PF 3: its own element's u and g, and the u of the element a
        // resident wave later -- that CTA's S3 u-column loads then hit L2
        // instead of paying DRAM latency at its start; 27 KB per element at
        // n = 15, so the wave-ahead data is ~8 MB, not the 64 MB a whole
        // wave-ahead element costs in L2)
        if (L2PF == 3 && lane_ok && p == 0 && active) {
            prefetch_l2_bulk(u, e * NNN * 8, (e + 1) * NNN * 8, num_elements * NNN * 8);
            prefetch_l2_bulk(g, e * 6 * NNN * 8, (e + 1) * 6 * NNN * 8, num_elements * 6 * NNN * 8);
            if (pf_elems > 0 && e + pf_elems < num_elements)
                prefetch_l2_bulk(u, (e + pf_elems) * NNN * 8, (e + pf_elems + 1) * NNN * 8,
                                 num_elements * NNN * 8);
        } else if (L2PF && pf_elems >= 0 && lane_ok && p == 0 &&
                   (CGM == 2 && cgp.reverse ? e - pf_elems >= 0 : e + pf_elems < num_elements)) {
            const int64_t en = (CGM == 2 && cgp.reverse) ? e - pf_elems : e + pf_elems;
            prefetch_l2_bulk(u, en * NNN * 8, (en + 1) * NNN * 8, num_elements * NNN * 8);
            if constexpr (CGM != 0) {
                prefetch_l2_bulk(cgp.r, en * NNN * 8, (en + 1) * NNN * 8, num_elements * NNN * 8);
                prefetch_l2_bulk(cgp.x, en * NNN * 8, (en + 1) * NNN * 8, num_elements * NNN * 8);
            }
            prefetch_l2_bulk(g, en * 6 * NNN * 8, (en + 1) * 6 * NNN * 8,
                             num_elements * 6 * NNN * 8);
        }

        // ---- S3: k-pencil -- stage u, wt = D u_col -------------------------
        double wt[N];
#pragma unroll
        for (int k = 0; k < N; ++k)
            if (GMODE != 2 && lane_ok) U[k * LSU + kp] = ucol[k];
        pencil_gemv<N, FOLD, false>(D, kStS3, ucol, wt);
        __syncthreads();

        // ---- S1: i-pencil (j,k): wr[i] = sum_l D[i][l] U[k][j][l] ----------
        if (lane_ok) {
            double row[N];
            stack_row_ld<N>(U + ip_k * LSU + ip_j * RS, row);
            double out[N];
            pencil_gemv<N, FOLD, false>(D, kStS1, row, out);
            stack_row_st<N>(A + ip_k * LSA + ip_j * RS, out);
        }
        // ---- S2: j-pencil (i,k): ws[j] = sum_l D[j][l] U[k][l][i] ----------
        {
            double out[N];
            if (lane_ok) {
                double col[N];
                const double* src = U + jp_k * LSU + jp_i;
#pragma unroll
                for (int l = 0; l < N; ++l) col[l] = src[l * RS];
                pencil_gemv<N, FOLD, false>(D, kStS2, col, out);
            }
            if constexpr (ALIAS) __syncthreads();  // every U read done: B overwrites it
            if (lane_ok) {
                double* dst = B + jp_k * LSB + jp_i;
#pragma unroll
                for (int j = 0; j < N; ++j) dst[j * RS] = out[j];
            }
        }
        __syncthreads();

        // ---- S4: k-pencil metric per layer; ut scattered into Wt ----------
        if constexpr (GMODE >= 1) mbar_wait(gbar, 0);
        double Wt[N], utk[N];
#pragma unroll
        for (int k = 0; k < N; ++k) Wt[k] = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            double gc[6];
            if constexpr (GMODE >= 1) {
#pragma unroll
                for (int m = 0; m < 6; ++m) gc[m] = G[m * NNN + k * NN + p];
            } else {
                // register ring: consume layer k, refill the slot with layer k+PD
#pragma unroll
                for (int m = 0; m < 6; ++m) gc[m] = gq[k % PD][m];
                if (k + PD < N) {
#pragma unroll
                    for (int m = 0; m < 6; ++m)
                        gq[k % PD][m] = active ? __ldg(ge + m * NNN + (k + PD) * NN) : 0.0;
                }
            }
            if (lane_ok) {
                const double a = A[k * LSA + kp];
                const double b = B[k * LSB + kp];
                const double t = wt[k];
                const double ur = fma(gc[2], t, fma(gc[1], b, gc[0] * a));
                const double us = fma(gc[4], t, fma(gc[3], b, gc[1] * a));
                const double ut = fma(gc[5], t, fma(gc[4], b, gc[2] * a));
                A[k * LSA + kp] = ur;
                B[k * LSB + kp] = us;
                if constexpr (FOLD) {
                    utk[k] = ut;  // folded D^T applied once all layers are known
                } else {
#pragma unroll
                    for (int kk = 0; kk < N; ++kk)
                        Wt[kk] = fma(D.d[kStS4][k * N + kk], ut, Wt[kk]);
                }
            } else if constexpr (FOLD) {
                utk[k] = 0.0;
            }
        }
        if constexpr (FOLD) pencil_gemv<N, true, true>(D, kStS4, utk, Wt);
        __syncthreads();

        // ---- S5: i-pencil: A row <- D^T A row ------------------------------
        if (lane_ok) {
            double row[N];
            double* rp = A + ip_k * LSA + ip_j * RS;
            stack_row_ld<N>(rp, row);
            double out[N];
            pencil_gemv<N, FOLD, true>(D, kStS5, row, out);
            stack_row_st<N>(rp, out);
        }
        // ---- S6: j-pencil: B col <- D^T B col ------------------------------
        if (lane_ok) {
            double col[N];
            double* cp = B + jp_k * LSB + jp_i;
#pragma unroll
            for (int l = 0; l < N; ++l) col[l] = cp[l * RS];
            double out[N];
            pencil_gemv<N, FOLD, true>(D, kStS6, col, out);
#pragma unroll
            for (int j = 0; j < N; ++j) cp[j * RS] = out[j];
        }
        // next batch's u columns: in flight across the barrier and S7
        if (PERSIST && GMODE != 2) load_ucol(batch + gridDim.x);
        __syncthreads();

        // ---- S7: k-pencil: w = A + B + Wt ----------------------------------
        if constexpr (WBULK) {
            // WBULK: w staged contiguously in the (dead) metric block, then
            // ONE bulk store of the element (large writes; for mapped host
            // buffers, large PCIe write packets)
            static_assert(GMODE == 1 && SLOTS == 1 && CGM == 0 && !PERSIST && N % 2 == 0,
                          "WBULK: staged metric block reused, one element per CTA");
            if (active) {
#pragma unroll
                for (int k = 0; k < N; ++k)
                    G[k * NN + p] = (A[k * LSA + kp] + B[k * LSB + kp]) + Wt[k];
            }
            fence_async_smem();
            __syncthreads();
            if (tid == 0) {
                bulk_s2g(w + e * NNN, G, NNN * 8);
                bulk_wait_read();
            }
        } else if (active) {
            double* we = w + e * NNN + p;
#pragma unroll
            for (int k = 0; k < N; ++k) {
                const double v = (A[k * LSA + kp] + B[k * LSB + kp]) + Wt[k];
                __stcs(we + k * NN, v);
                if constexpr (CGM != 0)  // U = p_new; scaled by pap_s^2 (fin_pap)
                    pap_acc = fma(pap_s * U[k * LSU + kp], pap_s * v, pap_acc);
            }
        }
        // (no barrier needed: the next S3 writes only U, last read before the
        //  second barrier of this iteration; A/B are next written after S3's
        //  barrier)
    }
    if constexpr (CGM != 0) {
        // <p, A p>: CTA partial -> partials[blockIdx.x]; the last CTA to
        // arrive sums them in a fixed order and settles alpha (cg.py:163-170)
        __shared__ double red_sh[THREADS / 32];
        __shared__ bool red_last;
        griddep_launch();  // late trigger: the dependent launches as this grid drains
        const double tot = block_sum<THREADS>(pap_acc, red_sh);
#ifdef SEM_TRACE
        if (CGM == 2 && tid == 0) {
            unsigned long long* _tr = reinterpret_cast<unsigned long long*>(cgp.st + 1) +
                                      (0 * 128 + (cgp.st->it & 127)) * 3;
            atomicMin(_tr, _sem_t0);
            atomicMin(_tr + 1, _sem_t1);
            atomicMax(_tr + 2, sem_gtimer());
        }
#endif
        if (cgp.deferred) {
            // the CTA retires at once: a per-CTA fence + atomic would hold
            // its shared memory for a full memory round trip
            if (tid == 0) cgp.partials[blockIdx.x] = tot;
            return;
        }
        if (tid == 0) {
            cgp.partials[blockIdx.x] = tot;
            __threadfence();
            red_last = atomicAdd(cgp.counter, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (!red_last) return;
        __threadfence();
        double v = 0.0;
#pragma unroll 8
        for (int b = tid; b < (int)gridDim.x; b += THREADS) v += __ldcg(cgp.partials + b);
        const double pap = block_sum<THREADS>(v, red_sh);
        if (tid == 0) {
            sem_cg_state* st = cgp.st;
            *cgp.counter = 0u;
            if constexpr (CGM == 3) {  // this rank's partial; combined across ranks later
                st->local_sum = (cgp.accumulate ? st->local_sum : 0.0) + pap;
                return;
            }
            st->x_pending = 0;  // every CTA applied it above
            const int k = pap_scale_exp(st->rtz);  // pap is scaled by 2^(2k)
            st->pap = ldexp(pap, -2 * k);
            if (pap <= 0.0) {   // cg.py:164-169 breakdown
                st->stop = 2;
                st->breakdown_it = st->it + 1;
            } else {
                st->alpha = ldexp(st->rtz, 2 * k) / pap;
            }
        }
    }
}

}  // namespace sem
