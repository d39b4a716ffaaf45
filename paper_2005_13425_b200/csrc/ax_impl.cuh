#pragma once
#include <string.h>
// Local Poisson operator Ax on B200 (sm_100a), FP64 -- kernel templates and
// per-n launch tables.  Instantiated per n in ax_inst.cu (one object per n
// group, compiled in parallel); dispatched from ax.cu.
//
// Algorithm: the LAYERED variant of sembench/kernels.py:267-410 (paper
// §IV-C): a 2-D layer of threads walks the k layers of an element in lock
// step; each thread keeps its u column and its w accumulator column in
// registers, the r/s contractions of a layer read the layer (and its
// phase-1 results) from shared memory, and the t contraction is a register
// GEMV whose D entries are compile-time constant-bank operands.
//
// B200-specific layout decisions:
//  * a thread owns an i-PAIR (i0, i0+1) of one (j) row, so every u / g / w
//    global access is a coalesced 128-bit vector (ld.global.nc.v2.f64) and
//    every shared-memory read of the layer is an LDS.128; odd n pads the
//    shared layer to an even row stride with a zero phantom column.
//  * D and D^T live in shared memory for the lane-varying (r, s) directions
//    and in kernel-parameter constant space for the warp-uniform (t)
//    direction -- so the t-direction costs no shared-memory traffic.
//  * several elements ("slots") per CTA, double-buffered layer arrays so a
//    layer needs two CTA barriers, and the next layer's six metric vectors
//    are prefetched into registers while the current one computes.
//
// Arithmetic differs from the reference only by FMA contraction and
// association (tolerance 1e-12 max-norm relative, sembench/verify.py:37-42).
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <atomic>

#include "sem_common.cuh"
#include "ax_pencil.cuh"
#include "ax_half.cuh"
#include "ax_split.cuh"
#include "box.cuh"

namespace sem {

template <int N>
struct DParam {
    double d[N * N];  // D[i][l] row-major (basis.diff)
};

__device__ __forceinline__ double2 ldg2(const double* p)
{
    double2 v;
    asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ double ldg1(const double* p)
{
    double v;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void stg2(double* p, double2 v)
{
    asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// Compile-time configuration per n.
template <int N>
struct AxCfg {
    static constexpr int NE = (N + 1) & ~1;        // padded row length (even)
    static constexpr int NP = NE / 2;              // i-pairs per row
    static constexpr int TPE = NP * N;             // threads per element
    static constexpr int NN = N * N;
    static constexpr int NNN = N * N * N;
    static constexpr int LAYER = NE * N;           // padded layer size (doubles)
    // elements per CTA: aim at ~256-448 threads
    static constexpr int SLOTS = (TPE >= 256) ? 1 : ((448 / TPE) < 1 ? 1 : (448 / TPE));
    static constexpr int THREADS = ((SLOTS * TPE + 31) / 32) * 32;
    static constexpr bool VEC = (N % 2) == 0;      // 16-B aligned global pairs
};

template <int N, int SLOTS>
struct AxSmem {
    static constexpr int NE = AxCfg<N>::NE;
    static constexpr int LAYER = AxCfg<N>::LAYER;
    alignas(16) double d[N * NE];    // d[i*NE + l]  = D[i][l]   (pad l>=N with 0)
    alignas(16) double dt[NE * NE];  // dt[l*NE + i] = D[i][l]   (pad i>=N with 0)
    alignas(16) double u[2][SLOTS][LAYER];
    alignas(16) double r[2][SLOTS][LAYER];
    alignas(16) double s[2][SLOTS][LAYER];
};

template <int N, int SLOTS, int THREADS>
__global__ void __launch_bounds__(THREADS)
ax_layered_kernel(const double* __restrict__ u, const double* __restrict__ g,
                  double* __restrict__ w, int64_t num_elements, const DParam<N> D)
{
    using C = AxCfg<N>;
    constexpr int NE = C::NE, NP = C::NP, TPE = C::TPE, NN = C::NN, NNN = C::NNN;
    constexpr bool VEC = C::VEC;
    __shared__ AxSmem<N, SLOTS> sm;

    const int tid = threadIdx.x;
    // D tables (padded with zeros so phantom rows/columns contribute 0)
    for (int t = tid; t < N * NE; t += THREADS) {
        const int i = t / NE, l = t % NE;
        sm.d[t] = (l < N) ? D.d[i * N + l] : 0.0;
    }
    for (int t = tid; t < NE * NE; t += THREADS) {
        const int l = t / NE, i = t % NE;
        sm.dt[t] = (i < N && l < N) ? D.d[i * N + l] : 0.0;
    }

    const int slot = tid / TPE;
    const int rem = tid - slot * TPE;
    const int j = rem / NP;
    const int i0 = 2 * (rem - j * NP);
    const int64_t e = (int64_t)blockIdx.x * SLOTS + slot;
    const bool active = (slot < SLOTS) && (e < num_elements);
    const bool second = (i0 + 1) < N;  // false only for the phantom of odd n
    const int sl = active ? slot : 0;

    const double* ue = u + (active ? e : 0) * NNN + j * N + i0;
    const double* ge = g + (active ? e : 0) * (6 * NNN) + j * N + i0;

    // u column of the pair, all layers (coalesced 128-bit loads)
    double2 uc[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        if (!active) {
            uc[k] = make_double2(0.0, 0.0);
        } else if (VEC) {
            uc[k] = ldg2(ue + k * NN);
        } else {
            uc[k].x = ldg1(ue + k * NN);
            uc[k].y = second ? ldg1(ue + k * NN + 1) : 0.0;
        }
    }
    double2 acc[N];
#pragma unroll
    for (int k = 0; k < N; ++k) acc[k] = make_double2(0.0, 0.0);

    auto load_g = [&](double2 (&gv)[6], int k) {
#pragma unroll
        for (int m = 0; m < 6; ++m) {
            const double* p = ge + m * NNN + k * NN;
            if (!active) {
                gv[m] = make_double2(0.0, 0.0);
            } else if (VEC) {
                gv[m] = ldg2(p);
            } else {
                gv[m].x = ldg1(p);
                gv[m].y = second ? ldg1(p + 1) : 0.0;
            }
        }
    };
    double2 gn[6];
    load_g(gn, 0);
    __syncthreads();

    const double2* d2 = reinterpret_cast<const double2*>(sm.d);
    const double2* dt2 = reinterpret_cast<const double2*>(sm.dt);

#pragma unroll
    for (int k = 0; k < N; ++k) {
        const int b = k & 1;
        double* su = sm.u[b][sl];
        double* sr = sm.r[b][sl];
        double* ss = sm.s[b][sl];
        if (active) *reinterpret_cast<double2*>(su + j * NE + i0) = uc[k];
        double2 gc[6];
#pragma unroll
        for (int m = 0; m < 6; ++m) gc[m] = gn[m];
        if (k + 1 < N) load_g(gn, k + 1);
        __syncthreads();

        // ---- phase 1: directional derivatives at layer k ----
        const double2* su2 = reinterpret_cast<const double2*>(su);
        double wr0 = 0.0, wr1 = 0.0, ws0 = 0.0, ws1 = 0.0, wt0 = 0.0, wt1 = 0.0;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const double2 ur = su2[(j * NE) / 2 + q];                 // U[j][2q..2q+1]
            const double2 da = dt2[((2 * q) * NE + i0) / 2];          // D[i0..i0+1][2q]
            const double2 dj = d2[(j * NE) / 2 + q];                  // D[j][2q..2q+1]
            const double2 ua = su2[((2 * q) * NE + i0) / 2];          // U[2q][i0..i0+1]
            wr0 = fma(da.x, ur.x, wr0);
            wr1 = fma(da.y, ur.x, wr1);
            ws0 = fma(dj.x, ua.x, ws0);
            ws1 = fma(dj.x, ua.y, ws1);
            if (2 * q + 1 < N) {
                const double2 db = dt2[((2 * q + 1) * NE + i0) / 2];  // D[i0..][2q+1]
                const double2 ub = su2[((2 * q + 1) * NE + i0) / 2];  // U[2q+1][i0..]
                wr0 = fma(db.x, ur.y, wr0);
                wr1 = fma(db.y, ur.y, wr1);
                ws0 = fma(dj.y, ub.x, ws0);
                ws1 = fma(dj.y, ub.y, ws1);
            }
        }
#pragma unroll
        for (int l = 0; l < N; ++l) {
            const double dkl = D.d[k * N + l];  // warp-uniform: constant bank
            wt0 = fma(dkl, uc[l].x, wt0);
            wt1 = fma(dkl, uc[l].y, wt1);
        }
        // metric: (ur,us,ut) = G (wr,ws,wt), G = (g1 g2 g3; g2 g4 g5; g3 g5 g6)
        const double r0 = fma(gc[2].x, wt0, fma(gc[1].x, ws0, gc[0].x * wr0));
        const double r1 = fma(gc[2].y, wt1, fma(gc[1].y, ws1, gc[0].y * wr1));
        const double s0 = fma(gc[4].x, wt0, fma(gc[3].x, ws0, gc[1].x * wr0));
        const double s1 = fma(gc[4].y, wt1, fma(gc[3].y, ws1, gc[1].y * wr1));
        const double t0 = fma(gc[5].x, wt0, fma(gc[4].x, ws0, gc[2].x * wr0));
        const double t1 = fma(gc[5].y, wt1, fma(gc[4].y, ws1, gc[2].y * wr1));
        if (active) {
            *reinterpret_cast<double2*>(sr + j * NE + i0) = make_double2(r0, r1);
            *reinterpret_cast<double2*>(ss + j * NE + i0) = make_double2(s0, s1);
        }
        __syncthreads();

        // ---- phase 2: transposed contractions ----
        const double2* sr2 = reinterpret_cast<const double2*>(sr);
        const double2* ss2 = reinterpret_cast<const double2*>(ss);
        double ar0 = 0.0, ar1 = 0.0, as0 = 0.0, as1 = 0.0;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const double2 rr = sr2[(j * NE) / 2 + q];                 // ur[j][2q..]
            const double2 da = d2[((2 * q) * NE + i0) / 2];           // D[2q][i0..i0+1]
            const double2 dj = dt2[(j * NE) / 2 + q];                 // D[2q..2q+1][j]
            const double2 sa = ss2[((2 * q) * NE + i0) / 2];          // us[2q][i0..]
            ar0 = fma(da.x, rr.x, ar0);
            ar1 = fma(da.y, rr.x, ar1);
            as0 = fma(dj.x, sa.x, as0);
            as1 = fma(dj.x, sa.y, as1);
            if (2 * q + 1 < N) {
                const double2 db = d2[((2 * q + 1) * NE + i0) / 2];   // D[2q+1][i0..]
                const double2 sb = ss2[((2 * q + 1) * NE + i0) / 2];
                ar0 = fma(db.x, rr.y, ar0);
                ar1 = fma(db.y, rr.y, ar1);
                as0 = fma(dj.y, sb.x, as0);
                as1 = fma(dj.y, sb.y, as1);
            }
        }
        acc[k].x += ar0 + as0;
        acc[k].y += ar1 + as1;
#pragma unroll
        for (int kk = 0; kk < N; ++kk) {
            const double dkk = D.d[k * N + kk];  // D^T[kk][k]
            acc[kk].x = fma(dkk, t0, acc[kk].x);
            acc[kk].y = fma(dkk, t1, acc[kk].y);
        }
    }

    if (active) {
        double* we = w + e * NNN + j * N + i0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            if (VEC) {
                stg2(we + k * NN, acc[k]);
            } else {
                we[k * NN] = acc[k].x;
                if (second) we[k * NN + 1] = acc[k].y;
            }
        }
    }
}

template <int N>
static int launch_ax(const double* u, const double* g, const double* dx, double* w,
                     int64_t E, cudaStream_t stream)
{
    using C = AxCfg<N>;
    DParam<N> D;
    for (int t = 0; t < N * N; ++t) D.d[t] = dx[t];
    if (E == 0) return 0;
    const int64_t blocks = (E + C::SLOTS - 1) / C::SLOTS;
    if (blocks > 0x7fffffffLL) {
        set_error("sem_ax: too many elements (%lld)", (long long)E);
        return SEM_E_INVALID;
    }
    ax_layered_kernel<N, C::SLOTS, C::THREADS>
        <<<(unsigned)blocks, C::THREADS, 0, stream>>>(u, g, w, E, D);
    SEM_CHECK_LAUNCH("sem_ax launch");
    return 0;
}

constexpr int kAxCarveout = -1;

// Kernel-parameter D tables (one copy per stage) and their even-odd forms.
// Returns whether D is centro-antisymmetric to 1e-13 relative, i.e. whether
// the folded contraction is usable (it is for every GLL basis).
template <int N>
static bool fill_dparam_compute(DParamP<N>& P, const double* dx);

// The kernel-parameter form of D for this n, recomputed only when the
// caller's D differs from the last one seen by this host thread (every call
// of a solve passes the same basis; the fold / antisymmetry check is a few
// microseconds of host time per launch otherwise).
template <int N>
static bool fill_dparam(DParamP<N>& P, const double* dx)
{
    struct Cached {
        bool valid = false, antisym = false;
        double dx[N * N];
        DParamP<N> P;
    };
    static thread_local Cached c;
    if (c.valid && memcmp(c.dx, dx, sizeof(double) * N * N) == 0) {
        P = c.P;
        return c.antisym;
    }
    c.antisym = fill_dparam_compute<N>(c.P, dx);
    memcpy(c.dx, dx, sizeof(double) * N * N);
    c.valid = true;
    P = c.P;
    return c.antisym;
}

template <int N>
static bool fill_dparam_compute(DParamP<N>& P, const double* dx)
{
    constexpr int H = N / 2, c = (N - 1) / 2;
    double dev = 0.0, scale = 0.0;
    for (int i = 0; i < N; ++i)
        for (int l = 0; l < N; ++l) {
            const double v = dx[i * N + l];
            scale = fabs(v) > scale ? fabs(v) : scale;
            const double d = fabs(dx[(N - 1 - i) * N + (N - 1 - l)] + v);
            dev = d > dev ? d : dev;
        }
    for (int st = 0; st < 6; ++st) {
        for (int t = 0; t < N * N; ++t) P.d[st][t] = dx[t];
        const bool trans = (st == kStS4 || st == kStS5 || st == kStS6);
        auto M = [&](int i, int l) { return trans ? dx[l * N + i] : dx[i * N + l]; };
        for (int i = 0; i < H; ++i)
            for (int l = 0; l < H; ++l) {
                P.a[st][i * H + l] = 0.5 * (M(i, l) + M(i, N - 1 - l));
                P.b[st][i * H + l] = 0.5 * (M(i, l) - M(i, N - 1 - l));
            }
        if (N % 2 == 1) {
            for (int i = 0; i < H; ++i) P.mc[st][i] = M(i, c);
            for (int l = 0; l < H; ++l) P.mr[st][l] = 0.5 * (M(c, l) - M(c, N - 1 - l));
        }
    }
    return dev <= 1e-13 * scale;
}

// Phase stagger of co-resident CTAs (stagger_wait): the k-th resident CTA
// of every SM waits (k - 1) x kStaggerNs[N] at entry when the launch has at
// least 6 waves.  SEM_AX_STAGGER=ns[,lo,hi] overrides (tuning).
// Scanned at E = 4096 with the defaults of kDefaultVariant (tools/
// gpu_stagger.sh, profiles/r02_ax_stagger.txt; 1965 MHz): n = 12 73.0 ->
// 72.2 us, 13 97.9 -> 94.6, 14 132.0 -> 129.4, 15 163.3 -> 155.4, 16 180.6 ->
// 165.8 (two CTAs per SM); n = 10 (three per SM) 40.21 -> 40.04; n = 7, 9,
// 11 flat, so 0.  The optimum is a fraction of an element's time (~0.3-0.9)
// and sharp: the values sit in the middle of each n's gain band.
constexpr int kStaggerNs[17] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1300, 0, 3000, 5500, 4000, 10000, 11500};
template <int N>
static void stagger_cfg(int minb, int64_t nbatches, int& ns, int& lo, int& hi)
{
    static const char* env = getenv("SEM_AX_STAGGER");
    ns = 0;
    lo = sm_count();
    hi = minb * sm_count();
    if (env) {
        hi = 2 * sm_count();
        sscanf(env, "%d,%d,%d", &ns, &lo, &hi);
        return;
    }
    if (minb >= 2 && nbatches >= 6 * (int64_t)minb * sm_count()) ns = kStaggerNs[N];
}

template <int N, int SLOTS, int MINB, bool PERSIST, int PD = 1, int L2PF = 0, int GMODE = 0,
          bool FOLD = false, int CGM = 0, bool ALIAS = false, bool WBULK = false>
static int launch_pencil(const double* u, const double* g, const double* dx, double* w,
                         int64_t E, cudaStream_t stream, CgpArgs cgp = CgpArgs{})
{
    using C = PencilCfg<N>;
    constexpr int THREADS = ((SLOTS * C::NN + 31) / 32) * 32;
    constexpr size_t SMEM = sizeof(double) * ((size_t)SLOTS * slot_doubles<N, ALIAS>() +
                                              (GMODE ? (size_t)SLOTS * 6 * C::NNN + 6 : 0));
    static_assert(SMEM * MINB <= 227 * 1024, "pencil kernel shared memory");
    DParamP<N> D;
    const bool antisym = fill_dparam<N>(D, dx);
    if constexpr (FOLD) {
        if (!antisym)  // the even-odd form needs a centro-antisymmetric D
            return launch_pencil<N, SLOTS, MINB, PERSIST, PD, L2PF, GMODE, false, CGM, ALIAS, WBULK>(
                u, g, dx, w, E, stream, cgp);
    }
    if (E == 0) return 0;
    auto kern = ax_pencil_kernel<N, SLOTS, THREADS, MINB, PERSIST, PD, L2PF, GMODE, FOLD, CGM, ALIAS,
                                 WBULK>;
    // function attributes live in each device's context: configure once per
    // (template instance, device); a benign race only repeats the setting
    static std::atomic<uint64_t> configured{0};
    int dev = 0;
    if (cudaError_t err = cudaGetDevice(&dev)) return fail_cuda(err, "sem_ax: cudaGetDevice");
    const uint64_t bit = 1ull << (dev & 63);
    if (!(configured.load(std::memory_order_acquire) & bit)) {
        cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)SMEM);
        if (err != cudaSuccess) return fail_cuda(err, "sem_ax: cudaFuncSetAttribute");
        // smem/L1 split: the streaming u/g loads need L1 capacity for their
        // in-flight lines, so the carveout is a tuning knob (measured in
        // profiles/; SEM_AX_CARVEOUT overrides, -1 = driver default)
        int carve = kAxCarveout;
        if (const char* env = getenv("SEM_AX_CARVEOUT")) carve = atoi(env);
        if (carve >= 0) {
            err = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
            if (err != cudaSuccess) return fail_cuda(err, "sem_ax: carveout");
        }
        configured.fetch_or(bit, std::memory_order_release);
    }
    const int64_t nbatches = (E + SLOTS - 1) / SLOTS;
    const int64_t resident = (int64_t)sm_count() * MINB;
    const int64_t grid = PERSIST ? (nbatches < resident ? nbatches : resident) : nbatches;
    // prefetch distance: the batch that replaces this one on its SM
    int64_t pf = L2PF == 2 ? 0
               : L2PF == 3 ? ((nbatches > resident) ? resident * SLOTS : 0)
                           : ((nbatches > resident) ? resident * SLOTS : -1);
    static const char* pf_env = getenv("SEM_AX_PFDIST");  // tuning probe
    if (pf_env) pf = atoll(pf_env);
    if (cgp.grid_out) *cgp.grid_out = (unsigned)grid;
    if constexpr (CGM == 0) {
        if (!PERSIST) stagger_cfg<N>(MINB, nbatches, cgp.stagger_ns, cgp.stagger_lo, cgp.stagger_hi);
    } else if constexpr (CGM == 2) {  // tuning probe: SEM_CG_STAGGER=ns[,lo,hi]
        static const char* cg_env = getenv("SEM_CG_STAGGER");
        if (cg_env) {
            cgp.stagger_lo = sm_count();
            cgp.stagger_hi = 2 * sm_count();
            sscanf(cg_env, "%d,%d,%d", &cgp.stagger_ns, &cgp.stagger_lo, &cgp.stagger_hi);
        }
    }
    // plain Ax as a programmatic dependent (CGM == 0): the pre-wait L2
    // prefetch of the CTA's own blocks (pdl == 2) pays for short launches and
    // cost ~0.6% on long ones (E = 1024: 13.2 -> 12.9 us; E = 4096: 41.7 ->
    // 41.9 us; profiles/r02_ax_pdl_ab.txt), so it is kept below ~200 MB
    if (CGM == 0 && cgp.pdl == 2 && E * (int64_t)C::NNN * 64 > (int64_t)200e6) cgp.pdl = 1;
    if (cgp.pdl) {
        cudaError_t err = launch_k(kern, dim3((unsigned)grid), dim3(THREADS), SMEM, stream, true,
                                   u, g, w, E, D, pf, cgp);
        if (err != cudaSuccess) return fail_cuda(err, "sem_ax (pencil, PDL) launch");
        return 0;
    }
    kern<<<(unsigned)grid, THREADS, SMEM, stream>>>(u, g, w, E, D, pf, cgp);
    SEM_CHECK_LAUNCH("sem_ax (pencil) launch");
    return 0;
}

template <int N, int SLOTS, int MINB, bool PERSIST, int PD = 1, int L2PF = 0, int GMODE = 0,
          bool FOLD = false, int CGM = 0, bool ALIAS = false, bool WBULK = false>
static int try_pencil(const double* u, const double* g, const double* dx, double* w, int64_t E,
                      cudaStream_t stream, CgpArgs cgp = CgpArgs{})
{
    if constexpr (SLOTS >= 1 && SLOTS * N * N <= 1024 &&
                  (GMODE < 2 || (N % 2 == 0 && PencilCfg<N>::RS == N)) &&
                  (GMODE < 4 || (SLOTS == 1 && CGM != 0)) &&
                  (!ALIAS || (!PERSIST && CGM == 0 && GMODE < 2)) &&
                  (!WBULK || (GMODE == 1 && SLOTS == 1 && CGM == 0 && !PERSIST && N % 2 == 0)) &&
                  sizeof(double) * ((size_t)SLOTS * slot_doubles<N, ALIAS>() +
                                    (GMODE ? (size_t)SLOTS * 6 * N * N * N + 6 : 0)) * MINB <= 227 * 1024)
        return launch_pencil<N, SLOTS, MINB, PERSIST, PD, L2PF, GMODE, FOLD, CGM, ALIAS, WBULK>(
            u, g, dx, w, E, stream, cgp);
    else {
        note_fallback();
        return launch_pencil<N, PencilCfg<N>::SLOTS, 1, false, 1, false, 0, false, CGM>(
            u, g, dx, w, E, stream, cgp);
    }
}

// Half-pencil kernel (ax_half.cuh): two threads per k-pencil, large n.
template <int N, int MINB, int PD, bool FOLD>
static int launch_half(const double* u, const double* g, const double* dx, double* w, int64_t E,
                       cudaStream_t stream, bool uahead = false)
{
    using C = HalfCfg<N>;
    if constexpr (C::THREADS > 1024 || C::SMEM * MINB > 227 * 1024) {
        note_fallback();
        return try_pencil<N, 1, 2, false, 2, 2, 0, true>(u, g, dx, w, E, stream);
    } else {
        DParamP<N> D;
        const bool antisym = fill_dparam<N>(D, dx);
        if constexpr (FOLD) {
            if (!antisym) return launch_half<N, MINB, PD, false>(u, g, dx, w, E, stream, uahead);
        }
        if (E == 0) return 0;
        if (E > 0x7fffffffLL) {
            set_error("sem_ax: too many elements (%lld)", (long long)E);
            return SEM_E_INVALID;
        }
        auto kern = ax_half_kernel<N, MINB, PD, FOLD>;
        static std::atomic<uint64_t> configured{0};
        int dev = 0;
        if (cudaError_t err = cudaGetDevice(&dev)) return fail_cuda(err, "sem_ax: cudaGetDevice");
        const uint64_t bit = 1ull << (dev & 63);
        if (!(configured.load(std::memory_order_acquire) & bit)) {
            cudaError_t err = cudaFuncSetAttribute(
                kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
            if (err != cudaSuccess) return fail_cuda(err, "sem_ax: cudaFuncSetAttribute");
            configured.fetch_or(bit, std::memory_order_release);
        }
        const int64_t resident = (int64_t)sm_count() * MINB;
        int sns = 0, slo = 0, shi = 0;
        stagger_cfg<N>(MINB, E, sns, slo, shi);
        kern<<<(unsigned)E, C::THREADS, C::SMEM, stream>>>(u, g, w, E, D,
                                                           uahead && E > resident ? resident : 0, sns,
                                                           slo, shi);
        SEM_CHECK_LAUNCH("sem_ax (half-pencil) launch");
        return 0;
    }
}

// Split-element kernel (ax_split.cuh): the two k-halves of an element on a
// 2-CTA cluster.
template <int N, int MINB, int GM, bool FOLD, bool ALIAS>
static int launch_split(const double* u, const double* g, const double* dx, double* w, int64_t E,
                        cudaStream_t stream, int pdl)
{
    using C = SplitCfg<N, ALIAS>;
    constexpr size_t SMEM = C::template smem<GM>();
    if constexpr (C::THREADS > 1024 || (SMEM + 1024) * MINB > 228 * 1024 || (GM && N % 2 != 0)) {
        note_fallback();
        return try_pencil<N, PencilCfg<N>::SLOTS, 1, false>(u, g, dx, w, E, stream);
    } else {
        DParamP<N> D;
        const bool antisym = fill_dparam<N>(D, dx);
        if constexpr (FOLD) {
            if (!antisym) return launch_split<N, MINB, GM, false, ALIAS>(u, g, dx, w, E, stream, pdl);
        }
        if (E == 0) return 0;
        if (E > 0x3fffffffLL) {
            set_error("sem_ax: too many elements (%lld)", (long long)E);
            return SEM_E_INVALID;
        }
        auto kern = ax_split_kernel<N, MINB, GM, FOLD, ALIAS>;
        static std::atomic<uint64_t> configured{0};
        int dev = 0;
        if (cudaError_t err = cudaGetDevice(&dev)) return fail_cuda(err, "sem_ax: cudaGetDevice");
        const uint64_t bit = 1ull << (dev & 63);
        if (!(configured.load(std::memory_order_acquire) & bit)) {
            cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)SMEM);
            if (err != cudaSuccess) return fail_cuda(err, "sem_ax: cudaFuncSetAttribute");
            configured.fetch_or(bit, std::memory_order_release);
        }
        cudaError_t err = launch_k(kern, dim3((unsigned)(2 * E)), dim3(C::THREADS), SMEM, stream,
                                   pdl != 0, u, g, w, E, D, pdl);
        if (err != cudaSuccess) return fail_cuda(err, "sem_ax (split) launch");
        return 0;
    }
}

// variant 0: the tuned default for this n (kDefaultVariant);
// 1: per-point layered kernel (first B200 version, kept for ablation);
// 2..19: pencil tuning points <elements per CTA, CTAs per SM, metric
// prefetch depth, persistent, L2 bulk prefetch>.
// Default tuning point per n (tools/ax_sweep.py on B200, E=4096; see
// profiles/r01_ax_sweep.txt, r01_ax_sweep_self_pf_raw.jsonl, CUDA-graph
// timed): index = n, value = variant id.  n >= 12: folded register ring with
// the CTA's own element bulk-prefetched into L2 at start (+10..30%); n = 15,
// 16 with the B stack aliasing U (profiles/r01_ax_row_stride.txt: 171 -> 163
// and 185 -> 182 us).
// Round 2 (two full sweeps, tools/gpu_psweep.sh, profiles/r02_ax_psweep.txt):
// n = 2 -> 10, 4 -> 17 (-21%: 3.9 vs 5.0 us), 7 -> 40, 8 -> 40, 9 -> 41
// (1.6-3.1%, the same winner in both sweeps); n = 12 -> 75 (half-pencil
// with the u block a resident wave ahead in L2: 73.2 vs 75.5 us), n = 13 ->
// 74 (the same prefetch on the register-ring pencil: 97.3 vs 99.4 us),
// confirmed by a second run (profiles/r02_ax_uahead.txt).
constexpr int kDefaultVariant[17] = {0, 0, 10, 5, 17, 34, 38, 40, 40, 41, 34, 41, 75, 74, 59, 62, 61};

template <int N>
static int ax_n(const double* u, const double* g, const double* dx, double* w, int64_t E,
                int variant, int pdl, cudaStream_t stream)
{
    constexpr int S = PencilCfg<N>::SLOTS;
    if (variant == 0) variant = kDefaultVariant[N];
    // pencil kernels launched as programmatic dependents: their CTAs wait
    // (griddepcontrol.wait) for the predecessor at entry, so a grid can be
    // resident while the previous kernel in the stream drains
    CgpArgs pa{};
    pa.pdl = pdl;
    switch (variant) {
        case 19: return try_pencil<N, S, 1, false>(u, g, dx, w, E, stream, pa);
        case 20: return try_pencil<N, 1, 4, false, 3>(u, g, dx, w, E, stream, pa);
        case 21: return try_pencil<N, 1, 4, false, 4>(u, g, dx, w, E, stream, pa);
        case 22: return try_pencil<N, 1, 4, false, 5>(u, g, dx, w, E, stream, pa);
        case 23: return try_pencil<N, 1, 5, false, 2>(u, g, dx, w, E, stream, pa);
        case 24: return try_pencil<N, 1, 3, false, 5>(u, g, dx, w, E, stream, pa);
        case 25: return try_pencil<N, 1, 3, false, 1, false, 1>(u, g, dx, w, E, stream, pa);
        case 26: return try_pencil<N, 1, 2, false, 1, false, 1>(u, g, dx, w, E, stream, pa);
        case 27: return try_pencil<N, 1, 3, false, 1, false, 2>(u, g, dx, w, E, stream, pa);
        case 28: return try_pencil<N, 1, 4, false, 1, false, 1>(u, g, dx, w, E, stream, pa);
        case 29: return try_pencil<N, 1, 4, false, 1, false, 2>(u, g, dx, w, E, stream, pa);
        case 30: return try_pencil<N, (S + 1) / 2, 2, false, 1, false, 1>(u, g, dx, w, E, stream, pa);
        case 31: return try_pencil<N, (S + 1) / 2, 2, false, 1, false, 2>(u, g, dx, w, E, stream, pa);
        case 32: return try_pencil<N, (S + 2) / 3, 3, false, 1, false, 2>(u, g, dx, w, E, stream, pa);
        case 33: return try_pencil<N, 2, 2, false, 1, false, 2>(u, g, dx, w, E, stream, pa);
        // even-odd folded contractions (centro-antisymmetric D only)
        case 34: return try_pencil<N, 1, 3, false, 1, false, 1, true>(u, g, dx, w, E, stream, pa);
        case 35: return try_pencil<N, 1, 2, false, 1, false, 1, true>(u, g, dx, w, E, stream, pa);
        case 36: return try_pencil<N, 1, 5, false, 3, false, 0, true>(u, g, dx, w, E, stream, pa);
        case 37: return try_pencil<N, 1, 4, false, 1, false, 1, true>(u, g, dx, w, E, stream, pa);
        case 38: return try_pencil<N, 1, 3, false, 1, false, 2, true>(u, g, dx, w, E, stream, pa);
        case 39: return try_pencil<N, (S + 1) / 2, 2, false, 1, false, 1, true>(u, g, dx, w, E, stream, pa);
        // + bulk L2 prefetch of the element a resident wave ahead
        case 40: return try_pencil<N, 1, 3, false, 1, true, 1, true>(u, g, dx, w, E, stream, pa);
        case 41: return try_pencil<N, 1, 2, false, 1, true, 1, true>(u, g, dx, w, E, stream, pa);
        // large n: folded contractions with the metric register ring
        case 42: return try_pencil<N, 1, 2, false, 1, false, 0, true>(u, g, dx, w, E, stream, pa);
        case 43: return try_pencil<N, 1, 2, false, 2, false, 0, true>(u, g, dx, w, E, stream, pa);
        case 44: return try_pencil<N, 1, 2, false, 1, true, 0, true>(u, g, dx, w, E, stream, pa);
        case 45: return try_pencil<N, 1, 3, false, 1, false, 0, true>(u, g, dx, w, E, stream, pa);
        case 46: return try_pencil<N, 1, 1, false, 2, false, 0, true>(u, g, dx, w, E, stream, pa);
        // large n: register ring + the CTA's own element bulk-prefetched to L2
        case 47: return try_pencil<N, 1, 2, false, 1, 2, 0, true>(u, g, dx, w, E, stream, pa);
        case 48: return try_pencil<N, 1, 2, false, 2, 2, 0, true>(u, g, dx, w, E, stream, pa);
        case 49: return try_pencil<N, 1, 2, false, 1, 2, 0, false>(u, g, dx, w, E, stream, pa);
        case 50: return try_pencil<N, 1, 3, false, 1, 2, 0, true>(u, g, dx, w, E, stream, pa);
        case 51: return try_pencil<N, 1, 1, false, 3, 2, 0, true>(u, g, dx, w, E, stream, pa);
        case 52: return try_pencil<N, 1, 3, false, 1, 2, 1, true>(u, g, dx, w, E, stream, pa);
        case 53: return try_pencil<N, 1, 2, false, 1, 2, 1, true>(u, g, dx, w, E, stream, pa);
        case 54: return try_pencil<N, 1, 2, false, 3, 2, 0, true>(u, g, dx, w, E, stream, pa);
        case 55: return try_pencil<N, 1, 2, false, 4, 2, 0, true>(u, g, dx, w, E, stream, pa);
        // half-pencil kernel (two threads per k-pencil)
        case 56: return launch_half<N, 1, 2, true>(u, g, dx, w, E, stream);
        case 57: return launch_half<N, 2, 2, true>(u, g, dx, w, E, stream);
        case 58: return launch_half<N, 1, 3, true>(u, g, dx, w, E, stream);
        case 59: return launch_half<N, 2, 1, true>(u, g, dx, w, E, stream);
        case 60: return launch_half<N, 1, 4, true>(u, g, dx, w, E, stream);
        // large n, the B stack aliasing U (dead after S1/S2: one stack less per
        // element, one extra barrier): register ring + own element L2-prefetched
        case 61: return try_pencil<N, 1, 2, false, 2, 2, 0, true, 0, true>(u, g, dx, w, E, stream, pa);
        case 62: return try_pencil<N, 1, 2, false, 3, 2, 0, true, 0, true>(u, g, dx, w, E, stream, pa);
        // TMA-staged metric + w written back by one bulk store per element
        case 63: return try_pencil<N, 1, 3, false, 1, false, 1, true, 0, false, true>(u, g, dx, w, E, stream, pa);
        case 64: return try_pencil<N, 1, 2, false, 1, false, 1, true, 0, false, true>(u, g, dx, w, E, stream, pa);
        // split element: the two k-halves on a 2-CTA cluster (ax_split.cuh)
        case 65: return launch_split<N, 6, 1, true, true>(u, g, dx, w, E, stream, pdl);
        case 66: return launch_split<N, 5, 1, true, false>(u, g, dx, w, E, stream, pdl);
        case 67: return launch_split<N, 4, 0, true, true>(u, g, dx, w, E, stream, pdl);
        case 68: return launch_split<N, 6, 0, true, true>(u, g, dx, w, E, stream, pdl);
        case 69: return launch_split<N, 3, 0, true, true>(u, g, dx, w, E, stream, pdl);
        case 70: return launch_split<N, 8, 0, true, true>(u, g, dx, w, E, stream, pdl);
        // large n: as 61 / 62 / 54 / 55 / 59 with the u block of the element
        // a resident wave ahead also prefetched into L2 (L2PF 3)
        case 71: return try_pencil<N, 1, 2, false, 2, 3, 0, true, 0, true>(u, g, dx, w, E, stream, pa);
        case 72: return try_pencil<N, 1, 2, false, 3, 3, 0, true, 0, true>(u, g, dx, w, E, stream, pa);
        case 73: return try_pencil<N, 1, 2, false, 3, 3, 0, true>(u, g, dx, w, E, stream, pa);
        case 74: return try_pencil<N, 1, 2, false, 4, 3, 0, true>(u, g, dx, w, E, stream, pa);
        case 75: return launch_half<N, 2, 1, true>(u, g, dx, w, E, stream, true);
        case 1: return launch_ax<N>(u, g, dx, w, E, stream);
        case 2: return try_pencil<N, S, 1, true>(u, g, dx, w, E, stream, pa);
        case 3: return try_pencil<N, (S + 1) / 2, 2, false>(u, g, dx, w, E, stream, pa);
        case 4: return try_pencil<N, (S + 1) / 2, 2, false, 2>(u, g, dx, w, E, stream, pa);
        case 5: return try_pencil<N, (S + 1) / 2, 2, false, 3>(u, g, dx, w, E, stream, pa);
        case 6: return try_pencil<N, (S + 2) / 3, 3, false>(u, g, dx, w, E, stream, pa);
        case 7: return try_pencil<N, (S + 2) / 3, 3, false, 2>(u, g, dx, w, E, stream, pa);
        case 8: return try_pencil<N, (S + 2) / 3, 3, false, 3>(u, g, dx, w, E, stream, pa);
        case 9: return try_pencil<N, 1, 6, false, 2>(u, g, dx, w, E, stream, pa);
        case 10: return try_pencil<N, (S + 2) / 3, 3, false, 1, true>(u, g, dx, w, E, stream, pa);
        case 11: return try_pencil<N, S + 1, 1, false, 2>(u, g, dx, w, E, stream, pa);
        case 12: return try_pencil<N, 1, 7, false, 1>(u, g, dx, w, E, stream, pa);
        case 13: return try_pencil<N, 1, 7, false, 2>(u, g, dx, w, E, stream, pa);
        case 14: return try_pencil<N, 1, 7, false, 3>(u, g, dx, w, E, stream, pa);
        case 15: return try_pencil<N, 1, 5, false, 3>(u, g, dx, w, E, stream, pa);
        case 16: return try_pencil<N, 1, 6, false, 3>(u, g, dx, w, E, stream, pa);
        case 17: return try_pencil<N, (S + 1) / 2, 2, false, 4>(u, g, dx, w, E, stream, pa);
        default:
            set_error("sem_ax: unknown variant %d", variant);
            return SEM_E_INVALID;
    }
}

// CG iteration head fused with Ax (p = beta p + r; w = A_local p): the tuned
// configuration of each n with the metric staged by TMA and u through
// registers (the p update happens while the column is loaded), x update and
// <p, A p> fused too (ax_pencil.cuh).  CGM = 2: single-GPU solver; CGM = 3:
// z-slab rank of the multi-GPU solver.
template <int N, int CGM>
static int ax_cg_n(const double* g, const double* dx, double* w, int64_t E, CgpArgs a,
                   cudaStream_t s)
{
    double* p = a.p;
    if constexpr (N >= 8 && N <= 11) {
        // tuning hook (SEM_CG_AX_CFG, tools/cg_phases.py): alternative
        // tilings of the fused CG Ax for the headline degrees
        static const int cfg = getenv("SEM_CG_AX_CFG") ? atoi(getenv("SEM_CG_AX_CFG")) : 0;
        switch (cfg) {
            case 1: return try_pencil<N, 1, 4, false, 1, false, 0, true, CGM>(p, g, dx, w, E, s, a);
            case 2: return try_pencil<N, 1, 5, false, 2, false, 0, true, CGM>(p, g, dx, w, E, s, a);
            case 3: return try_pencil<N, 2, 2, false, 1, false, 0, true, CGM>(p, g, dx, w, E, s, a);
            case 4: return try_pencil<N, 1, 3, false, 1, false, 1, true, CGM>(p, g, dx, w, E, s, a);
            case 5: return try_pencil<N, 1, 2, false, 1, false, 1, true, CGM>(p, g, dx, w, E, s, a);
            // GMODE 4: all bulk copies issued before the CG scalars are read
            case 9: return try_pencil<N, 1, 3, false, 1, true, 4, true, CGM>(p, g, dx, w, E, s, a);
            case 10: return try_pencil<N, 1, 3, false, 1, false, 4, true, CGM>(p, g, dx, w, E, s, a);
            default: break;
        }
    }
    // default: TMA-staged metric, folded contractions, and a bulk L2 prefetch
    // of the element that replaces this one on its SM (its g, p, r and x):
    // the CG prologue reads three fields besides g, and warming L2 a wave
    // ahead cut the fused Ax from 88 to 79 us at E = 4096 and from 608 to
    // 502 us at E = 32768 (tools/cg_tune.sh, profiles/r01_cg_tune.txt)
    //
    // n = 6, 10 (even, unpadded stack rows): p, r and x are bulk-copied too,
    // and every copy is issued before the CG scalars are read (GMODE 4;
    // tools/cg_tune5.sh: E = 4096 77.2 -> 73.0 us, E = 32768 457 -> 451 us)
    if constexpr (N >= 6 && N <= 10 && N % 2 == 0 && PencilCfg<N>::RS == N)
        return try_pencil<N, 1, 3, false, 1, true, 4, true, CGM>(p, g, dx, w, E, s, a);
    else if constexpr (N == 11)  // 96 KB of shared memory per CTA: two per SM
        // (three did not fit and fell back to the generic tiling: 184 -> 140 us
        // per CG iteration at E = 4096; other n measured flat in the CTAs per
        // SM, profiles/r01_cg_minb.txt)
        return try_pencil<N, 1, 2, false, 1, true, 1, true, CGM>(p, g, dx, w, E, s, a);
    else if constexpr (N >= 5 && N <= 11)
        return try_pencil<N, 1, 3, false, 1, true, 1, true, CGM>(p, g, dx, w, E, s, a);
    else if constexpr (N == 4)
        return try_pencil<N, 1, 2, false, 1, false, 1, false, CGM>(p, g, dx, w, E, s, a);
    else if constexpr (N >= 12)  // register ring + own element prefetched to L2
        return try_pencil<N, 1, 2, false, 2, 2, 0, true, CGM>(p, g, dx, w, E, s, a);
    else
        return try_pencil<N, 1, 2, false, 1, false, 0, false, CGM>(p, g, dx, w, E, s, a);
}

}  // namespace sem
