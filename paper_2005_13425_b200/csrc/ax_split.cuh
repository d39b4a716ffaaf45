// Split-element Ax kernel: the two k-halves of one element on the two CTAs
// of a 2-CTA thread-block cluster, coupled through distributed shared memory.
//
// Why: with one element per CTA (ax_pencil.cuh) the unit of work is a whole
// element -- 56 n^3 B of loads, then all the contractions -- so at E = 1024
// (2.3 waves of 3 CTAs per SM at n = 10) the last partial wave runs one
// element per SM with nothing else to overlap, and at large n the 3 n^3
// doubles of layer stacks cap residency at 2 elements per SM.  Splitting an
// element across a CTA pair halves the per-CTA load, stacks and latency, so
// twice as many (half-size) units are resident and the tail is half as long.
//
// The contractions along r and s stay inside a k-layer; only the t direction
// couples the halves:
//   * wt = D u along k needs the whole u column: each CTA reads it (the
//     peer's half is an L2 hit -- DRAM traffic is unchanged);
//   * w_t = D^T ut along k needs ut of every layer: each CTA forms the
//     partial sum over ITS layers for ALL kk, pushes the peer's half into the
//     peer's shared memory and adds the partial it receives -- one exchange
//     of n^3/2 doubles per element.  The pushes are asynchronous remote
//     stores (st.async) that complete transaction bytes on the receiver's
//     mbarrier, so no cluster-wide fence is needed: a cluster barrier with a
//     release arrive compiled to MEMBAR.ALL.GPU and made "membar" the
//     second-largest stall (ncu, profiles/r02_split_ncu.txt).
//
// CTA c of the pair owns layers [K0, K0 + NK) (c = 0: the first KA = ceil(n/2)).
//   S3  k-pencil (i,j): u column (all n layers) -> regs; own layers -> U;
//       wt[own k] = D u_col                                         | sync
//   S1  i-pencils (j,k) of own layers: U row -> D -> A   (threads [0, n NK))
//   S2  j-pencils (i,k) of own layers: U col -> D -> B   (threads [JOFF, ..))
//                                                                   | sync
//   S4  k-pencil per own layer: metric (staged by TMA, GM = 1) -> ur -> A,
//       us -> B, ut -> partial w_t[kk] for all kk (regs)
//       push partial w_t[peer layers] -> peer X (st.async, peer's mbarrier)
//   S5  i-pencils: A row <- D^T ;  S6 j-pencils: B col <- D^T    | sync
//       wait on the own X mbarrier
//   S7  k-pencil: w = A + B + (own partial + X) on own layers -> HBM
#pragma once
#include "ax_pencil.cuh"

namespace sem {

template <int N, bool ALIAS>
struct SplitCfg {
    using P = PencilCfg<N>;
    static constexpr int NN = N * N, NNN = N * N * N;
    static constexpr int KA = (N + 1) / 2;  // layers of CTA 0; CTA 1 has N - KA
    static constexpr int RS = P::RS, LSU = P::LSU, LSA = P::LSA, LSB = P::LSB;
    // i-pencils on threads [0, n KA), j-pencils from the next warp boundary
    static constexpr int JOFF = ((N * KA + 31) / 32) * 32;
    static constexpr int TNEED = (NN > JOFF + N * KA) ? NN : JOFF + N * KA;
    static constexpr int THREADS = ((TNEED + 31) / 32) * 32;
    // shared memory (doubles): U, A, [B], then the staged metric (GM = 1),
    // then X (the partial w_t received from the peer), then one mbarrier
    static constexpr int STACKS = KA * (LSU + LSA + (ALIAS ? 0 : LSB));
    static constexpr int G_OFF = (STACKS + 1) / 2 * 2;
    template <int GM>
    static constexpr int x_off() { return G_OFF + (GM ? 6 * KA * NN : 0); }
    template <int GM>
    static constexpr int bar_off() { return (x_off<GM>() + KA * NN + 1) / 2 * 2; }
    template <int GM>
    static constexpr size_t smem() { return sizeof(double) * ((size_t)bar_off<GM>() + 2); }
    // mbarriers: [0] the staged metric (GM = 1), [1] X (the peer's partial)
};

__device__ __forceinline__ unsigned cluster_ctarank()
{
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_arrive_relaxed()
{
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait()
{
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `local` in CTA `rank` of this cluster
__device__ __forceinline__ uint32_t map_peer(const void* local, unsigned rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
    return r;
}
// asynchronous remote store completing 8 transaction bytes on the remote
// CTA's mbarrier `rbar`
__device__ __forceinline__ void st_async_f64(uint32_t addr, double v, uint32_t rbar)
{
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(addr),
                 "d"(v), "r"(rbar)
                 : "memory");
}

// One CTA's half of an element: CH = its rank in the pair (compile time, so
// every D operand stays a constant-bank index).
template <int N, int CH, int GM, bool FOLD, bool ALIAS>
__device__ __forceinline__ void split_half(const double* __restrict__ u,
                                           const double* __restrict__ g, double* __restrict__ w,
                                           int64_t e, int64_t num_elements, const DParamP<N>& D,
                                           double* smem, bool pdl)
{
    using C = SplitCfg<N, ALIAS>;
    constexpr int NN = C::NN, NNN = C::NNN, KA = C::KA, RS = C::RS, LSU = C::LSU,
                  LSA = C::LSA, LSB = C::LSB, JOFF = C::JOFF;
    constexpr int K0 = CH ? KA : 0, NK = CH ? N - KA : KA;      // own layers
    constexpr int KO = CH ? 0 : KA, NKO = CH ? KA : N - KA;     // the peer's layers
    double* U = smem;
    double* A = U + KA * LSU;
    double* B = ALIAS ? U : A + KA * LSA;
    double* G = smem + C::G_OFF;
    double* X = smem + C::template x_off<GM>();
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::template bar_off<GM>());
    uint64_t* xbar = bar + 1;

    const int tid = threadIdx.x;
    const bool kp_ok = tid < NN;                  // k-pencil (i,j) = tid
    const int kp = (tid / N) * RS + tid % N;
    const bool ip_ok = tid < N * NK;              // i-pencil (j,k) of an own layer
    const int jq = tid - JOFF;
    const bool jp_ok = jq >= 0 && jq < N * NK;    // j-pencil (i,k) of an own layer

    if (tid == 0) {
        if (GM) mbar_init(bar, 1);
        mbar_init(xbar, 1);
        mbar_expect_tx(xbar, (unsigned)(NK * NN * 8));  // the peer's partial of our layers
    }
    __syncthreads();
    cluster_arrive_relaxed();  // X's mbarrier is live: the peer may push after its wait
    if (pdl) {                 // programmatic dependent: the predecessor must be complete
        griddep_wait();
        griddep_launch();
    }
    if constexpr (GM) {
        if (tid == 0) {  // own layers of the six metric fields, one bulk copy each
            mbar_expect_tx(bar, (unsigned)(6 * NK * NN * 8));
#pragma unroll
            for (int m = 0; m < 6; ++m)
                bulk_g2s(G + m * KA * NN, g + e * 6 * NNN + m * NNN + K0 * NN, NK * NN * 8, bar);
        }
    } else {
        if (tid == 0) {  // own layers of the metric straight into L2
#pragma unroll
            for (int m = 0; m < 6; ++m) {
                const int64_t lo = (e * 6 * NNN + m * NNN + K0 * NN) * 8;
                prefetch_l2_bulk(g, lo, lo + NK * NN * 8, num_elements * 6 * NNN * 8);
            }
        }
    }

    // ---- S3: u column -> regs, own layers -> U; wt on own layers ----------
    double ucol[N], wt[NK];
    {
        const double* src = u + e * NNN + (kp_ok ? tid : 0);
#pragma unroll
        for (int k = 0; k < N; ++k) ucol[k] = kp_ok ? __ldg(src + k * NN) : 0.0;
    }
    if (kp_ok) {
#pragma unroll
        for (int m = 0; m < NK; ++m) U[m * LSU + kp] = ucol[K0 + m];
    }
#pragma unroll
    for (int m = 0; m < NK; ++m) {
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) s = fma(D.d[kStS3][(K0 + m) * N + l], ucol[l], s);
        wt[m] = s;
    }
    double gq[6];  // GM = 0: metric of the next own layer (register ring of depth 1)
    if constexpr (!GM) {
#pragma unroll
        for (int c = 0; c < 6; ++c)
            gq[c] = kp_ok ? __ldg(g + e * 6 * NNN + c * NNN + K0 * NN + tid) : 0.0;
    }
    __syncthreads();

    // ---- S1 / S2 on own layers (disjoint thread ranges) --------------------
    {
        double out[N];
        if (ip_ok) {
            const int j = tid % N, m = tid / N;
            double row[N];
            stack_row_ld<N>(U + m * LSU + j * RS, row);
            pencil_gemv<N, FOLD, false>(D, kStS1, row, out);
            stack_row_st<N>(A + m * LSA + j * RS, out);
        } else if (jp_ok) {
            const int i = jq % N, m = jq / N;
            double col[N];
            const double* src = U + m * LSU + i;
#pragma unroll
            for (int l = 0; l < N; ++l) col[l] = src[l * RS];
            pencil_gemv<N, FOLD, false>(D, kStS2, col, out);
        }
        if constexpr (ALIAS) __syncthreads();  // every U read done: B overwrites it
        if (jp_ok) {
            const int i = jq % N, m = jq / N;
            double* dst = B + m * LSB + i;
#pragma unroll
            for (int j = 0; j < N; ++j) dst[j * RS] = out[j];
        }
    }
    __syncthreads();

    // ---- S4: metric per own layer; partial w_t over own layers, all kk ----
    if constexpr (GM) mbar_wait(bar, 0);
    double Wp[N];
#pragma unroll
    for (int kk = 0; kk < N; ++kk) Wp[kk] = 0.0;
#pragma unroll
    for (int m = 0; m < NK; ++m) {
        double gc[6];
        if constexpr (GM) {
#pragma unroll
            for (int c = 0; c < 6; ++c) gc[c] = kp_ok ? G[c * KA * NN + m * NN + tid] : 0.0;
        } else {
#pragma unroll
            for (int c = 0; c < 6; ++c) gc[c] = gq[c];
            if (m + 1 < NK) {
#pragma unroll
                for (int c = 0; c < 6; ++c)
                    gq[c] = kp_ok ? __ldg(g + e * 6 * NNN + c * NNN + (K0 + m + 1) * NN + tid) : 0.0;
            }
        }
        if (kp_ok) {
            const double a = A[m * LSA + kp];
            const double b = B[m * LSB + kp];
            const double t = wt[m];
            const double ur = fma(gc[2], t, fma(gc[1], b, gc[0] * a));
            const double us = fma(gc[4], t, fma(gc[3], b, gc[1] * a));
            const double ut = fma(gc[5], t, fma(gc[4], b, gc[2] * a));
            A[m * LSA + kp] = ur;
            B[m * LSB + kp] = us;
#pragma unroll
            for (int kk = 0; kk < N; ++kk) Wp[kk] = fma(D.d[kStS4][(K0 + m) * N + kk], ut, Wp[kk]);
        }
    }
    // the peer's layers of the partial -> the peer's X (its mbarrier is live)
    cluster_wait();
    if (kp_ok) {
        const uint32_t px = map_peer(X + tid, CH ^ 1);
        const uint32_t pb = map_peer(xbar, CH ^ 1);
#pragma unroll
        for (int m = 0; m < NKO; ++m) st_async_f64(px + (uint32_t)(m * NN * 8), Wp[KO + m], pb);
    }
    __syncthreads();

    // ---- S5 / S6 on own layers ---------------------------------------------
    if (ip_ok) {
        const int j = tid % N, m = tid / N;
        double row[N], out[N];
        double* rp = A + m * LSA + j * RS;
        stack_row_ld<N>(rp, row);
        pencil_gemv<N, FOLD, true>(D, kStS5, row, out);
        stack_row_st<N>(rp, out);
    } else if (jp_ok) {
        const int i = jq % N, m = jq / N;
        double col[N], out[N];
        double* cp = B + m * LSB + i;
#pragma unroll
        for (int l = 0; l < N; ++l) col[l] = cp[l * RS];
        pencil_gemv<N, FOLD, true>(D, kStS6, col, out);
#pragma unroll
        for (int j = 0; j < N; ++j) cp[j * RS] = out[j];
    }
    __syncthreads();
    mbar_wait(xbar, 0);  // our X holds the peer's partial

    // ---- S7: w = A + B + w_t on own layers ----------------------------------
    if (kp_ok) {
        double* we = w + e * NNN + K0 * NN + tid;
#pragma unroll
        for (int m = 0; m < NK; ++m)
            __stcs(we + m * NN, (A[m * LSA + kp] + B[m * LSB + kp]) + (Wp[K0 + m] + X[m * NN + tid]));
    }
}

template <int N, int MINB, int GM, bool FOLD, bool ALIAS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(SplitCfg<N, ALIAS>::THREADS, MINB)
ax_split_kernel(const double* __restrict__ u, const double* __restrict__ g, double* __restrict__ w,
                int64_t num_elements, const DParamP<N> D, int pdl)
{
    static_assert(!GM || N % 2 == 0, "bulk metric copies need 16-byte layer blocks (even n)");
    extern __shared__ __align__(16) double smem[];
    const int64_t e = (int64_t)blockIdx.x >> 1;  // both CTAs of a pair exist even past E
    if (e >= num_elements) return;               // (grid = 2E: never taken)
    if (cluster_ctarank() == 0)
        split_half<N, 0, GM, FOLD, ALIAS>(u, g, w, e, num_elements, D, smem, pdl != 0);
    else
        split_half<N, 1, GM, FOLD, ALIAS>(u, g, w, e, num_elements, D, smem, pdl != 0);
}

}  // namespace sem
