// "Half-pencil" Ax kernel for large n (n >= 12): the pencil algorithm of
// ax_pencil.cuh with TWO threads per k-pencil.
//
// Why: at n >= 13 the pencil kernel holds n-long register arrays per thread
// (u column, wt, Wt, ut) and 3n^3 doubles of layer stacks per element, so a
// CTA of n^2 threads needs ~128 registers and two elements fill an SM: 512
// threads, too few loads in flight (profiles/r01_ax_n16_ncu.txt).  Here the
// k-direction work of a pencil (i,j) is split between two threads, one per
// half of the k layers (h = 0: k < KH, h = 1: k >= KH), so the per-thread
// arrays are KH long and a CTA has 2 x n^2 threads; the i- and j-pencil
// stages run concurrently on the two thread halves.
//
//   S3  (h): own half of the u column HBM -> U                          | sync
//       (h): wt[k in half] = sum_l D[k][l] U[l]  (streamed from smem)
//   S1  (h=0 warps): i-pencil rows of U -> D -> A
//   S2  (h=1 warps): j-pencil columns of U -> D -> B                      | sync
//   S4  (h): per own layer, metric (register ring, own element prefetched
//       to L2 at CTA start): ur -> A, us -> B, ut -> UT (aliases U)       | sync
//       (h): Wt[k in half] = sum_k' D[k'][k] UT[k']
//   S5  (h=0): A rows <- D^T ;  S6 (h=1): B columns <- D^T               | sync
//   S7  (h): w = A + B + Wt on own layers -> HBM
//
// The two halves start on warp boundaries (NP = n^2 rounded up to 32), so h
// is warp-uniform and every D operand is a compile-time constant-bank index.
#pragma once
#include "ax_pencil.cuh"

namespace sem {

template <int N>
struct HalfCfg {
    static constexpr int NN = N * N, NNN = N * N * N;
    static constexpr int KH = (N + 1) / 2;            // layers of half 0
    static constexpr int NP = ((NN + 31) / 32) * 32;  // threads per half
    static constexpr int THREADS = 2 * NP;
    using P = PencilCfg<N>;
    // unpadded rows (RS = N) and layer strides == N (mod 16).  Measured
    // (profiles/r01_ax_row_stride.txt): the pencil kernel's padded rows
    // (RS == 2 mod 4) cost this kernel 7-10% at n = 12, an odd stride 7-16%.
    static constexpr int RS = N, LSA = NN;
    static constexpr int LSB = NN + (((N - NN) % 16) + 16) % 16;
    static constexpr int LSU = LSB;
    static constexpr size_t SMEM = sizeof(double) * (size_t)N * (LSU + LSA + LSB);
};

// the k-direction work of one half-pencil: H = 0 (k < KH) or 1 (k >= KH)
template <int N, int H, int PD>
__device__ __forceinline__ void half_k_stages_s3(const DParamP<N>& D, const double* U, int p,
                                                 double (&wt)[HalfCfg<N>::KH])
{
    using C = HalfCfg<N>;
    constexpr int K0 = H * C::KH, NK = H ? N - C::KH : C::KH;
#pragma unroll
    for (int m = 0; m < C::KH; ++m) wt[m] = 0.0;
#pragma unroll
    for (int l = 0; l < N; ++l) {
        const double ul = U[l * C::LSU + p];
#pragma unroll
        for (int m = 0; m < NK; ++m) wt[m] = fma(D.d[kStS3][(K0 + m) * N + l], ul, wt[m]);
    }
}

template <int N, int H>
__device__ __forceinline__ void half_k_wt(const DParamP<N>& D, const double* UT, int p,
                                          double (&Wt)[HalfCfg<N>::KH])
{
    using C = HalfCfg<N>;
    constexpr int K0 = H * C::KH, NK = H ? N - C::KH : C::KH;
#pragma unroll
    for (int m = 0; m < C::KH; ++m) Wt[m] = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const double t = UT[k * C::LSU + p];
#pragma unroll
        for (int m = 0; m < NK; ++m) Wt[m] = fma(D.d[kStS4][k * N + K0 + m], t, Wt[m]);
    }
}

template <int N, int MINB, int PD, bool FOLD>
__global__ void __launch_bounds__(HalfCfg<N>::THREADS, MINB)
ax_half_kernel(const double* __restrict__ u, const double* __restrict__ g,
               double* __restrict__ w, int64_t num_elements, const DParamP<N> D,
               int64_t uahead = 0, int stagger_ns = 0, int stagger_lo = 0, int stagger_hi = 0)
{
    stagger_wait(stagger_ns, stagger_lo, stagger_hi);
    using C = HalfCfg<N>;
    constexpr int NN = C::NN, NNN = C::NNN, KH = C::KH, LSU = C::LSU, LSA = C::LSA,
                  LSB = C::LSB, NP = C::NP, RS = C::RS;
    extern __shared__ __align__(16) double smem[];
    double* U = smem;             // u stack; after S1/S2 it holds ut (UT)
    double* A = U + N * LSU;
    double* B = A + N * LSA;

    const int tid = threadIdx.x;
    const int h = tid / NP;       // warp-uniform half
    const int q = tid - h * NP;   // k-pencil / i-pencil / j-pencil index
    const bool ok = q < NN;
    const int kq = (q / N) * RS + q % N;  // k-pencil (i, j) = q: offset in a stack layer
    const int64_t e = blockIdx.x;
    const double* ue = u + e * NNN;
    const double* ge = g + e * 6 * NNN;
    if (tid == 0) {  // the whole element streams into L2 at once
        prefetch_l2_bulk(u, e * NNN * 8, (e + 1) * NNN * 8, num_elements * NNN * 8);
        prefetch_l2_bulk(g, e * 6 * NNN * 8, (e + 1) * 6 * NNN * 8, num_elements * 6 * NNN * 8);
        // and the u block of the element a resident wave later (uahead > 0)
        if (uahead > 0 && e + uahead < num_elements)
            prefetch_l2_bulk(u, (e + uahead) * NNN * 8, (e + uahead + 1) * NNN * 8,
                             num_elements * NNN * 8);
    }
    const int K0 = h * KH, NK = h ? N - KH : KH;

    // ---- S3: own half of the u column -> U; metric ring of the first layers
    double gq[PD][6];
    if (ok) {
#pragma unroll
        for (int m = 0; m < KH; ++m)
            if (m < NK) U[(K0 + m) * LSU + kq] = __ldg(ue + (K0 + m) * NN + q);
#pragma unroll
        for (int d = 0; d < PD; ++d)
#pragma unroll
            for (int c = 0; c < 6; ++c)
                gq[d][c] = (d < NK) ? __ldg(ge + c * NNN + (K0 + d) * NN + q) : 0.0;
    }
    __syncthreads();
    double wt[KH];
    if (ok) {
        if (h == 0) half_k_stages_s3<N, 0, PD>(D, U, kq, wt);
        else half_k_stages_s3<N, 1, PD>(D, U, kq, wt);
    }
    // ---- S1 (h = 0): i-pencil (j,k) = q ; S2 (h = 1): j-pencil (i,k) = q
    if (ok) {
        const int a = q % N, k = q / N;
        double in[N], out[N];
        if (h == 0) {
            const double* src = U + k * LSU + a * RS;  // row (j = a, k)
#pragma unroll
            for (int l = 0; l < N; ++l) in[l] = src[l];
            pencil_gemv<N, FOLD, false>(D, kStS1, in, out);
            double* dst = A + k * LSA + a * RS;
#pragma unroll
            for (int i = 0; i < N; ++i) dst[i] = out[i];
        } else {
            const double* src = U + k * LSU + a;      // column (i = a, k)
#pragma unroll
            for (int l = 0; l < N; ++l) in[l] = src[l * RS];
            pencil_gemv<N, FOLD, false>(D, kStS2, in, out);
            double* dst = B + k * LSB + a;
#pragma unroll
            for (int j = 0; j < N; ++j) dst[j * RS] = out[j];
        }
    }
    __syncthreads();

    // ---- S4: metric on own layers; ut -> UT (the U stack is dead now)
    if (ok) {
#pragma unroll
        for (int m = 0; m < KH; ++m) {
            if (m < NK) {
                const int k = K0 + m;
                double gc[6];
#pragma unroll
                for (int c = 0; c < 6; ++c) gc[c] = gq[m % PD][c];
                if (m + PD < NK) {
#pragma unroll
                    for (int c = 0; c < 6; ++c)
                        gq[m % PD][c] = __ldg(ge + c * NNN + (k + PD) * NN + q);
                }
                const double av = A[k * LSA + kq], bv = B[k * LSB + kq], tv = wt[m];
                A[k * LSA + kq] = fma(gc[2], tv, fma(gc[1], bv, gc[0] * av));
                B[k * LSB + kq] = fma(gc[4], tv, fma(gc[3], bv, gc[1] * av));
                U[k * LSU + kq] = fma(gc[5], tv, fma(gc[4], bv, gc[2] * av));
            }
        }
    }
    __syncthreads();
    double Wt[KH];
    if (ok) {
        if (h == 0) half_k_wt<N, 0>(D, U, kq, Wt);
        else half_k_wt<N, 1>(D, U, kq, Wt);
    }
    // ---- S5 (h = 0): A rows <- D^T ; S6 (h = 1): B columns <- D^T
    if (ok) {
        const int a = q % N, k = q / N;
        double in[N], out[N];
        if (h == 0) {
            double* rp = A + k * LSA + a * RS;
#pragma unroll
            for (int l = 0; l < N; ++l) in[l] = rp[l];
            pencil_gemv<N, FOLD, true>(D, kStS5, in, out);
#pragma unroll
            for (int i = 0; i < N; ++i) rp[i] = out[i];
        } else {
            double* cp = B + k * LSB + a;
#pragma unroll
            for (int l = 0; l < N; ++l) in[l] = cp[l * RS];
            pencil_gemv<N, FOLD, true>(D, kStS6, in, out);
#pragma unroll
            for (int j = 0; j < N; ++j) cp[j * RS] = out[j];
        }
    }
    __syncthreads();

    // ---- S7: w = A + B + Wt on own layers
    if (ok) {
        double* we = w + e * NNN + q;
#pragma unroll
        for (int m = 0; m < KH; ++m) {
            if (m < NK) {
                const int k = K0 + m;
                __stcs(we + k * NN, (A[k * LSA + kq] + B[k * LSB + kq]) + Wt[m]);
            }
        }
    }
}

}  // namespace sem
