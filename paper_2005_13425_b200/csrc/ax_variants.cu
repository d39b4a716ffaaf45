// The reference's two other storage strategies for Ax, on B200 (sm_100a):
// the GPU analogs of the paper's slower baselines (§IV-A, §IV-B), kept so
// `variant="reference"` / `"scratch"` run what they name and the paper's
// kernel ordering can be reproduced on B200.
//
//  REFERENCE (sembench/kernels.py:159-205): three launches over all
//    elements -- derivative pass writes full-size ur/us/ut, geometric pass
//    rewrites them in place with the metric, transpose pass contracts them
//    into w.  13 D words read + 7 D written (kernels.py:36), so it is HBM
//    bound at ~2.5x the LAYERED kernel's traffic.  On return ur/us/ut hold the
//    metric-scaled gradients, exactly as the reference leaves its workspace.
//  SCRATCH (kernels.py:213-259): one CTA per element stages u and D in shared
//    memory, phase 1 (gradients + metric, g read per point) writes three
//    element-sized shared blocks, phase 2 contracts them with D read
//    transposed.  7 D read + 1 D written; refuses n > 10 like the reference.
//
// Both replay the reference's operation order with unfused multiply / add
// (mul_rn / add_rn), so results are BIT-IDENTICAL to sembench (pinned through
// the oracle, tests/test_gpu_parity.py).  One thread per point, consecutive
// threads on consecutive i: every global access is coalesced.
#include "sem_common.cuh"

namespace sem {
namespace {

template <int N>
struct DMat {
    double d[N * N];  // D[i][l] row-major (basis.diff); D^T[i][l] = d[l*N+i]
};

constexpr int kVarThreads = 256;

template <int N>
__device__ __forceinline__ void stage(double* dst, const double* src, int count)
{
    for (int q = threadIdx.x; q < count; q += blockDim.x) dst[q] = src[q];
}

// ---- REFERENCE pass 1: ur/us/ut = D u along r / s / t (kernels.py:163-177)
template <int N>
__global__ void __launch_bounds__(kVarThreads)
    ref_deriv_kernel(const double* __restrict__ u, double* __restrict__ ur,
                     double* __restrict__ us, double* __restrict__ ut, const DMat<N> D)
{
    constexpr int NNN = N * N * N;
    __shared__ double su[NNN];
    const int64_t base = (int64_t)blockIdx.x * NNN;
    stage<N>(su, u + base, NNN);
    __syncthreads();
    for (int p = threadIdx.x; p < NNN; p += blockDim.x) {
        const int i = p % N, j = (p / N) % N, k = p / (N * N);
        double ar = 0.0, as = 0.0, at = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) {
            ar = add_rn(ar, mul_rn(D.d[i * N + l], su[(k * N + j) * N + l]));
            as = add_rn(as, mul_rn(D.d[j * N + l], su[(k * N + l) * N + i]));
            at = add_rn(at, mul_rn(D.d[k * N + l], su[(l * N + j) * N + i]));
        }
        ur[base + p] = ar;
        us[base + p] = as;
        ut[base + p] = at;
    }
}

// ---- REFERENCE pass 2: in-place metric combination (kernels.py:179-193)
template <int N>
__global__ void __launch_bounds__(kVarThreads)
    ref_geom_kernel(const double* __restrict__ g, double* __restrict__ ur,
                    double* __restrict__ us, double* __restrict__ ut, int64_t points)
{
    constexpr int NNN = N * N * N;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < points;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = q / NNN;
        const double* ge = g + e * 6 * NNN + (q - e * NNN);
        const double wr = ur[q], ws = us[q], wt = ut[q];
        const double g1 = __ldg(ge), g2 = __ldg(ge + NNN), g3 = __ldg(ge + 2 * NNN);
        const double g4 = __ldg(ge + 3 * NNN), g5 = __ldg(ge + 4 * NNN);
        const double g6 = __ldg(ge + 5 * NNN);
        ur[q] = add_rn(add_rn(mul_rn(g1, wr), mul_rn(g2, ws)), mul_rn(g3, wt));
        us[q] = add_rn(add_rn(mul_rn(g2, wr), mul_rn(g4, ws)), mul_rn(g5, wt));
        ut[q] = add_rn(add_rn(mul_rn(g3, wr), mul_rn(g5, ws)), mul_rn(g6, wt));
    }
}

// ---- REFERENCE pass 3: w = sum_l Dt.. ur + Dt.. us + Dt.. ut, the three
// terms interleaved per l (kernels.py:195-203)
template <int N>
__global__ void __launch_bounds__(kVarThreads)
    ref_transpose_kernel(const double* __restrict__ ur, const double* __restrict__ us,
                         const double* __restrict__ ut, double* __restrict__ w, const DMat<N> Dt)
{
    constexpr int NNN = N * N * N;
    extern __shared__ double sm[];
    double *sr = sm, *ss = sm + NNN, *st = sm + 2 * NNN;
    const int64_t base = (int64_t)blockIdx.x * NNN;
    stage<N>(sr, ur + base, NNN);
    stage<N>(ss, us + base, NNN);
    stage<N>(st, ut + base, NNN);
    __syncthreads();
    for (int p = threadIdx.x; p < NNN; p += blockDim.x) {
        const int i = p % N, j = (p / N) % N, k = p / (N * N);
        double acc = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) {
            acc = add_rn(acc, mul_rn(Dt.d[i * N + l], sr[(k * N + j) * N + l]));
            acc = add_rn(acc, mul_rn(Dt.d[j * N + l], ss[(k * N + l) * N + i]));
            acc = add_rn(acc, mul_rn(Dt.d[k * N + l], st[(l * N + j) * N + i]));
        }
        w[base + p] = acc;
    }
}

// ---- SCRATCH: one element per CTA, both phases in shared memory
// (kernels.py:213-259; phase 2 reads D transposed, sd[l][i])
template <int N>
__global__ void __launch_bounds__(kVarThreads)
    scratch_kernel(const double* __restrict__ u, const double* __restrict__ g,
                   double* __restrict__ w, const DMat<N> D)
{
    constexpr int NNN = N * N * N;
    extern __shared__ double sm[];
    double *su = sm, *sr = sm + NNN, *ss = sm + 2 * NNN, *st = sm + 3 * NNN;
    const int64_t e = blockIdx.x;
    const int64_t base = e * NNN;
    const double* ge = g + e * 6 * NNN;
    stage<N>(su, u + base, NNN);
    __syncthreads();
    for (int p = threadIdx.x; p < NNN; p += blockDim.x) {
        const int i = p % N, j = (p / N) % N, k = p / (N * N);
        double wr = 0.0, ws = 0.0, wt = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) {
            wr = add_rn(wr, mul_rn(D.d[i * N + l], su[(k * N + j) * N + l]));
            ws = add_rn(ws, mul_rn(D.d[j * N + l], su[(k * N + l) * N + i]));
            wt = add_rn(wt, mul_rn(D.d[k * N + l], su[(l * N + j) * N + i]));
        }
        const double g1 = __ldg(ge + p), g2 = __ldg(ge + NNN + p), g3 = __ldg(ge + 2 * NNN + p);
        const double g4 = __ldg(ge + 3 * NNN + p), g5 = __ldg(ge + 4 * NNN + p);
        const double g6 = __ldg(ge + 5 * NNN + p);
        sr[p] = add_rn(add_rn(mul_rn(g1, wr), mul_rn(g2, ws)), mul_rn(g3, wt));
        ss[p] = add_rn(add_rn(mul_rn(g2, wr), mul_rn(g4, ws)), mul_rn(g5, wt));
        st[p] = add_rn(add_rn(mul_rn(g3, wr), mul_rn(g5, ws)), mul_rn(g6, wt));
    }
    __syncthreads();
    for (int p = threadIdx.x; p < NNN; p += blockDim.x) {
        const int i = p % N, j = (p / N) % N, k = p / (N * N);
        double acc = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) {
            acc = add_rn(acc, mul_rn(D.d[l * N + i], sr[(k * N + j) * N + l]));
            acc = add_rn(acc, mul_rn(D.d[l * N + j], ss[(k * N + l) * N + i]));
            acc = add_rn(acc, mul_rn(D.d[l * N + k], st[(l * N + j) * N + i]));
        }
        w[base + p] = acc;
    }
}

template <int N>
DMat<N> load_mat(const double* m)
{
    DMat<N> D;
    for (int q = 0; q < N * N; ++q) D.d[q] = m[q];
    return D;
}

template <int N>
int set_smem(const void* kern, size_t bytes)
{
    if (bytes <= 48 * 1024) return 0;
    cudaError_t err =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    return err == cudaSuccess ? 0 : fail_cuda(err, "ax variant: shared-memory opt-in");
}

template <int N>
int reference_n(const double* u, const double* g, const double* dx, const double* dxt,
                double* ur, double* us, double* ut, double* w, int64_t E, cudaStream_t s)
{
    constexpr int NNN = N * N * N;
    const int64_t points = E * NNN;
    ref_deriv_kernel<N><<<(unsigned)E, kVarThreads, 0, s>>>(u, ur, us, ut, load_mat<N>(dx));
    SEM_CHECK_LAUNCH("sem_ax_reference: derivative pass");
    const int64_t want = (points + kVarThreads - 1) / kVarThreads;
    const int64_t cap = (int64_t)sm_count() * 8;
    ref_geom_kernel<N><<<(unsigned)(want < cap ? want : cap), kVarThreads, 0, s>>>(g, ur, us, ut,
                                                                                  points);
    SEM_CHECK_LAUNCH("sem_ax_reference: geometric pass");
    const size_t smem = 3 * NNN * sizeof(double);
    if (int rc = set_smem<N>((const void*)ref_transpose_kernel<N>, smem)) return rc;
    ref_transpose_kernel<N><<<(unsigned)E, kVarThreads, smem, s>>>(ur, us, ut, w,
                                                                   load_mat<N>(dxt));
    SEM_CHECK_LAUNCH("sem_ax_reference: transpose pass");
    return 0;
}

template <int N>
int scratch_n(const double* u, const double* g, const double* dx, double* w, int64_t E,
              cudaStream_t s)
{
    constexpr int NNN = N * N * N;
    const size_t smem = 4 * NNN * sizeof(double);
    if (int rc = set_smem<N>((const void*)scratch_kernel<N>, smem)) return rc;
    scratch_kernel<N><<<(unsigned)E, kVarThreads, smem, s>>>(u, g, w, load_mat<N>(dx));
    SEM_CHECK_LAUNCH("sem_ax_scratch");
    return 0;
}

}  // namespace
}  // namespace sem

extern "C" int sem_ax_reference(const double* u, const double* g, const double* dx,
                                const double* dxt, double* ur, double* us, double* ut, double* w,
                                int64_t num_elements, int32_t n, sem_stream_t stream)
{
    using namespace sem;
    if (num_elements == 0) return 0;  // nothing to do; empty tensors may carry null pointers
    if (!u || !g || !dx || !dxt || !ur || !us || !ut || !w || num_elements < 0) {
        set_error("sem_ax_reference: null pointer or negative element count");
        return SEM_E_INVALID;
    }
    if (num_elements > 0x7fffffff) {
        set_error("sem_ax_reference: %lld elements exceed the grid limit",
                  (long long)num_elements);
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    if (num_elements == 0) return 0;
    switch (n) {
#define SEM_REF_CASE(NV) \
    case NV: return reference_n<NV>(u, g, dx, dxt, ur, us, ut, w, num_elements, s);
        SEM_REF_CASE(2) SEM_REF_CASE(3) SEM_REF_CASE(4) SEM_REF_CASE(5) SEM_REF_CASE(6)
        SEM_REF_CASE(7) SEM_REF_CASE(8) SEM_REF_CASE(9) SEM_REF_CASE(10) SEM_REF_CASE(11)
        SEM_REF_CASE(12) SEM_REF_CASE(13) SEM_REF_CASE(14) SEM_REF_CASE(15) SEM_REF_CASE(16)
#undef SEM_REF_CASE
        default:
            set_error("sem_ax_reference: n=%d outside the supported range [2, 16]", n);
            return SEM_E_INVALID;
    }
}

extern "C" int sem_ax_scratch(const double* u, const double* g, const double* dx, double* w,
                              int64_t num_elements, int32_t n, sem_stream_t stream)
{
    using namespace sem;
    if (num_elements == 0) return 0;  // nothing to do; empty tensors may carry null pointers
    if (!u || !g || !dx || !w || num_elements < 0) {
        set_error("sem_ax_scratch: null pointer or negative element count");
        return SEM_E_INVALID;
    }
    if (num_elements > 0x7fffffff) {
        set_error("sem_ax_scratch: %lld elements exceed the grid limit", (long long)num_elements);
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    if (num_elements == 0) return 0;
    switch (n) {
#define SEM_SCR_CASE(NV) \
    case NV: return scratch_n<NV>(u, g, dx, w, num_elements, s);
        SEM_SCR_CASE(2) SEM_SCR_CASE(3) SEM_SCR_CASE(4) SEM_SCR_CASE(5) SEM_SCR_CASE(6)
        SEM_SCR_CASE(7) SEM_SCR_CASE(8) SEM_SCR_CASE(9) SEM_SCR_CASE(10)
#undef SEM_SCR_CASE
        default:
            set_error("sem_ax_scratch: n=%d outside [2, %d] (the scratch capacity, "
                      "sembench/kernels.py:448-455)", n, SEM_SCRATCH_MAX_POINTS);
            return SEM_E_INVALID;
    }
}
