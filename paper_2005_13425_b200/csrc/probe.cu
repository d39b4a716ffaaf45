// Streaming-copy bandwidth probe: the device analog of the reference's
// `_stream_copy` (sembench/perf.py:156-159, dst[i] = src[i]) that
// measure_bandwidth times to anchor the paper's measured roofline (§V).
//
// HBM-bound by construction: 16 B per thread per step as two-double vectors
// (ld.global.nc.v2 / st.global.cs.v2 -- the destination is streamed, not
// kept in L2), 4 independent vectors in flight per thread per iteration, a
// grid of (SM count x 8) CTAs of 256 threads striding over the buffer.
#include "sem_common.cuh"

namespace sem {
namespace {

constexpr int kCopyThreads = 256;
constexpr int kCopyUnroll = 4;

__global__ void __launch_bounds__(kCopyThreads)
    stream_copy_kernel(double2* __restrict__ dst, const double2* __restrict__ src, int64_t nvec)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; q + (kCopyUnroll - 1) * stride < nvec; q += kCopyUnroll * stride) {
        double2 v[kCopyUnroll];
#pragma unroll
        for (int r = 0; r < kCopyUnroll; ++r) v[r] = __ldcs(src + q + r * stride);
#pragma unroll
        for (int r = 0; r < kCopyUnroll; ++r) __stcs(dst + q + r * stride, v[r]);
    }
    for (; q < nvec; q += stride) __stcs(dst + q, __ldcs(src + q));
}

__global__ void copy_tail_kernel(double* __restrict__ dst, const double* __restrict__ src,
                                 int64_t from, int64_t count)
{
    const int64_t q = from + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q < count) dst[q] = src[q];
}

}  // namespace
}  // namespace sem

extern "C" int sem_stream_copy(double* dst, const double* src, int64_t count, sem_stream_t stream)
{
    using namespace sem;
    if (!dst || !src || count < 0) {
        set_error("sem_stream_copy: bad arguments");
        return SEM_E_INVALID;
    }
    if (count == 0) return 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    const bool aligned = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) &
                          15) == 0;
    const int64_t nvec = aligned ? count / 2 : 0;
    if (nvec > 0) {
        const int64_t want = (nvec + kCopyThreads - 1) / kCopyThreads;
        const int64_t cap = 8LL * sm_count();
        stream_copy_kernel<<<(unsigned)(want < cap ? want : cap), kCopyThreads, 0, s>>>(
            reinterpret_cast<double2*>(dst), reinterpret_cast<const double2*>(src), nvec);
        SEM_CHECK_LAUNCH("sem_stream_copy");
    }
    const int64_t rest = count - 2 * nvec;
    if (rest > 0) {
        const int64_t blocks = (rest + 255) / 256;
        if (blocks > 0x7fffffff) {
            set_error("sem_stream_copy: misaligned buffers too large");
            return SEM_E_INVALID;
        }
        copy_tail_kernel<<<(unsigned)blocks, 256, 0, s>>>(dst, src, 2 * nvec, count);
        SEM_CHECK_LAUNCH("sem_stream_copy tail");
    }
    return 0;
}
