// Device-side input builders, bit-identical to the reference's host code.
//
// random_field (sembench/fields.py:42-54) is a counter-based SplitMix64
// stream: value q = 2 * ((mix(seed + q)) >> 11) * 2^-53 - 1, so it can be
// generated in place on the GPU (no multi-GB host build + H2D at E=32768).
// build_geom (sembench/mesh.py:72-91) for the affine box map is
// g1 = g4 = g6 = ((w_k * w_j) * w_i) * (h / 2), g2 = g3 = g5 = 0.
#include "sem_common.cuh"

namespace sem {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void random_field_kernel(double* __restrict__ out, int64_t count, uint64_t seed)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < count; q += stride) {
        const uint64_t bits = splitmix64(seed + (uint64_t)q);
        const double u01 = __dmul_rn((double)(bits >> 11), 1.0 / 9007199254740992.0);
        out[q] = __dsub_rn(__dmul_rn(2.0, u01), 1.0);
    }
}

struct Weights16 {
    double w[16];
};

__global__ void box_geom_kernel(double* __restrict__ g, int64_t E, int n, Weights16 wt,
                                double half_h)
{
    const int nnn = n * n * n;
    const int64_t total = E * 6 * nnn;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += stride) {
        const int r = (int)(q % nnn);
        const int comp = (int)((q / nnn) % 6);
        double v = 0.0;
        if (comp == 0 || comp == 3 || comp == 5) {
            const int k = r / (n * n), j = (r / n) % n, i = r % n;
            v = __dmul_rn(__dmul_rn(__dmul_rn(wt.w[k], wt.w[j]), wt.w[i]), half_h);
        }
        g[q] = v;
    }
}

}  // namespace sem

extern "C" int sem_random_field(double* out, int64_t count, uint64_t seed, sem_stream_t stream)
{
    if (!out || count < 0) {
        sem::set_error("sem_random_field: bad arguments");
        return SEM_E_INVALID;
    }
    if (count == 0) return 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = sem::bind_stream_device(s)) return rc;
    const int64_t want = (count + 255) / 256;
    const unsigned grid = (unsigned)(want < 32LL * sem::sm_count() ? want : 32LL * sem::sm_count());
    sem::random_field_kernel<<<grid, 256, 0, s>>>(out, count, seed);
    SEM_CHECK_LAUNCH("sem_random_field launch");
    return 0;
}

extern "C" int sem_box_geom(double* g, int64_t num_elements, int32_t n, const double* weights,
                            double extent, sem_stream_t stream)
{
    if (!g || !weights || num_elements < 0 || n < 2 || n > 16) {
        sem::set_error("sem_box_geom: bad arguments");
        return SEM_E_INVALID;
    }
    if (num_elements == 0) return 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = sem::bind_stream_device(s)) return rc;
    sem::Weights16 wt{};
    for (int q = 0; q < n; ++q) wt.w[q] = weights[q];
    const int64_t total = num_elements * 6 * (int64_t)n * n * n;
    const int64_t want = (total + 255) / 256;
    const unsigned grid = (unsigned)(want < 32LL * sem::sm_count() ? want : 32LL * sem::sm_count());
    sem::box_geom_kernel<<<grid, 256, 0, s>>>(g, num_elements, n, wt, extent / 2.0);
    SEM_CHECK_LAUNCH("sem_box_geom launch");
    return 0;
}
