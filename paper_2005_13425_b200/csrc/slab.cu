// Multi-GPU z-slab assembly primitives (halo protocol of dist.py).
//
// The global element order e = ix + ex*(iy + ey*iz) makes contiguous element
// ranges z-slabs, so rank r owns global layers [gz0, gz0+ez).  A node on the
// interface plane between ranks r-1 and r has copies in layer gz0-1 (k=n-1,
// rank r-1) and layer gz0 (k=0, rank r); in the reference's bincount order
// (ascending element id, sembench/assembly.py:116) ALL of rank r-1's copies
// come first.  So the reference sum is reproduced bit-for-bit by
//   1. rank r-1: plane_top  = ordered in-plane sum of its copies, from +0.0,
//   2. rank r:   plane_bottom = that prefix continued with its own copies,
//   3. rank r sends the totals back to rank r-1 (its top-face values).
// Planes are indexed gy * (ex*(n-1)+1) + gx on the global x/y lattice.
#include "box.cuh"

namespace sem {

int dssum_slab(const double* f, double* out, const double* bot, const double* top, const Box& b,
               int n, bool mask, cudaStream_t s);
int mask_slab(const double* f, double* out, const Box& b, int n, cudaStream_t s);

// copies of global lattice coordinate gc along one axis: (element, local)
template <int N>
__device__ __forceinline__ AxisCopies lattice_copies(int gc, int ecount)
{
    AxisCopies a;
    const int last = ecount * (N - 1);
    const int q = gc / (N - 1), l = gc - q * (N - 1);
    if (gc == last) {
        a.cnt = 1; a.e0 = ecount - 1; a.l0 = N - 1; a.e1 = a.e0; a.l1 = a.l0;
    } else if (l == 0 && gc > 0) {
        a.cnt = 2; a.e0 = q - 1; a.l0 = N - 1; a.e1 = q; a.l1 = 0;
    } else {
        a.cnt = 1; a.e0 = q; a.l0 = l; a.e1 = q; a.l1 = l;
    }
    return a;
}

template <int N>
__global__ void slab_plane_kernel(const double* __restrict__ f,
                                  const double* __restrict__ prefix, double* __restrict__ out,
                                  int ex, int ey, int layer, int k)
{
    constexpr int NN = N * N, NNN = N * N * N;
    const int nx = ex * (N - 1) + 1, ny = ey * (N - 1) + 1;
    const int64_t total = (int64_t)nx * ny;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += stride) {
        const int gy = (int)(q / nx), gx = (int)(q - (int64_t)gy * nx);
        const AxisCopies ax = lattice_copies<N>(gx, ex);
        const AxisCopies ay = lattice_copies<N>(gy, ey);
        double s = prefix ? __ldg(prefix + q) : 0.0;
#pragma unroll
        for (int yc = 0; yc < 2; ++yc) {
            if (yc >= ay.cnt) break;
            const int iy = yc ? ay.e1 : ay.e0, j = yc ? ay.l1 : ay.l0;
#pragma unroll
            for (int xc = 0; xc < 2; ++xc) {
                if (xc >= ax.cnt) break;
                const int ix = xc ? ax.e1 : ax.e0, i = xc ? ax.l1 : ax.l0;
                const int64_t e = ((int64_t)layer * ey + iy) * ex + ix;
                s = add_rn(s, __ldg(f + e * NNN + k * NN + j * N + i));
            }
        }
        out[q] = s;
    }
}

template <int N>
static int launch_plane(const double* f, const double* prefix, double* out, int ex, int ey,
                        int layer, int k, cudaStream_t s)
{
    const int64_t total = (int64_t)(ex * (N - 1) + 1) * (ey * (N - 1) + 1);
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = 8LL * sm_count();
    if (blocks > cap) blocks = cap;
    slab_plane_kernel<N><<<(unsigned)(blocks > 0 ? blocks : 1), 256, 0, s>>>(f, prefix, out, ex,
                                                                             ey, layer, k);
    SEM_CHECK_LAUNCH("slab plane launch");
    return 0;
}

}  // namespace sem

using namespace sem;

extern "C" int sem_slab_plane_top(const double* f, double* plane, int32_t ex, int32_t ey,
                                  int32_t ez, int32_t n, sem_stream_t stream)
{
    if (int rc = check_box(ex, ey, ez, n, "sem_slab_plane_top")) return rc;
    if (!f || !plane) { set_error("sem_slab_plane_top: null pointer"); return SEM_E_INVALID; }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    SEM_SWITCH_N(n, return launch_plane<NV>(f, nullptr, plane, ex, ey, ez - 1, NV - 1, s));
}

extern "C" int sem_slab_plane_bottom(const double* f, const double* prefix, double* totals,
                                     int32_t ex, int32_t ey, int32_t ez, int32_t n,
                                     sem_stream_t stream)
{
    if (int rc = check_box(ex, ey, ez, n, "sem_slab_plane_bottom")) return rc;
    if (!f || !totals) { set_error("sem_slab_plane_bottom: null pointer"); return SEM_E_INVALID; }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    SEM_SWITCH_N(n, return launch_plane<NV>(f, prefix, totals, ex, ey, 0, 0, s));
}

extern "C" int sem_dssum_slab(const double* f, double* out, const double* bottom_totals,
                              const double* top_totals, int32_t ex, int32_t ey, int32_t ez,
                              int32_t n, int32_t gz0, int32_t ez_global, int32_t apply_mask,
                              sem_stream_t stream)
{
    if (int rc = check_box(ex, ey, ez, n, "sem_dssum_slab")) return rc;
    if (!f || !out || f == out || gz0 < 0 || ez_global < gz0 + ez) {
        set_error("sem_dssum_slab: bad arguments");
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    const Box b{ex, ey, ez, gz0, ez_global};
    return dssum_slab(f, out, bottom_totals, top_totals, b, n, apply_mask != 0, s);
}

extern "C" int sem_mask_slab(const double* f, double* out, int32_t ex, int32_t ey, int32_t ez,
                             int32_t n, int32_t gz0, int32_t ez_global, sem_stream_t stream)
{
    if (int rc = check_box(ex, ey, ez, n, "sem_mask_slab")) return rc;
    if (!f || !out || gz0 < 0 || ez_global < gz0 + ez) {
        set_error("sem_mask_slab: bad arguments");
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    const Box b{ex, ey, ez, gz0, ez_global};
    return mask_slab(f, out, b, n, s);
}
