// Direct-stiffness summation (dssum) and Dirichlet mask on a structured box.
//
// Reference: sembench/assembly.py:113-129.  dssum there is
//     acc = np.bincount(global_id, weights=f); out = acc[global_id]
// i.e. every class of coincident nodes is summed in ASCENDING LOCAL INDEX
// order starting from +0.0.  Each element holds at most one copy of a global
// node, so ascending local index == ascending element id, which on the box
// is lexicographic (iz, iy, ix).  This kernel gathers the (1, 2, 4 or 8)
// copies of each point in exactly that order, so its output is bit-identical
// to the reference -- including the +0.0 start (a lone -0.0 becomes +0.0).
//
// Out-of-place, one CTA per element (grid-stride), threads over the n^3
// points so the own-copy read and the write are coalesced; neighbour copies
// are L2 hits.  The global lattice (ids, multiplicity, mask) is recomputed
// from coordinates, so no index array is read.
#include "box.cuh"
#include "reduce.cuh"
#include "cols.cuh"

namespace sem {


// MASK: multiply by the 0/1 mask (reference mask() is f*mask).
template <int N, bool MASK>
__global__ void __launch_bounds__(ColCfg<N>::THREADS)
dssum_box_kernel(const double* __restrict__ f, double* __restrict__ out, int64_t E, Box b,
                 const double* __restrict__ bot, const double* __restrict__ top)
{
    constexpr int NN = N * N, NNN = N * N * N;
    col_loop<N>(E, b, [&](int64_t e, const ElemCoord& c, const ColXY<N>& t) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
            double s = col_dssum<N>(f, t, c, k, b, bot, top);
            if (MASK) s = mul_rn(s, col_mask<N>(t, c, k, b));
            out[e * NNN + k * NN + t.p] = s;
        }
    });
}

template <int N>
__global__ void __launch_bounds__(ColCfg<N>::THREADS)
mask_box_kernel(const double* __restrict__ f, double* __restrict__ out, int64_t E, Box b)
{
    constexpr int NN = N * N, NNN = N * N * N;
    col_loop<N>(E, b, [&](int64_t e, const ElemCoord& c, const ColXY<N>& t) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const int64_t idx = e * NNN + k * NN + t.p;
            out[idx] = mul_rn(__ldg(f + idx), col_mask<N>(t, c, k, b));
        }
    });
}

template <int N>
static unsigned box_grid(int64_t E)
{
    return col_grid<N>(E, 16 * sm_count());
}

template <int N>
static int launch_dssum(const double* f, double* out, int64_t E, Box b, bool mask,
                        cudaStream_t s, const double* bot = nullptr, const double* top = nullptr)
{
    if (E == 0) return 0;
    if (mask)
        dssum_box_kernel<N, true><<<box_grid<N>(E), ColCfg<N>::THREADS, 0, s>>>(f, out, E, b, bot, top);
    else
        dssum_box_kernel<N, false><<<box_grid<N>(E), ColCfg<N>::THREADS, 0, s>>>(f, out, E, b, bot, top);
    SEM_CHECK_LAUNCH("sem_dssum_box launch");
    return 0;
}

template <int N>
static int launch_mask(const double* f, double* out, int64_t E, Box b, cudaStream_t s)
{
    if (E == 0) return 0;
    mask_box_kernel<N><<<box_grid<N>(E), ColCfg<N>::THREADS, 0, s>>>(f, out, E, b);
    SEM_CHECK_LAUNCH("sem_mask_box launch");
    return 0;
}

int check_box(int ex, int ey, int ez, int n, const char* who)
{
    if (ex < 1 || ey < 1 || ez < 1) {
        set_error("%s: element counts must be positive (got %d x %d x %d)", who, ex, ey, ez);
        return SEM_E_INVALID;
    }
    if (n < 2 || n > 16) {
        set_error("%s: n=%d outside the supported range [2, 16]", who, n);
        return SEM_E_INVALID;
    }
    return 0;
}

int dssum_box(const double* f, double* out, int ex, int ey, int ez, int n, bool mask,
              cudaStream_t s)
{
    const Box b{ex, ey, ez, 0, ez};
    const int64_t E = (int64_t)ex * ey * ez;
    SEM_SWITCH_N(n, return launch_dssum<NV>(f, out, E, b, mask, s));
}

int mask_box(const double* f, double* out, int ex, int ey, int ez, int n, cudaStream_t s)
{
    const Box b{ex, ey, ez, 0, ez};
    const int64_t E = (int64_t)ex * ey * ez;
    SEM_SWITCH_N(n, return launch_mask<NV>(f, out, E, b, s));
}

int dssum_slab(const double* f, double* out, const double* bot, const double* top, const Box& b,
               int n, bool mask, cudaStream_t s)
{
    const int64_t E = (int64_t)b.ex * b.ey * b.ez;
    SEM_SWITCH_N(n, return launch_dssum<NV>(f, out, E, b, mask, s, bot, top));
}

int mask_slab(const double* f, double* out, const Box& b, int n, cudaStream_t s)
{
    const int64_t E = (int64_t)b.ex * b.ey * b.ez;
    SEM_SWITCH_N(n, return launch_mask<NV>(f, out, E, b, s));
}

int ax_dispatch(const double* u, const double* g, const double* dx, double* w, int64_t E,
                int n, int variant, cudaStream_t stream);

}  // namespace sem

extern "C" int sem_dssum_box(const double* f, double* out, int32_t ex, int32_t ey,
                             int32_t ez, int32_t n, int32_t apply_mask, sem_stream_t stream)
{
    if (int rc = sem::check_box(ex, ey, ez, n, "sem_dssum_box")) return rc;
    if (!f || !out || f == out) {
        sem::set_error("sem_dssum_box: null pointer or in-place call (out must differ from f)");
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = sem::bind_stream_device(s)) return rc;
    return sem::dssum_box(f, out, ex, ey, ez, n, apply_mask != 0, s);
}

extern "C" int sem_mask_box(const double* f, double* out, int32_t ex, int32_t ey, int32_t ez,
                            int32_t n, sem_stream_t stream)
{
    if (int rc = sem::check_box(ex, ey, ez, n, "sem_mask_box")) return rc;
    if (!f || !out) {
        sem::set_error("sem_mask_box: null pointer");
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = sem::bind_stream_device(s)) return rc;
    return sem::mask_box(f, out, ex, ey, ez, n, s);
}

extern "C" int sem_apply_global(const double* u, const double* g, const double* dx,
                                const double* dxt, double* w, double* scratch, int32_t ex,
                                int32_t ey, int32_t ez, int32_t n, sem_stream_t stream)
{
    if (int rc = sem::check_box(ex, ey, ez, n, "sem_apply_global")) return rc;
    if (!u || !g || !dx || !dxt || !w || !scratch || w == scratch || u == w) {
        sem::set_error("sem_apply_global: null or aliasing pointers");
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = sem::bind_stream_device(s)) return rc;
    const int64_t E = (int64_t)ex * ey * ez;
    // mask(u) -> w ; A_local -> scratch ; mask(dssum(scratch)) -> w
    if (int rc = sem::mask_box(u, w, ex, ey, ez, n, s)) return rc;
    if (int rc = sem::ax_dispatch(w, g, dx, scratch, E, n, 0, s)) return rc;
    return sem::dssum_box(scratch, w, ex, ey, ez, n, true, s);
}
