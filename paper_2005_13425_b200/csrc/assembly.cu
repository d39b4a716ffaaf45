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
#include "flat.cuh"
#include "rows.cuh"

namespace sem {


// MASK: multiply by the 0/1 mask (reference mask() is f*mask).
template <int N, bool MASK>
__global__ void __launch_bounds__(kRowThreads)
dssum_box_kernel(const double* __restrict__ f, double* __restrict__ out, int64_t E, Box b,
                 const double* __restrict__ bot, const double* __restrict__ top)
{
    constexpr int NN = N * N, NNN = N * N * N;
    for (int64_t row = (int64_t)blockIdx.x * kRowThreads + threadIdx.x; row < E * NN;
         row += (int64_t)gridDim.x * kRowThreads) {
        const Row<N> r = make_row<N>(row, b);
        double v[N];
        dssum_row<N>(f, r, b, bot, top, v);
        if (MASK) {
#pragma unroll
            for (int i = 0; i < N; ++i) v[i] = mul_rn(v[i], row_mask<N>(r, i));
        }
        store_row<N>(out + r.e * NNN + r.jk * N, v);
    }
}

template <int N>
__global__ void __launch_bounds__(PairCfg<N>::THREADS)
mask_box_kernel(const double* __restrict__ f, double* __restrict__ out, int64_t E, BoxFlat bf)
{
    constexpr int NP = PairCfg<N>::NP;
    const int64_t units = E * (int64_t)(N * N * N) / NP;
    for (int64_t u = (int64_t)blockIdx.x * PairCfg<N>::THREADS + threadIdx.x; u < units;
         u += (int64_t)gridDim.x * PairCfg<N>::THREADS) {
        const int64_t q0 = u * NP;
        ElemCoord c;
        int i, j, k;
        pair_point<N>(q0, bf, c, i, j, k);
        double v[NP];
        ld_pair<N>(f + q0, v);
#pragma unroll
        for (int h = 0; h < NP; ++h) v[h] = mul_rn(v[h], mask_of<N>(c, i + h, j, k, bf.b));
        st_pair<N>(out + q0, v);
    }
}

template <int N>
static unsigned box_grid(int64_t E)
{
    const int64_t blocks = (E * N * N + kRowThreads - 1) / kRowThreads;
    const int64_t cap = 16LL * sm_count();
    return (unsigned)(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

template <int N>
static int launch_dssum(const double* f, double* out, int64_t E, Box b, bool mask,
                        cudaStream_t s, const double* bot = nullptr, const double* top = nullptr)
{
    if (E == 0) return 0;
    if (mask)
        dssum_box_kernel<N, true><<<box_grid<N>(E), kRowThreads, 0, s>>>(f, out, E, b, bot, top);
    else
        dssum_box_kernel<N, false><<<box_grid<N>(E), kRowThreads, 0, s>>>(f, out, E, b, bot, top);
    SEM_CHECK_LAUNCH("sem_dssum_box launch");
    return 0;
}

template <int N>
static int launch_mask(const double* f, double* out, int64_t E, Box b, cudaStream_t s)
{
    if (E == 0) return 0;
    mask_box_kernel<N><<<flat_grid<N>(E, 16 * sm_count()), PairCfg<N>::THREADS, 0, s>>>(
        f, out, E, make_box_flat(b));
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
