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
                int n, int variant, cudaStream_t stream, int pdl = -1);

}  // namespace sem

extern "C" int sem_dssum_box(const double* f, double* out, int32_t ex, int32_t ey,
                             int32_t ez, int32_t n, int32_t apply_mask, sem_stream_t stream)
{
    if (int rc = sem::check_box(ex, ey, ez, n, "sem_dssum_box")) return rc;
    if (!f || !out || f == out) {
        sem::set_error("sem_dssum_box: null pointer or in-place call (out must differ from f)");
        return SEM_E_INVALID;
    }
    if (int rc = sem::check_fields_aligned("sem_dssum_box", n, nullptr, {f, out})) return rc;
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
    if (int rc = sem::check_fields_aligned("sem_mask_box", n, nullptr, {f, out})) return rc;
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

// ------------------------------------------------------------------------
// General numbering: the reference's dssum for ANY Topology.global_id
// (sembench/assembly.py:113-120), not just the box lattice.  The host builds
// a CSR of the id classes once per topology: seg_idx lists local flat
// indices grouped by global id, each group in ascending local index (a stable
// argsort of global_id), seg_off[s]..seg_off[s+1] delimits group s.  One
// thread per class sums its copies in that order from +0.0 -- np.bincount's
// order -- and scatters the total back to every copy: bit-identical for any
// numbering.  Not the hot path (the box kernels above are): indices are read
// coalesced, the f gathers / out scatters follow the caller's numbering.
namespace sem {

__global__ void __launch_bounds__(256)
dssum_csr_kernel(const double* __restrict__ f, double* __restrict__ out,
                 const int32_t* __restrict__ off, const int32_t* __restrict__ idx, int64_t nseg)
{
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nseg;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t b = off[s], e = off[s + 1];
        double acc = 0.0;
        for (int32_t q = b; q < e; ++q) acc = add_rn(acc, f[idx[q]]);
        for (int32_t q = b; q < e; ++q) out[idx[q]] = acc;
    }
}

__global__ void __launch_bounds__(256)
mask_array_kernel(const double* __restrict__ f, const double* __restrict__ m,
                  double* __restrict__ out, int64_t count)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < count;
         q += (int64_t)gridDim.x * blockDim.x)
        out[q] = mul_rn(f[q], m[q]);
}

static unsigned flat_blocks(int64_t count)
{
    const int64_t blocks = (count + 255) / 256;
    const int64_t cap = 16LL * sm_count();
    return (unsigned)(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

}  // namespace sem

extern "C" int sem_dssum_csr(const double* f, double* out, const int32_t* seg_off,
                             const int32_t* seg_idx, int64_t nseg, sem_stream_t stream)
{
    if (nseg < 0 || (nseg > 0 && (!f || !out || !seg_off || !seg_idx)) ||
        (nseg > 0 && f == out)) {
        sem::set_error("sem_dssum_csr: null pointer, negative count or in-place call");
        return SEM_E_INVALID;
    }
    if (nseg == 0) return 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = sem::bind_stream_device(s)) return rc;
    sem::dssum_csr_kernel<<<sem::flat_blocks(nseg), 256, 0, s>>>(f, out, seg_off, seg_idx, nseg);
    SEM_CHECK_LAUNCH("sem_dssum_csr launch");
    return 0;
}

extern "C" int sem_mask_array(const double* f, const double* mask, double* out, int64_t count,
                              sem_stream_t stream)
{
    if (count < 0 || (count > 0 && (!f || !mask || !out))) {
        sem::set_error("sem_mask_array: null pointer or negative count");
        return SEM_E_INVALID;
    }
    if (count == 0) return 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = sem::bind_stream_device(s)) return rc;
    sem::mask_array_kernel<<<sem::flat_blocks(count), 256, 0, s>>>(f, mask, out, count);
    SEM_CHECK_LAUNCH("sem_mask_array launch");
    return 0;
}

// ------------------------------------------------------------------------
// Interface consistency of mask(f) on the box: every copy of a shared,
// unmasked node holds the same value.  The fused CG computes <p, A p> as the
// element-local sum  sum_e p_e . (A_e p_e), which equals the reference's
// <p, mask(dssum(A p))>_c (cg.py:163) only for a continuous p; p inherits
// continuity from r = mask(f).  cg_solve runs this check once and takes the
// generic (assembled) path when it fails.  Each row compares its own values
// with every other copy (the same neighbour walk as dssum_row); equality is
// transitive, so checking each point against all its copies is complete.
namespace sem {

template <int N>
__global__ void __launch_bounds__(kRowThreads)
consistent_box_kernel(const double* __restrict__ f, int64_t E, Box b, int32_t* __restrict__ bad)
{
    constexpr int NN = N * N, NNN = N * N * N;
    bool ok = true;
    for (int64_t row = (int64_t)blockIdx.x * kRowThreads + threadIdx.x; row < E * NN;
         row += (int64_t)gridDim.x * kRowThreads) {
        const Row<N> r = make_row<N>(row, b);
        if (!r.yz_inner) continue;  // the whole row is masked: zero in every copy
        double own[N];
        load_row<N>(f + r.e * NNN + r.jk * N, own);
        const AxisCopies ay = axis_copies<N>(r.c.iy, r.j, b.ey);
        const AxisCopies az = axis_copies<N>(r.c.iz, r.k, b.ez);
        for (int zc = 0; zc < az.cnt; ++zc) {
            const int ez_ = zc ? az.e1 : az.e0, kk = zc ? az.l1 : az.l0;
            for (int yc = 0; yc < ay.cnt; ++yc) {
                const int ey_ = yc ? ay.e1 : ay.e0, jj = yc ? ay.l1 : ay.l0;
                const int64_t e2 = ((int64_t)ez_ * b.ey + ey_) * b.ex + r.c.ix;
                const double* src = f + e2 * NNN + (kk * N + jj) * N;
                double s[N];
                load_row<N>(src, s);
#pragma unroll
                for (int i = 0; i < N; ++i)
                    if (row_mask<N>(r, i) != 0.0 && s[i] != own[i]) ok = false;
                // the x-neighbour copies of the row's end points
                if (r.x_lo_in && __ldg(src - NNN + (N - 1)) != own[0]) ok = false;
                if (r.x_hi_in && __ldg(src + NNN) != own[N - 1]) ok = false;
            }
        }
    }
    if (!ok) atomicOr(bad, 1);
}

}  // namespace sem

namespace sem {
static int consistent_box(const double* f, int ex, int ey, int ez, int n, int32_t* flag,
                          cudaStream_t s)
{
    const Box b{ex, ey, ez, 0, ez};
    const int64_t E = (int64_t)ex * ey * ez;
    SEM_SWITCH_N(n, {
        consistent_box_kernel<NV><<<box_grid<NV>(E), kRowThreads, 0, s>>>(f, E, b, flag);
        SEM_CHECK_LAUNCH("sem_consistent_box launch");
        return 0;
    });
}
}  // namespace sem

extern "C" int sem_consistent_box(const double* f, int32_t ex, int32_t ey, int32_t ez, int32_t n,
                                  int32_t* flag_dev, sem_stream_t stream)
{
    if (int rc = sem::check_box(ex, ey, ez, n, "sem_consistent_box")) return rc;
    if (!f || !flag_dev) {
        sem::set_error("sem_consistent_box: null pointer");
        return SEM_E_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = sem::bind_stream_device(s)) return rc;
    cudaError_t err = cudaMemsetAsync(flag_dev, 0, sizeof(int32_t), s);
    if (err != cudaSuccess) return sem::fail_cuda(err, "sem_consistent_box: memset");
    return sem::consistent_box(f, ex, ey, ez, n, flag_dev, s);
}
