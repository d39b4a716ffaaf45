// Column-mapped box kernels: thread p = (j, i) of an element walks k.
//
// Every k-layer of an element is n^2 contiguous doubles, so threads p = 0..
// n^2-1 read and write each layer fully coalesced.  The lattice quantities
// are separable -- mask(i,j,k) = mx(i) my(j) mz(k), 1/mult = wx(i) wy(j)
// wz(k) -- so the (i, j) factors are per-thread constants and the k factor a
// per-element constant, and the ordered dssum gather needs neighbour copies
// only for threads on an element edge (x/y) or at k = 0, n-1 (z); a thread in
// the interior of the (i,j) face does one load per point.  The gather order
// is z-choice outer, y middle, x inner = ascending element id, i.e. the
// reference's bincount order (sembench/assembly.py:116), bit-identical.
#pragma once
#include "box.cuh"

namespace sem {

template <int N>
struct ColCfg {
    static constexpr int NN = N * N;
    static constexpr int THREADS = NN <= 128 ? 128 : 256;
    static constexpr int EPB = THREADS / NN;  // elements per block iteration
};

// per-thread (i, j) constants for one element
template <int N>
struct ColXY {
    int p, i, j;
    AxisCopies ax, ay;
    bool mxy;       // x and y Dirichlet mask
    double wxy;     // x and y inverse multiplicity
};

template <int N>
__device__ __forceinline__ ColXY<N> col_xy(int p, const ElemCoord& c, const Box& b)
{
    ColXY<N> t;
    t.p = p;
    t.j = p / N;
    t.i = p - t.j * N;
    t.ax = axis_copies<N>(c.ix, t.i, b.ex);
    t.ay = axis_copies<N>(c.iy, t.j, b.ey);
    t.mxy = axis_interior<N>(c.ix, t.i, b.ex) && axis_interior<N>(c.iy, t.j, b.ey);
    const int m = axis_mult<N>(c.ix, t.i, b.ex) * axis_mult<N>(c.iy, t.j, b.ey);
    t.wxy = m == 1 ? 1.0 : (m == 2 ? 0.5 : 0.25);
    return t;
}

template <int N>
__device__ __forceinline__ double col_mask(const ColXY<N>& t, const ElemCoord& c, int k,
                                           const Box& b)
{
    return (t.mxy && axis_interior<N>(c.iz + b.gz0, k, b.ez_global)) ? 1.0 : 0.0;
}

template <int N>
__device__ __forceinline__ double col_inv_mult(const ColXY<N>& t, const ElemCoord& c, int k,
                                               const Box& b)
{
    return axis_mult<N>(c.iz + b.gz0, k, b.ez_global) == 2 ? 0.5 * t.wxy : t.wxy;
}

// Ordered dssum of point (i, j, k) (k compile-time in the caller's unrolled
// loop).  Slab faces shared with another rank come from the halo planes.
template <int N>
__device__ __forceinline__ double col_dssum(const double* __restrict__ f, const ColXY<N>& t,
                                            const ElemCoord& c, int k, const Box& b,
                                            const double* __restrict__ bot,
                                            const double* __restrict__ top)
{
    constexpr int NNN = N * N * N;
    if ((bot != nullptr && c.iz == 0 && k == 0) ||
        (top != nullptr && c.iz == b.ez - 1 && k == N - 1)) {
        const double* plane = (c.iz == 0 && k == 0 && bot != nullptr) ? bot : top;
        const int nx = b.ex * (N - 1) + 1;
        return __ldg(plane + (int64_t)(c.iy * (N - 1) + t.j) * nx + (c.ix * (N - 1) + t.i));
    }
    const AxisCopies az = axis_copies<N>(c.iz, k, b.ez);
    double v[8];
    bool ok[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int zc = q >> 2, yc = (q >> 1) & 1, xc = q & 1;
        ok[q] = zc < az.cnt && yc < t.ay.cnt && xc < t.ax.cnt;
        const int ez_ = zc ? az.e1 : az.e0, kk = zc ? az.l1 : az.l0;
        const int ey_ = yc ? t.ay.e1 : t.ay.e0, jj = yc ? t.ay.l1 : t.ay.l0;
        const int ex_ = xc ? t.ax.e1 : t.ax.e0, ii = xc ? t.ax.l1 : t.ax.l0;
        const int64_t e2 = ((int64_t)ez_ * b.ey + ey_) * b.ex + ex_;
        v[q] = ok[q] ? __ldg(f + e2 * NNN + (kk * N + jj) * N + ii) : 0.0;
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
        if (ok[q]) s = add_rn(s, v[q]);
    return s;
}

// Iterate the (element, thread position) pairs of a fixed grid; body(e, c, t)
// runs for active lanes (t.p < n^2).  Inactive lanes just fall through, so
// block-wide reductions after the loop stay uniform.
template <int N, typename F>
__device__ __forceinline__ void col_loop(int64_t E, const Box& b, F&& body)
{
    using CC = ColCfg<N>;
    const int slot = threadIdx.x / CC::NN;
    const int p = threadIdx.x - slot * CC::NN;
    for (int64_t eb = (int64_t)blockIdx.x * CC::EPB; eb < E; eb += (int64_t)gridDim.x * CC::EPB) {
        const int64_t e = eb + slot;
        if (slot < CC::EPB && e < E) {
            const ElemCoord c = elem_coord(e, b);
            const ColXY<N> t = col_xy<N>(p, c, b);
            body(e, c, t);
        }
    }
}

template <int N>
static unsigned col_grid(int64_t E, int cap)
{
    const int64_t blocks = (E + ColCfg<N>::EPB - 1) / ColCfg<N>::EPB;
    return (unsigned)(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

}  // namespace sem
