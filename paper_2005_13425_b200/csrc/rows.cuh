// Row-granular box kernels: one thread per (j, k) row of an element.
//
// Along a row only the two end points (i = 0, n-1) can have x-neighbours,
// a non-unit x-multiplicity or a global x-boundary; the y/z copies, the y/z
// mask and the y/z multiplicity are constant over the row.  So the lattice
// arithmetic that the per-point kernels repeated for every point is done
// once per row, the row is moved with 128-bit loads/stores (n even), and
// the ordered dssum gather becomes "add whole source rows in (z, y) order,
// with the x-neighbour scalar spliced in at the two ends" -- the same
// ascending-element order as gather_sum (box.cuh), hence bit-identical.
#pragma once
#include "box.cuh"
#include "flat.cuh"

namespace sem {

#ifndef SEM_ROW_THREADS
#define SEM_ROW_THREADS 128
#endif
constexpr int kRowThreads = SEM_ROW_THREADS;

template <int N>
__device__ __forceinline__ void load_row(const double* __restrict__ p, double (&v)[N])
{
    if constexpr (N % 2 == 0) {
#pragma unroll
        for (int q = 0; q < N / 2; ++q) {
            const double2 t = __ldg(reinterpret_cast<const double2*>(p) + q);
            v[2 * q] = t.x;
            v[2 * q + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] = __ldg(p + i);
    }
}

// plain (cached) loads for fields this kernel also writes
template <int N>
__device__ __forceinline__ void load_row_rw(const double* p, double (&v)[N])
{
    if constexpr (N % 2 == 0) {
#pragma unroll
        for (int q = 0; q < N / 2; ++q) {
            const double2 t = reinterpret_cast<const double2*>(p)[q];
            v[2 * q] = t.x;
            v[2 * q + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] = p[i];
    }
}

template <int N>
__device__ __forceinline__ void store_row(double* p, const double (&v)[N])
{
    if constexpr (N % 2 == 0) {
#pragma unroll
        for (int q = 0; q < N / 2; ++q)
            reinterpret_cast<double2*>(p)[q] = make_double2(v[2 * q], v[2 * q + 1]);
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) p[i] = v[i];
    }
}

// Row descriptor: element coordinates plus everything constant along i.
template <int N>
struct Row {
    int64_t e;
    int jk, j, k;
    ElemCoord c;
    bool yz_inner;   // y and z Dirichlet mask == 1 for this row
    double inv_myz;  // 1 / (y multiplicity * z multiplicity), global lattice
    bool x_lo_in;    // i = 0 is not on the global x boundary (ix > 0)
    bool x_hi_in;    // i = n-1 is not on the global x boundary (ix < ex-1)
};

__device__ __forceinline__ const Box& box_of(const Box& b) { return b; }
__device__ __forceinline__ const Box& box_of(const BoxFlat& bf) { return bf.b; }
__device__ __forceinline__ ElemCoord elem_coord_of(int64_t e, const Box& b) { return elem_coord(e, b); }
// magic-number division (no 64-bit divide on the row's critical path)
__device__ __forceinline__ ElemCoord elem_coord_of(int64_t e, const BoxFlat& bf)
{
    return elem_coord_fast((uint32_t)e, bf);
}

template <int N, class BoxT>
__device__ __forceinline__ Row<N> make_row(int64_t row, const BoxT& bt)
{
    constexpr int NN = N * N;
    const Box& b = box_of(bt);
    Row<N> r;
    r.e = row / NN;
    r.jk = (int)(row - r.e * NN);
    r.k = r.jk / N;
    r.j = r.jk - r.k * N;
    r.c = elem_coord_of(r.e, bt);
    const int gz = r.c.iz + b.gz0;
    r.yz_inner = axis_interior<N>(r.c.iy, r.j, b.ey) && axis_interior<N>(gz, r.k, b.ez_global);
    const int m = axis_mult<N>(r.c.iy, r.j, b.ey) * axis_mult<N>(gz, r.k, b.ez_global);
    r.inv_myz = m == 1 ? 1.0 : (m == 2 ? 0.5 : 0.25);
    r.x_lo_in = r.c.ix > 0;
    r.x_hi_in = r.c.ix < b.ex - 1;
    return r;
}

// 1/multiplicity and mask of point i of the row (x factor only at the ends)
template <int N>
__device__ __forceinline__ double row_inv_mult(const Row<N>& r, int i)
{
    if ((i == 0 && r.x_lo_in) || (i == N - 1 && r.x_hi_in)) return 0.5 * r.inv_myz;
    return r.inv_myz;
}

template <int N>
__device__ __forceinline__ double row_mask(const Row<N>& r, int i)
{
    if (!r.yz_inner) return 0.0;
    if ((i == 0 && !r.x_lo_in) || (i == N - 1 && !r.x_hi_in)) return 0.0;
    return 1.0;
}

// Ordered dssum of one row: sources (z outer, y inner) in ascending element
// order; at i = 0 the x-lower copy (element ix-1, i = n-1) precedes the own
// copy, at i = n-1 the x-upper copy (element ix+1, i = 0) follows it.
// Faces shared with another rank (DIST) come from the halo planes.
template <int N>
__device__ __forceinline__ void dssum_row(const double* __restrict__ f, const Row<N>& r,
                                          const Box& b, const double* __restrict__ bot,
                                          const double* __restrict__ top, double (&v)[N])
{
    constexpr int NNN = N * N * N;
    const double* plane = nullptr;
    if (bot != nullptr && r.c.iz == 0 && r.k == 0) plane = bot;
    if (top != nullptr && r.c.iz == b.ez - 1 && r.k == N - 1) plane = top;
    if (plane != nullptr) {
        const int nx = b.ex * (N - 1) + 1;
        const double* pr = plane + (int64_t)(r.c.iy * (N - 1) + r.j) * nx + r.c.ix * (N - 1);
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] = __ldg(pr + i);
        return;
    }
    const AxisCopies ay = axis_copies<N>(r.c.iy, r.j, b.ey);
    const AxisCopies az = axis_copies<N>(r.c.iz, r.k, b.ez);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = 0.0;
#pragma unroll
    for (int zc = 0; zc < 2; ++zc) {
        if (zc >= az.cnt) break;
        const int ez_ = zc ? az.e1 : az.e0, kk = zc ? az.l1 : az.l0;
#pragma unroll
        for (int yc = 0; yc < 2; ++yc) {
            if (yc >= ay.cnt) break;
            const int ey_ = yc ? ay.e1 : ay.e0, jj = yc ? ay.l1 : ay.l0;
            const int64_t e2 = ((int64_t)ez_ * b.ey + ey_) * b.ex + r.c.ix;
            const double* src = f + e2 * NNN + (kk * N + jj) * N;
            double s[N];
            load_row<N>(src, s);
            const double lo = r.x_lo_in ? __ldg(src - NNN + (N - 1)) : 0.0;
            const double hi = r.x_hi_in ? __ldg(src + NNN) : 0.0;
            v[0] = r.x_lo_in ? add_rn(add_rn(v[0], lo), s[0]) : add_rn(v[0], s[0]);
#pragma unroll
            for (int i = 1; i < N - 1; ++i) v[i] = add_rn(v[i], s[i]);
            v[N - 1] = r.x_hi_in ? add_rn(add_rn(v[N - 1], s[N - 1]), hi)
                                 : add_rn(v[N - 1], s[N - 1]);
        }
    }
}

}  // namespace sem
