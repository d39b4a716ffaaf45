// Flat (fully coalesced) traversal of box fields for the streaming kernels.
//
// Thread q handles the point pair (2q, 2q+1) (n even: a pair never crosses a
// row, so it is one 128-bit load/store per field); its element is 2q / n^3
// (constant divisor) and the element's lattice coordinate uses precomputed
// magic-number division (FastDiv), so the only per-point lattice work left
// is the separable mask / multiplicity factor of (i, j, k).
#pragma once
#include "box.cuh"

namespace sem {

// n / d for 0 <= n < 2^31 by multiply-high (round-up method): q = (hi(n*m) + n) >> s
struct FastDiv {
    uint32_t d, m, s;
};

inline FastDiv make_fastdiv(uint32_t d)
{
    uint32_t s = 0;
    while ((uint64_t(1) << s) < d) ++s;
    const uint64_t m = ((uint64_t(1) << 32) * ((uint64_t(1) << s) - d)) / d + 1;
    return FastDiv{d, (uint32_t)m, s};
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f)
{
    return (__umulhi(n, f.m) + n) >> f.s;
}

struct BoxFlat {
    Box b;
    FastDiv fx;   // divide by ex
    FastDiv fxy;  // divide by ex*ey
};

inline BoxFlat make_box_flat(const Box& b)
{
    return BoxFlat{b, make_fastdiv((uint32_t)b.ex), make_fastdiv((uint32_t)(b.ex * b.ey))};
}

__device__ __forceinline__ ElemCoord elem_coord_fast(uint32_t e, const BoxFlat& bf)
{
    ElemCoord c;
    c.iz = (int)fdiv(e, bf.fxy);
    const uint32_t rem = e - (uint32_t)c.iz * bf.fxy.d;
    c.iy = (int)fdiv(rem, bf.fx);
    c.ix = (int)(rem - (uint32_t)c.iy * bf.fx.d);
    return c;
}

// separable lattice factors (global lattice along z)
template <int N>
__device__ __forceinline__ double inv_mult_of(const ElemCoord& c, int i, int j, int k, const Box& b)
{
    const int m = axis_mult<N>(c.ix, i, b.ex) * axis_mult<N>(c.iy, j, b.ey) *
                  axis_mult<N>(c.iz + b.gz0, k, b.ez_global);
    return m == 1 ? 1.0 : (m == 2 ? 0.5 : (m == 4 ? 0.25 : 0.125));
}

template <int N>
__device__ __forceinline__ double mask_of(const ElemCoord& c, int i, int j, int k, const Box& b)
{
    return (axis_interior<N>(c.ix, i, b.ex) && axis_interior<N>(c.iy, j, b.ey) &&
            axis_interior<N>(c.iz + b.gz0, k, b.ez_global))
               ? 1.0
               : 0.0;
}

// Per-pair context: point q0 = 2*qp (n even) or q0 = qp (n odd, NP = 1).
template <int N>
struct PairCfg {
    static constexpr int NP = (N % 2 == 0) ? 2 : 1;  // points per thread
    static constexpr int THREADS = 256;
};

template <int N>
__device__ __forceinline__ void pair_point(int64_t q0, const BoxFlat& bf, ElemCoord& c, int& i,
                                           int& j, int& k)
{
    constexpr int NN = N * N, NNN = N * N * N;
    const uint32_t e = (uint32_t)(q0 / NNN);
    const int r = (int)(q0 - (int64_t)e * NNN);
    k = r / NN;
    j = (r - k * NN) / N;
    i = r - k * NN - j * N;
    c = elem_coord_fast(e, bf);
}

template <int N>
__device__ __forceinline__ void ld_pair(const double* p, double (&v)[PairCfg<N>::NP])
{
    if constexpr (PairCfg<N>::NP == 2) {
        const double2 t = __ldg(reinterpret_cast<const double2*>(p));
        v[0] = t.x;
        v[1] = t.y;
    } else {
        v[0] = __ldg(p);
    }
}

template <int N>
__device__ __forceinline__ void ld_pair_rw(const double* p, double (&v)[PairCfg<N>::NP])
{
    if constexpr (PairCfg<N>::NP == 2) {
        const double2 t = *reinterpret_cast<const double2*>(p);
        v[0] = t.x;
        v[1] = t.y;
    } else {
        v[0] = *p;
    }
}

template <int N>
__device__ __forceinline__ void st_pair(double* p, const double (&v)[PairCfg<N>::NP])
{
    if constexpr (PairCfg<N>::NP == 2)
        *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    else
        *p = v[0];
}

// grid for the flat kernels: a function of E and n only (reproducible trees)
template <int N>
static unsigned flat_grid(int64_t E, int cap)
{
    const int64_t units = E * N * N * N / PairCfg<N>::NP;
    const int64_t blocks = (units + PairCfg<N>::THREADS - 1) / PairCfg<N>::THREADS;
    return (unsigned)(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

}  // namespace sem
