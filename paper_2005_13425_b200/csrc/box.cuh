// Structured-box lattice arithmetic shared by the assembly and CG kernels.
//
// The reference numbers global nodes by exact integer lattice coordinates
// (sembench/assembly.py:69-110).  On a box every shared node is found from
// its element coordinate and local index alone, so the device kernels never
// read a global_id / multiplicity / mask array: all three are recomputed
// from (ix, iy, iz, i, j, k) in registers.
#pragma once
#include "sem_common.cuh"

namespace sem {

// Element lattice of one field (a whole box, or a z-slab of a larger box).
struct Box {
    int ex, ey, ez;    // elements per axis in this field
    int gz0;           // global z element offset of this slab (0 = whole box)
    int ez_global;     // global elements along z
};

// Copies of a node along one axis: (element coordinate, local index) pairs
// in ascending element order.  cnt = 1 or 2.
struct AxisCopies {
    int cnt;
    int e0, l0, e1, l1;
};

template <int N>
__device__ __forceinline__ AxisCopies axis_copies(int ec, int l, int ecount)
{
    AxisCopies a;
    if (l == 0 && ec > 0) {
        a.cnt = 2; a.e0 = ec - 1; a.l0 = N - 1; a.e1 = ec; a.l1 = 0;
    } else if (l == N - 1 && ec < ecount - 1) {
        a.cnt = 2; a.e0 = ec; a.l0 = N - 1; a.e1 = ec + 1; a.l1 = 0;
    } else {
        a.cnt = 1; a.e0 = ec; a.l0 = l; a.e1 = ec; a.l1 = l;
    }
    return a;
}

// Dirichlet mask (assembly.py:92-97): 1 strictly inside the global grid.
template <int N>
__device__ __forceinline__ bool axis_interior(int ec_global, int l, int ecount_global)
{
    return !((ec_global == 0 && l == 0) || (ec_global == ecount_global - 1 && l == N - 1));
}

// Multiplicity along one axis (1 or 2) -- on the GLOBAL lattice.
template <int N>
__device__ __forceinline__ int axis_mult(int ec_global, int l, int ecount_global)
{
    return ((l == 0 && ec_global > 0) || (l == N - 1 && ec_global < ecount_global - 1)) ? 2 : 1;
}

struct ElemCoord {
    int ix, iy, iz;
};

__device__ __forceinline__ ElemCoord elem_coord(int64_t e, const Box& b)
{
    ElemCoord c;
    const int64_t exy = (int64_t)b.ex * b.ey;
    c.iz = (int)(e / exy);
    const int rem = (int)(e - (int64_t)c.iz * exy);
    c.iy = rem / b.ex;
    c.ix = rem - c.iy * b.ex;
    return c;
}

// Dispatch a runtime n in [2,16] to a compile-time NV.
#define SEM_SWITCH_N(n, ...)                                                          \
    switch (n) {                                                                      \
        case 2: { constexpr int NV = 2; __VA_ARGS__; }                                       \
        case 3: { constexpr int NV = 3; __VA_ARGS__; }                                       \
        case 4: { constexpr int NV = 4; __VA_ARGS__; }                                       \
        case 5: { constexpr int NV = 5; __VA_ARGS__; }                                       \
        case 6: { constexpr int NV = 6; __VA_ARGS__; }                                       \
        case 7: { constexpr int NV = 7; __VA_ARGS__; }                                       \
        case 8: { constexpr int NV = 8; __VA_ARGS__; }                                       \
        case 9: { constexpr int NV = 9; __VA_ARGS__; }                                       \
        case 10: { constexpr int NV = 10; __VA_ARGS__; }                                     \
        case 11: { constexpr int NV = 11; __VA_ARGS__; }                                     \
        case 12: { constexpr int NV = 12; __VA_ARGS__; }                                     \
        case 13: { constexpr int NV = 13; __VA_ARGS__; }                                     \
        case 14: { constexpr int NV = 14; __VA_ARGS__; }                                     \
        case 15: { constexpr int NV = 15; __VA_ARGS__; }                                     \
        case 16: { constexpr int NV = 16; __VA_ARGS__; }                                     \
        default: set_error("n=%d outside the supported range [2, 16]", (int)(n));     \
                 return SEM_E_INVALID;                                                \
    }

int check_box(int ex, int ey, int ez, int n, const char* who);

}  // namespace sem
