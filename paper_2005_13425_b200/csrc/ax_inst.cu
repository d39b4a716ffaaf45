// Per-n instantiation of the Ax kernels (ax_impl.cuh).  build.py compiles
// this file once per SEM_AX_GROUP so the heavy unrolled instantiations build
// in parallel; ax.cu dispatches to ax_entry_<n> / ax_cg_entry_<n>.
#include "ax_impl.cuh"

#ifndef SEM_AX_GROUP
#error "compile with -DSEM_AX_GROUP=<0..7>"
#endif

namespace sem {

#define SEM_AX_DEFINE(NV)                                                                    \
    int ax_entry_##NV(const double* u, const double* g, const double* dx, double* w,          \
                      int64_t E, int variant, int pdl, cudaStream_t s)                        \
    {                                                                                         \
        return ax_n<NV>(u, g, dx, w, E, variant, pdl, s);                                     \
    }                                                                                         \
    int ax_cg_entry_##NV(const double* g, const double* dx, double* w, int64_t E,             \
                         CgpArgs a, int mode, cudaStream_t s)                                 \
    {                                                                                         \
        return mode == 3 ? ax_cg_n<NV, 3>(g, dx, w, E, a, s) : ax_cg_n<NV, 2>(g, dx, w, E, a, s); \
    }

// groups balanced by compile cost (grows steeply with n)
#if SEM_AX_GROUP == 0
SEM_AX_DEFINE(16)
#elif SEM_AX_GROUP == 1
SEM_AX_DEFINE(15)
#elif SEM_AX_GROUP == 2
SEM_AX_DEFINE(14)
#elif SEM_AX_GROUP == 3
SEM_AX_DEFINE(13) SEM_AX_DEFINE(2)
#elif SEM_AX_GROUP == 4
SEM_AX_DEFINE(12) SEM_AX_DEFINE(3)
#elif SEM_AX_GROUP == 5
SEM_AX_DEFINE(11) SEM_AX_DEFINE(4) SEM_AX_DEFINE(5)
#elif SEM_AX_GROUP == 6
SEM_AX_DEFINE(10) SEM_AX_DEFINE(6)
#elif SEM_AX_GROUP == 7
SEM_AX_DEFINE(9) SEM_AX_DEFINE(8) SEM_AX_DEFINE(7)
#endif

}  // namespace sem
