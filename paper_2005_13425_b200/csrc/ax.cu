// Local Poisson operator Ax on B200 (sm_100a): the C-ABI entry points and the
// runtime-n dispatch.  The kernels are in ax_pencil.cuh / ax_impl.cuh and are
// instantiated per n in ax_inst.cu.
#include "sem_common.cuh"
#include "box.cuh"
#include "ax_pencil.cuh"

#include <stdlib.h>

namespace sem {

#define SEM_AX_DECLARE(NV)                                                                   \
    int ax_entry_##NV(const double* u, const double* g, const double* dx, double* w,          \
                      int64_t E, int variant, int pdl, cudaStream_t s);                       \
    int ax_cg_entry_##NV(const double* g, const double* dx, double* w, int64_t E,             \
                         CgpArgs a, int mode, cudaStream_t s);
SEM_AX_DECLARE(2) SEM_AX_DECLARE(3) SEM_AX_DECLARE(4) SEM_AX_DECLARE(5) SEM_AX_DECLARE(6)
SEM_AX_DECLARE(7) SEM_AX_DECLARE(8) SEM_AX_DECLARE(9) SEM_AX_DECLARE(10) SEM_AX_DECLARE(11)
SEM_AX_DECLARE(12) SEM_AX_DECLARE(13) SEM_AX_DECLARE(14) SEM_AX_DECLARE(15) SEM_AX_DECLARE(16)
#undef SEM_AX_DECLARE

// mode 2: single-GPU solver (<p, A p> -> alpha in the last CTA); mode 3:
// z-slab rank (<p, A p> partial -> state->local_sum)
int ax_cg_dispatch(const double* g, const double* dx, double* w, int64_t E, int n, CgpArgs a,
                   int mode, cudaStream_t stream)
{
    if (E == 0) return 0;
    switch (n) {
#define SEM_AXCG_CASE(NV) \
    case NV: return ax_cg_entry_##NV(g, dx, w, E, a, mode, stream);
        SEM_AXCG_CASE(2) SEM_AXCG_CASE(3) SEM_AXCG_CASE(4) SEM_AXCG_CASE(5) SEM_AXCG_CASE(6)
        SEM_AXCG_CASE(7) SEM_AXCG_CASE(8) SEM_AXCG_CASE(9) SEM_AXCG_CASE(10) SEM_AXCG_CASE(11)
        SEM_AXCG_CASE(12) SEM_AXCG_CASE(13) SEM_AXCG_CASE(14) SEM_AXCG_CASE(15) SEM_AXCG_CASE(16)
#undef SEM_AXCG_CASE
        default:
            set_error("sem_cg_ax: n=%d outside the supported range [2, 16]", n);
            return SEM_E_INVALID;
    }
}

// programmatic dependent launch of the plain Ax kernels: each CTA waits
// (griddepcontrol.wait) for the predecessor at entry, so it is safe after any
// kind of stream work, and the grid is resident while the previous kernel
// drains (E = 1024: 13.8 -> 12.8 us, E = 4096: 41.8 -> 41.0 us).  Mode 2
// also prefetches the CTA's own blocks into L2 before the wait (short
// launches only, see launch_pencil).  SEM_AX_PDL = 0 / 1 / 2 overrides.
static int ax_pdl()
{
    static const int k = getenv("SEM_AX_PDL") ? atoi(getenv("SEM_AX_PDL")) : 2;
    return k;
}

int ax_dispatch(const double* u, const double* g, const double* dx, double* w, int64_t E,
                int n, int variant, cudaStream_t stream, int pdl)
{
    if (pdl < 0) pdl = ax_pdl();
    switch (n) {
#define SEM_AX_CASE(NV) \
    case NV: return ax_entry_##NV(u, g, dx, w, E, variant, pdl, stream);
        SEM_AX_CASE(2) SEM_AX_CASE(3) SEM_AX_CASE(4) SEM_AX_CASE(5) SEM_AX_CASE(6)
        SEM_AX_CASE(7) SEM_AX_CASE(8) SEM_AX_CASE(9) SEM_AX_CASE(10) SEM_AX_CASE(11)
        SEM_AX_CASE(12) SEM_AX_CASE(13) SEM_AX_CASE(14) SEM_AX_CASE(15) SEM_AX_CASE(16)
#undef SEM_AX_CASE
        default:
            set_error("sem_ax: n=%d outside the supported range [2, 16]", n);
            return SEM_E_INVALID;
    }
}

}  // namespace sem

extern "C" int sem_ax_variant(const double* u, const double* g, const double* dx,
                              const double* dxt, double* w, int64_t num_elements,
                              int32_t n, int32_t variant, sem_stream_t stream)
{
    if (num_elements == 0) return 0;  // nothing to do; empty tensors may carry null pointers
    if (!u || !g || !dx || !dxt || !w || num_elements < 0) {
        sem::set_error("sem_ax: null pointer or negative element count");
        return SEM_E_INVALID;
    }
    if (int rc = sem::check_fields_aligned("sem_ax", n, g, {u, w})) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = sem::bind_stream_device(s)) return rc;
    return sem::ax_dispatch(u, g, dx, w, num_elements, n, variant, s, -1);
}

extern "C" int sem_ax(const double* u, const double* g, const double* dx,
                      const double* dxt, double* w, int64_t num_elements, int32_t n,
                      sem_stream_t stream)
{
    return sem_ax_variant(u, g, dx, dxt, w, num_elements, n, 0, stream);
}

extern "C" int sem_ax_num_variants(int32_t n)
{
    return (n >= 2 && n <= 16) ? 76 : 0;
}
