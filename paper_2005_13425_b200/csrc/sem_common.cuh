// Shared helpers for libsem (B200 / sm_100a).
#pragma once
#include <cstdint>
#include <initializer_list>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <utility>

#include "../../include/sem.h"

namespace sem {

// Error reporting: every C-ABI entry point returns 0 on success, else a
// cudaError_t (or SEM_E_* code) and leaves a message for sem_last_error().
void set_error(const char* fmt, ...);
int fail_cuda(cudaError_t err, const char* what);

// Make the calling thread's runtime device match the device owning `stream`
// (the library links cudart statically, so its current-device state is
// separate from torch's).
int bind_stream_device(cudaStream_t stream);

// a requested kernel tiling that does not fit (shared memory / threads) ran
// the generic fallback instead -- counted, so tests can assert the tuned
// defaults never take it (sem_fallback_count)
void note_fallback();

constexpr int kNumSMsB200 = 148;
int sm_count();

// Analytic structured-box helpers (sembench/assembly.py:69-110): element
// e = ex_i + ex*(ey_i + ey*ez_i); global lattice coordinate along x is
// ex_i*(n-1)+i, and a node is interior iff every coordinate is strictly inside
// the global point grid [0, ex*(n-1)].
struct BoxDims {
    int ex, ey, ez;   // elements per axis of THIS field (a z-slab for multi-GPU)
    int n;
    int gz0;          // global element-layer offset of this slab along z
    int ez_global;    // global element count along z
};

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor in
// the stream drains; griddep_wait() blocks until the predecessor grid has
// completed and its writes are visible, griddep_launch() lets this grid's
// own dependent start launching.  Both are no-ops without the attribute.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch()
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Phase stagger of co-resident CTAs (large-n Ax): CTAs lo..hi-1 -- the
// second CTA of every SM in the first wave -- idle at entry for ns
// nanoseconds at the 1965 MHz boost clock, counted in SM cycles (clock64) so
// the offset stays the same fraction of an element's time when the power cap
// lowers the clock.  The CTAs sharing an SM then run out of step: one
// streams its metric (S4) while the other is in its shared-memory
// contractions, and every later CTA inherits its slot's offset, so HBM
// demand is spread over the element instead of arriving in per-wave bursts.
// CTA b in [lo, hi) waits ns x (b / lo): with lo = the SM count, the k-th
// resident CTA of an SM waits (k - 1) ns (hi = 2 lo: the second CTA only).
__device__ __forceinline__ void stagger_wait(int ns, int lo, int hi)
{
    if (ns <= 0 || (int)blockIdx.x < lo || (int)blockIdx.x >= hi) return;
    const long long cycles = (long long)ns * ((int)blockIdx.x / lo) * 1965 / 1000;
    const long long t0 = clock64();
    do {
        __nanosleep(256);
    } while (clock64() - t0 < cycles);
}

// Timeline tracing of the fused CG chain (diagnostic builds only,
// -DSEM_TRACE; tools/cg_trace.py): per kernel kind and iteration slot, the
// earliest CTA entry, the earliest return from griddep_wait and the latest
// CTA exit (%globaltimer ns), kept in a caller-provided area right after
// the sem_cg_state struct.  Compiled out of the product build.
#ifdef SEM_TRACE
__device__ __forceinline__ unsigned long long sem_gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define SEM_TRACE_ENTRY(st) const unsigned long long _sem_t0 = sem_gtimer();
#define SEM_TRACE_WAITED(st) const unsigned long long _sem_t1 = sem_gtimer();
#define SEM_TRACE_EXIT(st, kid)                                                             \
    do {                                                                                    \
        if (threadIdx.x == 0) {                                                             \
            unsigned long long* _tr = reinterpret_cast<unsigned long long*>((st) + 1) +      \
                                      ((kid) * 128 + ((st)->it & 127)) * 3;                  \
            atomicMin(_tr, _sem_t0);                                                        \
            atomicMin(_tr + 1, _sem_t1);                                                    \
            atomicMax(_tr + 2, sem_gtimer());                                               \
        }                                                                                   \
    } while (0)
#else
#define SEM_TRACE_ENTRY(st)
#define SEM_TRACE_WAITED(st)
#define SEM_TRACE_EXIT(st, kid)
#endif

// Field-pointer alignment contract (checked before anything is enqueued, so
// a bad pointer is an error code, not a device fault that poisons the
// context): metric blocks move by bulk (TMA) copies -> 16 bytes; fields of an
// even n are moved as 16-byte row pairs / bulk layers -> 16 bytes (n^3 is
// even, so any element offset keeps it); odd n -> 8 bytes.
inline bool aligned_to(const void* p, unsigned bytes)
{
    return (reinterpret_cast<uintptr_t>(p) & (uintptr_t)(bytes - 1)) == 0;
}
inline int check_fields_aligned(const char* who, int n, const void* metric,
                                std::initializer_list<const void*> fields)
{
    if (metric && !aligned_to(metric, 16)) {
        set_error("%s: the metric must be 16-byte aligned", who);
        return SEM_E_INVALID;
    }
    const unsigned need = (n % 2 == 0) ? 16u : 8u;
    for (const void* f : fields)
        if (f && !aligned_to(f, need)) {
            set_error("%s: field pointers must be %u-byte aligned for n = %d", who, need, n);
            return SEM_E_INVALID;
        }
    return 0;
}

// Launch `kern` on `stream`, with programmatic stream serialization when
// `pdl` is set (the kernel must call griddep_wait() before touching anything
// its predecessors write).
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t stream, bool pdl, Args&&... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace sem

#define SEM_CHECK_LAUNCH(what)                                         \
    do {                                                               \
        cudaError_t _e = cudaGetLastError();                           \
        if (_e != cudaSuccess) return ::sem::fail_cuda(_e, what);      \
    } while (0)

// IEEE double ops that nvcc must not contract into FMA: the reference's
// vector updates are unfused multiply-then-add (sembench/cg.py:95-104).
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// Exact power-of-two scale for the fused <p, A p> sum: 2^k with rtz * 2^(2k)
// in [1, 8).  The CG kernels accumulate (s p) * (s w) and divide s^2 back out
// of rtz instead of pap, so in the normal range every product and partial
// sum is the unscaled one times an exact power of two (alpha bit-identical),
// while deep in FP64 underflow the scaled <p, A p> cannot flush to zero
// before <r, r> does -- breakdown is then decided by the sign of <p, A p>,
// not by which reduction tree underflows first.
__device__ __forceinline__ int pap_scale_exp(double rtz)
{
    if (!(rtz > 0.0) || !isfinite(rtz)) return 0;
    return -(ilogb(rtz) >> 1);
}

