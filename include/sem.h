/*
 * libsem -- B200-native (sm_100a) hot path of the Nekbone / sembench
 * spectral-element Poisson solve (arXiv 2005.13425): the local tensor-product
 * operator Ax, the direct-stiffness summation dssum + Dirichlet mask, and the
 * CG vector kernels (add2s1 / add2s2 / glsc3).
 *
 * Plain C ABI: device pointers are raw CUDA device addresses (a torch
 * tensor's data_ptr(), a cudaMalloc result, ...), sizes are int64, and every
 * call is enqueued on `stream` (a cudaStream_t; NULL = legacy default
 * stream) without synchronising the host.  Every entry point returns 0 on
 * success, otherwise a nonzero code with a message in sem_last_error().
 * No entry point allocates device memory; scratch is caller-provided.
 * Alignment: the metric g must be 16-byte aligned (it moves by bulk copies);
 * fields (u, w, f, x, r, p) must be 16-byte aligned for even n and 8-byte
 * aligned for odd n -- allocation bases always are, and since n^3 is even for
 * even n, element sub-ranges keep the property.  Violations return
 * SEM_E_INVALID before anything is enqueued.
 *
 * Reference interface each entry point replaces (the reference is the
 * Python/numba package `sembench`, paths relative to
 * /root/reference/pkg/src/sembench/):
 *
 *   sem_ax             kernels.py:413-468 apply_ax (LAYERED, :267-410)
 *   sem_ax_reference   kernels.py:159-205 _ax_reference (REFERENCE variant)
 *   sem_ax_scratch     kernels.py:213-259 _ax_scratch   (SCRATCH variant)
 *   sem_dssum_box      assembly.py:113-120 dssum  (bincount order, bit-exact)
 *   sem_mask_box       assembly.py:123-129 mask
 *   sem_apply_global   assembly.py:132-155 apply_global
 *   sem_add2s1         cg.py:101-104 _scale_add   p = beta*p + z
 *   sem_add2s2         cg.py:95-98   _axpy_into   x += alpha*y
 *   sem_glsc3*         cg.py:77-92,107-111 _wdot3 / weighted_dot
 *   sem_cg_*           cg.py:114-193 cg_solve loop (device-resident scalars)
 *   sem_random_field   fields.py:42-54 random_field (bit-exact SplitMix64)
 *   sem_box_geom       mesh.py:72-91 build_geom (bit-exact)
 *   sem_stream_copy    perf.py:156-159 _stream_copy (bandwidth probe)
 */
#ifndef SEM_H_
#define SEM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SEM_ABI_VERSION 1

/* Error codes besides cudaError_t values. */
#define SEM_E_INVALID 1001  /* bad argument (shape, n range, null pointer) */
#define SEM_E_BREAKDOWN 1002

typedef void *sem_stream_t; /* cudaStream_t */

int sem_abi_version(void);
const char *sem_last_error(void);

/* Supported points per dimension n (sembench/basis.py:17-18: 2..16). */
int sem_min_points(void);
int sem_max_points(void);
/* Number of launches since load whose requested kernel tiling did not fit
 * (shared memory / threads) and ran the generic tiling instead; the tuned
 * defaults never do (tests/test_gpu_parity.py).  Diagnostic only. */
int64_t sem_fallback_count(void);

/* ---------------------------------------------------------------- Ax ---- */
/* w[e] = A_local u[e] for every element (kernels.py:413-468).
 * u, w : [E][n][n][n] float64 device, i fastest; g : [E][6][n][n][n] float64
 * device (metric g1..g6 per point, mesh.py:40-57); dx, dxt : [n][n] float64
 * HOST arrays (basis.diff / basis.diff_t, 2 KB at most) -- they travel in the
 * kernel's constant parameter space.  u and w must not alias. */
int sem_ax(const double *u, const double *g, const double *dx, const double *dxt,
           double *w, int64_t num_elements, int32_t n, sem_stream_t stream);

/* Kernel-variant hook for benchmarks/ablation: variant 0 = default layered
 * kernel; other values select alternative tilings. */
int sem_ax_variant(const double *u, const double *g, const double *dx,
                   const double *dxt, double *w, int64_t num_elements, int32_t n,
                   int32_t variant, sem_stream_t stream);
int sem_ax_num_variants(int32_t n);

/* Host-buffer form (the reference's call shape: u and w in host memory).
 * If both u_host and w_host are page-locked (mapped), the kernel reads u and
 * writes w across PCIe itself in one launch.  Otherwise u_dev and w_dev
 * (E*n^3 device scratch vectors, always required) stage the data: the
 * element range is streamed in chunks of `chunk_elements` (<= 0: one chunk),
 * H2D of chunk c+1, Ax of chunk c and D2H of chunk c-1 running concurrently
 * on library-owned copy streams.
 * Asynchronous: w_host is complete once `stream` has been synchronised. */
int sem_ax_host(const double *u_host, const double *g, const double *dx,
                const double *dxt, double *w_host, int64_t num_elements, int32_t n,
                double *u_dev, double *w_dev, int64_t chunk_elements, sem_stream_t stream);

/* The reference's other two storage strategies (kernels.py:1-45), bit-exact
 * with sembench (same operation order, no FMA contraction).  REFERENCE: three
 * passes through caller-provided full-size intermediates ur, us, ut
 * ([E][n][n][n] device), which hold the metric-scaled gradients on return
 * (kernels.py:159-205).  SCRATCH: element staged in shared memory, n <=
 * SEM_SCRATCH_MAX_POINTS (kernels.py:213-259, :448-455). */
#define SEM_SCRATCH_MAX_POINTS 10
int sem_ax_reference(const double *u, const double *g, const double *dx,
                     const double *dxt, double *ur, double *us, double *ut, double *w,
                     int64_t num_elements, int32_t n, sem_stream_t stream);
int sem_ax_scratch(const double *u, const double *g, const double *dx, double *w,
                   int64_t num_elements, int32_t n, sem_stream_t stream);

/* ------------------------------------------------- assembly (box mesh) -- */
/* Element numbering e = ix + ex*(iy + ey*iz) and lattice ids of
 * assembly.py:69-110.  `out` may equal neither `f` (out-of-place).
 * apply_mask != 0 multiplies the summed value by the Dirichlet 0/1 mask
 * (i.e. returns mask(dssum(f))). */
int sem_dssum_box(const double *f, double *out, int32_t ex, int32_t ey, int32_t ez,
                  int32_t n, int32_t apply_mask, sem_stream_t stream);
int sem_mask_box(const double *f, double *out, int32_t ex, int32_t ey, int32_t ez,
                 int32_t n, sem_stream_t stream);
/* General numbering (any reference Topology.global_id, assembly.py:113-120):
 * the id classes as a CSR -- seg_idx = local flat indices grouped by global
 * id, each group in ascending local index (a stable argsort of global_id);
 * seg_off[nseg+1] delimits the groups.  Each class is summed in that order
 * from +0.0 (np.bincount's order) and the total written to every copy:
 * bit-identical to the reference for any numbering.  Out-of-place. */
int sem_dssum_csr(const double *f, double *out, const int32_t *seg_off,
                  const int32_t *seg_idx, int64_t nseg, sem_stream_t stream);
/* out = f * mask pointwise (assembly.py:123-129 with an arbitrary mask array). */
int sem_mask_array(const double *f, const double *mask, double *out, int64_t count,
                   sem_stream_t stream);
/* flag_dev[0] <- 0 if every unmasked shared node of f has equal copies
 * (f is interface-consistent on the box), else 1.  The fused CG's local
 * <p, A p> equals the reference's assembled one (cg.py:163) only for
 * consistent iterates; cg_solve checks mask(f) with this first. */
int sem_consistent_box(const double *f, int32_t ex, int32_t ey, int32_t ez, int32_t n,
                       int32_t *flag_dev, sem_stream_t stream);
/* mask(dssum(A_local(mask(u)))) with `scratch` an E*n^3 float64 buffer. */
int sem_apply_global(const double *u, const double *g, const double *dx,
                     const double *dxt, double *w, double *scratch, int32_t ex,
                     int32_t ey, int32_t ez, int32_t n, sem_stream_t stream);

/* ------------------------------------------------------ CG vector ops -- */
/* Bit-exact unfused updates (multiply rounded, then add rounded). */
int sem_add2s1(double *p, const double *z, double beta, int64_t m, sem_stream_t stream);
int sem_add2s2(double *x, const double *y, double alpha, int64_t m, sem_stream_t stream);

/* Deterministic weighted dot sum_i a_i*b_i*wt_i.  The result lands in
 * out_dev[0] (device).  `scratch` must hold sem_reduce_scratch_bytes(). */
int64_t sem_reduce_scratch_bytes(void);
int sem_glsc3(const double *a, const double *b, const double *wt, int64_t m,
              double *out_dev, void *scratch, sem_stream_t stream);
/* Same with wt = 1/multiplicity computed from the box lattice (no weight
 * array is read). */
int sem_glsc3_box(const double *a, const double *b, int32_t ex, int32_t ey,
                  int32_t ez, int32_t n, double *out_dev, void *scratch,
                  sem_stream_t stream);

/* --------------------------------------------------------- CG driver ---- */
/* Device-resident CG state (cg.py:139-186).  Layout shared with the host. */
typedef struct sem_cg_state {
    double rtz;        /* <r,r>_c of the current residual            */
    double rtz_old;
    double pap;
    double alpha;
    double beta;
    double tolerance;
    int32_t it;        /* iterations started so far                   */
    int32_t max_iterations;
    int32_t iterations_run;
    int32_t stop;      /* 0 running, 1 exact zero residual (cg.py:151),
                          2 breakdown <p,Ap> <= 0, 3 tolerance reached */
    int32_t breakdown_it;
    int32_t x_pending; /* single GPU: x += alpha p of the last completed
                          iteration not yet applied (sem_cg_finalize)     */
    double local_sum;  /* multi-GPU: this rank's partial of the last reduction */
} sem_cg_state;

/* Initialise: r = mask(f), x = p = 0, rtz = <r,r>_c, state fields. */
int sem_cg_init(const double *f, double *x, double *r, double *p, sem_cg_state *state,
                double *history, int32_t max_iterations, double tolerance,
                int32_t ex, int32_t ey, int32_t ez, int32_t n, void *scratch,
                sem_stream_t stream);
/* Enqueue `iterations` fused CG iterations on the box operator (single GPU):
 * per iteration the Ax kernel with the iteration head, x update and the
 * <p,Ap> block partials fused, a one-block settle (alpha), and the r update
 * with dssum + mask and <r,r>_c fused.  w is a 2*E*n^3 scratch
 * buffer; history receives sqrt(<r,r>_c) per iteration.  The x update of
 * the LAST iteration run is deferred: call sem_cg_finalize before reading x. */
int sem_cg_run(const double *g, const double *dx, const double *dxt, double *x,
               double *r, double *p, double *w, sem_cg_state *state, double *history,
               int32_t iterations, int32_t ex, int32_t ey, int32_t ez, int32_t n,
               void *scratch, sem_stream_t stream);
/* sem_cg_run for iterations first_iteration .. first_iteration+iterations-1
 * of a solve (1-based): the fused iteration alternates its element walk
 * direction by the parity of the global iteration number (L2 reuse between
 * consecutive Ax launches), so a solve split into several calls -- one per
 * callback, graph replays of a fixed chunk -- rounds exactly like one call.
 * sem_cg_run(...) == sem_cg_run_at(..., first_iteration = 1, ...). */
int sem_cg_run_at(const double *g, const double *dx, const double *dxt, double *x,
                  double *r, double *p, double *w, sem_cg_state *state, double *history,
                  int32_t iterations, int32_t first_iteration, int32_t ex, int32_t ey,
                  int32_t ez, int32_t n, void *scratch, sem_stream_t stream);
/* Apply the pending x += alpha p (if any; not after a breakdown) and clear it.
 * num_points = E*n^3. */
int sem_cg_finalize(double *x, const double *p, sem_cg_state *state, int64_t num_points,
                    sem_stream_t stream);
/* sem_cg_run with CUDA events between its launches (measurement only):
 * synchronises, then ADDS each phase's device milliseconds to phase_ms[0]
 * (Ax with the fused iteration head and <p,Ap>, plus the settle), [1] (r update with the
 * fused dssum + mask, <r,r>), [2] (unused). */
int sem_cg_run_phases(const double *g, const double *dx, const double *dxt, double *x,
                      double *r, double *p, double *w, sem_cg_state *state, double *history,
                      int32_t iterations, int32_t ex, int32_t ey, int32_t ez, int32_t n,
                      void *scratch, double *phase_ms, sem_stream_t stream);

/* ------------------------------------------- multi-GPU z-slab partition -- */
/* A rank owns global element layers [gz0, gz0+ez) of an ex*ey*ez_global box
 * (contiguous element range, e = ix + ex*(iy + ey*iz)).  Interface planes are
 * (ey*(n-1)+1) x (ex*(n-1)+1) arrays indexed gy*(ex*(n-1)+1) + gx.
 * Halo protocol (bit-exact with the reference's bincount order):
 *   plane_top    : ordered in-plane sum of this slab's top-face copies, from +0.0
 *   plane_bottom : `prefix` (the lower rank's plane_top, or NULL = +0.0)
 *                  continued with this slab's bottom-face copies = totals   */
int sem_slab_plane_top(const double *f, double *plane, int32_t ex, int32_t ey, int32_t ez,
                       int32_t n, sem_stream_t stream);
int sem_slab_plane_bottom(const double *f, const double *prefix, double *totals, int32_t ex,
                          int32_t ey, int32_t ez, int32_t n, sem_stream_t stream);
/* dssum on a slab: nodes on the bottom/top face shared with another rank take
 * bottom_totals / top_totals (NULL = no neighbour), the rest are gathered
 * locally; the mask and multiplicities use the GLOBAL lattice. */
int sem_dssum_slab(const double *f, double *out, const double *bottom_totals,
                   const double *top_totals, int32_t ex, int32_t ey, int32_t ez, int32_t n,
                   int32_t gz0, int32_t ez_global, int32_t apply_mask, sem_stream_t stream);
int sem_mask_slab(const double *f, double *out, int32_t ex, int32_t ey, int32_t ez, int32_t n,
                  int32_t gz0, int32_t ez_global, sem_stream_t stream);
/* this rank's partial of the weighted dot (global multiplicities) */
int sem_glsc3_slab(const double *a, const double *b, int32_t ex, int32_t ey, int32_t ez,
                   int32_t n, int32_t gz0, int32_t ez_global, double *out_dev, void *scratch,
                   sem_stream_t stream);
/* Distributed CG phases: each reduction leaves this rank's partial in
 * state->local_sum; after gathering all ranks' partials (rank order) into
 * `gathered`, sem_cg_finish(phase) combines them in rank order and performs
 * the phase's scalar step (0: rtz after init, 1: pap -> alpha / breakdown,
 * 2: <r,r> -> history, rtz, tolerance, x update owed). */
int sem_cg_init_slab(const double *f, double *x, double *r, double *p, sem_cg_state *state,
                     double *history, int32_t max_iterations, double tolerance, int32_t ex,
                     int32_t ey, int32_t ez, int32_t n, int32_t gz0, int32_t ez_global,
                     void *scratch, sem_stream_t stream);
/* The single-GPU iteration's two kernels on a slab (each rank, every
 * iteration): sem_cg_ax_slab on element ranges of the slab (edge layers
 * first, then the interior overlapping the halo exchange) = exact-zero exit,
 * beta, x += alpha_prev p_old (deferred), p = beta*p + r, w = A_local p and
 * this range's sum of p*(A_local p) added to (accumulate > 0) or stored in
 * (accumulate == 0) state->local_sum -- gather + sem_cg_finish(phase 1) then
 * settles alpha.  `partials` holds one double per element of the range
 * (device scratch).  accumulate < 0 only leaves the per-element-slot partials
 * there; one sem_cg_settle_slab over the slots of all of an iteration's
 * ranges then sets local_sum (one settle per iteration instead of one per
 * range).
 * sem_cg_update_slab = r += (-alpha) mask(dssum(w)) with the interface faces
 * from the halo totals, and this rank's <r,r>_c partial in local_sum
 * (phase 2).  sem_cg_finalize applies the last owed x update. */
int sem_cg_ax_slab(double *p, const double *r, double *x, const double *g, const double *dx,
                   const double *dxt, double *w, int64_t num_elements, int32_t n,
                   sem_cg_state *state, double *history, double *partials, void *scratch,
                   int32_t accumulate, sem_stream_t stream);
int sem_cg_settle_slab(const double *partials, int64_t count, sem_cg_state *state,
                       int32_t accumulate, sem_stream_t stream);
int sem_cg_update_slab(const double *w, double *r, const double *bottom_totals,
                       const double *top_totals, sem_cg_state *state, int32_t ex, int32_t ey,
                       int32_t ez, int32_t n, int32_t gz0, int32_t ez_global, void *scratch,
                       sem_stream_t stream);
int sem_cg_finish(sem_cg_state *state, const double *gathered, int32_t nranks, int32_t phase,
                  double *history, sem_stream_t stream);
/* sem_cg_finish(phase 1) folded into sem_cg_update_slab: every CTA combines
 * the ranks' <p,Ap> partials `gathered_pap[0..nranks)` in rank order and
 * derives alpha itself (breakdown -> stop = 2, r untouched), then the update.
 * One launch per iteration fewer (replaces sem_cg_finish(state, ., ., 1, .)
 * + sem_cg_update_slab; the sembench recurrence cg.py:163-172). */
int sem_cg_update_slab_alpha(const double *w, double *r, const double *bottom_totals,
                             const double *top_totals, sem_cg_state *state,
                             const double *gathered_pap, int32_t nranks, int32_t ex, int32_t ey,
                             int32_t ez, int32_t n, int32_t gz0, int32_t ez_global,
                             void *scratch, sem_stream_t stream);

/* ------------------------------------------------------ input builders -- */
int sem_random_field(double *out, int64_t count, uint64_t seed, sem_stream_t stream);
/* g for the affine box map: g1=g4=g6=(w_k*w_j)*w_i*(h/2), g2=g3=g5=0;
 * weights is a HOST array of n GLL weights. */
int sem_box_geom(double *g, int64_t num_elements, int32_t n, const double *weights,
                 double extent, sem_stream_t stream);

/* ------------------------------------------------------------ probe ---- */
/* dst[i] = src[i] for count doubles (device, non-overlapping): the streaming
 * copy that measure_bandwidth times (perf.py:156-203, paper §V). */
int sem_stream_copy(double *dst, const double *src, int64_t count, sem_stream_t stream);

/* ------------------------------------------------------- L2 residency -- */
/* Device limits in bytes: persisting-L2 carve-out maximum, access-policy
 * window maximum, L2 size. */
int sem_l2_props(int64_t *persist_max, int64_t *window_max, int64_t *l2_bytes);
/* Mark [base, base+bytes) L2-persisting (hit_ratio of its lines) for kernels
 * launched into / captured from `stream`; set_aside > 0 sizes the device's
 * persisting carve-out (clamped).  bytes == 0 clears the window and resets
 * the persisting lines.  Used by the fused CG (cg.py) to keep r and w in L2
 * between its launches; no reference counterpart (a B200 residency knob). */
int sem_l2_window(void *base, int64_t bytes, double hit_ratio, int64_t set_aside,
                  sem_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SEM_H_ */
