/* A plain C client of libsem (no Python, no torch in the process): the
 * drop-in boundary exercised the way a C / Go / Fortran host would bind it.
 *
 *   sem_client <dir>
 *
 * reads <dir>/meta.txt ("n ex ey ez iters rhs_seed"), <dir>/dx.bin,
 * <dir>/dxt.bin, <dir>/weights.bin (float64, n*n / n*n / n), then on the GPU:
 *   u = random_field(E, n, 1), g = random_field(6E, n, 2)     (sem_random_field)
 *   w = A_local u                                             (sem_ax)
 *   d = mask(dssum(u))                                        (sem_dssum_box)
 *   CG on the box: f = mask(dssum(random_field(E, n, rhs_seed))), affine
 *   geometry (sem_box_geom), `iters` iterations (sem_cg_init / sem_cg_run /
 *   sem_cg_finalize)
 * and writes <dir>/w.bin, <dir>/dssum.bin, <dir>/hist.bin, <dir>/x.bin.
 * tests/test_c_client.py compares them with the CPU oracle. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "sem.h"

#define CK(call)                                                                   \
    do {                                                                           \
        int rc_ = (call);                                                          \
        if (rc_ != 0) {                                                            \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, sem_last_error()); \
            return 2;                                                              \
        }                                                                          \
    } while (0)
#define CU(call)                                                                   \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess) {                                                   \
            fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));            \
            return 3;                                                              \
        }                                                                          \
    } while (0)

static int read_f64(const char* dir, const char* name, double* out, size_t count)
{
    char path[1024];
    snprintf(path, sizeof path, "%s/%s", dir, name);
    FILE* f = fopen(path, "rb");
    if (!f) return -1;
    size_t got = fread(out, sizeof(double), count, f);
    fclose(f);
    return got == count ? 0 : -1;
}

static int write_dev(const char* dir, const char* name, const double* dev, size_t count)
{
    double* host = (double*)malloc(count * sizeof(double));
    if (!host || cudaMemcpy(host, dev, count * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
        return -1;
    char path[1024];
    snprintf(path, sizeof path, "%s/%s", dir, name);
    FILE* f = fopen(path, "wb");
    if (!f) return -1;
    fwrite(host, sizeof(double), count, f);
    fclose(f);
    free(host);
    return 0;
}

int main(int argc, char** argv)
{
    if (argc != 2) {
        fprintf(stderr, "usage: %s <dir>\n", argv[0]);
        return 1;
    }
    const char* dir = argv[1];
    char path[1024];
    snprintf(path, sizeof path, "%s/meta.txt", dir);
    FILE* mf = fopen(path, "r");
    int n, ex, ey, ez, iters;
    unsigned long long rhs_seed;
    if (!mf || fscanf(mf, "%d %d %d %d %d %llu", &n, &ex, &ey, &ez, &iters, &rhs_seed) != 6) {
        fprintf(stderr, "bad meta.txt\n");
        return 1;
    }
    fclose(mf);
    if (sem_abi_version() != SEM_ABI_VERSION) {
        fprintf(stderr, "ABI mismatch\n");
        return 1;
    }
    const int64_t E = (int64_t)ex * ey * ez, m = E * n * n * n;
    double dx[256], dxt[256], wts[16];
    if (read_f64(dir, "dx.bin", dx, (size_t)n * n) || read_f64(dir, "dxt.bin", dxt, (size_t)n * n) ||
        read_f64(dir, "weights.bin", wts, (size_t)n)) {
        fprintf(stderr, "missing basis files\n");
        return 1;
    }
    cudaStream_t s;
    CU(cudaStreamCreate(&s));
    double *u, *g, *w, *d, *f, *x, *r, *p, *wcg, *hist, *gbox;
    void *state, *scratch;
    CU(cudaMalloc((void**)&u, m * sizeof(double)));
    CU(cudaMalloc((void**)&g, 6 * m * sizeof(double)));
    CU(cudaMalloc((void**)&w, m * sizeof(double)));
    CU(cudaMalloc((void**)&d, m * sizeof(double)));
    CU(cudaMalloc((void**)&f, m * sizeof(double)));
    CU(cudaMalloc((void**)&x, m * sizeof(double)));
    CU(cudaMalloc((void**)&r, m * sizeof(double)));
    CU(cudaMalloc((void**)&p, m * sizeof(double)));
    CU(cudaMalloc((void**)&wcg, 2 * m * sizeof(double)));
    CU(cudaMalloc((void**)&gbox, 6 * m * sizeof(double)));
    CU(cudaMalloc((void**)&hist, (iters > 0 ? iters : 1) * sizeof(double)));
    CU(cudaMalloc(&state, sizeof(sem_cg_state)));
    CU(cudaMalloc(&scratch, (size_t)sem_reduce_scratch_bytes()));
    CU(cudaMemset(scratch, 0, (size_t)sem_reduce_scratch_bytes()));

    /* Ax and dssum on seeded random fields */
    CK(sem_random_field(u, m, 1, s));
    CK(sem_random_field(g, 6 * m, 2, s));
    CK(sem_ax(u, g, dx, dxt, w, E, n, s));
    CK(sem_dssum_box(u, d, ex, ey, ez, n, 1, s));

    /* CG on the box: f = mask(dssum(random_field(rhs_seed))) */
    CK(sem_random_field(r, m, rhs_seed, s));
    CK(sem_dssum_box(r, f, ex, ey, ez, n, 1, s));
    CK(sem_box_geom(gbox, E, n, wts, 1.0, s));
    CK(sem_cg_init(f, x, r, p, (sem_cg_state*)state, hist, iters, 0.0, ex, ey, ez, n, scratch, s));
    CK(sem_cg_run(gbox, dx, dxt, x, r, p, wcg, (sem_cg_state*)state, hist, iters, ex, ey, ez, n,
                  scratch, s));
    CK(sem_cg_finalize(x, p, (sem_cg_state*)state, m, s));
    CU(cudaStreamSynchronize(s));
    sem_cg_state st;
    CU(cudaMemcpy(&st, state, sizeof st, cudaMemcpyDeviceToHost));
    if (st.iterations_run != iters || st.stop != 0) {
        fprintf(stderr, "CG ran %d iterations, stop %d\n", st.iterations_run, st.stop);
        return 4;
    }
    if (write_dev(dir, "w.bin", w, m) || write_dev(dir, "dssum.bin", d, m) ||
        write_dev(dir, "hist.bin", hist, iters) || write_dev(dir, "x.bin", x, m)) {
        fprintf(stderr, "write failed\n");
        return 5;
    }

    /* host buffers, the reference's call shape: pageable (malloc) arrays go
     * through the chunked copy-engine pipeline, mapped page-locked arrays
     * through the one-launch zero-copy kernel */
    double* uh = (double*)malloc(m * sizeof(double));
    double* wh = (double*)malloc(m * sizeof(double));
    double *up, *wp;
    CU(cudaHostAlloc((void**)&up, m * sizeof(double), cudaHostAllocMapped));
    CU(cudaHostAlloc((void**)&wp, m * sizeof(double), cudaHostAllocMapped));
    CU(cudaMemcpy(uh, u, m * sizeof(double), cudaMemcpyDeviceToHost));
    memcpy(up, uh, m * sizeof(double));
    CK(sem_ax_host(uh, g, dx, dxt, wh, E, n, d, wcg, 2, s));  /* 2-element chunks */
    CK(sem_ax_host(up, g, dx, dxt, wp, E, n, d, wcg, 0, s));
    CU(cudaStreamSynchronize(s));
    /* weighted dot and the unfused vector updates */
    double* dot;
    CU(cudaMalloc((void**)&dot, sizeof(double)));
    CK(sem_glsc3_box(u, w, ex, ey, ez, n, dot, scratch, s));
    CK(sem_add2s1(w, u, 0.75, m, s));   /* w = 0.75 w + u */
    CK(sem_add2s2(u, g, -1.25, m, s));  /* u += -1.25 g[:m] */
    CU(cudaStreamSynchronize(s));
    char p2[1024];
    FILE* fo;
    snprintf(p2, sizeof p2, "%s/w_host.bin", dir);
    if (!(fo = fopen(p2, "wb"))) return 5;
    fwrite(wh, sizeof(double), m, fo);
    fclose(fo);
    snprintf(p2, sizeof p2, "%s/w_mapped.bin", dir);
    if (!(fo = fopen(p2, "wb"))) return 5;
    fwrite(wp, sizeof(double), m, fo);
    fclose(fo);
    if (write_dev(dir, "dot.bin", dot, 1) || write_dev(dir, "add2s1.bin", w, m) ||
        write_dev(dir, "add2s2.bin", u, m)) {
        fprintf(stderr, "write failed\n");
        return 5;
    }
    printf("sem_client ok: E=%lld n=%d iterations=%d\n", (long long)E, n, st.iterations_run);
    return 0;
}
