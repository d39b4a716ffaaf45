// Deterministic two-stage reductions (fixed grid, fixed tree order).
//
// The reference's glsc3 (sembench/cg.py:77-92) folds 65536-point chunks
// sequentially; replicating that order on a GPU would serialise 65536-long
// dependency chains, so the device instead uses a FIXED reduction tree: a
// constant number of blocks (kReduceBlocks, independent of the GPU), a fixed
// per-thread stride pattern, a warp-shuffle tree and an in-order combine of
// block partials by the last block to finish.  Results are bit-reproducible
// run to run and across devices, and agree with the reference to rounding.
#pragma once
#include "sem_common.cuh"

namespace sem {

constexpr int kReduceBlocks = 1184;  // 8 x 148; a constant so the tree is fixed
constexpr int kReduceBlocksMax = 4 * kReduceBlocks;  // capacity of the partial slots
constexpr int kReduceThreads = 256;
constexpr int kMaxReductions = 4;    // independent accumulators per kernel

// scratch layout: double partials[kMaxReductions][kReduceBlocksMax]; uint32 counter
struct ReduceScratch {
    double partials[kMaxReductions][kReduceBlocksMax];
    unsigned int counter;
    unsigned int pad[15];
};

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    return v;
}

// Block-wide sum in a fixed order; result valid in thread 0.
template <int THREADS>
__device__ __forceinline__ double block_sum(double v, double* sh /* >= THREADS/32 */)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double t = 0.0;
    if (wid == 0) {
        t = (lane < THREADS / 32) ? sh[lane] : 0.0;
        t = warp_sum(t);
    }
    __syncthreads();
    return t;
}

// Publish NR block partials; the last block to arrive combines them in
// block order and calls fin(totals, ctx) from thread 0, where ctx = pre()
// was evaluated by that thread BEFORE the partials are loaded (pre issues the
// loads fin needs -- e.g. state fields -- so they share the partials' round
// trip instead of following the sum).
template <int NR, int THREADS, typename Pre, typename Fin>
__device__ __forceinline__ void reduce_publish_and_finish_pre(const double (&vals)[NR],
                                                              ReduceScratch* rs, Pre pre, Fin fin)
{
    __shared__ double sh[THREADS / 32];
    __shared__ bool am_last;
    double tot[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) tot[q] = block_sum<THREADS>(vals[q], sh);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < NR; ++q) rs->partials[q][blockIdx.x] = tot[q];
        // acq_rel arrival: releases this block's partials (thread 0 wrote
        // them) and, in the last block, acquires every earlier block's; the
        // barrier below then orders the other threads' loads after it (the
        // semaphore pattern) -- no separate SC fences
        unsigned prev;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                     : "=r"(prev) : "l"(&rs->counter) : "memory");
        am_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last) return;
    decltype(pre()) ctx{};
    if (threadIdx.x == 0) ctx = pre();
    double fin_tot[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
        double v = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += THREADS)
            v += __ldcg(&rs->partials[q][b]);
        fin_tot[q] = block_sum<THREADS>(v, sh);
    }
    if (threadIdx.x == 0) {
        rs->counter = 0u;
        fin(fin_tot, ctx);
    }
}

// The same without a prefetch: fin(totals) from thread 0 of the last block.
template <int NR, int THREADS, typename Fin>
__device__ __forceinline__ void reduce_publish_and_finish(const double (&vals)[NR],
                                                          ReduceScratch* rs, Fin fin)
{
    reduce_publish_and_finish_pre<NR, THREADS>(
        vals, rs, [] { return 0; }, [&](const double (&t)[NR], int) { fin(t); });
}

// Deferred form: publish this block's NR totals only (no fence, no arrival
// counter, the block retires at once); a following kernel combines them.
template <int NR, int THREADS>
__device__ __forceinline__ void reduce_publish_only(const double (&vals)[NR], ReduceScratch* rs)
{
    __shared__ double sh[THREADS / 32];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
        const double t = block_sum<THREADS>(vals[q], sh);
        if (threadIdx.x == 0) rs->partials[q][blockIdx.x] = t;
    }
}

// Sum count partials in a fixed order with one block of THREADS threads
// (every load independent, so the whole set is in flight at once); the
// total is valid in thread 0.
template <int THREADS>
__device__ __forceinline__ double settle_sum(const double* __restrict__ partials, int count)
{
    __shared__ double sh[THREADS / 32];
    double v = 0.0;
    // 128-bit loads (the partial arrays are 16-byte aligned)
    const double2* p2 = reinterpret_cast<const double2*>(partials);
#pragma unroll 4
    for (int b = threadIdx.x; b < count / 2; b += THREADS) {
        const double2 t = __ldcg(p2 + b);
        v += t.x;
        v += t.y;
    }
    if ((count & 1) && threadIdx.x == 0) v += __ldcg(partials + count - 1);
    return block_sum<THREADS>(v, sh);
}

}  // namespace sem
