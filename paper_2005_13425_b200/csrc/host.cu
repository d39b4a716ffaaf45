// Host-buffer entry point: w_host = A_local u_host with the PCIe transfers
// pipelined against the kernel.
//
// A reference-style caller holds u and w in host memory.  Copying the whole
// field in, computing, and copying it out serialises ~0.7 ms of H2D, 45 us
// of compute and ~0.7 ms of D2H.  Here the element range is cut into chunks
// and three streams run H2D of chunk c+1, Ax of chunk c and D2H of chunk c-1
// concurrently (PCIe is full duplex), so the call costs ~max(H2D, D2H).
// The chunk loop runs in C (no per-chunk host-language overhead); the two
// copy streams and an event pool are created once per device and reused.
#include <mutex>

#include "sem_common.cuh"

namespace sem {

int ax_dispatch(const double* u, const double* g, const double* dx, double* w, int64_t E,
                int n, int variant, cudaStream_t stream);

namespace {

constexpr int kMaxDevices = 64;
constexpr int kEventPool = 2 * 256 + 2;

struct DevicePipes {
    bool ready = false;
    cudaStream_t s_in = nullptr, s_out = nullptr;
    cudaEvent_t ev[kEventPool];
};

DevicePipes g_pipes[kMaxDevices];
std::mutex g_pipes_mu;
std::mutex g_enqueue_mu;

int get_pipes(DevicePipes** out)
{
    int dev = 0;
    cudaError_t err = cudaGetDevice(&dev);
    if (err != cudaSuccess) return fail_cuda(err, "sem_ax_host: cudaGetDevice");
    if (dev < 0 || dev >= kMaxDevices) {
        set_error("sem_ax_host: device index %d out of range", dev);
        return SEM_E_INVALID;
    }
    std::lock_guard<std::mutex> lock(g_pipes_mu);
    DevicePipes& p = g_pipes[dev];
    if (!p.ready) {
        err = cudaStreamCreateWithFlags(&p.s_in, cudaStreamNonBlocking);
        if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&p.s_out, cudaStreamNonBlocking);
        for (int i = 0; i < kEventPool && err == cudaSuccess; ++i)
            err = cudaEventCreateWithFlags(&p.ev[i], cudaEventDisableTiming);
        if (err != cudaSuccess) return fail_cuda(err, "sem_ax_host: stream/event setup");
        p.ready = true;
    }
    *out = &p;
    return 0;
}

}  // namespace
}  // namespace sem

extern "C" int sem_ax_host(const double* u_host, const double* g, const double* dx,
                           const double* dxt, double* w_host, int64_t num_elements, int32_t n,
                           double* u_dev, double* w_dev, int64_t chunk_elements,
                           sem_stream_t stream)
{
    using namespace sem;
    if (!u_host || !g || !dx || !dxt || !w_host || !u_dev || !w_dev || num_elements < 0 ||
        n < 2 || n > 16) {
        set_error("sem_ax_host: bad arguments");
        return SEM_E_INVALID;
    }
    if (num_elements == 0) return 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (int rc = bind_stream_device(s)) return rc;
    DevicePipes* P = nullptr;
    if (int rc = get_pipes(&P)) return rc;
    // one enqueue at a time per process: the copy streams and event pool are
    // shared, and stream ordering keeps back-to-back calls correct
    std::lock_guard<std::mutex> lock(g_enqueue_mu);
    const int64_t per = (int64_t)n * n * n;
    int64_t chunk = chunk_elements > 0 ? chunk_elements : num_elements;
    int64_t nchunks = (num_elements + chunk - 1) / chunk;
    if (nchunks > 256) {  // bounded by the event pool
        chunk = (num_elements + 255) / 256;
        nchunks = (num_elements + chunk - 1) / chunk;
    }
    cudaError_t err;
    // the copy streams start after everything already queued on `stream`
    err = cudaEventRecord(P->ev[0], s);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(P->s_in, P->ev[0], 0);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(P->s_out, P->ev[0], 0);
    if (err != cudaSuccess) return fail_cuda(err, "sem_ax_host: ordering");
    for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t e0 = c * chunk;
        const int64_t e1 = (e0 + chunk < num_elements) ? e0 + chunk : num_elements;
        const int64_t a = e0 * per;
        const size_t bytes = (size_t)((e1 - e0) * per) * sizeof(double);
        cudaEvent_t ev_in = P->ev[2 + 2 * c], ev_k = P->ev[3 + 2 * c];
        err = cudaMemcpyAsync(u_dev + a, u_host + a, bytes, cudaMemcpyHostToDevice, P->s_in);
        if (err == cudaSuccess) err = cudaEventRecord(ev_in, P->s_in);
        if (err == cudaSuccess) err = cudaStreamWaitEvent(s, ev_in, 0);
        if (err != cudaSuccess) return fail_cuda(err, "sem_ax_host: H2D");
        if (int rc = ax_dispatch(u_dev + a, g + e0 * 6 * per, dx, w_dev + a, e1 - e0, n, 0, s))
            return rc;
        err = cudaEventRecord(ev_k, s);
        if (err == cudaSuccess) err = cudaStreamWaitEvent(P->s_out, ev_k, 0);
        if (err == cudaSuccess)
            err = cudaMemcpyAsync(w_host + a, w_dev + a, bytes, cudaMemcpyDeviceToHost, P->s_out);
        if (err != cudaSuccess) return fail_cuda(err, "sem_ax_host: D2H");
    }
    // the caller's stream completes only when the last D2H has landed
    err = cudaEventRecord(P->ev[1], P->s_out);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(s, P->ev[1], 0);
    if (err != cudaSuccess) return fail_cuda(err, "sem_ax_host: completion");
    return 0;
}
