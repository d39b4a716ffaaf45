// Host-buffer entry point: w_host = A_local u_host with the PCIe transfers
// pipelined against the kernel.
//
// A reference-style caller holds u and w in host memory.  Copying the whole
// field in, computing, and copying it out serialises ~0.7 ms of H2D, 45 us
// of compute and ~0.7 ms of D2H.  When both host buffers are page-locked
// (mapped into the device address space) the Ax kernel itself loads u from
// and stores w to host memory: one launch, the PCIe reads of later elements
// overlap the writes of earlier ones, no copy-engine handoffs.  Pageable
// buffers (or SEM_HOST_MODE=0) take the streamed path: the element range is
// cut into chunks and three streams run H2D of chunk c+1, Ax of chunk c and
// D2H of chunk c-1 concurrently (PCIe is full duplex).  The chunk loop runs
// in C; the copy streams and an event pool are created once per device.
#include <cstdlib>
#include <mutex>

#include "sem_common.cuh"

namespace sem {

int ax_dispatch(const double* u, const double* g, const double* dx, double* w, int64_t E,
                int n, int variant, cudaStream_t stream, int pdl = -1);

namespace {

constexpr int kMaxDevices = 64;
constexpr int kMaxChunks = 256;
// Default transfer mode (tools/e2e_probe.py, B200 + PCIe Gen5, E=4096 p=9):
// 0 = chunked copy engines both ways (0.97 ms), 1 = the kernel reads u and
// writes w in mapped host memory itself (0.94 ms; 0.91 ms without the Python
// wrapper), 2 = copy-engine u + mapped w (0.94 ms at 4 MB chunks), 3 = mapped
// u + copy-engine w (1.17 ms).
constexpr int kHostMode = 1;
constexpr int kEventPool = 2 * kMaxChunks + 2;

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

// Device address of a mapped page-locked host buffer, or nullptr (pageable).
double* mapped(const double* host)
{
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, host) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (at.type != cudaMemoryTypeHost || at.devicePointer == nullptr) return nullptr;
    return static_cast<double*>(at.devicePointer);
}

// Uniform chunk sizes (elements) for a streamed call; returns the count.
// (A geometric ramp at both ends of the pipeline measured slower on B200 +
// PCIe Gen5: every extra chunk costs more than the fill it saves.)
int chunk_schedule(int64_t num_elements, int64_t base, int64_t* sizes)
{
    if (base <= 0 || base > num_elements) base = num_elements;
    if ((num_elements + base - 1) / base > kMaxChunks)
        base = (num_elements + kMaxChunks - 1) / kMaxChunks;
    int k = 0;
    for (int64_t e0 = 0; e0 < num_elements; e0 += base)
        sizes[k++] = (e0 + base < num_elements) ? base : num_elements - e0;
    return k;
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
    // Which side of the link each field crosses by copy engine and which by
    // the kernel's own loads/stores of mapped page-locked memory (UVA).
    // Pageable buffers have no device mapping and always use the copy engine.
    // read per call (tests switch it between calls): one environment lookup
    int mode = kHostMode;
    if (const char* env = getenv("SEM_HOST_MODE")) mode = atoi(env);
    double* u_map = mapped(u_host);
    double* w_map = mapped(w_host);
    const bool zc_in = (mode == 1 || mode == 3) && u_map;
    const bool zc_out = (mode == 1 || mode == 2) && w_map;
    if (zc_in && zc_out) {  // one launch: PCIe reads and writes of all elements overlap
        // n = 10: each element's w leaves by ONE bulk (TMA) store -- larger
        // PCIe write packets than per-thread stores (tools/wbulk_probe.py:
        // 0.894 vs 0.904 ms; on device memory the bulk store is 5% slower,
        // so device-resident calls keep the default)
        const int zv = (n == 10) ? 63 : 0;
        return ax_dispatch(u_map, g, dx, w_map, num_elements, n, zv, s, 1);  // no L2 prefetch of host memory
    }
    int64_t sizes[kMaxChunks];
    const int nchunks = chunk_schedule(num_elements, chunk_elements, sizes);
    cudaError_t err;
    // the copy streams start after everything already queued on `stream`
    // (only the copy streams this mode uses join: inside CUDA-graph capture a
    // stream that waits on the capture and never rejoins it is an error)
    err = cudaEventRecord(P->ev[0], s);
    if (err == cudaSuccess && !zc_in) err = cudaStreamWaitEvent(P->s_in, P->ev[0], 0);
    if (err == cudaSuccess && !zc_out) err = cudaStreamWaitEvent(P->s_out, P->ev[0], 0);
    if (err != cudaSuccess) return fail_cuda(err, "sem_ax_host: ordering");
    int64_t e0 = 0;
    for (int c = 0; c < nchunks; ++c) {
        const int64_t e1 = e0 + sizes[c];
        const int64_t a = e0 * per;
        const size_t bytes = (size_t)((e1 - e0) * per) * sizeof(double);
        cudaEvent_t ev_in = P->ev[2 + 2 * c], ev_k = P->ev[3 + 2 * c];
        const double* ku = zc_in ? u_map + a : u_dev + a;
        double* kw = zc_out ? w_map + a : w_dev + a;
        if (!zc_in) {
            err = cudaMemcpyAsync(u_dev + a, u_host + a, bytes, cudaMemcpyHostToDevice, P->s_in);
            if (err == cudaSuccess) err = cudaEventRecord(ev_in, P->s_in);
            if (err == cudaSuccess) err = cudaStreamWaitEvent(s, ev_in, 0);
            if (err != cudaSuccess) return fail_cuda(err, "sem_ax_host: H2D");
        }
        const int cv = (zc_out && n == 10) ? 63 : 0;  // bulk-stored w into mapped memory
        if (int rc = ax_dispatch(ku, g + e0 * 6 * per, dx, kw, e1 - e0, n, cv, s)) return rc;
        if (!zc_out) {
            err = cudaEventRecord(ev_k, s);
            if (err == cudaSuccess) err = cudaStreamWaitEvent(P->s_out, ev_k, 0);
            if (err == cudaSuccess)
                err = cudaMemcpyAsync(w_host + a, w_dev + a, bytes, cudaMemcpyDeviceToHost,
                                      P->s_out);
            if (err != cudaSuccess) return fail_cuda(err, "sem_ax_host: D2H");
        }
        e0 = e1;
    }
    if (zc_out) return 0;  // the kernels on `stream` wrote w_host themselves
    // the caller's stream completes only when the last D2H has landed
    err = cudaEventRecord(P->ev[1], P->s_out);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(s, P->ev[1], 0);
    if (err != cudaSuccess) return fail_cuda(err, "sem_ax_host: completion");
    return 0;
}
