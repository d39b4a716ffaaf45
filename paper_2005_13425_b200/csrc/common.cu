// Error state, device binding and ABI metadata for libsem.
#include <stdarg.h>
#include <string.h>

#include <atomic>

#include "sem_common.cuh"

namespace sem {

static thread_local char g_last_error[512] = "";
static std::atomic<long long> g_fallbacks{0};

void note_fallback() { g_fallbacks.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char* fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
}

int fail_cuda(cudaError_t err, const char* what)
{
    set_error("%s: %s (%s)", what, cudaGetErrorString(err), cudaGetErrorName(err));
    return static_cast<int>(err);
}

int bind_stream_device(cudaStream_t stream)
{
    // The legacy/per-thread default streams belong to the current device.
    if (stream == nullptr || stream == cudaStreamLegacy || stream == cudaStreamPerThread)
        return 0;
    // Fast path: same stream as the previous call on this thread -> its
    // device is already current (no runtime call, so this is also safe
    // inside CUDA-graph capture).
    static thread_local cudaStream_t last_stream = nullptr;
    static thread_local int last_device = -1;
    if (stream == last_stream && last_device >= 0) return 0;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone)
        return 0;  // capturing: the capturing thread already has the right device
    int dev = -1;
    cudaError_t err = cudaStreamGetDevice(stream, &dev);
    if (err != cudaSuccess) return fail_cuda(err, "cudaStreamGetDevice");
    int cur = -1;
    err = cudaGetDevice(&cur);
    if (err != cudaSuccess) return fail_cuda(err, "cudaGetDevice");
    if (cur != dev) {
        err = cudaSetDevice(dev);
        if (err != cudaSuccess) return fail_cuda(err, "cudaSetDevice");
    }
    last_stream = stream;
    last_device = dev;
    return 0;
}

int sm_count()
{
    // cached per device: attribute queries are not needed on the launch path
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return kNumSMsB200;
    if (cache[dev] > 0) return cache[dev];
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
        return kNumSMsB200;
    cache[dev] = n;
    return n;
}

}  // namespace sem

extern "C" int sem_abi_version(void) { return SEM_ABI_VERSION; }
extern "C" const char* sem_last_error(void) { return sem::g_last_error; }
extern "C" int sem_min_points(void) { return 2; }

extern "C" int64_t sem_fallback_count(void) { return (int64_t)sem::g_fallbacks.load(); }
extern "C" int sem_max_points(void) { return 16; }
