// Error state, device binding and ABI metadata for libsem.
#include <stdarg.h>
#include <string.h>

#include <algorithm>
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

// ------------------------------------------------------- L2 residency --
// Device L2 persistence limits (bytes): the largest set-aside for persisting
// lines and the largest access-policy window.
extern "C" int sem_l2_props(int64_t* persist_max, int64_t* window_max, int64_t* l2_bytes)
{
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev)) return sem::fail_cuda(e, "sem_l2_props: cudaGetDevice");
    int pm = 0, wm = 0, l2 = 0;
    cudaDeviceGetAttribute(&pm, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&wm, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    if (persist_max) *persist_max = pm;
    if (window_max) *window_max = wm;
    if (l2_bytes) *l2_bytes = l2;
    return 0;
}

// Mark [base, base + bytes) as L2-persisting for kernels launched into
// `stream` (and kernels captured from it): hit_ratio of the window's lines
// get the persisting property, the rest stream.  set_aside > 0 sizes the
// device's persisting carve-out (clamped to the device maximum); bytes == 0
// clears the window and releases the persisting lines.
extern "C" int sem_l2_window(void* base, int64_t bytes, double hit_ratio, int64_t set_aside,
                             sem_stream_t stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    if (int rc = sem::bind_stream_device(s)) return rc;
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev)) return sem::fail_cuda(e, "sem_l2_window: cudaGetDevice");
    cudaStreamAttrValue v = {};
    if (bytes > 0) {
        int pm = 0, wm = 0;
        cudaDeviceGetAttribute(&pm, cudaDevAttrMaxPersistingL2CacheSize, dev);
        cudaDeviceGetAttribute(&wm, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        if (set_aside > 0) {
            const size_t sa = (size_t)std::min<int64_t>(set_aside, (int64_t)pm);
            if (cudaError_t e = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, sa))
                return sem::fail_cuda(e, "sem_l2_window: cudaDeviceSetLimit");
        }
        v.accessPolicyWindow.base_ptr = base;
        v.accessPolicyWindow.num_bytes = (size_t)std::min<int64_t>(bytes, (int64_t)wm);
        v.accessPolicyWindow.hitRatio = (float)(hit_ratio < 0 ? 0 : hit_ratio > 1 ? 1 : hit_ratio);
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    } else {
        v.accessPolicyWindow.num_bytes = 0;
        v.accessPolicyWindow.hitProp = cudaAccessPropertyNormal;
        v.accessPolicyWindow.missProp = cudaAccessPropertyNormal;
    }
    if (cudaError_t e = cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v))
        return sem::fail_cuda(e, "sem_l2_window: cudaStreamSetAttribute");
    if (bytes <= 0) {
        if (cudaError_t e = cudaCtxResetPersistingL2Cache())
            return sem::fail_cuda(e, "sem_l2_window: cudaCtxResetPersistingL2Cache");
    }
    return 0;
}
