// runtime.cu -- device runtime of the targetDP layer: allocation, copies,
// streams, events and syncTarget with the deferred kernel error word.
//
// Reference counterparts: target_malloc/target_free/copy_to_target/
// copy_from_target (pkg/src/latkit/memory.py:231-274) and sync_target
// (pkg/src/latkit/execution.py:271-281).  The reference's "target" is a host
// arena; here it is B200 HBM.
#include <atomic>
#include <map>
#include <utility>
#include <climits>
#include <cstring>
#include <mutex>

#include "ltk_common.cuh"

namespace ltk {

static thread_local char g_msg[512] = "";
static std::atomic<long long> g_launches{0};

int fail(int status, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_msg, sizeof g_msg, fmt, ap);
    va_end(ap);
    return status;
}

int cuda_fail(cudaError_t err, const char *what) {
    snprintf(g_msg, sizeof g_msg, "%s: %s (%s)", what, cudaGetErrorString(err),
             cudaGetErrorName(err));
    return err == cudaErrorMemoryAllocation ? LTK_ERR_ALLOC : LTK_ERR_DEVICE;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// One error word per (device, stream), allocated on first use.
static std::mutex g_word_mu;
static std::map<std::pair<int, cudaStream_t>, long long *> g_words;

long long *stream_word(cudaStream_t st) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lk(g_word_mu);
    auto key = std::make_pair(dev, st);
    auto it = g_words.find(key);
    if (it != g_words.end()) return it->second;
    long long *w = nullptr;
    if (cudaMalloc(&w, sizeof(long long)) != cudaSuccess) return nullptr;
    // zeroed in stream order, before any kernel of `st` can use it
    if (cudaMemsetAsync(w, 0, sizeof(long long), st) != cudaSuccess) {
        cudaFree(w);
        return nullptr;
    }
    g_words[key] = w;
    return w;
}

void release_stream_word(cudaStream_t st) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    std::lock_guard<std::mutex> lk(g_word_mu);
    auto it = g_words.find(std::make_pair(dev, st));
    if (it == g_words.end()) return;
    cudaFree(it->second);
    g_words.erase(it);
}

int take_word(long long *word, cudaStream_t st, long long *site) {
    *site = -1;
    long long v = 0;
    LTK_CUDA(cudaMemcpyAsync(&v, word, sizeof v, cudaMemcpyDeviceToHost, st));
    LTK_CUDA(cudaStreamSynchronize(st));
    if (v != 0) {
        LTK_CUDA(cudaMemsetAsync(word, 0, sizeof v, st));
        LTK_CUDA(cudaStreamSynchronize(st));
        *site = LLONG_MAX - v;
    }
    return LTK_OK;
}

}  // namespace ltk

using namespace ltk;

extern "C" {

int ltk_abi_version(void) { return LTK_ABI_VERSION; }
const char *ltk_last_error(void) { return g_msg; }
int64_t ltk_launch_count(void) { return g_launches.load(); }

int ltk_device_count(int *count) {
    LTK_CUDA(cudaGetDeviceCount(count));
    return LTK_OK;
}

int ltk_set_device(int device) {
    LTK_CUDA(cudaSetDevice(device));
    return LTK_OK;
}

int ltk_get_device(int *device) {
    LTK_CUDA(cudaGetDevice(device));
    return LTK_OK;
}

int ltk_device_info(int device, char *name, int *sm_count, int64_t *total_mem, int *cc_major,
                    int *cc_minor) {
    cudaDeviceProp prop;
    LTK_CUDA(cudaGetDeviceProperties(&prop, device));
    if (name) {
        strncpy(name, prop.name, 255);
        name[255] = 0;
    }
    if (sm_count) *sm_count = prop.multiProcessorCount;
    if (total_mem) *total_mem = (int64_t)prop.totalGlobalMem;
    if (cc_major) *cc_major = prop.major;
    if (cc_minor) *cc_minor = prop.minor;
    return LTK_OK;
}

int ltk_malloc(void **ptr, size_t bytes) {
    *ptr = nullptr;
    if (bytes == 0) bytes = 256;
    cudaError_t e = cudaMalloc(ptr, bytes);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        *ptr = nullptr;
        return fail(LTK_ERR_ALLOC, "cudaMalloc of %zu bytes failed: %s", bytes,
                    cudaGetErrorString(e));
    }
    // target_malloc zero-initialises (memory.py:231-241).  cudaMemset runs on
    // the legacy stream, which does not order against the library's
    // non-blocking streams: wait for it, or a later copy on another stream
    // could be overwritten by the late zero fill.
    LTK_CUDA(cudaMemset(*ptr, 0, bytes));
    LTK_CUDA(cudaStreamSynchronize(0));
    return LTK_OK;
}

int ltk_free(void *ptr) {
    LTK_CUDA(cudaFree(ptr));
    return LTK_OK;
}

int ltk_mem_info(size_t *free_bytes, size_t *total_bytes) {
    LTK_CUDA(cudaMemGetInfo(free_bytes, total_bytes));
    return LTK_OK;
}

int ltk_memset0(void *ptr, size_t bytes, void *stream) {
    LTK_CUDA(cudaMemsetAsync(ptr, 0, bytes, as_stream(stream)));
    return LTK_OK;
}

int ltk_h2d(void *dst, const void *src, size_t bytes, void *stream) {
    LTK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, as_stream(stream)));
    return LTK_OK;
}

int ltk_d2h(void *dst, const void *src, size_t bytes, void *stream) {
    LTK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, as_stream(stream)));
    return LTK_OK;
}

int ltk_d2d(void *dst, const void *src, size_t bytes, void *stream) {
    LTK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, as_stream(stream)));
    return LTK_OK;
}

int ltk_host_register(void *ptr, size_t bytes) {
    LTK_CUDA(cudaHostRegister(ptr, bytes, cudaHostRegisterDefault));
    return LTK_OK;
}

int ltk_host_unregister(void *ptr) {
    LTK_CUDA(cudaHostUnregister(ptr));
    return LTK_OK;
}

int ltk_host_alloc(void **ptr, size_t bytes) {
    LTK_CUDA(cudaMallocHost(ptr, bytes));
    return LTK_OK;
}

int ltk_host_free(void *ptr) {
    LTK_CUDA(cudaFreeHost(ptr));
    return LTK_OK;
}

int ltk_stream_create(void **stream) {
    cudaStream_t s;
    LTK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    *stream = s;
    return LTK_OK;
}

int ltk_stream_destroy(void *stream) {
    LTK_CUDA(cudaStreamSynchronize(as_stream(stream)));
    release_stream_word(as_stream(stream));
    LTK_CUDA(cudaStreamDestroy(as_stream(stream)));
    return LTK_OK;
}

int ltk_stream_sync(void *stream) {
    LTK_CUDA(cudaStreamSynchronize(as_stream(stream)));
    return LTK_OK;
}

int ltk_event_create(void **event, int timing) {
    cudaEvent_t e;
    LTK_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
    *event = e;
    return LTK_OK;
}

int ltk_event_destroy(void *event) {
    LTK_CUDA(cudaEventDestroy(reinterpret_cast<cudaEvent_t>(event)));
    return LTK_OK;
}

int ltk_event_record(void *event, void *stream) {
    LTK_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(event), as_stream(stream)));
    return LTK_OK;
}

int ltk_event_query(void *event, int *done) {
    cudaError_t e = cudaEventQuery(reinterpret_cast<cudaEvent_t>(event));
    if (e == cudaSuccess) {
        *done = 1;
        return LTK_OK;
    }
    if (e == cudaErrorNotReady) {
        (void)cudaGetLastError();
        *done = 0;
        return LTK_OK;
    }
    return cuda_fail(e, "cudaEventQuery");
}

int ltk_event_sync(void *event) {
    LTK_CUDA(cudaEventSynchronize(reinterpret_cast<cudaEvent_t>(event)));
    return LTK_OK;
}

int ltk_event_elapsed(void *start, void *stop, float *ms) {
    LTK_CUDA(cudaEventElapsedTime(ms, reinterpret_cast<cudaEvent_t>(start),
                                  reinterpret_cast<cudaEvent_t>(stop)));
    return LTK_OK;
}

int ltk_stream_wait_event(void *stream, void *event) {
    LTK_CUDA(cudaStreamWaitEvent(as_stream(stream), reinterpret_cast<cudaEvent_t>(event), 0));
    return LTK_OK;
}

int ltk_sync(void *stream, int64_t *site) {
    *site = -1;
    cudaStream_t st = as_stream(stream);
    LTK_CUDA(cudaStreamSynchronize(st));
    long long *w = stream_word(st);
    if (!w) return fail(LTK_ERR_DEVICE, "stream error word unavailable");
    long long v = -1;
    LTK_RC0(take_word(w, st, &v));
    if (v >= 0) {
        *site = v;
        return fail(LTK_ERR_SINGULAR, "rho <= 0 at lattice site %lld", v);
    }
    return LTK_OK;
}

}  // extern "C"
