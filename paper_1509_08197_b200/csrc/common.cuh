// Shared helpers for the HDP stereo sm_100a library: status codes, a
// thread-local error message, stream-ordered scratch buffers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/hdp_stereo.h"

namespace hdp {

void set_error(const char* fmt, ...);

struct Status {
    int code = HDP_OK;
};

#define HDP_CHECK_CUDA(expr)                                                          \
    do {                                                                             \
        cudaError_t _e = (expr);                                                     \
        if (_e != cudaSuccess) {                                                     \
            ::hdp::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,              \
                             cudaGetErrorString(_e));                                \
            return HDP_ERR_CUDA;                                                     \
        }                                                                            \
    } while (0)

#define HDP_CHECK_LAUNCH() HDP_CHECK_CUDA(cudaGetLastError())

#define HDP_REQUIRE(cond, code, ...)                                                 \
    do {                                                                             \
        if (!(cond)) {                                                               \
            ::hdp::set_error(__VA_ARGS__);                                           \
            return (code);                                                           \
        }                                                                            \
    } while (0)

#define HDP_TRY(expr)                                                                \
    do {                                                                             \
        int _s = (expr);                                                             \
        if (_s != HDP_OK) return _s;                                                 \
    } while (0)

// Keep freed pool blocks cached across stream synchronisations (the default
// release threshold of 0 would hand every block back to the driver at each
// sync and re-map it on the next allocation).
void keep_pool_memory();

// Process-wide count of this library's kernel launches (diagnostics for the
// bench's gpu_launches claim; CUB launches are not counted).
void note_launch();

// Stream-ordered device scratch (cudaMallocAsync from the device's default
// pool, which caches freed blocks, so steady-state calls do not hit the
// driver allocator).
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        release();
        p = o.p; n = o.n; s = o.s; o.p = nullptr;
        return *this;
    }
    int alloc(size_t count, cudaStream_t stream) {
        release();
        keep_pool_memory();
        s = stream;
        n = count;
        if (count == 0) return HDP_OK;
        HDP_CHECK_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T), stream));
        return HDP_OK;
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
    }
    ~DevBuf() { release(); }
    T* get() const { return p; }
};

// HDP_TRACE=1: host-side timestamps (ms since the previous mark) on stderr,
// synchronising the stream at each mark so the interval is GPU-complete.
struct Tracer {
    bool on = false;
    double last = 0.0;
    cudaStream_t st = nullptr;
    static double now_ms();
    explicit Tracer(cudaStream_t s);
    void mark(const char* what);
};

inline int grid_for(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > (int64_t)1 << 30) g = 1 << 30;
    return (int)g;
}

inline int ceil_log2(int64_t x) {
    int r = 0;
    while (((int64_t)1 << r) < x) r++;
    return r;
}

}  // namespace hdp
