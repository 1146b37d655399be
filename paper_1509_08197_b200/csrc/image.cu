// Image-side kernels: uint8 -> f64, pyramid block mean, prepared planes,
// dense matching cost, grid edge weights/keys.  All HBM-bound streaming
// kernels: one thread per output element, coalesced along the row.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <chrono>
#include <cstdlib>

#include "common.cuh"
#include "prims.cuh"

namespace hdp {

static thread_local char g_err[1024] = "";

void keep_pool_memory() {
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        // no hidden cross-stream waits: the pool may otherwise hand a block
        // freed on one stream (the HDP prior's side stream, say) to another
        // after inserting a wait on the first stream's pending work, which
        // stalls the level loop behind a long kernel it never depends on
        int no = 0;
        cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
    }
    done_dev = dev;
}

}  // namespace hdp
// Grow the stream-ordered pool once to `bytes` (allocate and free one block):
// the pool keeps what it has (keep_pool_memory), so later allocations up to
// that size are carved from memory the process already owns instead of going
// to the driver for new physical memory in the middle of a step.
extern "C" int hdp_pool_reserve(int64_t bytes, void* stream) {
    hdp::keep_pool_memory();
    if (bytes <= 0) return HDP_OK;
    void* p = nullptr;
    HDP_CHECK_CUDA(cudaMallocAsync(&p, (size_t)bytes, (cudaStream_t)stream));
    HDP_CHECK_CUDA(cudaFreeAsync(p, (cudaStream_t)stream));
    HDP_CHECK_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    return HDP_OK;
}
namespace hdp {
static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

double Tracer::now_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch()).count();
}
Tracer::Tracer(cudaStream_t s) : st(s) {
    const char* e = getenv("HDP_TRACE");
    on = e && e[0] == '1';
    if (on) {
        cudaStreamSynchronize(st);
        last = now_ms();
    }
}
void Tracer::mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    double t = now_ms();
    fprintf(stderr, "[hdp] %-28s %8.3f ms\n", what, t - last);
    last = t;
}

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

// numpy add.reduce / reduceat order for a short run: first element seeds the
// accumulator, the rest is numpy's pairwise_sum (sequential below 8, eight
// accumulators up to 128).  treestereo pyramid.py:71 (np.add.reduceat).
__device__ __forceinline__ double np_sum_run(const double* a, int n, int64_t stride) {
    if (n <= 0) return 0.0;
    double first = a[0];
    int m = n - 1;
    const double* r = a + stride;
    double rest;
    if (m < 8) {
        rest = 0.0;
        for (int i = 0; i < m; i++) rest = __dadd_rn(rest, r[i * stride]);
    } else {
        double acc[8];
        for (int j = 0; j < 8; j++) acc[j] = r[j * stride];
        int i = 8;
        for (; i < m - (m % 8); i += 8)
            for (int j = 0; j < 8; j++) acc[j] = __dadd_rn(acc[j], r[(i + j) * stride]);
        rest = __dadd_rn(__dadd_rn(__dadd_rn(acc[0], acc[1]), __dadd_rn(acc[2], acc[3])),
                         __dadd_rn(__dadd_rn(acc[4], acc[5]), __dadd_rn(acc[6], acc[7])));
        for (; i < m; i++) rest = __dadd_rn(rest, r[i * stride]);
    }
    return __dadd_rn(first, rest);
}

__global__ void k_u8_to_f64(const uint8_t* __restrict__ src, double* __restrict__ dst, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = (double)src[i];
}

// Row pass of block_mean: rows[b, i, x, k] = reduceat over rows i*S..
__global__ void k_block_rows(const double* __restrict__ src, double* __restrict__ rows, int batch,
                             int h, int w, int c, int s, int oh) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = (int64_t)batch * oh * w * c;
    if (t >= total) return;
    int k = t % c;
    int64_t rest = t / c;
    int x = rest % w;
    rest /= w;
    int i = rest % oh;
    int b = rest / oh;
    int r0 = i * s;
    int r1 = min(r0 + s, h);
    const double* base = src + (((int64_t)b * h + r0) * w + x) * c + k;
    rows[t] = np_sum_run(base, r1 - r0, (int64_t)w * c);
}

__global__ void k_block_cols(const double* __restrict__ rows, double* __restrict__ dst, int batch,
                             int h, int w, int c, int s, int oh, int ow) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = (int64_t)batch * oh * ow * c;
    if (t >= total) return;
    int k = t % c;
    int64_t rest = t / c;
    int j = rest % ow;
    rest /= ow;
    int i = rest % oh;
    int b = rest / oh;
    int c0 = j * s, c1 = min(c0 + s, w);
    int rc = min(s, h - i * s);
    const double* base = rows + (((int64_t)b * oh + i) * w + c0) * c + k;
    double sum = np_sum_run(base, c1 - c0, c);
    dst[t] = __ddiv_rn(sum, (double)(rc * (c1 - c0)));
}

__device__ __forceinline__ double gray_at(const double* px, int c) {
    if (c == 3) {
        double u0 = __ddiv_rn(px[0], 255.0), u1 = __ddiv_rn(px[1], 255.0),
               u2 = __ddiv_rn(px[2], 255.0);
        // OpenBLAS dgemv order of `unit @ GRAY_WEIGHTS` (cost_volume.py:65)
        return __fma_rn(u2, 0.114, __fma_rn(u0, 0.299, __dmul_rn(u1, 0.587)));
    }
    return __ddiv_rn(px[0], 255.0);
}

// prepare_layer (cost_volume.py:62-69), one thread per pixel.
__global__ void k_prepare(const double* __restrict__ img, int batch, int h, int w, int c,
                          double* __restrict__ unit, double* __restrict__ gray,
                          double* __restrict__ grad, float4* __restrict__ packed) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t n = (int64_t)batch * h * w;
    if (t >= n) return;
    int x = t % w;
    const double* px = img + t * c;
    double u[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < c; k++) u[k] = __ddiv_rn(px[k], 255.0);
    double g;
    if (w == 1) {
        g = 0.0;
    } else if (x == 0) {
        g = __dsub_rn(gray_at(px + c, c), gray_at(px, c));
    } else if (x == w - 1) {
        g = __dsub_rn(gray_at(px, c), gray_at(px - c, c));
    } else {
        g = __ddiv_rn(__dsub_rn(gray_at(px + c, c), gray_at(px - c, c)), 2.0);
    }
    if (unit)
        for (int k = 0; k < c; k++) unit[t * c + k] = u[k];
    if (grad) grad[t] = g;
    if (gray) gray[t] = gray_at(px, c);
    if (packed) packed[t] = make_float4((float)u[0], (float)u[1], (float)u[2], (float)g);
}

// prepare_layer from uint8 directly (the pipeline's level 0): unit = RN(I/255)
// from a 256-entry table built with the same IEEE division, gray and the
// central-difference gradient in k_prepare's exact operation order, so the
// packed plane is bit-identical to u8 -> f64 -> k_prepare.
__device__ __forceinline__ double gray_lut(const uint8_t* px, int c, const double* lut) {
    if (c == 3) return __fma_rn(lut[px[2]], 0.114, __fma_rn(lut[px[0]], 0.299, __dmul_rn(lut[px[1]], 0.587)));
    return lut[px[0]];
}
__global__ void __launch_bounds__(256) k_prepare_u8(const uint8_t* __restrict__ img, int batch, int h, int w,
                                                    int c, float4* __restrict__ packed) {
    __shared__ double lut[256];
    lut[threadIdx.x] = __ddiv_rn((double)threadIdx.x, 255.0);
    __syncthreads();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = (int64_t)batch * h * w;
    if (t >= n) return;
    const int x = (int)(t % w);
    const uint8_t* px = img + t * c;
    double g;
    if (w == 1) {
        g = 0.0;
    } else if (x == 0) {
        g = __dsub_rn(gray_lut(px + c, c, lut), gray_lut(px, c, lut));
    } else if (x == w - 1) {
        g = __dsub_rn(gray_lut(px, c, lut), gray_lut(px - c, c, lut));
    } else {
        g = __ddiv_rn(__dsub_rn(gray_lut(px + c, c, lut), gray_lut(px - c, c, lut)), 2.0);
    }
    const double u0 = lut[px[0]];
    const double u1 = c == 3 ? lut[px[1]] : 0.0, u2 = c == 3 ? lut[px[2]] : 0.0;
    packed[t] = make_float4((float)u0, (float)u1, (float)u2, (float)g);
}

// build_edge_list from uint8 (weights = max channel |difference|, integers:
// exactly k_grid_edges' values)
__global__ void k_grid_edges_u8(const uint8_t* __restrict__ img, int batch, int h, int w, int c,
                                int32_t* __restrict__ eu, int32_t* __restrict__ ev, float* __restrict__ ew,
                                uint64_t* __restrict__ key) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t n = (int64_t)h * w;
    if (t >= (int64_t)batch * n) return;
    int b = t / n;
    int64_t p = t % n;
    int r = p / w, col = p % w;
    int64_t E = 2 * n - h - w;
    int64_t ebase = (int64_t)b * E;
    const uint8_t* px = img + t * c;
    if (col + 1 < w) {
        int m = 0;
        for (int k = 0; k < c; k++) m = max(m, abs((int)px[k] - (int)px[c + k]));
        int64_t idx = (r < h - 1) ? (int64_t)r * (2 * w - 1) + 2 * col : (int64_t)(h - 1) * (2 * w - 1) + col;
        float wf = (float)m;
        eu[ebase + idx] = (int32_t)t;
        ev[ebase + idx] = (int32_t)(t + 1);
        if (ew) ew[ebase + idx] = wf;
        key[ebase + idx] = ((uint64_t)__float_as_uint(wf) << 32) | (uint64_t)idx;
    }
    if (r + 1 < h) {
        int m = 0;
        for (int k = 0; k < c; k++) m = max(m, abs((int)px[k] - (int)px[(int64_t)w * c + k]));
        int64_t idx = (int64_t)r * (2 * w - 1) + 2 * col + (col < w - 1 ? 1 : 0);
        float wf = (float)m;
        eu[ebase + idx] = (int32_t)t;
        ev[ebase + idx] = (int32_t)(t + w);
        if (ew) ew[ebase + idx] = wf;
        key[ebase + idx] = ((uint64_t)__float_as_uint(wf) << 32) | (uint64_t)idx;
    }
}

__device__ __forceinline__ float cost_f32(float4 L, float4 R, int c, float alpha, float tc,
                                          float tg) {
    float color;
    if (c == 3)
        color = (fabsf(L.x - R.x) + fabsf(L.y - R.y) + fabsf(L.z - R.z)) * (1.0f / 3.0f);
    else
        color = fabsf(L.x - R.x);
    float gd = fabsf(L.w - R.w);
    return (1.0f - alpha) * fminf(tc, color) + alpha * fminf(tg, gd);
}

// Dense cost (cost_grid over xs), disparity innermost; a warp covers 32
// consecutive disparities of one pixel so the store is coalesced.
__global__ void k_cost_volume(const float4* __restrict__ pl, const float4* __restrict__ pr,
                              int batch, int h, int w, int c, const int32_t* __restrict__ xs,
                              int nx, float alpha, float tc, float tg, float* __restrict__ out) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = (int64_t)batch * h * w * nx;
    if (t >= total) return;
    int j = t % nx;
    int64_t g = t / nx;
    int col = g % w;
    int x = xs[j];
    float border = (1.0f - alpha) * tc + alpha * tg;
    float v = border;
    if (col - x >= 0) v = cost_f32(pl[g], pr[g - x], c, alpha, tc, tg);
    out[t] = v;
}

// Grid edges in the reference scan order (spanning_forest.py:61-93).
__global__ void k_grid_edges(const double* __restrict__ img, int batch, int h, int w, int c,
                             int32_t* __restrict__ eu, int32_t* __restrict__ ev,
                             float* __restrict__ ew, uint64_t* __restrict__ key) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t n = (int64_t)h * w;
    if (t >= (int64_t)batch * n) return;
    int b = t / n;
    int64_t p = t % n;
    int r = p / w, col = p % w;
    int64_t E = 2 * n - h - w;
    int64_t ebase = (int64_t)b * E;
    const double* px = img + t * c;
    if (col + 1 < w) {
        double m = 0.0;
        for (int k = 0; k < c; k++) m = fmax(m, fabs(px[k] - px[c + k]));
        int64_t idx = (r < h - 1) ? (int64_t)r * (2 * w - 1) + 2 * col
                                  : (int64_t)(h - 1) * (2 * w - 1) + col;
        float wf = (float)m;
        eu[ebase + idx] = (int32_t)t;
        ev[ebase + idx] = (int32_t)(t + 1);
        if (ew) ew[ebase + idx] = wf;
        key[ebase + idx] = ((uint64_t)__float_as_uint(wf) << 32) | (uint64_t)idx;
    }
    if (r + 1 < h) {
        double m = 0.0;
        for (int k = 0; k < c; k++) m = fmax(m, fabs(px[k] - px[(int64_t)w * c + k]));
        int64_t idx = (int64_t)r * (2 * w - 1) + 2 * col + (col < w - 1 ? 1 : 0);
        float wf = (float)m;
        eu[ebase + idx] = (int32_t)t;
        ev[ebase + idx] = (int32_t)(t + w);
        if (ew) ew[ebase + idx] = wf;
        key[ebase + idx] = ((uint64_t)__float_as_uint(wf) << 32) | (uint64_t)idx;
    }
}

__global__ void k_iota32(int64_t n, int32_t* a) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int32_t)i;
}

// keys of hdp_aggregate_wta: u64 = ord(f32 cost) << 32 | d, ord the
// order-preserving map of IEEE floats onto u32; with signed_order the top bit
// is flipped so that int64 order equals u64 order (NCCL reduces int64)
__global__ void k_keys_unpack(const uint64_t* __restrict__ keys, int64_t n, int signed_order, int32_t* disp,
                              float* min_cost) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    uint64_t k = keys[t] ^ (signed_order ? 0x8000000000000000ull : 0ull);
    uint32_t u = (uint32_t)(k >> 32);
    // inverse of the order-preserving encoding used by hdp_aggregate_wta
    uint32_t b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
    if (disp) disp[t] = (int32_t)(k & 0xffffffffu);
    if (min_cost) min_cost[t] = __uint_as_float(b);
}

__global__ void k_keys_pack(const int32_t* __restrict__ disp, const float* __restrict__ min_cost, int64_t n,
                            int signed_order, uint64_t* __restrict__ keys) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    uint32_t b = __float_as_uint(min_cost[t]);
    uint32_t o = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    uint64_t k = ((uint64_t)o << 32) | (uint32_t)disp[t];
    keys[t] = k ^ (signed_order ? 0x8000000000000000ull : 0ull);
}

}  // namespace hdp

using namespace hdp;

extern "C" {

int hdp_abi_version(void) { return HDP_ABI_VERSION; }

int64_t hdp_launch_count(void) { return (int64_t)launch_count(); }

const char* hdp_last_error(void) { return g_err; }

int hdp_u8_to_f64(const uint8_t* src, double* dst, int64_t n, void* stream) {
    if (n <= 0) return HDP_OK;
    k_u8_to_f64<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(src, dst, n); note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

int hdp_block_mean(const double* src, double* dst, int batch, int h, int w, int c, int s,
                   void* stream) {
    HDP_REQUIRE(s >= 2 && s <= 129, HDP_ERR_CONFIG, "block_size must be in [2, 129], got %d", s);
    HDP_REQUIRE(batch >= 1 && h >= 1 && w >= 1 && c >= 1, HDP_ERR_DATA, "empty image");
    cudaStream_t st = (cudaStream_t)stream;
    int oh = (h + s - 1) / s, ow = (w + s - 1) / s;
    DevBuf<double> rows;
    HDP_TRY(rows.alloc((size_t)batch * oh * w * c, st));
    int64_t n1 = (int64_t)batch * oh * w * c;
    k_block_rows<<<grid_for(n1, 256), 256, 0, st>>>(src, rows.get(), batch, h, w, c, s, oh); note_launch();
    HDP_CHECK_LAUNCH();
    int64_t n2 = (int64_t)batch * oh * ow * c;
    k_block_cols<<<grid_for(n2, 256), 256, 0, st>>>(rows.get(), dst, batch, h, w, c, s, oh, ow); note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

int hdp_prepare(const double* img, int batch, int h, int w, int c, double* unit, double* gray,
                double* grad, float* packed, void* stream) {
    HDP_REQUIRE(c == 1 || c == 3, HDP_ERR_DATA, "channels must be 1 or 3, got %d", c);
    int64_t n = (int64_t)batch * h * w;
    if (n <= 0) return HDP_OK;
    k_prepare<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(img, batch, h, w, c, unit,
                                                                   gray, grad, (float4*)packed); note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

int hdp_prepare_u8(const uint8_t* img, int batch, int h, int w, int c, float* packed, void* stream) {
    HDP_REQUIRE(c == 1 || c == 3, HDP_ERR_DATA, "channels must be 1 or 3, got %d", c);
    int64_t n = (int64_t)batch * h * w;
    if (n <= 0) return HDP_OK;
    k_prepare_u8<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(img, batch, h, w, c, (float4*)packed);
    note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

int hdp_grid_edges_u8(const uint8_t* img, int batch, int h, int w, int c, int32_t* eu, int32_t* ev, float* ew,
                      uint64_t* key, void* stream) {
    int64_t n = (int64_t)h * w;
    HDP_REQUIRE(2 * n - h - w < ((int64_t)1 << 32), HDP_ERR_CONFIG, "too many edges per pair");
    HDP_REQUIRE((int64_t)batch * n < ((int64_t)1 << 31), HDP_ERR_CONFIG, "too many nodes");
    if (batch * n <= 0) return HDP_OK;
    k_grid_edges_u8<<<grid_for(batch * n, 256), 256, 0, (cudaStream_t)stream>>>(img, batch, h, w, c, eu, ev, ew,
                                                                                key); note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

int hdp_cost_volume(const float* packed_l, const float* packed_r, int batch, int h, int w, int c,
                    const int32_t* xs, int nx, float alpha, float tau_c, float tau_g, float* out,
                    void* stream) {
    HDP_REQUIRE(c == 1 || c == 3, HDP_ERR_DATA, "channels must be 1 or 3, got %d", c);
    int64_t total = (int64_t)batch * h * w * nx;
    if (total <= 0) return HDP_OK;
    k_cost_volume<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(
        (const float4*)packed_l, (const float4*)packed_r, batch, h, w, c, xs, nx, alpha, tau_c,
        tau_g, out); note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

int hdp_grid_edges(const double* img, int batch, int h, int w, int c, int32_t* eu, int32_t* ev,
                   float* ew, uint64_t* key, void* stream) {
    int64_t n = (int64_t)h * w;
    HDP_REQUIRE(2 * n - h - w < ((int64_t)1 << 32), HDP_ERR_CONFIG, "too many edges per pair");
    HDP_REQUIRE((int64_t)batch * n < ((int64_t)1 << 31), HDP_ERR_CONFIG, "too many nodes");
    if (batch * n <= 0) return HDP_OK;
    k_grid_edges<<<grid_for(batch * n, 256), 256, 0, (cudaStream_t)stream>>>(img, batch, h, w, c,
                                                                             eu, ev, ew, key); note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

int hdp_argsort_u64(const uint64_t* keys, int64_t n, int32_t* perm, void* stream) {
    HDP_REQUIRE(n >= 0 && n < ((int64_t)1 << 31), HDP_ERR_CONFIG, "bad key count");
    if (n == 0) return HDP_OK;
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf<uint64_t> kout;
    DevBuf<int32_t> idx;
    HDP_TRY(kout.alloc(n, st));
    HDP_TRY(idx.alloc(n, st));
    k_iota32<<<grid_for(n, 256), 256, 0, st>>>(n, idx.get()); note_launch();
    HDP_CHECK_LAUNCH();
    return sort_pairs(keys, kout.get(), idx.get(), perm, n, 0, 64, st);
}

int hdp_keys_unpack(const uint64_t* keys, int64_t n, int signed_order, int32_t* disp, float* min_cost,
                    void* stream) {
    if (n <= 0) return HDP_OK;
    k_keys_unpack<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(keys, n, signed_order, disp, min_cost);
    note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

int hdp_keys_pack(const int32_t* disp, const float* min_cost, int64_t n, int signed_order, uint64_t* keys,
                  void* stream) {
    if (n <= 0) return HDP_OK;
    HDP_REQUIRE(disp && min_cost && keys, HDP_ERR_CONFIG, "null buffer");
    k_keys_pack<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(disp, min_cost, n, signed_order, keys);
    note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

}  // extern "C"
