// Boundary helpers: float64 edge weights for the EdgeList API type, and the
// 3x3 median prefilter of the reference's M+* method variants.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"

namespace hdp {

// spanning_forest.py:61-93 weights in float64 (EdgeList.weight), scan order.
__global__ void k_edge_w64(const double* __restrict__ img, int batch, int h, int w, int c,
                           double* __restrict__ ew) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t n = (int64_t)h * w;
    if (t >= (int64_t)batch * n) return;
    int b = t / n;
    int64_t p = t % n;
    int r = p / w, col = p % w;
    int64_t ebase = (int64_t)b * (2 * n - h - w);
    const double* px = img + t * c;
    if (col + 1 < w) {
        double m = 0.0;
        for (int k = 0; k < c; k++) m = fmax(m, fabs(px[k] - px[c + k]));
        int64_t idx = (r < h - 1) ? (int64_t)r * (2 * w - 1) + 2 * col
                                  : (int64_t)(h - 1) * (2 * w - 1) + col;
        ew[ebase + idx] = m;
    }
    if (r + 1 < h) {
        double m = 0.0;
        for (int k = 0; k < c; k++) m = fmax(m, fabs(px[k] - px[(int64_t)w * c + k]));
        ew[ebase + (int64_t)r * (2 * w - 1) + 2 * col + (col < w - 1 ? 1 : 0)] = m;
    }
}

// apply_median_prefilter (spanning_forest.py:342-347): scipy.ndimage
// median_filter size 3, mode "reflect" (half-sample symmetric: index -1 reads
// index 0), per channel.  Integer exact.
__global__ void k_median3(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int batch,
                          int h, int w, int c) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = (int64_t)batch * h * w * c;
    if (t >= total) return;
    int k = t % c;
    int64_t pix = t / c;
    int x = pix % w;
    int64_t rest = pix / w;
    int y = rest % h;
    int b = rest / h;
    uint8_t v[9];
    int q = 0;
    for (int dy = -1; dy <= 1; dy++) {
        int yy = min(max(y + dy, 0), h - 1);
        for (int dx = -1; dx <= 1; dx++) {
            int xx = min(max(x + dx, 0), w - 1);
            v[q++] = src[(((int64_t)b * h + yy) * w + xx) * c + k];
        }
    }
    // partial selection: 5 passes of min-extraction give the 5th smallest
    for (int i = 0; i < 5; i++) {
        int mi = i;
        for (int j = i + 1; j < 9; j++)
            if (v[j] < v[mi]) mi = j;
        uint8_t tmp = v[i];
        v[i] = v[mi];
        v[mi] = tmp;
    }
    dst[t] = v[4];
}

// error_rate (evaluation.py:27-54) for a batch: per pair the number of
// evaluated pixels (valid in both maps, not occluded) and, per threshold t,
// how many of them have |pred - gt| >= t.  Integer counts (the percentage is
// formed on the host exactly as the reference does).  One CTA per (pair,
// slice of pixels), block reduction, one atomic per counter per CTA.
constexpr int kMaxThr = 8;
__global__ void k_error_counts(const int32_t* __restrict__ pred, const int32_t* __restrict__ gt,
                               const uint8_t* __restrict__ pvalid, const uint8_t* __restrict__ gvalid,
                               const uint8_t* __restrict__ occ, int64_t npix, const int32_t* __restrict__ thr,
                               int n_thr, unsigned long long* __restrict__ counts) {
    const int b = blockIdx.y;
    unsigned long long c[kMaxThr + 1];
#pragma unroll
    for (int i = 0; i <= kMaxThr; i++) c[i] = 0;
    int th[kMaxThr];
#pragma unroll
    for (int i = 0; i < kMaxThr; i++) th[i] = i < n_thr ? thr[i] : 0x7fffffff;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = (int64_t)b * npix + p;
        bool ev = (!pvalid || pvalid[q]) && (!gvalid || gvalid[q]) && (!occ || !occ[q]);
        if (!ev) continue;
        c[0]++;
        const long long d = (long long)pred[q] - (long long)gt[q];
        const long long ad = d < 0 ? -d : d;
#pragma unroll
        for (int i = 0; i < kMaxThr; i++) c[i + 1] += ad >= th[i] ? 1ull : 0ull;
    }
    __shared__ unsigned long long red[kMaxThr + 1];
    if (threadIdx.x <= kMaxThr) red[threadIdx.x] = 0;
    __syncthreads();
#pragma unroll
    for (int i = 0; i <= kMaxThr; i++) {
        unsigned long long v = c[i];
        for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&red[i], v);
    }
    __syncthreads();
    if (threadIdx.x <= n_thr && red[threadIdx.x]) atomicAdd(&counts[(int64_t)b * (n_thr + 1) + threadIdx.x],
                                                              red[threadIdx.x]);
}

// occlusion_from_gt (evaluation.py:57-76): a valid left pixel with disparity d
// is occluded when c - d is off the image, the right map is invalid there, or
// |d_left - d_right| > 1.  Pixels without left ground truth stay unmarked.
__global__ void k_occlusion(const int32_t* __restrict__ gl, const int32_t* __restrict__ gr,
                            const uint8_t* __restrict__ lvalid, const uint8_t* __restrict__ rvalid, int batch,
                            int h, int w, uint8_t* __restrict__ occ) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = (int64_t)h * w;
    if (t >= (int64_t)batch * n) return;
    const int64_t rowbase = t - (t % n) + ((t % n) / w) * w;  // first pixel of this row
    const int col = (int)((t % n) % w);
    const long long dl = gl[t];
    const long long target = (long long)col - dl;
    bool consistent = false;
    if (target >= 0 && target < w) {
        const int64_t q = rowbase + target;
        const bool rok = !rvalid || rvalid[q];
        const long long dr = gr[q];
        const long long diff = dl - dr;
        consistent = rok && (diff <= 1 && diff >= -1);
    }
    const bool lv = !lvalid || lvalid[t];
    occ[t] = (lv && !consistent) ? 1 : 0;
}

// first minimum of every row of an (n, m) float64 matrix (np.argmin: the
// lowest index among equal minima); one warp per row
__global__ void k_rows_argmin(const double* __restrict__ rows, int64_t n, int m, int32_t* __restrict__ arg,
                              double* __restrict__ best) {
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= n) return;
    double b = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    int bj = 0x7fffffff;
    for (int j = lane; j < m; j += 32) {
        const double v = rows[r * m + j];
        if (v < b) {
            b = v;
            bj = j;
        }
    }
    for (int o = 16; o >= 1; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, b, o);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (ob < b || (ob == b && oj < bj)) {
            b = ob;
            bj = oj;
        }
    }
    if (lane == 0) {
        arg[r] = bj == 0x7fffffff ? 0 : bj;  // a row of +inf only: column 0, as np.argmin
        best[r] = bj == 0x7fffffff ? rows[r * m] : b;
    }
}

// ragged gather of a dense (pixels, ncols) f32 grid: output row r takes pixel
// node[r] and the columns cols[cstart[r] .. cstart[r] + cnt[r]), written as
// float64 at out + off[r]
__global__ void k_gather_ragged(const float* __restrict__ grid, int ncols, int64_t nrows,
                                const int64_t* __restrict__ node, const int64_t* __restrict__ off,
                                const int32_t* __restrict__ cstart, const int32_t* __restrict__ cnt,
                                const int32_t* __restrict__ cols, double* __restrict__ out) {
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= nrows) return;
    const float* src = grid + node[r] * ncols;
    const int32_t* cl = cols + cstart[r];
    double* dst = out + off[r];
    for (int j = lane; j < cnt[r]; j += 32) dst[j] = (double)src[cl[j]];
}

}  // namespace hdp

using namespace hdp;

extern "C" int hdp_error_counts(const int32_t* pred, const int32_t* gt, const uint8_t* pred_valid,
                                const uint8_t* gt_valid, const uint8_t* occlusion, int batch, int64_t npix,
                                const int32_t* thresholds, int n_thr, int64_t* counts, void* stream) {
    HDP_REQUIRE(n_thr >= 1 && n_thr <= kMaxThr, HDP_ERR_CONFIG, "1..%d thresholds, got %d", kMaxThr, n_thr);
    HDP_REQUIRE(pred && gt && thresholds && counts, HDP_ERR_CONFIG, "null buffer");
    cudaStream_t st = (cudaStream_t)stream;
    HDP_CHECK_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * batch * (n_thr + 1), st));
    if (batch <= 0 || npix <= 0) return HDP_OK;
    const unsigned gx = (unsigned)std::min<int64_t>((npix + 255) / 256, 1184);
    k_error_counts<<<dim3(gx, (unsigned)batch), 256, 0, st>>>(pred, gt, pred_valid, gt_valid, occlusion, npix,
                                                             thresholds, n_thr, (unsigned long long*)counts);
    note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

extern "C" int hdp_occlusion_from_gt(const int32_t* gt_left, const int32_t* gt_right, const uint8_t* left_valid,
                                     const uint8_t* right_valid, int batch, int h, int w, uint8_t* occlusion,
                                     void* stream) {
    HDP_REQUIRE(gt_left && gt_right && occlusion, HDP_ERR_CONFIG, "null buffer");
    const int64_t n = (int64_t)batch * h * w;
    if (n <= 0) return HDP_OK;
    k_occlusion<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(gt_left, gt_right, left_valid, right_valid, batch,
                                                                  h, w, occlusion);
    note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

extern "C" int hdp_grid_edge_weights64(const double* img, int batch, int h, int w, int c, double* ew,
                                       void* stream) {
    int64_t n = (int64_t)batch * h * w;
    if (n <= 0) return HDP_OK;
    k_edge_w64<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(img, batch, h, w, c, ew); note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

extern "C" int hdp_median3x3(const uint8_t* src, uint8_t* dst, int batch, int h, int w, int c,
                             void* stream) {
    int64_t n = (int64_t)batch * h * w * c;
    if (n <= 0) return HDP_OK;
    k_median3<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(src, dst, batch, h, w, c); note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

extern "C" int hdp_rows_first_argmin(const double* rows, int64_t n, int m, int32_t* arg, double* best,
                                     void* stream) {
    HDP_REQUIRE(rows && arg && best && m >= 1, HDP_ERR_CONFIG, "null buffer or empty rows");
    if (n <= 0) return HDP_OK;
    k_rows_argmin<<<grid_for(n * 32, 256), 256, 0, (cudaStream_t)stream>>>(rows, n, m, arg, best); note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

extern "C" int hdp_gather_ragged(const float* grid, int ncols, int64_t nrows, const int64_t* node,
                                 const int64_t* off, const int32_t* cstart, const int32_t* cnt,
                                 const int32_t* cols, double* out, void* stream) {
    HDP_REQUIRE(grid && node && off && cstart && cnt && cols && out && ncols >= 1, HDP_ERR_CONFIG, "null buffer");
    if (nrows <= 0) return HDP_OK;
    k_gather_ragged<<<grid_for(nrows * 32, 256), 256, 0, (cudaStream_t)stream>>>(grid, ncols, nrows, node, off, cstart,
                                                                               cnt, cols, out); note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}
