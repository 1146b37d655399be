// Boundary helpers: float64 edge weights for the EdgeList API type, and the
// 3x3 median prefilter of the reference's M+* method variants.
#include <cuda_runtime.h>

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

}  // namespace hdp

using namespace hdp;

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
