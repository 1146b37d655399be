// Sampled disparity prior, float64 bit-exact with the reference.
//
// Replaces estimate_prior's matching part (hdp_model.py:425-470 with
// _window_indices :366-374, _matched_window_cost :377-394, _windowed_wta
// :397-422).  One warp per sample centre: lanes take disparities x, x+32, ...,
// each lane evaluates the window-mean cost in exactly numpy's order
// (sequential 3-channel mean, separate multiply/add, numpy pairwise sum of
// the window, strict '<' over ascending x), and a lexicographic (cost, x)
// shuffle reduction reproduces the reference's first-minimum scan.  The
// cross-checked winners are histogrammed with integer atomics.  FP64 compute
// bound; inputs are L1/L2 resident.
#include <cuda_runtime.h>

#include "common.cuh"

namespace hdp {

struct PriorArgs {
    const double* ul;
    const double* gl;
    const double* ur;
    const double* gr;
    int h, w, c, d_max, stride, window, max_offset;
    int nrc, ncc;  // centre grid
    double one_minus_alpha, alpha, tc, tg, border;
    double inv_c, inv_win;  // RN(1/c), RN(1/window^2) for div_rn_by
    unsigned long long* counts;
    unsigned long long* kept;
    // 7 x 7 path: per pixel a 32-byte record (u0, u1, u2, grad) of each image
    // (channels past C unused), stored as two planes of 16-byte halves so
    // that 32 lanes reading 32 consecutive pixels touch 512 contiguous bytes
    const double2* pl;  // left: (u0, u1) plane, then the (u2, grad) plane
    const double2* pr;
    int64_t plane;      // elements per plane
    // filter-and-verify (7 x 7, d_max < 256): the same records rounded to f32
    const float4* pl32;
    const float4* pr32;
    float eps32;        // f32 window means within eps32 of the f32 minimum are verified in f64
    // u8 filter records (level 0: every unit value is k / 255): (packed channel bytes, f32 gradient);
    // *nonint != 0 when some value is not a multiple of 1 / 255 (the kernel then filters from pl32)
    const uint2* pl8;
    const uint2* pr8;
    const int* nonint;
};

__global__ void k_pack_px(const double* __restrict__ u, const double* __restrict__ g, int64_t n, int c,
                          double2* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = make_double2(u[i * c], c > 1 ? u[i * c + 1] : 0.0);
    out[n + i] = make_double2(c > 2 ? u[i * c + 2] : 0.0, g[i]);
}

// All three record sets of one image in one pass over its planes (the
// default 7 x 7 filter path): f64 planes, f32 records, byte records.
__global__ void k_pack_all(const double* __restrict__ u, const double* __restrict__ g, int64_t n, int c,
                           double2* __restrict__ out64, float4* __restrict__ out32, uint2* __restrict__ out8,
                           int* __restrict__ nonint) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double u0 = u[i * c], u1 = c > 1 ? u[i * c + 1] : 0.0, u2 = c > 2 ? u[i * c + 2] : 0.0, gg = g[i];
    out64[i] = make_double2(u0, u1);
    out64[n + i] = make_double2(u2, gg);
    out32[i] = make_float4((float)u0, (float)u1, (float)u2, (float)gg);
    if (out8) {
        const double v[3] = {u0 * 255.0, u1 * 255.0, u2 * 255.0};
        unsigned pk = 0;
        bool bad = false;
        for (int k = 0; k < c; k++) {
            const double r = rint(v[k]);
            bad = bad || !(fabs(v[k] - r) <= 1e-9) || r < 0.0 || r > 255.0;
            pk |= (unsigned)(bad ? 0 : (int)r) << (8 * k);
        }
        out8[i] = make_uint2(pk, __float_as_uint((float)gg));
        if (bad) *nonint = 1;
    }
}

// 3 channels, two pixels per thread with 16-byte loads and stores (the planes
// are 16-byte aligned: cudaMalloc'd / torch tensors); n even
__global__ void k_pack_px3(const double2* __restrict__ u, const double2* __restrict__ g, int64_t n2,
                           double2* __restrict__ out, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n2) return;
    const double2 a = __ldg(u + 3 * i), b = __ldg(u + 3 * i + 1), c = __ldg(u + 3 * i + 2), gg = __ldg(g + i);
    // pixel 2i: (a.x, a.y, b.x), pixel 2i + 1: (b.y, c.x, c.y)
    out[2 * i] = make_double2(a.x, a.y);
    out[2 * i + 1] = make_double2(b.y, c.x);
    out[n + 2 * i] = make_double2(b.x, gg.x);
    out[n + 2 * i + 1] = make_double2(c.y, gg.y);
}

// RN(x / b) for b > 0 given y = RN(1 / b): q = RN(x y) is within one ulp of
// x / b, the remainder r = x - q b is exact in one FMA, and RN(q + r y) is the
// correctly rounded quotient (Markstein's theorem; no overflow or underflow
// for the [0, 3] sums here).  Three FP64 instructions instead of the
// reciprocal-iteration sequence of an IEEE division; hdp_check_exact_division
// compares it with __ddiv_rn.
__device__ __forceinline__ double div_rn_by(double x, double b, double y) {
    const double q = __dmul_rn(x, y);
    const double r = __fma_rn(-q, b, x);
    return __fma_rn(r, y, q);
}

__device__ __forceinline__ double px_cost(const PriorArgs& a, const double* su, const double* sg,
                                          const double* du, const double* dg, int64_t p,
                                          int64_t q) {
    double acc = fabs(__dsub_rn(su[p * a.c], du[q * a.c]));
    for (int k = 1; k < a.c; k++) acc = __dadd_rn(acc, fabs(__dsub_rn(su[p * a.c + k], du[q * a.c + k])));
    double color = div_rn_by(acc, (double)a.c, a.inv_c);
    double gd = fabs(__dsub_rn(sg[p], dg[q]));
    double v = __dmul_rn(a.one_minus_alpha, color < a.tc ? color : a.tc);
    double t = __dmul_rn(a.alpha, gd < a.tg ? gd : a.tg);
    return __dadd_rn(v, t);
}

// window-mean cost of matching centre (cr, cc) of `src` against `dst` at
// column offset sign*x (hdp_model.py:377-394), numpy summation order.
__device__ double window_cost(const PriorArgs& a, const double* su, const double* sg,
                              const double* du, const double* dg, int64_t base, int cr, int cc,
                              int sign, int x) {
    // numpy's mean over the window: pairwise_sum of all nwin values from the
    // identity 0 (eight accumulators, nwin <= 121 <= 128), then / nwin
    int half = a.window / 2;
    int nwin = a.window * a.window;
    int main_n = nwin < 8 ? 0 : nwin - (nwin % 8);
    double res = 0.0;
    double acc[8];
    int q = 0;
    for (int dr = -half; dr <= half; dr++) {
        int r = min(max(cr + dr, 0), a.h - 1);
        for (int dc = -half; dc <= half; dc++) {
            int col = min(max(cc + dc, 0), a.w - 1);
            int dcol = col + sign * x;
            double v;
            if (dcol >= 0 && dcol < a.w) {
                int64_t p = base + (int64_t)r * a.w + col;
                int64_t qq = base + (int64_t)r * a.w + dcol;
                v = px_cost(a, su, sg, du, dg, p, qq);
            } else {
                v = a.border;
            }
            if (nwin < 8) {
                res = __dadd_rn(res, v);  // pairwise_sum below 8: 0 + a0 + a1 ...
            } else if (q < 8) {
                acc[q] = v;
            } else if (q < main_n) {
                acc[q & 7] = __dadd_rn(acc[q & 7], v);
            } else {
                if (q == main_n) {
                    res = __dadd_rn(__dadd_rn(__dadd_rn(acc[0], acc[1]), __dadd_rn(acc[2], acc[3])),
                                    __dadd_rn(__dadd_rn(acc[4], acc[5]), __dadd_rn(acc[6], acc[7])));
                }
                res = __dadd_rn(res, v);
            }
            q++;
        }
    }
    if (nwin >= 8 && main_n == nwin) {
        res = __dadd_rn(__dadd_rn(__dadd_rn(acc[0], acc[1]), __dadd_rn(acc[2], acc[3])),
                        __dadd_rn(__dadd_rn(acc[4], acc[5]), __dadd_rn(acc[6], acc[7])));
    }
    return div_rn_by(res, (double)nwin, a.inv_win);
}

// warp-wide windowed WTA: first minimum over x = 0..d_max
__device__ int warp_wta(const PriorArgs& a, const double* su, const double* sg, const double* du,
                        const double* dg, int64_t base, int cr, int cc, int sign) {
    int lane = threadIdx.x & 31;
    double best = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    int bx = 0x7fffffff;
    for (int x = lane; x <= a.d_max; x += 32) {
        double v = window_cost(a, su, sg, du, dg, base, cr, cc, sign, x);
        if (v < best) {
            best = v;
            bx = x;
        }
    }
    for (int o = 16; o >= 1; o >>= 1) {
        double ob = __shfl_xor_sync(0xffffffffu, best, o);
        int ox = __shfl_xor_sync(0xffffffffu, bx, o);
        if (ob < best || (ob == best && ox < bx)) {
            best = ob;
            bx = ox;
        }
    }
    return bx;
}

// The 7 x 7 window (the reference default) with numpy's summation split over
// lanes: element q >= 1 of the window goes to accumulator (q - 1) & 7, and each
// accumulator is a sequential sum of 6 elements, so lane group g (8 lanes)
// evaluates disparity x0 + g and lane k of the group accumulates chain k;
// the pairwise tree ((a0+a1)+(a2+a3))+((a4+a5)+(a6+a7)) is three xor-shuffle
// levels (IEEE addition is commutative), lane 0 adds `first`.  A lane's six
// window elements are fixed per centre: their row offsets, columns and source
// pixels (C channels + gradient) are loaded into registers once, so the
// disparity loop only loads the matched pixels and runs the cost arithmetic.
template <int C>
__device__ __forceinline__ double rec_cost(const double4 L, const double4 R, double tc, double tg, double oma,
                                           double al, double inv_c) {
    double acc = fabs(__dsub_rn(L.x, R.x));
    if (C > 1) acc = __dadd_rn(acc, fabs(__dsub_rn(L.y, R.y)));
    if (C > 2) acc = __dadd_rn(acc, fabs(__dsub_rn(L.z, R.z)));
    const double color = C == 1 ? acc : div_rn_by(acc, (double)C, inv_c);
    const double gd = fabs(__dsub_rn(L.w, R.w));
    const double v = __dmul_rn(oma, color < tc ? color : tc);
    const double t2 = __dmul_rn(al, gd < tg ? gd : tg);
    return __dadd_rn(v, t2);
}

__device__ __forceinline__ double4 ld_rec(const double2* plane01, int64_t plane, int64_t i) {
    const double2 a = __ldg(plane01 + i), b = __ldg(plane01 + plane + i);
    return make_double4(a.x, a.y, b.x, b.y);
}

// The 7 x 7 window (the reference default): one warp per sample centre, one
// disparity per lane (x = lane, lane + 32, ...).  A lane evaluates all 49
// window elements of its disparity in numpy's order: element q < 48 goes to
// accumulator q & 7 (six sequential additions each), then
// ((a0+a1)+(a2+a3))+((a4+a5)+(a6+a7)), then + element 48, divided by 49 --
// numpy's mean: pairwise_sum of all 49 values from the identity (numpy 2.x;
// oracle or_np_sum, pinned against numpy in test_oracle_golden).  The
// window's source pixels are staged once per centre in shared memory (read
// as broadcasts); the matched pixels of the 32 lanes are 32 consecutive
// 32-byte records.  Fully unrolled: no shuffles, no divergent lanes, the
// geometry is compile-time per element.
constexpr int kPriorWarps = 8;

// Window-mean cost of one lane's disparity (offset `off` = sign * x) over
// the staged 7 x 7 window.  Element q = 7 dr + dc < 48 goes to accumulator
// q & 7 = (dc - dr) mod 8: V[dc] names that accumulator in row dr when V is
// rotated right by one register per row; element 48 (dr = dc = 6) is added
// after the tree.  Accumulators start at +0 (0 + v == v exactly).  FAST: every
// matched column is inside the image (no tests).
template <int C, bool FAST>
__device__ __forceinline__ double window_at(const double4* win, const double2* db, int64_t plane, int ro0,
                                            const int* colv, int off, int cr, int h, int w, double tc, double tg,
                                            double oma, double al, double inv_c, double inv_win, double border) {
    auto elem = [&](int dr, int ro, int dc) -> double {
        const int dcol = colv[dc] + off;
        if (FAST || (dcol >= 0 && dcol < w))
            return rec_cost<C>(win[7 * dr + dc], ld_rec(db, plane, ro + dcol), tc, tg, oma, al, inv_c);
        return border;
    };
    double V[8];
#pragma unroll
    for (int j = 0; j < 8; j++) V[j] = 0.0;
#pragma unroll
    for (int dc = 0; dc < 7; dc++) V[dc] = elem(0, ro0, dc);
    double last = 0.0;  // element 48
#pragma unroll 1
    for (int dr = 1; dr < 7; dr++) {
        const int ro = min(max(cr + dr - 3, 0), h - 1) * w;
        const double t = V[7];
#pragma unroll
        for (int j = 7; j > 0; j--) V[j] = V[j - 1];
        V[0] = t;
#pragma unroll
        for (int dc = 0; dc < 6; dc++) V[dc] = __dadd_rn(V[dc], elem(dr, ro, dc));
        const double e6 = elem(dr, ro, 6);
        if (dr < 6) V[6] = __dadd_rn(V[6], e6);
        else last = e6;
    }
    // after row 6, accumulator i is V[(i + 6) mod 8]
    const double res = __dadd_rn(__dadd_rn(__dadd_rn(V[6], V[7]), __dadd_rn(V[0], V[1])),
                                 __dadd_rn(__dadd_rn(V[2], V[3]), __dadd_rn(V[4], V[5])));
    return div_rn_by(__dadd_rn(res, last), 49.0, inv_win);
}

// Filter-and-verify WTA (exact): every disparity's 7 x 7 window mean is
// first computed in f32 from f32-rounded records; the f64 argmin (first
// minimum) is among the disparities whose f32 mean lies within eps32 of the
// f32 minimum, because |mean32 - mean64| <= eps32 / 2 for every disparity
// (inputs in [0, 1] / [-1, 1]: per element <= 4e-7 through the truncated
// colour and gradient terms, <= 2e-5 over the 49-value sum, < 5e-7 on the
// mean; eps32 = 1e-5 scaled by the border cost); only those candidates are
// evaluated in f64 in numpy's order (window_at), and the first minimum among
// them is the f64 first minimum over all disparities.
// u8 records: the channel sum of absolute differences is one VABSDIFF4 with
// the accumulator preloaded with the bits of 2^23, so the result reads as the
// float 2^23 + SAD (exact, SAD <= 765); tcs = tc * 255 C, omas = (1 - alpha) / (255 C)
__device__ __forceinline__ float rec_cost8(const uint2 L, const uint2 R, float tcs, float tg, float omas, float al,
                                           float acc) {
    unsigned r;
    asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(r) : "r"(L.x), "r"(R.x), "r"(0x4B000000u));
    const float sad = __uint_as_float(r) - 8388608.0f;
    const float g = fabsf(__uint_as_float(L.y) - __uint_as_float(R.y));
    acc = fmaf(omas, fminf(sad, tcs), acc);
    return fmaf(al, fminf(g, tg), acc);
}

constexpr int kFiltMax = 256;  // disparities per warp in the filter's shared arrays

// One candidate's exact f64 window mean with the 49 elements spread over the
// lanes: lane q holds element q (eA) and, for q <= 16, element 32 + q (eB).
// numpy's order: accumulator k = ((((e_k + e_{k+8}) + e_{k+16}) + e_{k+24}) +
// e_{k+32}) + e_{k+40}, then ((a0+a1)+(a2+a3))+((a4+a5)+(a6+a7)) (xor
// shuffles: IEEE addition is commutative), + e_48, / 49.  Valid on every lane.
__device__ __forceinline__ double window_mean_lanes(double eA, double eB, double inv_win) {
    const unsigned full = 0xffffffffu;
    const int k = threadIdx.x & 7;
    double s = __shfl_sync(full, eA, k);
    s = __dadd_rn(s, __shfl_sync(full, eA, k + 8));
    s = __dadd_rn(s, __shfl_sync(full, eA, k + 16));
    s = __dadd_rn(s, __shfl_sync(full, eA, k + 24));
    s = __dadd_rn(s, __shfl_sync(full, eB, k));
    s = __dadd_rn(s, __shfl_sync(full, eB, k + 8));
    s = __dadd_rn(s, __shfl_xor_sync(full, s, 1));
    s = __dadd_rn(s, __shfl_xor_sync(full, s, 2));
    s = __dadd_rn(s, __shfl_xor_sync(full, s, 4));
    const double last = __shfl_sync(full, eB, 16);
    return div_rn_by(__dadd_rn(s, last), 49.0, inv_win);
}

// Pass 1 of the filter: the f32 window mean of every disparity into c32,
// returns this lane's minimum.  Rec = uint2 (byte records, level 0) or float4
// (f32 records).  tcs / omas: the colour truncation and weight rescaled to
// the record's channel sum (tc 255 C and (1 - alpha) / (255 C) for bytes, tc C
// and (1 - alpha) / C for floats).
template <int C>
__device__ __forceinline__ float rec_acc(const float4 L, const float4 R, float tcs, float tg, float omas, float al,
                                         float acc) {
    float cs = fabsf(L.x - R.x);
    if (C > 1) cs += fabsf(L.y - R.y);
    if (C > 2) cs += fabsf(L.z - R.z);
    acc = fmaf(omas, fminf(cs, tcs), acc);
    return fmaf(al, fminf(fabsf(L.w - R.w), tg), acc);
}
template <int C>
__device__ __forceinline__ float rec_acc(const uint2 L, const uint2 R, float tcs, float tg, float omas, float al,
                                         float acc) {
    return rec_cost8(L, R, tcs, tg, omas, al, acc);
}

template <int C, typename Rec>
__device__ __forceinline__ float filter_means(const Rec* __restrict__ db, const Rec* wl, float tcs, float tg, float omas,
                                              float al, float border32, int cr, int cc, int sign, int h, int w,
                                              int d_max, const int* colv, int safe, int out, float* c32) {
    const int lane = threadIdx.x & 31;
    float mn = __int_as_float(0x7f800000);
    const bool interior = cc - 3 >= 0 && cc + 3 <= w - 1;  // the window's columns are consecutive
    // four 32-disparity blocks per round
    for (int xg = 0; xg <= d_max; xg += 128) {
        if constexpr (sizeof(Rec) == 8) {
            // byte records, four active blocks inside the image: the blocks share
            // the window's left records, and the next block's matched records are
            // in flight while this block's costs are evaluated
            if (interior && min(xg + 127, d_max) <= safe && xg + 96 <= d_max) {
                float acc[4];
                int off[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    acc[u] = 0.0f;
                    off[u] = sign * min(xg + 32 * u + lane, d_max);
                }
                Rec Ra[7], Rb[7];
                {
                    const Rec* rp = db + min(max(cr - 3, 0), h - 1) * w + (cc - 3) + off[0];
#pragma unroll
                    for (int dc = 0; dc < 7; dc++) Ra[dc] = __ldg(rp + dc);
                }
#pragma unroll 1
                for (int dr = 0; dr < 7; dr++) {
                    const int ro = min(max(cr + dr - 3, 0), h - 1) * w + (cc - 3);
                    const int ron = min(max(cr + min(dr + 1, 6) - 3, 0), h - 1) * w + (cc - 3);
                    Rec Lr[7];
#pragma unroll
                    for (int dc = 0; dc < 7; dc++) Lr[dc] = wl[7 * dr + dc];
#pragma unroll
                    for (int dc = 0; dc < 7; dc++) Rb[dc] = __ldg(db + ro + off[1] + dc);
#pragma unroll
                    for (int dc = 0; dc < 7; dc++) acc[0] = rec_acc<C>(Lr[dc], Ra[dc], tcs, tg, omas, al, acc[0]);
#pragma unroll
                    for (int dc = 0; dc < 7; dc++) Ra[dc] = __ldg(db + ro + off[2] + dc);
#pragma unroll
                    for (int dc = 0; dc < 7; dc++) acc[1] = rec_acc<C>(Lr[dc], Rb[dc], tcs, tg, omas, al, acc[1]);
#pragma unroll
                    for (int dc = 0; dc < 7; dc++) Rb[dc] = __ldg(db + ro + off[3] + dc);
#pragma unroll
                    for (int dc = 0; dc < 7; dc++) acc[2] = rec_acc<C>(Lr[dc], Ra[dc], tcs, tg, omas, al, acc[2]);
#pragma unroll
                    for (int dc = 0; dc < 7; dc++) Ra[dc] = __ldg(db + ron + off[0] + dc);  // row 6: reloaded, unused
#pragma unroll
                    for (int dc = 0; dc < 7; dc++) acc[3] = rec_acc<C>(Lr[dc], Rb[dc], tcs, tg, omas, al, acc[3]);
                }
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int x = xg + 32 * u + lane;
                    if (x <= d_max) {
                        const float m = acc[u] * (1.0f / 49.0f);
                        c32[x] = m;
                        mn = fminf(mn, m);
                    }
                }
                continue;
            }
        }
        // block by block: inside the image (no tests), entirely past the border
        // (every element costs `border`), or mixed (per-element tests)
#pragma unroll 1
        for (int u = 0; u < 4; u++) {
            const int xb = xg + 32 * u;
            if (xb > d_max) break;
            const int offu = sign * min(xb + lane, d_max);
            float accu = 0.0f;
            if (interior && min(xb + 31, d_max) <= safe) {
                // half rows software-pipelined: columns 4..6 of this row and 0..3 of
                // the next are in flight while the other half is evaluated
                Rec Ra[4], Rb[3];
                {
                    const Rec* rp = db + min(max(cr - 3, 0), h - 1) * w + (cc - 3) + offu;
#pragma unroll
                    for (int dc = 0; dc < 4; dc++) Ra[dc] = __ldg(rp + dc);
                }
#pragma unroll 1
                for (int dr = 0; dr < 7; dr++) {
                    const Rec* rp = db + min(max(cr + dr - 3, 0), h - 1) * w + (cc - 3) + offu;
                    const Rec* rn = db + min(max(cr + min(dr + 1, 6) - 3, 0), h - 1) * w + (cc - 3) + offu;
#pragma unroll
                    for (int dc = 0; dc < 3; dc++) Rb[dc] = __ldg(rp + 4 + dc);
#pragma unroll
                    for (int dc = 0; dc < 4; dc++) accu = rec_acc<C>(wl[7 * dr + dc], Ra[dc], tcs, tg, omas, al, accu);
#pragma unroll
                    for (int dc = 0; dc < 4; dc++) Ra[dc] = __ldg(rn + dc);  // row 6: reloaded, unused
#pragma unroll
                    for (int dc = 0; dc < 3; dc++)
                        accu = rec_acc<C>(wl[7 * dr + 4 + dc], Rb[dc], tcs, tg, omas, al, accu);
                }
            } else if (xb > out) {
                accu = 49.0f * border32;
            } else {
#pragma unroll 1
                for (int dr = 0; dr < 7; dr++) {
                    const int ro = min(max(cr + dr - 3, 0), h - 1) * w;
#pragma unroll
                    for (int dc = 0; dc < 7; dc++) {
                        const int dcol = colv[dc] + offu;
                        if (dcol >= 0 && dcol < w)
                            accu = rec_acc<C>(wl[7 * dr + dc], __ldg(db + ro + dcol), tcs, tg, omas, al, accu);
                        else
                            accu += border32;
                    }
                }
            }
            const int x = xb + lane;
            if (x <= d_max) {
                const float m = accu * (1.0f / 49.0f);
                c32[x] = m;
                mn = fminf(mn, m);
            }
        }
    }
    return mn;
}

// candidates above this count are verified one per lane (window_at), fewer with
// the window's elements spread over the lanes (window_mean_lanes)
constexpr int kLaneVerifyMax = 12;

template <int C>
__device__ int warp_wta7_filter(const PriorArgs& a, const double2* src, const double2* dst, const float4* src32,
                                const float4* dst32, const uint2* src8, const uint2* dst8, bool use8,
                                int64_t base, int cr, int cc, int sign, double4* win,
                                float4* win32, uint2* win8, float* c32, int* cand) {
    const int lane = threadIdx.x & 31;
    int rowo[7], colv[7];
#pragma unroll
    for (int i = 0; i < 7; i++) {
        rowo[i] = min(max(cr + i - 3, 0), a.h - 1) * a.w;
        colv[i] = min(max(cc + i - 3, 0), a.w - 1);
    }
    for (int q = lane; q < 49; q += 32) {
        const int dr = q / 7, dc = q - 7 * dr;
        const int64_t px = base + (int64_t)rowo[dr] + colv[dc];
        win[q] = ld_rec(src, a.plane, px);
        if (use8) win8[q] = __ldg(src8 + px);
        else win32[q] = __ldg(src32 + px);
    }
    __syncwarp();
    const int w = a.w, h = a.h, d_max = a.d_max;
    const float tg = (float)a.tg, al = (float)a.alpha;
    const float border32 = (float)a.border;
    // disparities whose matched columns are inside the image for every element
    const int safe = sign < 0 ? colv[0] : a.w - 1 - colv[6];
    // disparities above `out` match every element outside the image
    const int out = sign < 0 ? colv[6] : a.w - 1 - colv[0];
    // pass 1: f32 window means of every disparity
    float mn;
    if (use8)
        mn = filter_means<C>(dst8 + base, win8, (float)(a.tc * 255.0 * C), tg, (float)(a.one_minus_alpha / (255.0 * C)),
                             al, border32, cr, cc, sign, h, w, d_max, colv, safe, out, c32);
    else
        mn = filter_means<C>(dst32 + base, win32, (float)(a.tc * C), tg, (float)(a.one_minus_alpha / C), al, border32, cr,
                             cc, sign, h, w, d_max, colv, safe, out, c32);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    __syncwarp();
    // pass 2: candidates, compacted in ascending disparity order
    const float thr = mn + a.eps32;
    int ncand = 0;
    for (int x0 = 0; x0 <= d_max; x0 += 32) {
        const int x = x0 + lane;
        const bool is = x <= d_max && c32[x] <= thr;
        const unsigned bal = __ballot_sync(0xffffffffu, is);
        if (is) cand[ncand + __popc(bal & ((1u << lane) - 1u))] = x;
        ncand += __popc(bal);
    }
    __syncwarp();
    // pass 3: exact f64 means of the candidates, first minimum
    const double2* db = dst + base;
    const int64_t plane = a.plane;
    const double dtc = a.tc, dtg = a.tg, doma = a.one_minus_alpha, dal = a.alpha, border = a.border;
    const double inv_c = a.inv_c, inv_win = a.inv_win;
    double best = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    int bx = 0x7fffffff;
    if (ncand <= kLaneVerifyMax) {
        // few candidates (the usual case): one at a time, elements over the lanes
        const int qB = min(32 + lane, 48);
        const int drA = lane / 7, dcA = lane - 7 * drA, drB = qB / 7, dcB = qB - 7 * drB;
        const int roA = min(max(cr + drA - 3, 0), h - 1) * w, roB = min(max(cr + drB - 3, 0), h - 1) * w;
        const int colA = min(max(cc + dcA - 3, 0), w - 1), colB = min(max(cc + dcB - 3, 0), w - 1);
        const double4 LA = win[lane], LB = win[qB];
        for (int i = 0; i < ncand; i++) {
            const int x = cand[i];
            const int da = colA + sign * x, dbc = colB + sign * x;
            double eA = border, eB = border;
            if (da >= 0 && da < w) eA = rec_cost<C>(LA, ld_rec(db, plane, roA + da), dtc, dtg, doma, dal, inv_c);
            if (lane <= 16 && dbc >= 0 && dbc < w)
                eB = rec_cost<C>(LB, ld_rec(db, plane, roB + dbc), dtc, dtg, doma, dal, inv_c);
            const double v = window_mean_lanes(eA, eB, inv_win);
            if (v < best) {  // candidates ascend: strict < keeps the first minimum
                best = v;
                bx = x;
            }
        }
        __syncwarp();  // the shared arrays are rewritten by the next call
        return bx;
    }
    for (int i0 = 0; i0 < ncand; i0 += 32) {
        const bool ok = i0 + lane < ncand;
        const int x = cand[ok ? i0 + lane : i0];
        const bool fast = __all_sync(0xffffffffu, x <= safe);
        const int off = sign * x;
        const double v = fast ? window_at<C, true>(win, db, plane, rowo[0], colv, off, cr, h, w, dtc, dtg, doma, dal,
                                                   inv_c, inv_win, border)
                              : window_at<C, false>(win, db, plane, rowo[0], colv, off, cr, h, w, dtc, dtg, doma,
                                                    dal, inv_c, inv_win, border);
        if (ok && (v < best || (v == best && x < bx))) {
            best = v;
            bx = x;
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int ox = __shfl_xor_sync(0xffffffffu, bx, o);
        if (ob < best || (ob == best && ox < bx)) {
            best = ob;
            bx = ox;
        }
    }
    __syncwarp();  // the shared arrays are rewritten by the next call
    return bx;
}

template <int C>
__device__ int warp_wta7(const PriorArgs& a, const double2* src, const double2* dst, int64_t base, int cr, int cc,
                         int sign, double4* win) {
    const int lane = threadIdx.x & 31;
    int rowo[7], colv[7];
#pragma unroll
    for (int i = 0; i < 7; i++) {
        rowo[i] = min(max(cr + i - 3, 0), a.h - 1) * a.w;
        colv[i] = min(max(cc + i - 3, 0), a.w - 1);
    }
    for (int q = lane; q < 49; q += 32) {
        const int dr = q / 7, dc = q - 7 * dr;
        win[q] = ld_rec(src, a.plane, base + (int64_t)min(max(cr + dr - 3, 0), a.h - 1) * a.w +
                                          min(max(cc + dc - 3, 0), a.w - 1));
    }
    __syncwarp();
    const double2* db = dst + base;
    const int64_t plane = a.plane;
    const double tc = a.tc, tg = a.tg, oma = a.one_minus_alpha, al = a.alpha, border = a.border;
    const double inv_c = a.inv_c, inv_win = a.inv_win;
    // disparities whose matched columns are inside the image for every element
    const int safe = sign < 0 ? colv[0] : a.w - 1 - colv[6];
    double best = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    int bx = 0x7fffffff;
    const int w = a.w, h = a.h, d_max = a.d_max;
    for (int x0 = 0; x0 <= d_max; x0 += 32) {
        const int x = x0 + lane;
        const int off = sign * min(x, d_max);  // lanes past d_max: an in-range disparity, result unused
        const double v = (x0 + 31 <= safe && x0 + 31 <= d_max)  // warp-uniform: no border tests
                             ? window_at<C, true>(win, db, plane, rowo[0], colv, off, cr, h, w, tc, tg, oma, al,
                                                  inv_c, inv_win, border)
                             : window_at<C, false>(win, db, plane, rowo[0], colv, off, cr, h, w, tc, tg, oma, al,
                                                   inv_c, inv_win, border);
        if (x <= d_max && v < best) {  // x ascends per lane: strict < keeps the first minimum
            best = v;
            bx = x;
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int ox = __shfl_xor_sync(0xffffffffu, bx, o);
        if (ob < best || (ob == best && ox < bx)) {
            best = ob;
            bx = ox;
        }
    }
    __syncwarp();  // `win` is rewritten by the next call
    return bx;
}

struct FiltSmem {
    float4 win32[49];
    uint2 win8[49];
    float c32[kFiltMax];
    int cand[kFiltMax];
};

template <int W7>  // 0: any window; 1 / 3: 7 x 7 window, 1 / 3 channels
__device__ __forceinline__ void prior_centre(const PriorArgs& a, int64_t per, int64_t wid, double4* win,
                                             FiltSmem* fs, bool use8) {
    int b = (int)(wid / per);
    int k = (int)(wid % per);
    int i = k / a.ncc, j = k % a.ncc;
    int rs = i * a.stride, cs = j * a.stride;
    int cr = (rs + min(rs + a.stride, a.h) - 1) / 2;
    int cc = (cs + min(cs + a.stride, a.w) - 1) / 2;
    int64_t base = (int64_t)b * a.h * a.w;
    int dl;
    if constexpr (W7 > 0) {
        dl = a.pl32 ? warp_wta7_filter<W7>(a, a.pl, a.pr, a.pl32, a.pr32, a.pl8, a.pr8, use8, base, cr, cc, -1, win,
                                           fs->win32, fs->win8, fs->c32, fs->cand)
                    : warp_wta7<W7>(a, a.pl, a.pr, base, cr, cc, -1, win);
    } else {
        dl = warp_wta(a, a.ul, a.gl, a.ur, a.gr, base, cr, cc, -1);
    }
    int mc = cc - dl;
    if (mc < 0) return;  // infeasible (hdp_model.py:458-459)
    int dr;
    if constexpr (W7 > 0) {
        dr = a.pl32 ? warp_wta7_filter<W7>(a, a.pr, a.pl, a.pr32, a.pl32, a.pr8, a.pl8, use8, base, cr, mc, +1, win,
                                           fs->win32, fs->win8, fs->c32, fs->cand)
                    : warp_wta7<W7>(a, a.pr, a.pl, base, cr, mc, +1, win);
    } else {
        dr = warp_wta(a, a.ur, a.gr, a.ul, a.gl, base, cr, mc, +1);
    }
    int diff = dl - dr;
    if (diff < 0) diff = -diff;
    if ((threadIdx.x & 31) == 0 && diff <= a.max_offset) {
        atomicAdd(&a.counts[(int64_t)b * (a.d_max + 1) + dl], 1ull);
        atomicAdd(&a.kept[b], 1ull);
    }
}

template <int W7>
#ifndef HDP_PRIOR_MINB
#define HDP_PRIOR_MINB 3
#endif
__global__ void __launch_bounds__(256, HDP_PRIOR_MINB) k_prior(PriorArgs a, int batch) {
    const int64_t per = (int64_t)a.nrc * a.ncc;
    const int64_t nwarp = (int64_t)gridDim.x * (blockDim.x >> 5);
    __shared__ double4 win[kPriorWarps][49];  // the 7 x 7 path's staged window, per warp
    __shared__ FiltSmem fsm[W7 > 0 ? kPriorWarps : 1];  // the filter pass (7 x 7)
    // grid-stride over sample centres (a capped grid leaves SMs to other streams)
    const bool use8 = W7 > 0 && a.pl8 != nullptr && __ldg(a.nonint) == 0;  // uniform over the grid
    for (int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wid < per * batch; wid += nwarp)
        prior_centre<W7>(a, per, wid, win[threadIdx.x >> 5], &fsm[W7 > 0 ? threadIdx.x >> 5 : 0], use8);
}
// numpy's pairwise_sum (eight accumulators for blocks <= 128, halves rounded
// to multiples of 8 above; oracle/hdp_oracle.c np_pairwise): sequential
// device code with exactly that association order.
__device__ double np_pairwise_dev(const double* a, int n) {
    // iterative form of the recursion: an explicit stack of (offset, count)
    double part[16];
    int off[16], cnt[16], state[16];
    int sp = 0;
    off[0] = 0;
    cnt[0] = n;
    state[0] = 0;
    double ret = 0.0;
    while (sp >= 0) {
        const int o = off[sp], m = cnt[sp];
        if (m <= 128) {
            double r;
            if (m < 8) {
                r = 0.0;
                for (int i = 0; i < m; i++) r += a[o + i];
            } else {
                double q[8];
                for (int j = 0; j < 8; j++) q[j] = a[o + j];
                int i;
                for (i = 8; i < m - (m % 8); i += 8)
                    for (int j = 0; j < 8; j++) q[j] += a[o + i + j];
                r = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
                for (; i < m; i++) r += a[o + i];
            }
            ret = r;
            sp--;
            // hand the value to the parent frame
            while (sp >= 0) {
                if (state[sp] == 1) {  // left half done: remember it, do the right half
                    part[sp] = ret;
                    state[sp] = 2;
                    int n2 = cnt[sp] / 2;
                    n2 -= n2 % 8;
                    off[sp + 1] = off[sp] + n2;
                    cnt[sp + 1] = cnt[sp] - n2;
                    state[sp + 1] = 0;
                    sp++;
                    break;
                }
                ret = part[sp] + ret;  // both halves done
                sp--;
            }
        } else {
            int n2 = m / 2;
            n2 -= n2 % 8;
            state[sp] = 1;
            off[sp + 1] = o;
            cnt[sp + 1] = n2;
            state[sp + 1] = 0;
            sp++;
        }
    }
    return ret;
}
// add.reduce over a contiguous axis (sum / mean): pairwise over all n values
// from the identity (numpy 2.x; oracle or_np_sum)
__device__ __forceinline__ double np_sum_dev(const double* a, int n) { return np_pairwise_dev(a, n); }

// priors from the cross-checked counts (hdp_model.py:465-470): hist = counts
// + 1, hist / hist.sum(); no kept sample -> 1 / (d + 1).  One warp per pair,
// hist staged in shared memory, lane 0 sums in numpy's order.
constexpr int kBayesMaxCols = 256;
__global__ void __launch_bounds__(256) k_priors(const long long* __restrict__ counts, const long long* __restrict__ kept,
                                                int batch, int d1, double* __restrict__ out) {
    __shared__ double hist[8][kBayesMaxCols];
    __shared__ double tot[8];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int b = blockIdx.x * 8 + wib;
    if (b >= batch) return;
    const bool none = kept[b] == 0;
    for (int i = lane; i < d1; i += 32) hist[wib][i] = (double)counts[(int64_t)b * d1 + i] + 1.0;
    __syncwarp();
    if (lane == 0) tot[wib] = np_sum_dev(hist[wib], d1);
    __syncwarp();
    const double uni = 1.0 / (double)d1;
    for (int i = lane; i < d1; i += 32) out[(int64_t)b * d1 + i] = none ? uni : hist[wib][i] / tot[wib];
}

// bayes_child_given_parent (hdp_model.py:334-363) for every (pair, row):
// joint = cond[r, :] * prior[b, :], row_sum in numpy's order, a row without
// mass becomes all ones (so 1 / cols), out = joint / row_sum.  One warp per row.
__global__ void __launch_bounds__(256) k_bayes(const double* __restrict__ cond, const double* __restrict__ priors,
                                               int batch, int rows, int cols, double* __restrict__ out,
                                               int* __restrict__ n_dead) {
    __shared__ double joint[8][kBayesMaxCols];
    __shared__ double tot[8];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t row = (int64_t)blockIdx.x * 8 + wib;
    if (row >= (int64_t)batch * rows) return;
    const int b = (int)(row / rows), r = (int)(row % rows);
    for (int i = lane; i < cols; i += 32)
        joint[wib][i] = __dmul_rn(cond[(int64_t)r * cols + i], priors[(int64_t)b * cols + i]);
    __syncwarp();
    if (lane == 0) {
        double t = np_sum_dev(joint[wib], cols);
        if (t <= 0.0) {
            for (int i = 0; i < cols; i++) joint[wib][i] = 1.0;
            t = np_sum_dev(joint[wib], cols);
            if (n_dead) atomicAdd(n_dead + b, 1);
        }
        tot[wib] = t;
    }
    __syncwarp();
    for (int i = lane; i < cols; i += 32) out[row * cols + i] = __ddiv_rn(joint[wib][i], tot[wib]);
}

__global__ void k_assign_rows(const int32_t* __restrict__ pd, int batch, int ph, int pw, int h,
                              int w, int s, int n_rows, int32_t* __restrict__ rows, int* bad) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t n = (int64_t)h * w;
    if (t >= (int64_t)batch * n) return;
    int b = t / n;
    int64_t p = t % n;
    int r = p / w, col = p % w;
    int32_t v = pd[((int64_t)b * ph + r / s) * pw + col / s];
    if (v < 0 || v >= n_rows) {
        atomicAdd(bad, 1);
        v = 0;
    }
    rows[t] = v;
}

// predict_intervals (hdp_model.py:498-525) for every (pair, parent row) on
// the device: one warp per row of the Bayes matrix.  The stable descending
// order is a rank count (greater values first, equal values in index order --
// np.argsort(-P, kind="stable")); lane 0 then runs the running mass in that
// order exactly as np.cumsum (sequential) and stops at the first
// P / (c + P) < delta; the chosen ranks become the row's bitset, one ballot
// per 32 columns (lane l of register r holds column 32 r + l).
constexpr int kPmMaxCols = 256;
__global__ void __launch_bounds__(256) k_predict_masks(const double* __restrict__ bayes, int64_t nrows, int ncols,
                                                       double delta, uint32_t* __restrict__ masks, int nw) {
    __shared__ double sv[8][kPmMaxCols];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t row = (int64_t)blockIdx.x * 8 + wib;
    if (row >= nrows) return;
    const double* pr = bayes + row * ncols;
    double v[8];
    int rk[8];
#pragma unroll
    for (int r = 0; r < 8; r++) {
        const int j = 32 * r + lane;
        v[r] = j < ncols ? pr[j] : 0.0;
        rk[r] = 0;
    }
#pragma unroll
    for (int rj = 0; rj < 8; rj++) {
        if (32 * rj >= ncols) break;
        for (int sj = 0; sj < 32; sj++) {
            const int j = 32 * rj + sj;
            if (j >= ncols) break;
            const double vj = __shfl_sync(0xffffffffu, v[rj], sj);
#pragma unroll
            for (int r = 0; r < 8; r++) {
                const int i = 32 * r + lane;
                rk[r] += (vj > v[r] || (vj == v[r] && j < i)) ? 1 : 0;
            }
        }
    }
#pragma unroll
    for (int r = 0; r < 8; r++)
        if (32 * r + lane < ncols) sv[wib][rk[r]] = v[r];
    __syncwarp();
    int k = ncols;
    if (lane == 0) {
        double c = sv[wib][0];
        for (int t = 1; t < ncols; t++) {
            const double p = sv[wib][t];
            if (__ddiv_rn(p, __dadd_rn(c, p)) < delta) {
                k = t;
                break;
            }
            c = __dadd_rn(c, p);
        }
    }
    k = __shfl_sync(0xffffffffu, k, 0);
#pragma unroll
    for (int r = 0; r < 8; r++) {
        const unsigned word = __ballot_sync(0xffffffffu, 32 * r + lane < ncols && rk[r] < k);
        if (lane == 0 && r < nw) masks[row * nw + r] = word;
    }
}

}  // namespace hdp

using namespace hdp;

extern "C" int hdp_predict_masks(const double* bayes, int64_t nrows, int ncols, double delta, uint32_t* masks,
                                 int nw, void* stream) {
    HDP_REQUIRE(ncols >= 1 && ncols <= kPmMaxCols, HDP_ERR_CONFIG, "interval table has %d columns (max %d)", ncols,
                kPmMaxCols);
    HDP_REQUIRE(nw == (ncols + 31) / 32, HDP_ERR_CONFIG, "mask words %d do not cover %d columns", nw, ncols);
    if (nrows <= 0) return HDP_OK;
    k_predict_masks<<<(unsigned)((nrows + 7) / 8), 256, 0, (cudaStream_t)stream>>>(bayes, nrows, ncols, delta, masks,
                                                                                   nw);
    note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

extern "C" int hdp_prior_counts(const double* unit_l, const double* grad_l, const double* unit_r,
                                const double* grad_r, int batch, int h, int w, int c, int d_max,
                                int stride, int window, int max_offset, double alpha, double tau_c,
                                double tau_g, int64_t* counts, int64_t* kept, int max_ctas, void* stream) {
    HDP_REQUIRE(stride >= 1 && window >= 1 && window % 2 == 1, HDP_ERR_CONFIG,
                "sample_stride must be >= 1 and window odd and positive");
    HDP_REQUIRE(window * window <= 129, HDP_ERR_CONFIG, "window larger than 11 not supported");
    HDP_REQUIRE(c == 1 || c == 3, HDP_ERR_DATA, "channels must be 1 or 3");
    HDP_REQUIRE(d_max >= 0, HDP_ERR_CONFIG, "d_max must be >= 0");
    cudaStream_t st = (cudaStream_t)stream;
    HDP_CHECK_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * batch * (d_max + 1), st));
    HDP_CHECK_CUDA(cudaMemsetAsync(kept, 0, sizeof(int64_t) * batch, st));
    PriorArgs a;
    a.ul = unit_l; a.gl = grad_l; a.ur = unit_r; a.gr = grad_r;
    a.h = h; a.w = w; a.c = c; a.d_max = d_max; a.stride = stride; a.window = window;
    a.max_offset = max_offset;
    a.nrc = (h + stride - 1) / stride;
    a.ncc = (w + stride - 1) / stride;
    a.one_minus_alpha = 1.0 - alpha;
    a.alpha = alpha; a.tc = tau_c; a.tg = tau_g;
    a.border = (1.0 - alpha) * tau_c + alpha * tau_g;  // cost_volume.py:48-50, host IEEE
    a.counts = (unsigned long long*)counts;
    a.kept = (unsigned long long*)kept;
    int64_t warps = (int64_t)a.nrc * a.ncc * batch;
    if (warps == 0) return HDP_OK;
    unsigned grid = (unsigned)grid_for(warps * 32, 256);
    if (max_ctas > 0 && (unsigned)max_ctas < grid) grid = (unsigned)max_ctas;
    a.inv_c = 1.0 / (double)c;  // host IEEE: RN(1/c)
    a.inv_win = 1.0 / (double)(window * window);
    DevBuf<double2> pk;
    DevBuf<float4> pk32;
    DevBuf<uint2> pk8;
    DevBuf<int> nonint;
    a.pl = a.pr = nullptr;
    a.pl8 = a.pr8 = nullptr;
    a.nonint = nullptr;
    a.pl32 = a.pr32 = nullptr;
    a.eps32 = 0.0f;
    a.plane = (int64_t)batch * h * w;
    if (window == 7) {
        const int64_t n = a.plane;
        HDP_TRY(pk.alloc(4 * n, st));
        a.pl = pk.get();
        a.pr = pk.get() + 2 * n;
        const char* e = getenv("HDP_PRIOR_FILTER");  // diagnostics / tests: 0 = every disparity in f64
        const bool filt = !(e && e[0] == '0');
        // the f32 error bound assumes unit-scaled inputs (|u|, |grad| <= 1)
        // and the default-sized truncations; eps32 scales with the border cost
        if (filt && d_max < kFiltMax && a.border > 0.0 && a.border < 1.0) {
            HDP_TRY(pk32.alloc(2 * n, st));
            a.pl32 = pk32.get();
            a.pr32 = pk32.get() + n;
            a.eps32 = (float)(1e-5 * std::max(1.0, a.border / 0.00977));
            // level 0 of a uint8 pair: byte records for the filter (HDP_PRIOR_U8=0: diagnostics / tests)
            const char* e8 = getenv("HDP_PRIOR_U8");
            if (!(e8 && e8[0] == '0')) {
                HDP_TRY(pk8.alloc(2 * n, st));
                HDP_TRY(nonint.alloc(1, st));
                HDP_CHECK_CUDA(cudaMemsetAsync(nonint.get(), 0, sizeof(int), st));
                a.pl8 = pk8.get();
                a.pr8 = pk8.get() + n;
                a.nonint = nonint.get();
            }
            // one pass per image writes all its record sets
            k_pack_all<<<grid_for(n, 256), 256, 0, st>>>(unit_l, grad_l, n, c, pk.get(), pk32.get(),
                                                         a.pl8 ? pk8.get() : nullptr, nonint.get()); note_launch();
            k_pack_all<<<grid_for(n, 256), 256, 0, st>>>(unit_r, grad_r, n, c, pk.get() + 2 * n, pk32.get() + n,
                                                         a.pl8 ? pk8.get() + n : nullptr, nonint.get()); note_launch();
        } else {
            const bool v2 = c == 3 && n % 2 == 0 && ((uintptr_t)unit_l | (uintptr_t)grad_l | (uintptr_t)unit_r |
                                                     (uintptr_t)grad_r) % 16 == 0;
            if (v2) {
                k_pack_px3<<<grid_for(n / 2, 256), 256, 0, st>>>((const double2*)unit_l, (const double2*)grad_l, n / 2,
                                                                pk.get(), n); note_launch();
                k_pack_px3<<<grid_for(n / 2, 256), 256, 0, st>>>((const double2*)unit_r, (const double2*)grad_r, n / 2,
                                                                pk.get() + 2 * n, n); note_launch();
            } else {
                k_pack_px<<<grid_for(n, 256), 256, 0, st>>>(unit_l, grad_l, n, c, pk.get()); note_launch();
                k_pack_px<<<grid_for(n, 256), 256, 0, st>>>(unit_r, grad_r, n, c, pk.get() + 2 * n); note_launch();
            }
        }
    }
    if (window == 7 && c == 3)
        k_prior<3><<<grid, 256, 0, st>>>(a, batch);
    else if (window == 7)
        k_prior<1><<<grid, 256, 0, st>>>(a, batch);
    else
        k_prior<0><<<grid, 256, 0, st>>>(a, batch);
    note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

namespace hdp {
__global__ void k_check_div(int64_t n, unsigned long long seed, unsigned long long* bad) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // splitmix64 -> x in [0, 4): random mantissas over every binade below 4,
    // plus sums of three |k/255 - j/255| differences (the prior's inputs)
    unsigned long long z = seed + (unsigned long long)i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    double x;
    if (i & 1) {
        const int e = (int)(z >> 52) % 40;  // exponent: [2^-38, 4)
        x = ldexp(1.0 + (double)(z & 0xFFFFFFFFFFFFFull) * 0x1p-52, 1 - e);
    } else {
        const int k0 = z & 255, k1 = (z >> 8) & 255, k2 = (z >> 16) & 255;
        const int j0 = (z >> 24) & 255, j1 = (z >> 32) & 255, j2 = (z >> 40) & 255;
        x = __dadd_rn(__dadd_rn(fabs(__dsub_rn(k0 / 255.0, j0 / 255.0)), fabs(__dsub_rn(k1 / 255.0, j1 / 255.0))),
                      fabs(__dsub_rn(k2 / 255.0, j2 / 255.0)));
    }
    const double b[3] = {3.0, 49.0, 25.0};
    for (int t = 0; t < 3; t++)
        if (div_rn_by(x, b[t], 1.0 / b[t]) != __ddiv_rn(x, b[t])) atomicAdd(bad, 1ull);
}
}  // namespace hdp

extern "C" int hdp_check_exact_division(int64_t n, uint64_t seed, int64_t* mismatches, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf<unsigned long long> bad;
    HDP_TRY(bad.alloc(1, st));
    HDP_CHECK_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(unsigned long long), st));
    if (n > 0) {
        k_check_div<<<grid_for(n, 256), 256, 0, st>>>(n, seed, bad.get());
        note_launch();
    }
    HDP_CHECK_LAUNCH();
    HDP_CHECK_CUDA(cudaMemcpyAsync(mismatches, bad.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    HDP_CHECK_CUDA(cudaStreamSynchronize(st));
    return HDP_OK;
}

extern "C" int hdp_assign_rows(const int32_t* parent_disp, int batch, int ph, int pw, int h, int w,
                               int s, int n_rows, int32_t* pixel_row, void* stream) {
    HDP_REQUIRE(s >= 2, HDP_ERR_CONFIG, "block_size must be >= 2");
    HDP_REQUIRE(ph == (h + s - 1) / s && pw == (w + s - 1) / s, HDP_ERR_INTERNAL,
                "parent map %dx%d does not cover child %dx%d at block %d", ph, pw, h, w, s);
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf<int> bad;
    HDP_TRY(bad.alloc(1, st));
    HDP_CHECK_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), st));
    int64_t n = (int64_t)batch * h * w;
    k_assign_rows<<<grid_for(n, 256), 256, 0, st>>>(parent_disp, batch, ph, pw, h, w, s, n_rows,
                                                    pixel_row, bad.get()); note_launch();
    HDP_CHECK_LAUNCH();
    int hb = 0;
    HDP_CHECK_CUDA(cudaMemcpyAsync(&hb, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
    HDP_CHECK_CUDA(cudaStreamSynchronize(st));
    HDP_REQUIRE(hb == 0, HDP_ERR_INTERNAL, "%d parent disparities outside the %d-row table", hb,
                n_rows);
    return HDP_OK;
}

extern "C" int hdp_priors_from_counts(const int64_t* counts, const int64_t* kept, int batch, int d1, double* priors,
                                      void* stream) {
    HDP_REQUIRE(batch >= 1 && d1 >= 1, HDP_ERR_CONFIG, "bad prior shape");
    HDP_REQUIRE(d1 <= kBayesMaxCols, HDP_ERR_CONFIG, "disparity range above 255 not supported by hdp_priors_from_counts");
    k_priors<<<(batch + 7) / 8, 256, 0, (cudaStream_t)stream>>>((const long long*)counts, (const long long*)kept,
                                                               batch, d1, priors);
    note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

extern "C" int hdp_bayes(const double* cond, const double* priors, int batch, int rows, int cols, double* bayes,
                         int32_t* n_dead, void* stream) {
    HDP_REQUIRE(batch >= 1 && rows >= 1 && cols >= 1, HDP_ERR_CONFIG, "bad Bayes shape");
    HDP_REQUIRE(cols <= kBayesMaxCols, HDP_ERR_CONFIG, "disparity range above 255 not supported by hdp_bayes");
    const int64_t nrows = (int64_t)batch * rows;
    k_bayes<<<(unsigned)((nrows + 7) / 8), 256, 0, (cudaStream_t)stream>>>(cond, priors, batch, rows, cols, bayes,
                                                                         n_dead);
    note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}
