// Two-pass tree aggregation fused with the matching cost and winner-takes-all.
//
// Replaces masked_cost_volume + aggregate_tree + winner_takes_all_with_cost
// (cost_volume.py:183-236, aggregation.py:158-256) and the baseline's
// streamed chunk loop (aggregation.py:311-326).
//
//   up:   A_up(v) = E(v) + sum_c s_c A_up(c)
//   down: A(root) = A_up(root);  A(v) = s_v A(parent) + (1 - s_v^2) A_up(v)
//
// Work follows the heavy-path layout of forest.cu (phases = light depth,
// every heavy path contiguous, the rows of one path contiguous because all
// its nodes share the tree's lane count m; rows padded to 16 bytes).
//   E pre-pass  k_ecost_range_u / k_ecost_pix: E(v) for every node in pixel
//               order into the node's row (right-image window staged per tile)
//   up, per phase (deepest light depth first):
//     k_up_chunk  short paths, CTA-staged chunks (1-D TMA): A_up = b + s A_up(next),
//                 b = E + sum of the light children's s A_up
//     k_seg_up    long paths in 32-node segments, one warp per (segment, 32
//                 float4 columns); carries chained by deterministic decoupled
//                 look-back (bit-identical to the serial chain)
//   down, per phase (root phase first):
//     k_down_chunk / k_seg_down  A = s A(prev) + (1 - s^2) A_up, then the
//                 first argmin of every node folded into its (cost, d) key
//   k_keys_finish  keys -> disparity + min cost
// A is written back only where a light child will read it (or the volume is
// requested).  Fallbacks for layouts without chunks: k_light, k_scan_up_short,
// k_down_short; for cost rows given by the caller: k_ecompute.
#include <cuda_runtime.h>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <vector>

#include <algorithm>
#include <atomic>

#include "forest.cuh"
#include "prims.cuh"

namespace hdp {

struct AggArgs {
    const int4* lmeta;      // (node, lane offset, image column, m) per layout position
    const float* lsimf;     // similarity, sign = has light children
    const int32_t* lc_start;
    const int64_t* lc_row;
    const float* lc_sim;
    const int4* pinfo;      // per path of the launch list: (start, len, m, lane offset)
    const longlong2* prows; // (first row, parent's row or -1)
    const int2* seg_tab;    // (long-path index, segment index from the head)
    const SegDesc* seg_desc;  // per segment: rows, parent row, light-child range
    const int32_t* dlist;
    const int64_t* rowoff;
    const int32_t* lp_list;
    const int64_t* nodeoff;
    const int64_t* lc_rowoff;
    const int64_t* auxd;
    const float4* pl;
    const float4* pr;
    const float* cost_rows;
    int32_t npix;  // pixels per pair
    int32_t w;
    int c;
    int range_x0;  // >= 0: lane j is disparity range_x0 + j
    float alpha, tc, tg, border;
    float* aup;
    float* volume;
    unsigned long long* keys;
    unsigned long long* agg;    // per (segment, lane): local map value x_loc / y_loc (epoch-tagged)
    unsigned long long* aggp;   // per segment: local map product P / Q (epoch-tagged)
    unsigned long long* carry;  // per (segment, lane): (epoch << 32 | f32 bits), the
                                // epoch tag doubles as the readiness flag
    unsigned long long* segf;   // per (segment, column group): (local map, inclusive carry)
                                // published hints, epoch << 32 (the words above stay authoritative)
    unsigned epoch_up, epoch_down;
    int* tickets;        // per (phase, pass, group)
    int groups;  // 32-lane groups per node when sub == 32
    int sub;     // lanes per item for the packed mappings (power of 2 <= 32)
    int sub_shift;
    int atomic_keys;
    int store_all;  // store A for every node (volume requested), not only light parents
    int seg_light;  // the segment up pass gathers the light children itself (no k_light)
    int max_m;
    int max_mp;            // max_m rounded up to a multiple of 4 (carry stride)
    int qgroups;           // 32-float4 column groups of the widest row (segment kernels)
    int qsub, qsub_shift;  // chunk kernels: float4 lanes per path (power of 2 <= 32)
    int uni_mp;            // rowoff == nullptr (early raw cost): row of layout position k = k * uni_mp
    const uint2* pl8;      // byte records of the two images (k_pack_rec8), or null
    const uint2* pr8;
    const int* nonint8;    // != 0: some plane value is not a byte's image; the f32 records are used
};

__device__ __forceinline__ int lane_disp(const AggArgs& a, int doff, int j) {
    return a.range_x0 >= 0 ? a.range_x0 + j : a.dlist[doff + j];
}

__device__ __forceinline__ float raw_cost(const AggArgs& a, int32_t node, int col, int d, int j) {
    if (a.cost_rows) return a.cost_rows[a.nodeoff[node] + j];  // pixel-major ragged rows
    if (col - d < 0) return a.border;
    float4 L = __ldg(a.pl + node);
    float4 R = __ldg(a.pr + node - d);
    float color;
    if (a.c == 3)
        color = (fabsf(L.x - R.x) + fabsf(L.y - R.y) + fabsf(L.z - R.z)) * (1.0f / 3.0f);
    else
        color = fabsf(L.x - R.x);
    float gd = fabsf(L.w - R.w);
    return (1.0f - a.alpha) * fminf(a.tc, color) + a.alpha * fminf(a.tg, gd);
}

// Monotone float -> u32 so that u64 (ord(cost) << 32 | d) min == first argmin.
__device__ __forceinline__ uint32_t ord_f32(float f) {
    uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ unsigned long long pack_key(float y, int d) {
    return ((unsigned long long)ord_f32(y) << 32) | (uint32_t)d;
}

__device__ __forceinline__ void cp_async4(float* smem, const float* gmem, bool pred) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    int sz = pred ? 4 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Thread -> (item, lane j).  With sub < 32 (a power of two) several items
// share a warp, `sub` lanes each; otherwise one warp covers 32 lanes of one
// item and the lane group is blockIdx.y (no integer division anywhere).
struct Slot {
    int64_t item;
    int j;
};
__device__ __forceinline__ Slot slot_at(const AggArgs& a, int64_t t) {
    Slot s;
    if (a.sub < 32) {
        s.item = t >> a.sub_shift;
        s.j = (int)(t & (a.sub - 1));
    } else {
        s.item = t >> 5;
        s.j = (int)blockIdx.y * 32 + (int)(t & 31);
    }
    return s;
}
__device__ __forceinline__ Slot slot_of(const AggArgs& a) {
    return slot_at(a, (int64_t)blockIdx.x * blockDim.x + threadIdx.x);
}

constexpr int BU = 4;  // independent work items per thread (memory-level parallelism)

// Cost of the padding lanes of a row (rows hold ceil4(m) floats).  Large
// enough never to win an argmin, small enough that sums over a whole tree stay
// finite (no inf, so no 0 * inf anywhere in the recurrences).
constexpr float kPadCost = 1.0e30f;

// b(v) = E(v) for every node of a phase, BU independent (node, lane) items
// per thread; two load levels (metadata -> image planes).
__global__ void __launch_bounds__(256) k_ecompute(AggArgs a, int64_t k0, int64_t nk) {
    int64_t T = (int64_t)gridDim.x * blockDim.x;
    int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t row[BU];
    int4 mt[BU];
    int j[BU];
    bool ok[BU];
#pragma unroll
    for (int u = 0; u < BU; u++) {
        Slot s = slot_at(a, t0 + u * T);
        ok[u] = s.item < nk;
        j[u] = s.j;
        int64_t k = k0 + (ok[u] ? s.item : 0);
        mt[u] = a.lmeta[k];
        row[u] = a.rowoff[k];
        ok[u] = ok[u] && s.j < ((mt[u].w + 3) & ~3);  // pad lanes get 0
    }
    float v[BU];
#pragma unroll
    for (int u = 0; u < BU; u++) {
        bool lv = ok[u] && j[u] < mt[u].w;
        int d = lv ? lane_disp(a, mt[u].y, j[u]) : 0;
        v[u] = lv ? raw_cost(a, mt[u].x, mt[u].z, d, j[u]) : kPadCost;
    }
#pragma unroll
    for (int u = 0; u < BU; u++)
        if (ok[u]) a.aup[row[u] + j[u]] = v[u];
}

// b(v) = E(v) for every node at once, in pixel order: one CTA per (image
// row, kETile columns).  The right-image window the tile's lanes can reach
// (columns c0 - max_d .. c0 + kETile) is staged in shared memory once, so
// each hypothesis costs one shared load and one 4-byte global store into the
// node's layout row (the rows of one node are contiguous; m lanes -> m/32
// coalesced stores per warp).
constexpr int kETile = 128;

__device__ __forceinline__ float pix_cost(const AggArgs& a, float wc, const float4& L, const float4& R) {
    float color;
    if (a.c == 3)
        color = (fabsf(L.x - R.x) + fabsf(L.y - R.y) + fabsf(L.z - R.z)) * (1.0f / 3.0f);
    else
        color = fabsf(L.x - R.x);
    return wc * fminf(a.tc, color) + a.alpha * fminf(a.tg, fabsf(L.w - R.w));
}

// Range lanes (lane j is disparity range_x0 + j, every row the same width):
// one CTA per (image row, kETile columns); the tile's row offsets are looked
// up once into shared memory, then threads take flat (node, float4) items,
// four disparities and one 16-byte store each.
template <bool SMEM>
__global__ void __launch_bounds__(256) k_ecost_range(AggArgs a, const int32_t* __restrict__ lpos, int d_hi,
                                                     int m, unsigned inv) {
    extern __shared__ float4 win[];
    __shared__ long long srow[kETile];
    __shared__ float4 sL[kETile];
    const int64_t base = (int64_t)blockIdx.x * a.w;  // node id of column 0 of this image row
    const int c0 = (int)blockIdx.y * kETile;
    const int lo = max(0, c0 - d_hi), hi = min(a.w, c0 + kETile);
    const int nt = hi - c0;  // columns in this tile
    if (SMEM)
        for (int i = threadIdx.x; i < hi - lo; i += blockDim.x) win[i] = __ldg(a.pr + base + lo + i);
    for (int i = threadIdx.x; i < nt; i += blockDim.x) {
        srow[i] = __ldg(a.rowoff + __ldg(lpos + base + c0 + i));
        sL[i] = __ldg(a.pl + base + c0 + i);
    }
    __syncthreads();
    const float4* rrow = a.pr + base;  // right-image row (global fallback)
    // one warp per node, lanes over disparities: adjacent lanes read adjacent
    // window pixels (conflict-free 16-byte shared loads) and store adjacent
    // floats; the left pixel is loaded once per node
    const int mp = (m + 3) & ~3;
    const float wc = 1.0f - a.alpha;
    const int lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    (void)inv;
    for (int q = threadIdx.x >> 5; q < nt; q += nwarp) {
        const int col = c0 + q;
        const float4 L = sL[q];
        float* out = a.aup + srow[q];
        const int xl = col - a.range_x0;  // right-image column of lane 0
        for (int j = lane; j < mp; j += 32) {
            const int x = xl - j;
            float e;
            if (j >= m) e = kPadCost;
            else if (x < 0) e = a.border;
            else e = pix_cost(a, wc, L, SMEM ? win[x - lo] : __ldg(rrow + x));
            out[j] = e;
        }
    }
}

// Range lanes, rows of at most 32 U floats (the common case): the same tile,
// but the window is staged from virtual column c0 - x0 - (mp - 1) (columns
// left of the image zero-filled), so lane j of the node in tile column q reads
// window entry q + mp - 1 - j with no clamping: one base address per node,
// compile-time offsets for the U lane blocks, border / padding by selects.
// Roughly 15 instructions per hypothesis (was ~50: the k_ecost_range loop
// was issue-bound at 92 % in ncu).
// Byte records (uint8 pairs at full resolution): (channel bytes, f32 gradient)
// per pixel, 8 bytes instead of the 16-byte f32 record -- the pre-pass is
// bound by the shared-memory wavefronts of its window reads (ncu: LSU 97 %),
// which the narrower record halves.  The channel sum of absolute differences
// is one VABSDIFF4 whose accumulator holds the bits of 2^23: the result reads
// as the float 2^23 + SAD, exact.  k_pack_rec8 builds the records from the f32
// planes and raises *nonint8 if any channel is not exactly f32(k / 255).
struct CostK {
    float wc, alpha, tc, tg;  // f32 records
    float omas, tcs;          // byte records: (1 - alpha) / (255 C), tc * 255 C
    int c;
};
__device__ __forceinline__ float rec_cost(const CostK& k, const float4& L, const float4& R) {
    float color;
    if (k.c == 3)
        color = (fabsf(L.x - R.x) + fabsf(L.y - R.y) + fabsf(L.z - R.z)) * (1.0f / 3.0f);
    else
        color = fabsf(L.x - R.x);
    return k.wc * fminf(k.tc, color) + k.alpha * fminf(k.tg, fabsf(L.w - R.w));
}
__device__ __forceinline__ float rec_cost(const CostK& k, const uint2& L, const uint2& R) {
    unsigned r;
    asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(r) : "r"(L.x), "r"(R.x), "r"(0x4B000000u));
    const float sad = __uint_as_float(r) - 8388608.0f;
    const float g = fabsf(__uint_as_float(L.y) - __uint_as_float(R.y));
    return fmaf(k.alpha, fminf(g, k.tg), k.omas * fminf(sad, k.tcs));
}
__device__ __forceinline__ void rec_zero(float4& r) { r = make_float4(0.0f, 0.0f, 0.0f, 0.0f); }
__device__ __forceinline__ void rec_zero(uint2& r) { r = make_uint2(0u, 0u); }

__global__ void k_pack_rec8(const float4* __restrict__ planes, int64_t n, int c, uint2* __restrict__ out,
                            int* __restrict__ nonint) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 p = __ldg(planes + i);
    const float v[3] = {p.x, p.y, p.z};
    unsigned pk = 0;
    bool bad = false;
    for (int k = 0; k < c; k++) {
        const float r = rintf(v[k] * 255.0f);
        // exactly the f32 image of a byte: the planes hold f32(u8 / 255) (image.cu k_prepare*)
        const bool ok = r >= 0.0f && r <= 255.0f && (float)((double)r / 255.0) == v[k];
        bad = bad || !ok;
        pk |= (unsigned)(ok ? (int)r : 0) << (8 * k);
    }
    out[i] = make_uint2(pk, __float_as_uint(p.w));
    if (bad) *nonint = 1;
}

template <int U, typename Rec>
__device__ __forceinline__ void ecost_range_body(const AggArgs& a, const int32_t* __restrict__ lpos, int m,
                                                 const Rec* __restrict__ pl, const Rec* __restrict__ pr, Rec* win,
                                                 Rec* sL, long long* srow, const CostK& ck) {
    const int64_t base = (int64_t)blockIdx.x * a.w;  // node id of column 0 of this image row
    const int c0 = (int)blockIdx.y * kETile;
    const int mp = (m + 3) & ~3;
    const int v0 = c0 - a.range_x0 - (mp - 1);  // column of window entry 0
    const int hi = min(a.w, c0 + kETile);
    const int nt = hi - c0;
    const int nwin = hi - v0;
    for (int i = threadIdx.x; i < nwin; i += 256) {
        const int x = v0 + i;
        Rec r;
        rec_zero(r);
        if (x >= 0) r = __ldg(pr + base + x);
        win[i] = r;
    }
    for (int i = threadIdx.x; i < nt; i += 256) {
        const int32_t k = __ldg(lpos + base + c0 + i);
        srow[i] = a.rowoff ? __ldg(a.rowoff + k) : (long long)k * a.uni_mp;
        sL[i] = __ldg(pl + base + c0 + i);
    }
    __syncthreads();
    const float border = a.border;
    const int lane = threadIdx.x & 31;
    // blocks 0 .. U-2 are full (32 (U-1) < mp) and hold no padding lanes
    // (m > mp - 4 >= 32 (U-1) - 3 and mp is a multiple of 4 > 32 (U-1));
    // only the last block needs the row-end guard and the padding select
    const int jl = lane + 32 * (U - 1);
    for (int q = threadIdx.x >> 5; q < nt; q += 8) {
        const Rec L = sL[q];
        float* out = a.aup + srow[q] + lane;
        const int xl = c0 + q - a.range_x0;  // lanes j > xl reach left of the image
        const Rec* wp = win + (q + mp - 1 - lane);
        if (xl >= mp - 1) {  // warp-uniform: no lane reaches the border
#pragma unroll
            for (int u = 0; u < U - 1; u++) out[32 * u] = rec_cost(ck, L, wp[-32 * u]);
            if (jl < mp) {
                const float e = rec_cost(ck, L, wp[-32 * (U - 1)]);
                out[32 * (U - 1)] = jl >= m ? kPadCost : e;
            }
        } else {
#pragma unroll
            for (int u = 0; u < U - 1; u++) {
                const float e = rec_cost(ck, L, wp[-32 * u]);
                out[32 * u] = lane + 32 * u > xl ? border : e;
            }
            if (jl < mp) {
                float e = rec_cost(ck, L, wp[-32 * (U - 1)]);
                e = jl > xl ? border : e;
                out[32 * (U - 1)] = jl >= m ? kPadCost : e;
            }
        }
    }
}

template <int U>
__global__ void __launch_bounds__(256) k_ecost_range_u(AggArgs a, const int32_t* __restrict__ lpos, int m) {
    extern __shared__ float4 win[];
    __shared__ long long srow[kETile];
    __shared__ float4 sL[kETile];
    CostK ck;
    ck.wc = 1.0f - a.alpha;
    ck.alpha = a.alpha;
    ck.tc = a.tc;
    ck.tg = a.tg;
    ck.c = a.c;
    ck.omas = (1.0f - a.alpha) / (255.0f * (float)a.c);
    ck.tcs = a.tc * 255.0f * (float)a.c;
    if (a.pl8 != nullptr && __ldg(a.nonint8) == 0)  // uniform over the grid
        ecost_range_body<U, uint2>(a, lpos, m, a.pl8, a.pr8, reinterpret_cast<uint2*>(win),
                                   reinterpret_cast<uint2*>(sL), srow, ck);
    else
        ecost_range_body<U, float4>(a, lpos, m, a.pl, a.pr, win, sL, srow, ck);
}

// RANGE: lane j is disparity range_x0 + j (dense / slab lanes); otherwise the
// tree's lane list.  SMEM: the right-image window fits in shared memory.
template <bool RANGE, bool SMEM>
__global__ void __launch_bounds__(256) k_ecost_pix(AggArgs a, const int32_t* __restrict__ lpos, int d_hi) {
    extern __shared__ float4 win[];
    const int64_t base = (int64_t)blockIdx.x * a.w;  // node id of column 0 of this image row
    const int c0 = (int)blockIdx.y * kETile;
    const int lo = max(0, c0 - d_hi), hi = min(a.w, c0 + kETile);
    if (SMEM) {
        for (int i = threadIdx.x; i < hi - lo; i += blockDim.x) win[i] = __ldg(a.pr + base + lo + i);
        __syncthreads();
    }
    const float4* rrow = a.pr + base;  // right-image row (global fallback)
    const int lane = threadIdx.x & 31;
    const int per = 32 >> a.qsub_shift;  // nodes per warp pass
    const int sl = lane & (a.qsub - 1);
    const float wc = 1.0f - a.alpha;
    for (int q = (threadIdx.x >> 5) * per + (lane >> a.qsub_shift); q < kETile;
         q += (blockDim.x >> 5) * per) {
        const int col = c0 + q;
        if (col >= a.w) break;
        const int64_t node = base + col;
        const int kk = __ldg(lpos + node);
        const int4 mt = __ldg(a.lmeta + kk);
        float4* out = reinterpret_cast<float4*>(a.aup + __ldg(a.rowoff + kk));
        const float4 L = __ldg(a.pl + node);
        const int m = mt.w, mq = (m + 3) >> 2;
        for (int jq = sl; jq < mq; jq += a.qsub) {
            float e[4];
            if (RANGE) {
                const int x = col - (a.range_x0 + 4 * jq);  // right-image column of lane 4 jq
                if (x - 3 >= 0 && 4 * jq + 3 < m) {
#pragma unroll
                    for (int u = 0; u < 4; u++)
                        e[u] = pix_cost(a, wc, L, SMEM ? win[x - u - lo] : __ldg(rrow + x - u));
                } else {
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        if (4 * jq + u >= m) e[u] = kPadCost;
                        else if (x - u < 0) e[u] = a.border;
                        else e[u] = pix_cost(a, wc, L, SMEM ? win[x - u - lo] : __ldg(rrow + x - u));
                    }
                }
            } else {
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int j = 4 * jq + u;
                    if (j >= m) {
                        e[u] = kPadCost;
                        continue;
                    }
                    const int x = col - a.dlist[mt.y + j];
                    e[u] = x < 0 ? a.border : pix_cost(a, wc, L, SMEM ? win[x - lo] : __ldg(rrow + x));
                }
            }
            out[jq] = make_float4(e[0], e[1], e[2], e[3]);
        }
    }
}

// b(v) += sum_{light children c} s_c A_up(c) for the phase's light parents
// (children in ascending id order, their A_up final since the deeper phase).
// One `qsub`-lane group per parent, float4 columns; the parent's metadata and
// its first child's row are fetched before the remaining children are walked.
__global__ void __launch_bounds__(256) k_light(AggArgs a, int64_t p0, int64_t np) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t it = t >> a.qsub_shift;
    const int sl = (int)(t & (a.qsub - 1));
    if (it >= np) return;
    const int32_t k = a.lp_list[p0 + it];
    const int m = a.lmeta[k].w, mq = (m + 3) >> 2;
    const int32_t c0 = a.lc_start[k], c1 = a.lc_start[k + 1];
    float4* row = reinterpret_cast<float4*>(a.aup + a.rowoff[k]);
    const float s0 = a.lc_sim[c0];
    const float4* r0 = reinterpret_cast<const float4*>(a.aup + a.lc_row[c0]);
    for (int jq = sl; jq < mq; jq += a.qsub) {
        const float4 v0 = r0[jq];
        const float4 bv = row[jq];
        float4 x = make_float4(s0 * v0.x, s0 * v0.y, s0 * v0.z, s0 * v0.w);
        for (int32_t q = c0 + 1; q < c1; q++) {
            const float sq = a.lc_sim[q];
            const float4 v = reinterpret_cast<const float4*>(a.aup + a.lc_row[q])[jq];
            x.x += sq * v.x;
            x.y += sq * v.y;
            x.z += sq * v.z;
            x.w += sq * v.w;
        }
        row[jq] = make_float4(bv.x + x.x, bv.y + x.y, bv.z + x.z, bv.w + x.w);
    }
}

// Short-path kernels: one `sub`-lane group per path (sub == 32: one warp per
// path, the 32-lane groups looped inside the kernel).  Two lane groups are in
// flight per iteration and every row of the path is loaded before the chain
// runs, so a warp keeps 2 * (len + 1) independent loads outstanding.
struct ShortSlot {
    int64_t item;
    int sl;
};
__device__ __forceinline__ ShortSlot short_slot(const AggArgs& a) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    return ShortSlot{t >> a.sub_shift, (int)(t & (a.sub - 1))};
}

// A_up along short paths (2..kShortPath nodes), tail -> head.
__global__ void __launch_bounds__(256) k_scan_up_short(AggArgs a, int64_t s0, int64_t ns) {
    const ShortSlot s = short_slot(a);
    if (s.item >= ns) return;
    const int4 info = a.pinfo[s0 + s.item];
    const int len = info.y, m = info.z, mp = (m + 3) & ~3;
    if (len < 2) return;
    float* row0 = a.aup + a.prows[s0 + s.item].x;
    float sn[kShortPath];  // similarity of the node after q (0 past the tail)
#pragma unroll
    for (int q = 0; q < kShortPath; q++) sn[q] = q + 1 < len ? fabsf(a.lsimf[info.x + q + 1]) : 0.0f;
    for (int j = s.sl; j < m; j += 2 * a.sub) {
        const int j2 = j + a.sub;
        const bool h2 = j2 < m;
        float b0[kShortPath], b1[kShortPath];
#pragma unroll
        for (int q = 0; q < kShortPath; q++) {
            b0[q] = q < len ? row0[(int64_t)q * mp + j] : 0.0f;
            b1[q] = (q < len && h2) ? row0[(int64_t)q * mp + j2] : 0.0f;
        }
        float x0 = 0.0f, x1 = 0.0f;
#pragma unroll
        for (int q = kShortPath - 1; q >= 0; q--) {
            if (q < len) {
                x0 = b0[q] + sn[q] * x0;
                x1 = b1[q] + sn[q] * x1;
                row0[(int64_t)q * mp + j] = x0;
                if (h2) row0[(int64_t)q * mp + j2] = x1;
            }
        }
    }
}

// Diagnostics build (-DHDP_AGG_PROFILE): per-CTA / per-warp globaltimer stamps
// of the staging and compute steps, read back by hdp_debug_prof.
#ifdef HDP_AGG_PROFILE
constexpr unsigned kProfMax = 1u << 20;
__device__ unsigned long long g_prof[kProfMax * 8];
__device__ unsigned g_prof_n;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %smid;" : "=r"(r));
    return r;
}
#define PROF_DECL unsigned long long _pt0 = gtimer(), _pt1 = 0, _pt2 = 0, _pt3 = 0, _pt4 = 0
#define PROF_T(k) (_pt##k = gtimer())
#define PROF_PUT(kind, lead, aux)                                                                     \
    do {                                                                                              \
        if (lead) {                                                                                   \
            const unsigned _i = atomicAdd(&g_prof_n, 1u);                                             \
            if (_i < kProfMax) {                                                                      \
                unsigned long long* _r = g_prof + (size_t)_i * 8;                                     \
                _r[0] = ((unsigned long long)(kind) << 56) | ((unsigned long long)smid() << 40) |     \
                        (unsigned long long)(unsigned)(aux);                                          \
                _r[1] = _pt0; _r[2] = _pt1; _r[3] = _pt2; _r[4] = _pt3; _r[5] = _pt4; _r[6] = gtimer(); \
            }                                                                                         \
        }                                                                                             \
    } while (0)
#else
#define PROF_DECL
#define PROF_T(k)
#define PROF_PUT(kind, lead, aux)
#endif

// ---------------------------------------------------------------- segments

struct SegCtx {
    int32_t doff, mp;
    int64_t rowa, prow;  // first row of the segment, the path's parent row
    int32_t a, b;        // segment node range [a, b) (layout positions)
    int32_t e0, e1;      // light-child entries of the segment's nodes
    int s, nseg;
    bool has_next;       // more segments toward the tail
    int64_t gseg;        // global segment index
};

__device__ __forceinline__ SegCtx seg_ctx(const AggArgs& a, int64_t gseg) {
    const int4* p = reinterpret_cast<const int4*>(a.seg_desc + gseg);
    const int4 w0 = __ldg(p), w1 = __ldg(p + 1), w2 = __ldg(p + 2);
    SegCtx c;
    c.rowa = ((long long)(unsigned)w0.y << 32) | (unsigned)w0.x;
    c.prow = ((long long)(unsigned)w0.w << 32) | (unsigned)w0.z;
    c.a = w1.x;
    c.b = w1.x + w1.y;
    c.e0 = w1.z;
    c.e1 = w1.w;
    c.mp = w2.x;
    c.doff = w2.y;
    c.s = w2.z;
    c.nseg = w2.w;
    c.has_next = c.s + 1 < c.nseg;
    c.gseg = gseg;
    return c;
}

__device__ __forceinline__ int warp_ticket(int* ctr) {
    int t = 0;
    if ((threadIdx.x & 31) == 0) t = atomicAdd(ctr, 1);
    return __shfl_sync(0xffffffffu, t, 0);
}

// Carry words hold (epoch << 32 | value bits): a 64-bit store is a single
// transaction, so a reader that sees the epoch also sees the value -- no
// separate flag and no fences on the chain (decoupled look-back, flag in data).
__device__ __forceinline__ void put_carry(unsigned long long* p, unsigned epoch, float v) {
    unsigned long long w = ((unsigned long long)epoch << 32) | __float_as_uint(v);
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}

__device__ __forceinline__ float get_carry(const unsigned long long* p, unsigned epoch) {
    unsigned long long w;
    while (true) {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
        if ((unsigned)(w >> 32) == epoch) break;
        __nanosleep(20);
    }
    return __uint_as_float((unsigned)(w & 0xffffffffu));
}

// orders this thread's generic-proxy shared-memory accesses before later
// async-proxy (TMA) accesses: needed before a bulk copy reuses a buffer
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// 1-D TMA (bulk async copy) global -> shared, completing on an mbarrier
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps in the barrier
// instead of spinning through issue slots the resident compute warps need
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680u)
        : "memory");
}

__device__ __forceinline__ void put_carry4(unsigned long long* p, unsigned epoch, const float4& v) {
    put_carry(p, epoch, v.x);
    put_carry(p + 1, epoch, v.y);
    put_carry(p + 2, epoch, v.z);
    put_carry(p + 3, epoch, v.w);
}
__device__ __forceinline__ float4 get_carry4(const unsigned long long* p, unsigned epoch) {
    float4 v;
    v.x = get_carry(p, epoch);
    v.y = get_carry(p + 1, epoch);
    v.z = get_carry(p + 2, epoch);
    v.w = get_carry(p + 3, epoch);
    return v;
}

__device__ __forceinline__ bool try_carry4(const unsigned long long* p, unsigned epoch, float4& v) {
    unsigned long long w0, w1, w2, w3;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w0) : "l"(p) : "memory");
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w1) : "l"(p + 1) : "memory");
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w2) : "l"(p + 2) : "memory");
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w3) : "l"(p + 3) : "memory");
    v = make_float4(__uint_as_float((unsigned)w0), __uint_as_float((unsigned)w1),
                    __uint_as_float((unsigned)w2), __uint_as_float((unsigned)w3));
    return (unsigned)(w0 >> 32) == epoch && (unsigned)(w1 >> 32) == epoch &&
           (unsigned)(w2 >> 32) == epoch && (unsigned)(w3 >> 32) == epoch;
}
__device__ __forceinline__ bool try_carry1(const unsigned long long* p, unsigned epoch, float& v) {
    unsigned long long w;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    v = __uint_as_float((unsigned)w);
    return (unsigned)(w >> 32) == epoch;
}

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long w;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    return w;
}

// Carry-in of a segment by decoupled look-back over the segments at offsets
// dir, 2 dir, ... (toward the tail on the way up, toward the head on the way
// down).  The warp probes the hint flags of 32 predecessor segments at once
// (lane i: the segment i + 1 further away), takes the first whose inclusive
// carry is published -- or the path's end, where the carry is `edge` --
// provided every local map in between is published, then applies those maps
// in the serial chain's order, X = x_loc(k) + P(k) * X, so the result does not
// depend on timing.  The maps are read in batches of kApply with their own
// epoch tags checked (a hint is not ordered with the data it announces: a
// word not there yet is waited for).
#ifndef HDP_APPLY
#define HDP_APPLY 4
#endif
constexpr int kApply = HDP_APPLY;
__device__ __forceinline__ void wait_word(const unsigned long long* p, unsigned long long& w, unsigned epoch) {
    while ((unsigned)(w >> 32) != epoch) {
        __nanosleep(20);
        w = ld_relaxed(p);
    }
}
__device__ __forceinline__ float4 seg_lookback_w(const AggArgs& a, int64_t gseg, int dir, int kmax, unsigned epoch,
                                                 int jq, bool act, float4 edge, int g) {
    const size_t lw = (size_t)a.max_mp;
    const int lane = threadIdx.x & 31;
    int base = 1, kstop = kmax + 1;
    while (base <= kmax) {
        const int k = base + lane;
        bool inc = true, agg = false;  // past the path's end: the edge value
        if (k <= kmax) {
            const unsigned long long* fp = a.segf + 2 * ((gseg + (int64_t)dir * k) * a.qgroups + g);
            agg = (unsigned)(ld_relaxed(fp) >> 32) == epoch;
            inc = (unsigned)(ld_relaxed(fp + 1) >> 32) == epoch;
        }
        const unsigned binc = __ballot_sync(0xffffffffu, inc), bagg = __ballot_sync(0xffffffffu, agg);
        const int t = binc ? __ffs(binc) - 1 : 32;
        const unsigned need = t >= 32 ? 0xffffffffu : ((1u << t) - 1u);
        if ((bagg & need) == need) {
            if (t < 32) {
                kstop = base + t;
                break;
            }
            base += 32;  // 32 maps published: the inclusive carry is further away
            continue;
        }
        __nanosleep(32);
    }
    float4 X = edge;
    if (kstop <= kmax && act) {
        const unsigned long long* pi = a.carry + (gseg + (int64_t)dir * kstop) * lw + 4 * jq;
        unsigned long long w[4];
#pragma unroll
        for (int c = 0; c < 4; c++) w[c] = ld_relaxed(pi + c);
#pragma unroll
        for (int c = 0; c < 4; c++) wait_word(pi + c, w[c], epoch);
        X = make_float4(__uint_as_float((unsigned)w[0]), __uint_as_float((unsigned)w[1]),
                        __uint_as_float((unsigned)w[2]), __uint_as_float((unsigned)w[3]));
    }
    for (int kb = kstop - 1; kb >= 1; kb -= kApply) {
        const int nb = min(kApply, kb);
        unsigned long long wa[kApply][4], wp[kApply];
#pragma unroll
        for (int j = 0; j < kApply; j++) {
            if (j >= nb) break;
            const int64_t gk = gseg + (int64_t)dir * (kb - j);
            const unsigned long long* pa = a.agg + gk * lw + 4 * jq;
#pragma unroll
            for (int c = 0; c < 4; c++) wa[j][c] = act ? ld_relaxed(pa + c) : ((unsigned long long)epoch << 32);
            wp[j] = ld_relaxed(a.aggp + gk);
        }
#pragma unroll
        for (int j = 0; j < kApply; j++) {
            if (j >= nb) break;
            const int64_t gk = gseg + (int64_t)dir * (kb - j);
            if (act) {
                const unsigned long long* pa = a.agg + gk * lw + 4 * jq;
#pragma unroll
                for (int c = 0; c < 4; c++) wait_word(pa + c, wa[j][c], epoch);
            }
            wait_word(a.aggp + gk, wp[j], epoch);
            const float P = __uint_as_float((unsigned)wp[j]);
            X.x = __uint_as_float((unsigned)wa[j][0]) + P * X.x;
            X.y = __uint_as_float((unsigned)wa[j][1]) + P * X.y;
            X.z = __uint_as_float((unsigned)wa[j][2]) + P * X.z;
            X.w = __uint_as_float((unsigned)wa[j][3]) + P * X.w;
        }
    }
    return X;
}

// hint flags of this warp's (segment, column group): 0 = local map, 1 =
// inclusive carry (after the warp's lanes stored their words)
__device__ __forceinline__ void put_segf(const AggArgs& a, int64_t gseg, int g, int which, unsigned epoch) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
        unsigned long long* fp = a.segf + 2 * (gseg * a.qgroups + g) + which;
        const unsigned long long w = (unsigned long long)epoch << 32;
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(fp), "l"(w) : "memory");
    }
}

// warp-uniform index i in [0, 32]: value of node a + i held in lane i of lo
// (i < 32), or `past` for i == 32 (segments have at most kSeg = 32 nodes)
static_assert(kSeg == 32, "segment lanes hold one node each");
__device__ __forceinline__ float seg_pick(float lo, float past, int i) {
    const float l = __shfl_sync(0xffffffffu, lo, i & 31);
    return i < 32 ? l : past;
}

#ifndef HDP_SEG_WARPS
#define HDP_SEG_WARPS 4
#endif
constexpr int kSegWarps = HDP_SEG_WARPS;  // segment warps per CTA

// A segment's rows for this warp's column group: with one group (rows of at
// most 128 floats) the segment is one contiguous span of the row layout and
// arrives with a single bulk copy (row stride = the path's own mq in shared
// memory); otherwise each row's 32-column slice arrives by its own copy (row
// stride 32).  Returns the shared-memory row stride in float4.
__device__ __forceinline__ int seg_stage_issue(const AggArgs& a, const SegCtx& c, int g, float4* buf,
                                               unsigned long long* bar, int lane) {
    const int mq = c.mp >> 2;
    const int cnt = c.b - c.a;
    const float* src0 = a.aup + c.rowa;
    // every lane is done with the previous segment's buffer, and its generic
    // shared-memory accesses are ordered before the bulk copy's writes
    fence_proxy_async();
    __syncwarp();
    if (a.qgroups == 1) {
        if (lane == 0) {
            const unsigned bytes = (unsigned)cnt * (unsigned)c.mp * 4u;
            mbar_expect_tx(bar, bytes);
            bulk_g2s(buf, src0, bytes, bar);
        }
        return mq;
    }
    const int wq = min(32, mq - 32 * g);
    if (lane == 0) mbar_expect_tx(bar, (unsigned)cnt * (unsigned)wq * 16u);
    __syncwarp();
    for (int i = lane; i < cnt; i += 32)
        bulk_g2s(buf + i * 32, src0 + (int64_t)i * c.mp + 128 * g, (unsigned)wq * 16u, bar);
    return 32;
}
__device__ __forceinline__ void seg_stage_wait(unsigned long long* bar, unsigned& par) {
    mbar_wait(bar, par);
    par ^= 1u;
}
__device__ __forceinline__ int seg_stage(const AggArgs& a, const SegCtx& c, int g, float4* buf,
                                         unsigned long long* bar, unsigned& par, int lane) {
    const int rs = seg_stage_issue(a, c, g, buf, bar, lane);
    seg_stage_wait(bar, par);
    return rs;
}

// Up pass over one segment (tail -> head), one warp per (segment, 32 float4
// columns).  Segments are taken by ticket in reverse table order, so a
// path's tail segment comes first; the carry is X_a = x_loc(a) + P * X_b with
// P = prod s_{a+1..b}.
// light-child rows loaded per batch (registers: 4 per row)
#ifndef HDP_GATHER
#define HDP_GATHER 4
#endif
constexpr int kGather = HDP_GATHER;

__device__ __forceinline__ void seg_up_item(const AggArgs& a, const SegCtx& c, int g, float4* buf,
                                            unsigned long long* bar, unsigned& par, int lane) {
    PROF_DECL;
    const int mq = c.mp >> 2;
    if (g * 32 >= mq) return;
    const int jq = g * 32 + lane;
    const bool act = jq < mq;
    const int cnt = c.b - c.a;
    const bool has_next = c.has_next;
    const int rs = seg_stage_issue(a, c, g, buf, bar, lane);
    // while the segment's rows are in flight: the similarities, the light
    // children's CSR range and the first batch of their rows
    const float s_lo = (lane < cnt || (lane == cnt && has_next)) ? fabsf(a.lsimf[c.a + lane]) : 0.0f;
    const float s_past = (cnt == kSeg && has_next) ? fabsf(a.lsimf[c.b]) : 0.0f;
    int E0 = 0, E1 = 0, e0n = 0, e1n = 0;
    long long rowe = 0;
    float sime = 0.0f;
    float4 vpre[kGather];
    if (a.seg_light) {
        E0 = c.e0;
        E1 = c.e1;
        if (E1 > E0) {
            // per node: its entries [e0n, e1n) (lane cnt - 1 ends at E1)
            const int en = lane < cnt ? a.lc_start[c.a + lane] : E1;
            const int nx = __shfl_sync(0xffffffffu, en, (lane + 1) & 31);  // every lane shuffles
            e0n = en;
            e1n = lane == 31 ? E1 : nx;
            if (E0 + lane < E1) {
                rowe = a.lc_row[E0 + lane];
                sime = a.lc_sim[E0 + lane];
            }
#pragma unroll
            for (int j = 0; j < kGather; j++) {
                const long long r = __shfl_sync(0xffffffffu, rowe, j);
                vpre[j] = (E0 + j < E1 && act) ? reinterpret_cast<const float4*>(a.aup + r)[jq]
                                               : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            }
        }
    }
    seg_stage_wait(bar, par);
    PROF_T(1);
    if (a.seg_light) {
        // light children (final since the deeper phases) of the segment's nodes:
        // b(v) = E(v) + (s_c0 A_up(c0) + s_c1 A_up(c1) + ...), the operation
        // order of k_light.  The segment's entries are one contiguous CSR range.
        if (E1 > E0) {
            float4 xacc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            for (int eb = E0; eb < E1; eb += 32) {
                const int e = eb + lane, ne = min(32, E1 - eb);
                if (eb != E0) {
                    rowe = 0;
                    sime = 0.0f;
                    if (e < E1) {
                        rowe = a.lc_row[e];
                        sime = a.lc_sim[e];
                    }
                }
                for (int j0 = 0; j0 < ne; j0 += kGather) {
                    float4 v[kGather];
                    if (eb == E0 && j0 == 0) {
#pragma unroll
                        for (int j = 0; j < kGather; j++) v[j] = vpre[j];
                    } else {
#pragma unroll
                        for (int j = 0; j < kGather; j++) {
                            const long long r = __shfl_sync(0xffffffffu, rowe, (j0 + j) & 31);
                            v[j] = (j0 + j < ne && act) ? reinterpret_cast<const float4*>(a.aup + r)[jq]
                                                        : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < kGather; j++) {
                        if (j0 + j >= ne) break;
                        const int ee = eb + j0 + j;
                        const float sc = __shfl_sync(0xffffffffu, sime, j0 + j);
                        const unsigned own = __ballot_sync(0xffffffffu, lane < cnt && e0n <= ee && ee < e1n);
                        const int i = __ffs(own) - 1;
                        const bool first = ee == __shfl_sync(0xffffffffu, e0n, i);
                        const bool last = ee + 1 == __shfl_sync(0xffffffffu, e1n, i);
                        if (first) {
                            xacc = make_float4(sc * v[j].x, sc * v[j].y, sc * v[j].z, sc * v[j].w);
                        } else {
                            xacc.x += sc * v[j].x;
                            xacc.y += sc * v[j].y;
                            xacc.z += sc * v[j].z;
                            xacc.w += sc * v[j].w;
                        }
                        if (last && act) {
                            float4 b = buf[i * rs + lane];
                            b.x = b.x + xacc.x;
                            b.y = b.y + xacc.y;
                            b.z = b.z + xacc.z;
                            b.w = b.w + xacc.w;
                            buf[i * rs + lane] = b;
                        }
                    }
                }
            }
            __syncwarp();
        }
    }
    PROF_T(2);
    const float4 z = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    float4 x = z;
    float P = 1.0f;
    if (c.s > 0) {  // the head side will need this segment's map (local pass)
#pragma unroll 4
        for (int i = cnt - 1; i >= 0; i--) {
            const float sn = seg_pick(s_lo, s_past, i + 1);
            const float4 v = act ? buf[i * rs + lane] : z;
            x.x = v.x + sn * x.x;
            x.y = v.y + sn * x.y;
            x.z = v.z + sn * x.z;
            x.w = v.w + sn * x.w;
            P *= sn;
        }
        if (act) put_carry4(a.agg + c.gseg * a.max_mp + 4 * jq, a.epoch_up, x);
        if (lane == 0) put_carry(a.aggp + c.gseg, a.epoch_up, P);
        put_segf(a, c.gseg, g, 0, a.epoch_up);
    }
    PROF_T(3);
    float4 Xb = z;
    if (has_next)
        Xb = seg_lookback_w(a, c.gseg, +1, c.nseg - 1 - c.s, a.epoch_up, jq, act, z, g);
    PROF_T(4);
    if (c.s > 0) {
        if (act) {
            float4 o;
            o.x = x.x + P * Xb.x;
            o.y = x.y + P * Xb.y;
            o.z = x.z + P * Xb.z;
            o.w = x.w + P * Xb.w;
            put_carry4(a.carry + c.gseg * a.max_mp + 4 * jq, a.epoch_up, o);
        }
        put_segf(a, c.gseg, g, 1, a.epoch_up);
    }
    // final pass: exact recurrence from the true X_b
    float4* rows = reinterpret_cast<float4*>(a.aup + c.rowa) + jq;
    x = Xb;
#pragma unroll 4
    for (int i = cnt - 1; i >= 0; i--) {
        const float sn = seg_pick(s_lo, s_past, i + 1);
        const float4 v = act ? buf[i * rs + lane] : z;
        x.x = v.x + sn * x.x;
        x.y = v.y + sn * x.y;
        x.z = v.z + sn * x.z;
        x.w = v.w + sn * x.w;
        if (act) rows[(int64_t)i * mq] = x;
    }
    PROF_PUT(3, lane == 0, cnt | (c.s << 8) | ((has_next ? 1 : 0) << 30));
}

// Persistent: each warp takes segment tickets until the phase's are gone (a
// warp finishes its segment before taking the next, so every segment a
// look-back waits on is held by a running warp).
__global__ void __launch_bounds__(32 * kSegWarps) k_seg_up(AggArgs a, int64_t g0, int64_t ng, int* ctr,
                                                           int sq) {
    extern __shared__ float4 sbuf[];
    __shared__ unsigned long long bars[kSegWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = (int)blockIdx.y;
    float4* buf = sbuf + warp * kSeg * sq;
    if (lane == 0) mbar_init(&bars[warp], 1);
    __syncwarp();
    unsigned par = 0;
    // (taking the next ticket while the current segment runs was measured
    // slower: a ticket held by a busy warp stalls the look-backs behind it)
    for (;;) {
        const int t = warp_ticket(ctr + g);
        if (t >= ng) break;
        seg_up_item(a, seg_ctx(a, g0 + ng - 1 - t), g, buf, &bars[warp], par, lane);
    }
}

// Down pass over one segment (head -> tail).  The carry is
// Y_end = y_loc(b-1) + Q * Y_in with Q = prod_{t=a..b-1} s_t; the head of a
// root path uses s = 0 so that A(root) = A_up(root).  The first argmin of
// each node over this warp's columns is folded into the node's key (64-bit
// min when several warps share a row, a store otherwise); A is written back
// only where a light child will read it.
__device__ __forceinline__ void seg_down_item(const AggArgs& a, const SegCtx& c, int g, float4* buf,
                                              unsigned long long* bar, unsigned& par, int lane) {
    PROF_DECL;
    const int mq = c.mp >> 2;
    if (g * 32 >= mq) return;
    const int jq = g * 32 + lane;
    const bool act = jq < mq;
    const int cnt = c.b - c.a;
    const int rs = seg_stage_issue(a, c, g, buf, bar, lane);
    // while the rows are in flight: s (0 at a root head), light-children flag
    // and node id of node a + i, and the parent's row
    const float f_me = lane < cnt ? a.lsimf[c.a + lane] : 0.0f;
    const float s_lo = (c.s == 0 && lane == 0 && c.prow < 0) ? 0.0f : fabsf(f_me);
    const int n_lo = lane < cnt ? a.lmeta[c.a + lane].x : 0;
    unsigned lmask = __ballot_sync(0xffffffffu, lane < cnt && (__float_as_uint(f_me) >> 31));
    if (a.store_all) lmask = ~0u;
    const float4 z = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    float4 Ypar = z;  // A(parent) enters at the path's head (0 at a root)
    if (c.prow >= 0 && act) Ypar = reinterpret_cast<const float4*>(a.aup + c.prow)[jq];
    seg_stage_wait(bar, par);
    PROF_T(1);
    // local pass with Y_in = 0, only where the tail side needs this segment's map
    float4 yl = z;
    float Q = 1.0f;
    if (c.s + 1 < c.nseg) {
#pragma unroll 4
        for (int i = 0; i < cnt; i++) {
            const float sv = seg_pick(s_lo, 0.0f, i);
            const float w = 1.0f - sv * sv;
            const float4 v = act ? buf[i * rs + lane] : z;
            yl.x = sv * yl.x + w * v.x;
            yl.y = sv * yl.y + w * v.y;
            yl.z = sv * yl.z + w * v.z;
            yl.w = sv * yl.w + w * v.w;
            Q *= sv;
        }
        if (act) put_carry4(a.agg + c.gseg * a.max_mp + 4 * jq, a.epoch_down, yl);
        if (lane == 0) put_carry(a.aggp + c.gseg, a.epoch_down, Q);
        put_segf(a, c.gseg, g, 0, a.epoch_down);
    }
    PROF_T(2);
    const float4 Yin = c.s == 0 ? Ypar : seg_lookback_w(a, c.gseg, -1, c.s, a.epoch_down, jq, act, Ypar, g);
    PROF_T(3);
    if (c.s + 1 < c.nseg) {
        if (act) {
            float4 o;
            o.x = yl.x + Q * Yin.x;
            o.y = yl.y + Q * Yin.y;
            o.z = yl.z + Q * Yin.z;
            o.w = yl.w + Q * Yin.w;
            put_carry4(a.carry + c.gseg * a.max_mp + 4 * jq, a.epoch_down, o);
        }
        put_segf(a, c.gseg, g, 1, a.epoch_down);
    }
    float4* rows = reinterpret_cast<float4*>(a.aup + c.rowa) + jq;
    float4 y = Yin;
#pragma unroll 4
    for (int i = 0; i < cnt; i++) {
        const float sv = seg_pick(s_lo, 0.0f, i);
        const float w = 1.0f - sv * sv;
        const float4 v = act ? buf[i * rs + lane] : z;
        y.x = sv * y.x + w * v.x;
        y.y = sv * y.y + w * v.y;
        y.z = sv * y.z + w * v.z;
        y.w = sv * y.w + w * v.w;
        if (act) {
            if ((lmask >> i) & 1u) rows[(int64_t)i * mq] = y;
            buf[i * rs + lane] = y;  // A replaces A_up in the staged rows
        }
    }
    __syncwarp();
    // first minimum of every node over this warp's columns: four lanes per
    // node over interleaved float4 columns, then (value, index) minima
    if (a.keys) {
        const int wq = min(32, mq - 32 * g);  // float4 columns of this group
        const int sub = lane & 3;
        for (int i0 = 0; i0 < cnt; i0 += 8) {
            const int i = i0 + (lane >> 2);
            float best = __int_as_float(0x7f800000);
            int bj = 0x7fffffff;
            if (i < cnt) {
                for (int l = sub; l < wq; l += 4) {
                    const float4 yv = buf[i * rs + l];
                    const int j = 4 * (32 * g + l);  // padding lanes hold kPadCost and never win
                    if (yv.x < best) { best = yv.x; bj = j; }
                    if (yv.y < best) { best = yv.y; bj = j + 1; }
                    if (yv.z < best) { best = yv.z; bj = j + 2; }
                    if (yv.w < best) { best = yv.w; bj = j + 3; }
                }
            }
            uint32_t ob = bj == 0x7fffffff ? 0xffffffffu : ord_f32(best);
#pragma unroll
            for (int off = 1; off <= 2; off <<= 1) {
                const uint32_t o2 = __shfl_xor_sync(0xffffffffu, ob, off);
                const int j2 = __shfl_xor_sync(0xffffffffu, bj, off);
                if (o2 < ob || (o2 == ob && j2 < bj)) {
                    ob = o2;
                    bj = j2;
                }
            }
            const int node = __shfl_sync(0xffffffffu, n_lo, i & 31);
            if (i < cnt && sub == 0 && bj != 0x7fffffff) {
                const unsigned long long key = ((unsigned long long)ob << 32) | (uint32_t)lane_disp(a, c.doff, bj);
                if (a.atomic_keys)
                    atomicMin(&a.keys[node], key);
                else
                    a.keys[node] = key;
            }
        }
    }
    PROF_PUT(4, lane == 0, cnt | (c.s << 8) | ((c.s + 1 < c.nseg ? 1 : 0) << 30));
}

__global__ void __launch_bounds__(32 * kSegWarps) k_seg_down(AggArgs a, int64_t g0, int64_t ng, int* ctr,
                                                             int sq) {
    extern __shared__ float4 sbuf[];
    __shared__ unsigned long long bars[kSegWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = (int)blockIdx.y;
    float4* buf = sbuf + warp * kSeg * sq;
    if (lane == 0) mbar_init(&bars[warp], 1);
    __syncwarp();
    unsigned par = 0;
    for (;;) {
        const int t = warp_ticket(ctr + g);
        if (t >= ng) break;
        seg_down_item(a, seg_ctx(a, g0 + t), g, buf, &bars[warp], par, lane);
    }
}

// Short paths (1..kShortPath nodes): A = s A(parent) + (1 - s^2) A_up head ->
// tail fused with the first argmin of every node (aggregation.py:249,
// smallest disparity on ties: lanes ascend in disparity and each lane keeps
// its first minimum).  A is stored only for nodes with light children.
__global__ void __launch_bounds__(256) k_down_short(AggArgs a, int64_t s0, int64_t ns) {
    const ShortSlot s = short_slot(a);
    const bool valid = s.item < ns;
    const int4 info = valid ? a.pinfo[s0 + s.item] : make_int4(0, 0, 0, 0);
    const longlong2 rows = valid ? a.prows[s0 + s.item] : make_longlong2(0, -1);
    const int len = info.y, m = info.z, mp = (m + 3) & ~3;
    float sv[kShortPath];
    bool st[kShortPath];
#pragma unroll
    for (int q = 0; q < kShortPath; q++) {
        float f = q < len ? a.lsimf[info.x + q] : 0.0f;
        sv[q] = fabsf(f);
        st[q] = a.store_all || (__float_as_uint(f) >> 31);
    }
    if (rows.y < 0) sv[0] = 0.0f;  // root: A = A_up
    float* row0 = a.aup + rows.x;
    const float* prow = a.aup + (rows.y >= 0 ? rows.y : 0);
    uint32_t best[kShortPath];
    int bj[kShortPath];
#pragma unroll
    for (int q = 0; q < kShortPath; q++) {
        best[q] = 0xffffffffu;
        bj[q] = 0x7fffffff;
    }
    for (int j = s.sl; j < m; j += 2 * a.sub) {
        const int j2 = j + a.sub;
        const bool h2 = j2 < m;
        float u0[kShortPath], u1[kShortPath];
        float y0 = rows.y >= 0 ? prow[j] : 0.0f;
        float y1 = (rows.y >= 0 && h2) ? prow[j2] : 0.0f;
#pragma unroll
        for (int q = 0; q < kShortPath; q++) {
            u0[q] = q < len ? row0[(int64_t)q * mp + j] : 0.0f;
            u1[q] = (q < len && h2) ? row0[(int64_t)q * mp + j2] : 0.0f;
        }
#pragma unroll
        for (int q = 0; q < kShortPath; q++) {
            if (q < len) {
                y0 = sv[q] * y0 + (1.0f - sv[q] * sv[q]) * u0[q];
                y1 = sv[q] * y1 + (1.0f - sv[q] * sv[q]) * u1[q];
                if (st[q]) {
                    row0[(int64_t)q * mp + j] = y0;
                    if (h2) row0[(int64_t)q * mp + j2] = y1;
                }
                uint32_t o0 = ord_f32(y0);
                if (o0 < best[q]) {
                    best[q] = o0;
                    bj[q] = j;
                }
                uint32_t o1 = ord_f32(y1);
                if (h2 && o1 < best[q]) {
                    best[q] = o1;
                    bj[q] = j2;
                }
            }
        }
    }
    const int width = a.sub;
#pragma unroll
    for (int q = 0; q < kShortPath; q++) {
        if (!__any_sync(0xffffffffu, q < len)) break;
        uint32_t mn = best[q];
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            uint32_t t = __shfl_xor_sync(0xffffffffu, mn, off);
            if (off < width) mn = min(mn, t);
        }
        int jm = best[q] == mn ? bj[q] : 0x7fffffff;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            int t = __shfl_xor_sync(0xffffffffu, jm, off);
            if (off < width) jm = min(jm, t);
        }
        if (s.sl == 0 && q < len && a.keys && jm != 0x7fffffff)
            a.keys[a.lmeta[info.x + q].x] =
                ((unsigned long long)mn << 32) | (uint32_t)lane_disp(a, info.w, jm);
    }
}

// ------------------------------------------------------------ short chunks
//
// The short paths of a phase sit first in the phase's layout block, so their
// rows are one contiguous range; a chunk (forest.cuh) is a run of them whose
// rows, auxiliary rows (light children's A_up on the way up, the parent's A
// on the way down) and metadata fit in shared memory.  The CTA stages all of
// it first -- 16-byte loads for the row block, cp.async row gathers for the
// auxiliary rows, every load independent -- so the per-path walks that
// follow touch only shared memory, and global traffic is the chunk's rows in,
// the changed rows and the keys out.  One `sub`-lane group walks one path.

constexpr int kChunkThreads = 256;  // one CTA per chunk


struct ChunkSm {
    int4* info;         // per path: (start, len, m, lane offset)
    longlong2* prow;    // per path: (first row, parent's row or -1)
    long long* auxd;    // down: per path, auxd (parent-row slot)
    long long* lcr;     // up: per light-child entry (nl + 1), lc_rowoff
    long long* lcrow;   // up: per entry, global row of the child
    float* own;         // the chunk's rows
    float* aux;         // light children's rows (up) / parent rows (down)
    float* sim;         // per node: lsimf
    int* nodei;         // up: lc_start (nk + 1)
    float* lsim;        // up: per entry, similarity of the child
    int4* meta;         // down: per node, lmeta (node, lane offset, column, m)
    long long* nrow;    // down: per node, rowoff
};

template <bool UP>
__device__ __forceinline__ ChunkSm carve(const ChunkDesc& d, float4* sm4) {
    ChunkSm s;
    s.info = reinterpret_cast<int4*>(sm4);
    s.prow = reinterpret_cast<longlong2*>(sm4 + d.np);
    s.meta = reinterpret_cast<int4*>(sm4 + 2 * d.np);
    float4* p = sm4 + 2 * d.np + (UP ? 0 : d.nk);
    s.own = reinterpret_cast<float*>(p);
    p += d.n4;
    s.aux = reinterpret_cast<float*>(p);
    p += ((UP ? d.naux_up : d.naux_dn) + 3) >> 2;
    long long* l = reinterpret_cast<long long*>(p);
    s.auxd = l;
    l += UP ? 0 : (d.np + 1) & ~1;
    s.lcr = l;
    l += UP ? (d.nl + 2) & ~1 : 0;
    s.lcrow = l;
    l += UP ? (d.nl + 1) & ~1 : 0;
    s.nrow = l;
    l += UP ? 0 : (d.nk + 1) & ~1;
    float* q = reinterpret_cast<float*>(l);
    s.sim = q;
    q += d.nk;
    s.nodei = reinterpret_cast<int*>(q);
    q += d.nk + 1;
    s.lsim = q;
    return s;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4u(void* smem, const void* gmem) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_wait_one() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// 16-byte cp.async of a padded row of `cnt` floats (rows start 16-byte
// aligned), lanes of one warp striding the row
__device__ __forceinline__ void row_async(float* dst, const float* src, int cnt, int lane) {
    for (int j = lane * 4; j < cnt; j += 128) cp_async16(dst + j, src + j);
}

// The CTA stages its chunk with asynchronous copies only (no load waits on
// the issue path).  The row block and every auxiliary row (light children's
// A_up on the way up, the parent's A on the way down) arrive by 1-D TMA bulk
// copies completing on one mbarrier armed with the chunk's byte count; the
// small metadata arrays come by cp.async (group 1: what the auxiliary-row
// copies need, group 2: the rest).
template <bool UP>
__device__ __forceinline__ ChunkSm stage_chunk(const AggArgs& a, const ChunkDesc& d, float4* sm4,
                                               unsigned long long* bar, unsigned par) {
    ChunkSm s = carve<UP>(d, sm4);
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < d.np; i += nt) {
        cp_async16(s.info + i, a.pinfo + d.p0 + i);
        cp_async16(s.prow + i, a.prows + d.p0 + i);
        if (!UP) cp_async8(s.auxd + i, a.auxd + d.p0 + i);
    }
    if (UP) {
        for (int i = tid; i <= d.nl; i += nt) cp_async8(s.lcr + i, a.lc_rowoff + d.L0 + i);
        for (int i = tid; i < d.nl; i += nt) cp_async8(s.lcrow + i, a.lc_row + d.L0 + i);
    }
    cp_commit();
    for (int i = tid; i < d.nk; i += nt) cp_async4u(s.sim + i, a.lsimf + d.K0 + i);
    if (UP) {
        for (int i = tid; i <= d.nk; i += nt) cp_async4u(s.nodei + i, a.lc_start + d.K0 + i);
        for (int i = tid; i < d.nl; i += nt) cp_async4u(s.lsim + i, a.lc_sim + d.L0 + i);
    } else {
        for (int i = tid; i < d.nk; i += nt) {
            cp_async16(s.meta + i, a.lmeta + d.K0 + i);
            cp_async8(s.nrow + i, a.rowoff + d.K0 + i);
        }
    }
    cp_commit();
    __syncthreads();  // barrier initialised
    if (tid == 0) {
        mbar_expect_tx(bar, (unsigned)d.n4 * 16u + (unsigned)(UP ? d.naux_up : d.naux_dn) * 4u);
        bulk_g2s(s.own, a.aup + d.a0, (unsigned)d.n4 * 16u, bar);
    }
    cp_wait_one();
    __syncthreads();  // group 1 visible to every thread
    if (UP) {
        for (int e = tid; e < d.nl; e += nt) {
            const long long r0 = s.lcr[e];
            bulk_g2s(s.aux + (r0 - d.lcr0), a.aup + s.lcrow[e], (unsigned)(s.lcr[e + 1] - r0) * 4u, bar);
        }
    } else {
        for (int i = tid; i < d.np; i += nt) {
            const long long pr = s.prow[i].y;
            if (pr >= 0)
                bulk_g2s(s.aux + (s.auxd[i] - d.auxd0), a.aup + pr, (unsigned)((s.info[i].z + 3) & ~3) * 4u, bar);
        }
    }
    cp_wait_all();
    mbar_wait(bar, par);
    __syncthreads();
    return s;
}

// Up pass: tail -> head, A_up(q) = (E(q) + sum_light s_c A_up(c)) + s_{q+1} A_up(q+1)
// (the operation order of k_light + k_scan_up_short).  One thread per
// (path, float4 column); changed rows are stored, a lone leaf row (A_up = E)
// is left alone.
#ifndef HDP_UP_CHUNK_MINB
#define HDP_UP_CHUNK_MINB 5
#endif
__global__ void __launch_bounds__(kChunkThreads, HDP_UP_CHUNK_MINB) k_up_chunk(AggArgs a, const ChunkDesc* __restrict__ descs,
                                                            int64_t cbase, int64_t nc) {
    extern __shared__ float4 sm4[];
    __shared__ unsigned long long bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    unsigned par = 0;
    ChunkDesc dn;
    if (blockIdx.x < nc) dn = descs[cbase + blockIdx.x];
    for (int64_t ci = blockIdx.x; ci < nc; ci += gridDim.x) {
    PROF_DECL;
    const ChunkDesc d = dn;
    // a persistent CTA fetches its next descriptor while this chunk runs
    if (ci + gridDim.x < nc) dn = descs[cbase + ci + gridDim.x];
    if (d.np == 0) continue;
    PROF_T(1);
    const ChunkSm s = stage_chunk<true>(a, d, sm4, &bar, par);
    par ^= 1u;
    PROF_T(2);
    const float4* own4 = reinterpret_cast<const float4*>(s.own);
    const float4* aux4 = reinterpret_cast<const float4*>(s.aux);
    // with a uniform row width the (path, column) split is a multiply-high;
    // otherwise each path takes a 32-column stride of threads
    const int mqu = d.mqu;
    const int items = mqu > 0 ? d.np * mqu : d.np << a.qsub_shift;
    for (int t = threadIdx.x; t < items; t += blockDim.x) {
        int pi, jq;
        if (mqu > 0) {
            pi = mqu == 1 ? t : (int)__umulhi((unsigned)t, d.inv);
            jq = t - pi * mqu;
        } else {
            pi = t >> a.qsub_shift;
            jq = t & (a.qsub - 1);
        }
        const int4 info = s.info[pi];
        const int mq = (info.z + 3) >> 2;
        const long long r0 = s.prow[pi].x;
        const int k0 = info.x - d.K0;
        for (; jq < mq; jq += a.qsub) {
            const float4* col = own4 + ((r0 - d.a0) >> 2) + jq;
            float4* gcol = reinterpret_cast<float4*>(a.aup + r0) + jq;
            float4 xn = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            float sn = 0.0f;  // similarity of node q + 1
            for (int q = info.y - 1; q >= 0; q--) {
                const float f = s.sim[k0 + q];
                const bool has_l = __float_as_uint(f) >> 31;
                const bool tail = q + 1 == info.y;
                float4 b = col[q * mq];
                if (has_l) {
                    const int e0 = s.nodei[k0 + q] - d.L0, e1 = s.nodei[k0 + q + 1] - d.L0;
                    const float c0 = s.lsim[e0];
                    const float4 v0 = aux4[((int)(s.lcr[e0] - d.lcr0) >> 2) + jq];
                    float4 x = make_float4(c0 * v0.x, c0 * v0.y, c0 * v0.z, c0 * v0.w);
                    for (int e = e0 + 1; e < e1; e++) {
                        const float ce = s.lsim[e];
                        const float4 v = aux4[((int)(s.lcr[e] - d.lcr0) >> 2) + jq];
                        x.x += ce * v.x;
                        x.y += ce * v.y;
                        x.z += ce * v.z;
                        x.w += ce * v.w;
                    }
                    b.x = b.x + x.x;
                    b.y = b.y + x.y;
                    b.z = b.z + x.z;
                    b.w = b.w + x.w;
                }
                if (!tail) {
                    b.x = b.x + sn * xn.x;
                    b.y = b.y + sn * xn.y;
                    b.z = b.z + sn * xn.z;
                    b.w = b.w + sn * xn.w;
                }
                if (has_l || !tail) gcol[q * mq] = b;
                xn = b;
                sn = fabsf(f);
            }
            if (mqu > 0) break;  // uniform width: exactly one column per item
        }
    }
    fence_proxy_async();  // the next chunk's bulk copies overwrite shared memory
    __syncthreads();
#ifdef HDP_AGG_PROFILE
    PROF_T(3);
    PROF_PUT(1, threadIdx.x == 0, d.nk);
#endif
    }
}

// Down pass fused with the first argmin: head -> tail,
// A(q) = s_q A(q - 1) + (1 - s_q^2) A_up(q) with A(-1) = A(parent) (s = 0 at a
// root), one thread per (path, float4 column), A kept in shared memory and
// stored globally only where a light child will read it; then one thread
// per node scans its row for the first minimum (aggregation.py:249).
#ifndef HDP_DOWN_CHUNK_MINB
#define HDP_DOWN_CHUNK_MINB 5
#endif
__global__ void __launch_bounds__(kChunkThreads, HDP_DOWN_CHUNK_MINB) k_down_chunk(AggArgs a, const ChunkDesc* __restrict__ descs,
                                                              int64_t cbase, int64_t nc) {
    extern __shared__ float4 sm4[];
    __shared__ unsigned long long bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    unsigned par = 0;
    ChunkDesc dn;
    if (blockIdx.x < nc) dn = descs[cbase + blockIdx.x];
    for (int64_t ci = blockIdx.x; ci < nc; ci += gridDim.x) {
    PROF_DECL;
    const ChunkDesc d = dn;
    // a persistent CTA fetches its next descriptor while this chunk runs
    if (ci + gridDim.x < nc) dn = descs[cbase + ci + gridDim.x];
    if (d.np == 0) continue;
    PROF_T(1);
    const ChunkSm s = stage_chunk<false>(a, d, sm4, &bar, par);
    par ^= 1u;
    PROF_T(2);
    float4* own4 = reinterpret_cast<float4*>(s.own);
    const float4* aux4 = reinterpret_cast<const float4*>(s.aux);
    const int mqu = d.mqu;
    const int items = mqu > 0 ? d.np * mqu : d.np << a.qsub_shift;
    for (int t = threadIdx.x; t < items; t += blockDim.x) {
        int pi, jq;
        if (mqu > 0) {
            pi = mqu == 1 ? t : (int)__umulhi((unsigned)t, d.inv);
            jq = t - pi * mqu;
        } else {
            pi = t >> a.qsub_shift;
            jq = t & (a.qsub - 1);
        }
        const int4 info = s.info[pi];
        const int mq = (info.z + 3) >> 2;
        const longlong2 pr = s.prow[pi];
        const float* sim = s.sim + (info.x - d.K0);
        for (; jq < mq; jq += a.qsub) {
            float4* col = own4 + ((pr.x - d.a0) >> 2) + jq;
            float4* gcol = reinterpret_cast<float4*>(a.aup + pr.x) + jq;
            float4 yp = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            if (pr.y >= 0) yp = aux4[((s.auxd[pi] - d.auxd0) >> 2) + jq];
            for (int q = 0; q < info.y; q++) {
                const float f = sim[q];
                const float sv = (q == 0 && pr.y < 0) ? 0.0f : fabsf(f);  // root: A = A_up
                const float w = 1.0f - sv * sv;
                const float4 u = col[q * mq];
                float4 y;
                y.x = sv * yp.x + w * u.x;
                y.y = sv * yp.y + w * u.y;
                y.z = sv * yp.z + w * u.z;
                y.w = sv * yp.w + w * u.w;
                col[q * mq] = y;
                if (a.store_all || (__float_as_uint(f) >> 31)) gcol[q * mq] = y;
                yp = y;
            }
            if (mqu > 0) break;
        }
    }
    __syncthreads();
    PROF_T(3);
    if (a.max_mp >= 128) {
        // wide rows (a chunk holds few of them): one warp per node, lanes over
        // float4 columns, each lane keeping its first minimum, then redux
        const int lane = threadIdx.x & 31;
        for (int i = threadIdx.x >> 5; i < d.nk; i += blockDim.x >> 5) {
            const int4 mt = s.meta[i];
            const int m = mt.w, mq = (m + 3) >> 2;
            const float4* row = reinterpret_cast<const float4*>(s.own + (s.nrow[i] - d.a0));
            float best = __int_as_float(0x7f800000);  // +inf
            int bj = 0x7fffffff;
            for (int jq = lane; jq < mq; jq += 32) {
                const float4 y = row[jq];
                const int j = 4 * jq;  // padding lanes hold kPadCost and never win
                if (y.x < best) { best = y.x; bj = j; }
                if (y.y < best) { best = y.y; bj = j + 1; }
                if (y.z < best) { best = y.z; bj = j + 2; }
                if (y.w < best) { best = y.w; bj = j + 3; }
            }
            const uint32_t ob = bj == 0x7fffffff ? 0xffffffffu : ord_f32(best);
            const uint32_t mn = __reduce_min_sync(0xffffffffu, ob);
            const uint32_t jm = __reduce_min_sync(0xffffffffu, ob == mn ? (uint32_t)bj : 0xffffffffu);
            if (lane == 0 && a.keys)
                a.keys[mt.x] = ((unsigned long long)mn << 32) | (uint32_t)lane_disp(a, mt.y, (int)jm);
        }
    } else {
        // four threads per node, each keeping the first minimum of its
        // interleaved float4 columns, then (value, lane) minima over the four
        // (smallest value, then smallest index: np.argmin's first minimum)
        const int sub = threadIdx.x & 3;
        for (int i0 = 0; i0 < d.nk; i0 += kChunkThreads / 4) {
            const int i = i0 + (threadIdx.x >> 2);
            const bool ok = i < d.nk;
            int4 mt = make_int4(0, 0, 0, 0);
            float best = __int_as_float(0x7f800000);
            int bj = 0x7fffffff;
            if (ok) {
                mt = s.meta[i];
                const int mq = (mt.w + 3) >> 2;
                const float4* row = reinterpret_cast<const float4*>(s.own + (s.nrow[i] - d.a0));
                for (int jq = sub; jq < mq; jq += 4) {
                    const float4 y = row[jq];
                    const int j = 4 * jq;  // padding lanes hold kPadCost and never win
                    if (y.x < best) { best = y.x; bj = j; }
                    if (y.y < best) { best = y.y; bj = j + 1; }
                    if (y.z < best) { best = y.z; bj = j + 2; }
                    if (y.w < best) { best = y.w; bj = j + 3; }
                }
            }
            uint32_t ob = bj == 0x7fffffff ? 0xffffffffu : ord_f32(best);
#pragma unroll
            for (int off = 1; off <= 2; off <<= 1) {
                const uint32_t o2 = __shfl_xor_sync(0xffffffffu, ob, off);
                const int j2 = __shfl_xor_sync(0xffffffffu, bj, off);
                if (o2 < ob || (o2 == ob && j2 < bj)) {
                    ob = o2;
                    bj = j2;
                }
            }
            if (ok && sub == 0 && a.keys)
                a.keys[mt.x] = ((unsigned long long)ob << 32) | (uint32_t)lane_disp(a, mt.y, bj);
        }
    }
    fence_proxy_async();  // the next chunk's bulk copies overwrite shared memory
    __syncthreads();
#ifdef HDP_AGG_PROFILE
    PROF_T(4);
    PROF_PUT(2, threadIdx.x == 0, d.nk);
#endif
    }
}

// Pixel-major copy of the final aggregated volume (parity / API use only).
__global__ void __launch_bounds__(256) k_volume_copy(AggArgs a, int64_t n) {
    Slot s = slot_of(a);
    if (s.item >= n) return;
    int64_t k = s.item;
    int64_t row = a.rowoff[k];
    int m = a.lmeta[k].w;
    if (s.j >= m) return;
    a.volume[a.nodeoff[a.lmeta[k].x] + s.j] = a.aup[row + s.j];
}

// image column of every layout position for this call's geometry
__global__ void k_fill_cols(int64_t n, int4* lmeta, int32_t npix, int32_t w) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) lmeta[k].z = (lmeta[k].x % npix) % w;
}

__device__ __forceinline__ float unord_f32(uint32_t u) {
    uint32_t b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
    return __uint_as_float(b);
}

__global__ void k_keys_finish(int64_t n, const unsigned long long* __restrict__ keys,
                              int32_t* disp, float* min_cost) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    unsigned long long k = keys[i];
    if (disp) disp[i] = (int32_t)(k & 0xffffffffu);
    if (min_cost) min_cost[i] = unord_f32((uint32_t)(k >> 32));
}

// Per host thread and device: a second stream plus fork/join events.  Within
// a phase the short-path chunks and the long-path kernels touch disjoint rows,
// so they run concurrently (each alone leaves most of the GPU idle in the
// small phases and in the look-back chains).
struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    // segments of a phase that also has chunks: a high-priority stream, so the
    // block scheduler hands freed SM slots to pending segment CTAs first and the
    // two kinds actually run side by side (HDP_SEG_PRIO=0: off)
    cudaStream_t hi = nullptr;
    cudaEvent_t hjoin = nullptr;
};

static int side_stream(SideStream** out) {
    static thread_local SideStream per_dev[64];
    int dev = 0;
    HDP_CHECK_CUDA(cudaGetDevice(&dev));
    HDP_REQUIRE(dev >= 0 && dev < 64, HDP_ERR_CONFIG, "device ordinal %d out of range", dev);
    SideStream& ss = per_dev[dev];
    if (!ss.s) {
        HDP_CHECK_CUDA(cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking));
        HDP_CHECK_CUDA(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
        HDP_CHECK_CUDA(cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming));
        int lo = 0, hi = 0;
        HDP_CHECK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        HDP_CHECK_CUDA(cudaStreamCreateWithPriority(&ss.hi, cudaStreamNonBlocking, hi));
        HDP_CHECK_CUDA(cudaEventCreateWithFlags(&ss.hjoin, cudaEventDisableTiming));
    }
    *out = &ss;
    return HDP_OK;
}

static int fork_side(const SideStream* ss, cudaStream_t st) {
    HDP_CHECK_CUDA(cudaEventRecord(ss->fork, st));
    HDP_CHECK_CUDA(cudaStreamWaitEvent(ss->s, ss->fork, 0));
    return HDP_OK;
}

static int join_side(const SideStream* ss, cudaStream_t st) {
    HDP_CHECK_CUDA(cudaEventRecord(ss->join, ss->s));
    HDP_CHECK_CUDA(cudaStreamWaitEvent(st, ss->join, 0));
    return HDP_OK;
}
// one phase's chunks, small class then big class (forest.cu k_chunk_split)
template <typename G>
static int up_chunks(const AggArgs& sh, const hdp_forest* f, int64_t r, const G& cgrid, bool both, size_t ssmem,
                     size_t csmem, cudaStream_t s) {
    const int64_t c0 = f->chunk_off[r], nc = f->chunk_off[r + 1] - c0, nb = f->chunk_big[r], ns = nc - nb;
    // the small chunks that hold lone leaves only (the last chunk_lone[r] of
    // them) have nothing to do on the way up: A_up = E is already in place
    const int64_t nu = ns - (r < (int64_t)f->chunk_lone.size() ? f->chunk_lone[r] : 0);
    if (nu > 0) {
        k_up_chunk<<<cgrid(nu, both), kChunkThreads, ssmem, s>>>(sh, f->chunk_desc.get(), c0, nu); note_launch();
    }
    if (nb > 0) {
        k_up_chunk<<<cgrid(nb, both), kChunkThreads, csmem, s>>>(sh, f->chunk_desc.get(), c0 + ns, nb); note_launch();
    }
    return HDP_OK;
}
template <typename G>
static int down_chunks(const AggArgs& sh, const hdp_forest* f, int64_t r, const G& cgrid, bool both, size_t ssmem,
                       size_t csmem, cudaStream_t s) {
    const int64_t c0 = f->chunk_off[r], nc = f->chunk_off[r + 1] - c0, nb = f->chunk_big[r], ns = nc - nb;
    if (ns > 0) {
        k_down_chunk<<<cgrid(ns, both), kChunkThreads, ssmem, s>>>(sh, f->chunk_desc.get(), c0, ns); note_launch();
    }
    if (nb > 0) {
        k_down_chunk<<<cgrid(nb, both), kChunkThreads, csmem, s>>>(sh, f->chunk_desc.get(), c0 + ns, nb);
        note_launch();
    }
    return HDP_OK;
}

static int fork_hi(const SideStream* ss) {  // after fork_side: the fork event is recorded
    HDP_CHECK_CUDA(cudaStreamWaitEvent(ss->hi, ss->fork, 0));
    return HDP_OK;
}
static int join_hi(const SideStream* ss, cudaStream_t st) {
    HDP_CHECK_CUDA(cudaEventRecord(ss->hjoin, ss->hi));
    HDP_CHECK_CUDA(cudaStreamWaitEvent(st, ss->hjoin, 0));
    return HDP_OK;
}

static int env_int(const char* name, int dflt) {
    const char* e = getenv(name);  // diagnostics / tuning switches
    return e && *e ? atoi(e) : dflt;
}

static int pow2_at_least(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

// grid for the packed mappings: x covers items (sub lanes or one warp each,
// bu items per thread), y covers the 32-lane groups when sub == 32
static dim3 packed_grid(const AggArgs& a, int64_t items, int bu, int block) {
    int64_t th = a.sub < 32 ? items * a.sub : items * 32;
    th = (th + bu - 1) / bu;
    return dim3((unsigned)grid_for(th, block), a.sub < 32 ? 1u : (unsigned)a.groups, 1u);
}

}  // namespace hdp

using namespace hdp;

// HDP_AGG_TRACE=1: events between the aggregation's phases (no synchronisation
// until the end of the call), printed with each phase's chunk / segment counts
struct PhaseClock {
    bool on = false;
    cudaStream_t st;
    std::vector<cudaEvent_t> ev;
    std::vector<std::string> what;
    explicit PhaseClock(cudaStream_t s) : st(s) {
        const char* e = getenv("HDP_AGG_TRACE");
        on = e && e[0] == '1';
        if (on) mark("start", 0, 0);
    }
    void mark(const char* w, int64_t nc, int64_t ng) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        ev.push_back(e);
        char buf[96];
        snprintf(buf, sizeof(buf), "%-6s chunks %6lld segs %6lld", w, (long long)nc, (long long)ng);
        what.push_back(buf);
    }
    void report() {
        if (!on) return;
        cudaEventSynchronize(ev.back());
        for (size_t i = 1; i < ev.size(); i++) {
            float ms = 0.0f;
            cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
            fprintf(stderr, "[agg] %s %8.1f us\n", what[i].c_str(), 1e3 * ms);
        }
        for (auto e : ev) cudaEventDestroy(e);
        ev.clear();
    }
};

constexpr int kByteRecMinRow = 128;  // padded row width (floats) from which byte records are used

// Byte records for the range-lane raw cost (k_pack_rec8): both images' records in
// `buf` (2 n uint2), the exactness flag in `flag`; fills a.pl8 / a.pr8 / a.nonint8.
static int pack_byte_records(AggArgs& a, int64_t n, DevBuf<uint2>& buf, DevBuf<int>& flag, cudaStream_t st) {
    static const bool on = env_int("HDP_COST_U8", 1) != 0;  // diagnostics: 0 = always the f32 records
    a.pl8 = a.pr8 = nullptr;
    a.nonint8 = nullptr;
    if (!on) return HDP_OK;
    HDP_TRY(buf.alloc(2 * n, st));
    HDP_TRY(flag.alloc(1, st));
    HDP_CHECK_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), st));
    k_pack_rec8<<<grid_for(n, 256), 256, 0, st>>>(a.pl, n, a.c, buf.get(), flag.get()); note_launch();
    k_pack_rec8<<<grid_for(n, 256), 256, 0, st>>>(a.pr, n, a.c, buf.get() + n, flag.get()); note_launch();
    a.pl8 = buf.get();
    a.pr8 = buf.get() + n;
    a.nonint8 = flag.get();
    return HDP_OK;
}

// Early raw cost of the dense pipeline (forest.cuh EarlyCost): called by
// forest_build once the layout order is final.  Rows are uniform (range
// lanes), so a node's row is its layout position times the padded width.
int hdp::ecost_early(hdp_forest* f) {
    EarlyCost& e = f->early;
    cudaStream_t st = f->st;
    const int m = e.nx, mp = (m + 3) & ~3, U = (mp + 31) / 32;
    const size_t usmem = (size_t)(kETile + e.x0 + mp - 1) * sizeof(float4);
    if (!(usmem <= 48 * 1024 && U <= 17) || e.w <= 0 || f->n % e.w != 0 || (int64_t)e.h * e.w >= ((int64_t)1 << 31)) {
        e.want = 0;  // hdp_aggregate_wta runs its own pre-pass
        return HDP_OK;
    }
    HDP_TRY(e.rows.alloc(f->n * (int64_t)mp + 32, st));
    if (env_int("HDP_COST_U8", 1) != 0 && mp >= kByteRecMinRow) {
        HDP_TRY(e.rec8.alloc(2 * f->n, st));
        HDP_TRY(e.flag8.alloc(1, st));
        HDP_CHECK_CUDA(cudaMemsetAsync(e.flag8.get(), 0, sizeof(int), st));
    }
    HDP_CHECK_CUDA(cudaEventRecord(e.layout_ev, st));
    HDP_CHECK_CUDA(cudaStreamWaitEvent(e.side, e.layout_ev, 0));
    AggArgs a = {};
    a.pl = (const float4*)e.pl;
    a.pr = (const float4*)e.pr;
    a.npix = e.h * e.w;
    a.w = e.w;
    a.c = e.c;
    a.range_x0 = e.x0;
    a.alpha = e.alpha;
    a.tc = e.tau_c;
    a.tg = e.tau_g;
    a.border = (1.0f - e.alpha) * e.tau_c + e.alpha * e.tau_g;
    a.aup = e.rows.get();
    a.rowoff = nullptr;
    a.uni_mp = mp;
    a.pl8 = a.pr8 = nullptr;
    a.nonint8 = nullptr;
    if (e.flag8.get()) {  // byte records (allocated above on the forest's stream), packed on the side stream
        k_pack_rec8<<<grid_for(f->n, 256), 256, 0, e.side>>>(a.pl, f->n, a.c, e.rec8.get(), e.flag8.get()); note_launch();
        k_pack_rec8<<<grid_for(f->n, 256), 256, 0, e.side>>>(a.pr, f->n, a.c, e.rec8.get() + f->n, e.flag8.get());
        note_launch();
        a.pl8 = e.rec8.get();
        a.pr8 = e.rec8.get() + f->n;
        a.nonint8 = e.flag8.get();
    }
    dim3 g((unsigned)(f->n / e.w), (unsigned)((e.w + kETile - 1) / kETile));
    // shared-memory padding caps the grid's CTAs per SM (HDP_EARLY_SMEM_KB): the
    // build's latency-bound kernels beside it suffer less from a DRAM queue
    // that a full-occupancy write stream keeps saturated
    static const int pad_kb = env_int("HDP_EARLY_SMEM_KB", 0);
    const size_t esmem = std::max(usmem, (size_t)pad_kb * 1024);
    if (esmem > 48 * 1024) {
        switch (U) {
#define HDP_ECU(n) case n: cudaFuncSetAttribute(k_ecost_range_u<n>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)esmem); break;
            HDP_ECU(1) HDP_ECU(2) HDP_ECU(3) HDP_ECU(4) HDP_ECU(5) HDP_ECU(6) HDP_ECU(7) HDP_ECU(8)
            HDP_ECU(9) HDP_ECU(10) HDP_ECU(11) HDP_ECU(12) HDP_ECU(13) HDP_ECU(14) HDP_ECU(15)
            HDP_ECU(16) HDP_ECU(17)
#undef HDP_ECU
            default: break;
        }
    }
    switch (U) {
#define HDP_ECU(n) case n: k_ecost_range_u<n><<<g, 256, esmem, e.side>>>(a, f->lpos.get(), m); break;
        HDP_ECU(1) HDP_ECU(2) HDP_ECU(3) HDP_ECU(4) HDP_ECU(5) HDP_ECU(6) HDP_ECU(7) HDP_ECU(8)
        HDP_ECU(9) HDP_ECU(10) HDP_ECU(11) HDP_ECU(12) HDP_ECU(13) HDP_ECU(14) HDP_ECU(15)
        HDP_ECU(16) HDP_ECU(17)
#undef HDP_ECU
        default: break;
    }
    note_launch();
    HDP_CHECK_LAUNCH();
    HDP_CHECK_CUDA(cudaEventRecord(e.done_ev, e.side));
    e.done = 1;
    return HDP_OK;
}

#ifdef HDP_AGG_PROFILE
// records of 8 words: kind << 56 | smid << 40 | aux, then globaltimer stamps;
// returns the record count and resets it
extern "C" __attribute__((visibility("default"))) long long hdp_debug_prof(void* host, long long max_rec) {
    unsigned n = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&n, g_prof_n, sizeof(n));
    if (n > kProfMax) n = kProfMax;
    const long long k = n < max_rec ? n : max_rec;
    if (host && k > 0) cudaMemcpyFromSymbol(host, g_prof, (size_t)k * 64);
    const unsigned zero = 0;
    cudaMemcpyToSymbol(g_prof_n, &zero, sizeof(zero));
    return (long long)n;
}
#endif

extern "C" int hdp_aggregate_wta(hdp_forest* f, const float* packed_l, const float* packed_r,
                                 int h, int w, int c, float alpha, float tau_c, float tau_g,
                                 const float* cost_rows, int32_t* disp, float* min_cost,
                                 uint64_t* keys, float* volume, void* stream) {
    HDP_REQUIRE(f != nullptr && f->lanes_set, HDP_ERR_CONFIG, "forest lanes not set");
    HDP_REQUIRE(cost_rows || (packed_l && packed_r && h > 0 && w > 0), HDP_ERR_CONFIG,
                "need either cost rows or image planes");
    HDP_REQUIRE(cost_rows || (int64_t)h * w < ((int64_t)1 << 31), HDP_ERR_CONFIG, "image too large");
    cudaStream_t st = (cudaStream_t)stream;
    if (f->timing) HDP_CHECK_CUDA(cudaEventRecord(f->tev[0], st));
    AggArgs a;
    a.lmeta = f->lmeta.get();
    a.lsimf = f->lsimf.get();
    a.lc_start = f->lc_start.get();
    a.lc_row = f->lc_row.get();
    a.lc_sim = f->lc_sim.get();
    a.pinfo = nullptr;
    a.prows = nullptr;
    a.seg_tab = f->seg_tab.get();
    a.seg_desc = f->seg_desc.get();
    a.dlist = f->dlist.get();
    a.rowoff = f->rowoff.get();
    a.lp_list = f->lp_list.get();
    a.nodeoff = f->nodeoff.get();
    a.lc_rowoff = nullptr;
    a.auxd = nullptr;
    a.pl = (const float4*)packed_l;
    a.pr = (const float4*)packed_r;
    a.cost_rows = cost_rows;
    a.npix = (h > 0 && w > 0) ? h * w : 1;
    a.w = w > 0 ? w : 1;
    a.c = c;
    a.range_x0 = f->range_x0;
    a.alpha = alpha;
    a.tc = tau_c;
    a.tg = tau_g;
    a.border = (1.0f - alpha) * tau_c + alpha * tau_g;
    a.volume = volume;
    a.groups = (f->max_m + 31) / 32;
    a.max_m = f->max_m;
    a.max_mp = (f->max_m + 3) & ~3;
    a.qgroups = (a.max_mp / 4 + 31) / 32;
    DevBuf<unsigned long long> segfb;
    HDP_TRY(segfb.alloc(2 * f->n_segs * std::max(a.qgroups, 1) + 2, st));
    a.segf = segfb.get();
    a.sub = f->max_m <= 16 ? std::max(4, pow2_at_least(f->max_m)) : 32;  // >= one padded row
    a.sub_shift = 0;
    while ((1 << a.sub_shift) < a.sub) a.sub_shift++;
    {
        const int mq = (f->max_m + 3) >> 2;
        a.qsub = mq <= 16 ? pow2_at_least(mq) : 32;
        a.qsub_shift = 0;
        while ((1 << a.qsub_shift) < a.qsub) a.qsub_shift++;
    }
    PhaseClock pc(st);  // HDP_AGG_TRACE=1: per-stage device times on stderr
    DevBuf<float> aup;
    DevBuf<uint2> rec8;
    DevBuf<int> flag8;
    a.pl8 = a.pr8 = nullptr;
    a.nonint8 = nullptr;
    DevBuf<unsigned long long> carry;
    DevBuf<int> tickets;
    // the dense pipeline's early raw cost (forest.cuh EarlyCost): the rows are
    // already being filled on the side stream
    const bool early = f->early.done && !cost_rows && !volume && packed_l == f->early.pl &&
                       packed_r == f->early.pr && f->range_x0 == f->early.x0 && f->max_m == f->early.nx &&
                       h == f->early.h && w == f->early.w && c == f->early.c && alpha == f->early.alpha &&
                       tau_c == f->early.tau_c && tau_g == f->early.tau_g;
    if (early) {
        a.aup = f->early.rows.get();
        HDP_CHECK_CUDA(cudaStreamWaitEvent(st, f->early.done_ev, 0));
    } else {
        HDP_TRY(aup.alloc(f->total_rows + 32, st));
        a.aup = aup.get();
    }
    const int64_t nseg = f->n_segs;
    HDP_TRY(carry.alloc(nseg * a.max_mp + 1, st));
    DevBuf<unsigned long long> aggb, aggpb;
    HDP_TRY(aggb.alloc(nseg * a.max_mp + 1, st));
    HDP_TRY(aggpb.alloc(nseg + 1, st));
    a.agg = aggb.get();
    a.aggp = aggpb.get();
    HDP_TRY(tickets.alloc(2 * f->n_phases * a.groups + 1, st));
    HDP_CHECK_CUDA(cudaMemsetAsync(tickets.get(), 0,
                                   sizeof(int) * (2 * f->n_phases * a.groups + 1), st));
    // fresh epochs per call.  A carry word is (epoch << 32 | f32 bits) and the
    // tag doubles as the readiness flag, so a stale word in recycled pool
    // memory must never carry the current tag: epochs live in the NaN range
    // 0x7f800001..0x7fffffff, a pattern none of the library's buffers stores
    // in a 32-bit high word (finite floats, ids, sizes, sort keys), and every
    // call takes two fresh ones (4 M calls before the cycle repeats).
    static std::atomic<unsigned> g_epoch{0};
    const unsigned raw = g_epoch.fetch_add(1) % 0x3FFFFFu;
    const unsigned ep = 0x7f800001u + 2u * raw;
    a.carry = carry.get();
    a.epoch_up = ep;
    a.epoch_down = ep + 1;
    a.tickets = tickets.get();
    DevBuf<unsigned long long> kbuf;
    unsigned long long* kp = (unsigned long long*)keys;
    if (!kp) {
        HDP_TRY(kbuf.alloc(f->n, st));
        kp = kbuf.get();
    }
    a.keys = kp;
    // long-path nodes get one key contribution per 32-lane group
    a.atomic_keys = (f->n_segs > 0 && a.qgroups > 1) ? 1 : 0;
    static const bool poison = env_int("HDP_KEYS_POISON", 0) != 0;  // diagnostics: unwritten keys read as -1
    if (a.atomic_keys || poison) HDP_CHECK_CUDA(cudaMemsetAsync(kp, 0xff, sizeof(unsigned long long) * f->n, st));
    a.store_all = volume != nullptr;
    a.seg_light = f->chunks_ok ? 1 : 0;
    if (!cost_rows && (f->geom_w != a.w || f->geom_np != a.npix)) {
        k_fill_cols<<<grid_for(f->n, 256), 256, 0, st>>>(f->n, f->lmeta.get(), a.npix, a.w); note_launch();
        f->geom_w = a.w;
        f->geom_np = a.npix;
    }

    AggArgs lg = a;  // segment kernels: one warp per (segment, 32 float4 columns)
    // shared row stride (float4) of a staged segment: the widest row when one
    // column group covers it, else 32
    const int seg_sq = a.qgroups == 1 ? a.max_mp / 4 : 32;
    const size_t seg_smem = (size_t)kSegWarps * kSeg * seg_sq * sizeof(float4);
    if (seg_smem > 48 * 1024) {
        HDP_CHECK_CUDA(cudaFuncSetAttribute(k_seg_up, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)seg_smem));
        HDP_CHECK_CUDA(cudaFuncSetAttribute(k_seg_down, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)seg_smem));
    }
    lg.sub = 32;
    lg.pinfo = f->long_info.get();
    lg.prows = f->long_rows.get();
    AggArgs sh = a;
    sh.pinfo = f->short_info.get();
    sh.prows = f->short_rows.get();
    a.uni_mp = 0;
    if (early) {
    } else if (cost_rows) {
        k_ecompute<<<packed_grid(a, f->n, BU, 256), 256, 0, st>>>(a, 0, f->n); note_launch();
    } else {
        HDP_REQUIRE(f->n % a.w == 0, HDP_ERR_CONFIG, "node count is not a whole number of image rows");
        int64_t rows = f->n / a.w;
        HDP_REQUIRE(rows < ((int64_t)1 << 31), HDP_ERR_CONFIG, "too many image rows");
        size_t smem = (size_t)(kETile + f->max_d) * sizeof(float4);
        int use = smem <= 48 * 1024;
        dim3 g((unsigned)rows, (unsigned)((a.w + kETile - 1) / kETile));
        if (a.range_x0 >= 0) {
            const int m = f->max_m, mp = (m + 3) & ~3;
            const unsigned inv = (unsigned)((0x100000000ull + mp - 1) / mp);  // t / mp by multiply-high
            const int U = (mp + 31) / 32;
            const size_t usmem = (size_t)(kETile + a.range_x0 + mp - 1) * sizeof(float4);
            bool done = false;
            if (usmem <= 48 * 1024 && U <= 17) {
                done = true;
                // byte records pay for their pack pass when the rows are wide (C5:
                // pre-pass 2.49 -> 2.18 ms + 0.07 ms of packing; C2's 84-lane rows: a loss)
                if (mp >= kByteRecMinRow) HDP_TRY(pack_byte_records(a, f->n, rec8, flag8, st));
                switch (U) {
#define HDP_ECU(n) case n: k_ecost_range_u<n><<<g, 256, usmem, st>>>(a, f->lpos.get(), m); break;
                    HDP_ECU(1) HDP_ECU(2) HDP_ECU(3) HDP_ECU(4) HDP_ECU(5) HDP_ECU(6) HDP_ECU(7) HDP_ECU(8)
                    HDP_ECU(9) HDP_ECU(10) HDP_ECU(11) HDP_ECU(12) HDP_ECU(13) HDP_ECU(14) HDP_ECU(15)
                    HDP_ECU(16) HDP_ECU(17)
#undef HDP_ECU
                    default: done = false;
                }
            }
            if (done) {
            } else if (use) k_ecost_range<true><<<g, 256, smem, st>>>(a, f->lpos.get(), f->max_d, m, inv);
            else k_ecost_range<false><<<g, 256, 0, st>>>(a, f->lpos.get(), f->max_d, m, inv);
        } else {
            if (use) k_ecost_pix<false, true><<<g, 256, smem, st>>>(a, f->lpos.get(), f->max_d);
            else k_ecost_pix<false, false><<<g, 256, 0, st>>>(a, f->lpos.get(), f->max_d);
        }
        note_launch();
    }
    if (f->timing) HDP_CHECK_CUDA(cudaEventRecord(f->tev[1], st));
    pc.mark("ecost", 0, 0);
    const bool chunks = f->chunks_ok != 0;
    const size_t csmem = (size_t)((f->chunk_words + 3) & ~3ll) * sizeof(float);
    // the small-chunk class (forest.cuh kChunkSmallWords) launches with less
    // shared memory, so more of its CTAs are resident
    const size_t ssmem = std::min(csmem, (size_t)kChunkSmallWords * sizeof(float));
    sh.lc_rowoff = f->lc_rowoff.get();
    sh.auxd = f->auxd.get();
    if (chunks && csmem > 48 * 1024) {
        HDP_CHECK_CUDA(cudaFuncSetAttribute(k_up_chunk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
        HDP_CHECK_CUDA(cudaFuncSetAttribute(k_down_chunk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
    }
    SideStream* ss = nullptr;
    HDP_TRY(side_stream(&ss));
    // Chunk and segment kernels of one phase run side by side only if neither
    // takes every SM slot (the block scheduler dispatches one kernel's CTAs
    // before the next one's).  Both are persistent loops; HDP_CHUNK_SHARE /
    // HDP_SEG_SHARE (CTAs per SM) cap their grids when a phase has both kinds.
    // Measured at C2: capped grids (2 + 3 per SM) are slower than one kernel
    // after the other (register file), so the default is uncapped.
    int nsm = 148, dev = 0;
    HDP_CHECK_CUDA(cudaGetDevice(&dev));
    HDP_CHECK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    static const int chunk_share = env_int("HDP_CHUNK_SHARE", 0), seg_share = env_int("HDP_SEG_SHARE", 0);
    static const bool seg_prio = env_int("HDP_SEG_PRIO", 1) != 0;
    static const int chunk_persist = env_int("HDP_CHUNK_PERSIST", 0);  // CTAs per SM, 0 = one chunk per CTA
    auto cgrid = [&](int64_t nc, bool both) -> unsigned {
        int64_t g = both && chunk_share > 0 ? std::min<int64_t>(nc, (int64_t)chunk_share * nsm) : nc;
        if (chunk_persist > 0) g = std::min<int64_t>(g, (int64_t)chunk_persist * nsm);
        return (unsigned)g;
    };
    auto sgrid = [&](int64_t ng, bool both) -> unsigned {
        const int64_t need = grid_for(ng * 32, 32 * kSegWarps);
        return (unsigned)(both && seg_share > 0 ? std::min<int64_t>(need, (int64_t)seg_share * nsm) : need);
    };
    for (int64_t r = f->n_phases - 1; r >= 0; r--) {
        // light parents on short paths are handled inside k_up_chunk
        // light parents on short paths are handled by k_up_chunk, those on long
        // paths by k_seg_up (seg_light); k_light only in the fallback path
        int64_t p0 = f->lp_off[r], np = chunks ? 0 : f->lp_off[r + 1] - p0;
        int64_t c0 = f->chunk_off[r], nc = f->chunk_off[r + 1] - c0;
        int64_t g0 = f->seg_off[r], ng = f->seg_off[r + 1] - g0;
        const bool side = chunks && nc > 0 && (np > 0 || ng > 0);
        if (side) {
            HDP_TRY(fork_side(ss, st));
            HDP_TRY(up_chunks(sh, f, r, cgrid, ng > 0, ssmem, csmem, ss->s));
        }
        if (np > 0) {
            k_light<<<grid_for(np << a.qsub_shift, 256), 256, 0, st>>>(a, p0, np); note_launch();
        }
        if (ng > 0) {
            const bool hp = side && seg_prio;
            if (hp) HDP_TRY(fork_hi(ss));
            k_seg_up<<<dim3(sgrid(ng, side), lg.qgroups), 32 * kSegWarps, seg_smem, hp ? ss->hi : st>>>(
                lg, g0, ng, a.tickets + (2 * r) * a.groups, seg_sq); note_launch();
            if (hp) HDP_TRY(join_hi(ss, st));
        }
        int64_t s0 = f->short_off[r], ns = f->short_off[r + 1] - s0;
        if (side) {
            HDP_TRY(join_side(ss, st));
        } else if (chunks && nc > 0) {
            HDP_TRY(up_chunks(sh, f, r, cgrid, false, ssmem, csmem, st));
        } else if (!chunks && ns > 0) {
            k_scan_up_short<<<grid_for(ns * sh.sub, 256), 256, 0, st>>>(sh, s0, ns); note_launch();
        }
        pc.mark("up", nc, ng);
    }
    HDP_CHECK_LAUNCH();
    for (int64_t r = 0; r < f->n_phases; r++) {
        int64_t g0 = f->seg_off[r], ng = f->seg_off[r + 1] - g0;
        int64_t c0 = f->chunk_off[r], nc = f->chunk_off[r + 1] - c0;
        const bool side = chunks && nc > 0 && ng > 0;
        if (side) {
            HDP_TRY(fork_side(ss, st));
            HDP_TRY(down_chunks(sh, f, r, cgrid, ng > 0, ssmem, csmem, ss->s));
        }
        if (ng > 0) {
            const bool hp = side && seg_prio;
            if (hp) HDP_TRY(fork_hi(ss));
            k_seg_down<<<dim3(sgrid(ng, side), lg.qgroups), 32 * kSegWarps, seg_smem, hp ? ss->hi : st>>>(
                lg, g0, ng, a.tickets + (2 * r + 1) * a.groups, seg_sq); note_launch();
            if (hp) HDP_TRY(join_hi(ss, st));
        }
        int64_t s0 = f->short_off[r], ns = f->short_off[r + 1] - s0;
        if (side) {
            HDP_TRY(join_side(ss, st));
        } else if (chunks && nc > 0) {
            HDP_TRY(down_chunks(sh, f, r, cgrid, false, ssmem, csmem, st));
        } else if (!chunks && ns > 0) {
            k_down_short<<<grid_for(ns * sh.sub, 256), 256, 0, st>>>(sh, s0, ns); note_launch();
        }
        pc.mark("down", nc, ng);
    }
    HDP_CHECK_LAUNCH();
    if (volume) {
        k_volume_copy<<<packed_grid(a, f->n, 1, 256), 256, 0, st>>>(a, f->n); note_launch();
    }
    if (disp || min_cost) {
        k_keys_finish<<<grid_for(f->n, 256), 256, 0, st>>>(f->n, kp, disp, min_cost); note_launch();
    }
    pc.mark("finish", 0, 0);
    pc.report();
    if (f->timing) HDP_CHECK_CUDA(cudaEventRecord(f->tev[2], st));
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

extern "C" int hdp_forest_set_timing(hdp_forest* f, int on) {
    HDP_REQUIRE(f != nullptr, HDP_ERR_CONFIG, "null forest");
    if (on)
        for (auto& e : f->tev)
            if (!e) HDP_CHECK_CUDA(cudaEventCreate(&e));
    f->timing = on ? 1 : 0;
    return HDP_OK;
}

extern "C" int hdp_forest_stage_ms(const hdp_forest* f, float* cost_ms, float* aggregate_ms) {
    HDP_REQUIRE(f != nullptr && f->timing, HDP_ERR_CONFIG, "forest timing is off");
    HDP_CHECK_CUDA(cudaEventSynchronize(f->tev[2]));
    float a = 0.0f, b = 0.0f;
    HDP_CHECK_CUDA(cudaEventElapsedTime(&a, f->tev[0], f->tev[1]));
    HDP_CHECK_CUDA(cudaEventElapsedTime(&b, f->tev[1], f->tev[2]));
    if (cost_ms) *cost_ms = a;
    if (aggregate_ms) *aggregate_ms = b;
    return HDP_OK;
}
