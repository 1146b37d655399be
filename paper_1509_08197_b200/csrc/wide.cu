// Two-pass tree aggregation + first argmin for WIDE dense rows (a disparity
// range of >= HDP_WIDE_MIN lanes on every tree: the full-range baseline,
// run_baseline_pipeline, aggregation.py:274-358, and its disparity slabs).
//
// Same recurrences and heavy-path layout as aggregate.cu (_two_pass,
// aggregation.py:158-179), organised for rows of hundreds of lanes:
//
// * one warp per (path or segment, 128-lane slice of the row): every lane owns
//   one float4 column and streams the rows through registers -- no shared-
//   memory staging, so occupancy is set by registers alone and every warp
//   keeps its own loads in flight;
// * the raw matching cost E is computed in the up pass from the packed image
//   planes (no E volume in HBM: the up pass writes A_up once and reads only
//   the light children's rows);
// * long paths are cut into 32-node segments whose carries are resolved by
//   separate small kernels (no spinning look-back): the up pass stores the
//   local values x_loc (carry 0) and the per-node carry factor P'(k); the
//   carry kernel fixes the path head's row (the only row a parent reads) and
//   leaves X_in per segment, so the down pass rebuilds A_up = x_loc + P' X_in
//   on the fly; the down pass runs a local pass (segment maps), a carry pass,
//   and the final pass with the first argmin of every node folded into a
//   64-bit key (atomicMin over the row's slices).
//
// Per phase: up [short paths + segment local] -> up carry; down segment local
// -> down carry -> down [short paths + segment final].
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "forest.cuh"

namespace hdp {

namespace {

constexpr float kWidePad = 1.0e30f;  // padding lanes: never win, sums stay finite (aggregate.cu kPadCost)
constexpr int kWideThreads = 256;

struct WideArgs {
    const int4* lmeta;      // (node, lane offset, image column, m) per layout position
    const float* lsimf;     // similarity, sign bit = has light children
    const int32_t* lc_start;
    const int64_t* lc_row;
    const float* lc_sim;
    const int4* sinfo;      // short paths: (start, len, m, lane offset)
    const longlong2* srows; // (first row, parent row or -1)
    const SegDesc* seg;
    const float4* pl;
    const float4* pr;
    float* aup;             // rows of mp floats, layout order
    float* pprod;           // per position: carry factor P'(k) of long-path nodes
    float4* xin;            // per segment: up carry (A_up of the next segment's first node)
    float4* yloc;           // per segment: local down value at its last node
    float* qend;            // per segment: product of its similarities
    float4* yin;            // per segment: down carry entering it
    unsigned long long* keys;
    int mp, mq, m;          // padded row floats, float4 columns, lanes
    int slices;             // 32-column slices per row
    int x0;                 // disparity of lane 0
    int c;
    float alpha, tc, tg, border;
    int64_t s0, ns;         // short paths of the phase
    int64_t g0, ng;         // segments of the phase
};

__device__ __forceinline__ float wide_cost(const WideArgs& a, float4 L, int32_t node, int col, int x) {
    if (col - x < 0) return a.border;
    const float4 R = __ldg(a.pr + node - x);
    float color;
    if (a.c == 3)
        color = (fabsf(L.x - R.x) + fabsf(L.y - R.y) + fabsf(L.z - R.z)) * (1.0f / 3.0f);
    else
        color = fabsf(L.x - R.x);
    const float gd = fabsf(L.w - R.w);
    return (1.0f - a.alpha) * fminf(a.tc, color) + a.alpha * fminf(a.tg, gd);
}

__device__ __forceinline__ float4* wide_row(const WideArgs& a, int64_t k) {
    return reinterpret_cast<float4*>(a.aup + k * (int64_t)a.mp);
}

// rows read by a kernel are never written by the same kernel before the read
// (light children / parents belong to earlier launches; a position's own row
// is read before its thread overwrites it): non-coherent loads, so the
// compiler may hoist them over the stores of other rows
__device__ __forceinline__ float4 wide_ld(const float* p, int64_t row, int jq) {
    return __ldg(reinterpret_cast<const float4*>(p + row) + jq);
}

constexpr int kGrp = 8;  // nodes whose loads are issued together

// b(k) = E(k) + (s_c0 A_up(c0) + s_c1 A_up(c1) + ...) (the order of
// aggregate.cu's k_light) for this lane's float4 column jq; node / col / light
// range of k are given (warp-uniform)
__device__ __forceinline__ float4 wide_b(const WideArgs& a, int32_t node, int col, int e0, int e1, int jq) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e1 > e0) {
        // <= 3 light children on a 4-connected grid tree (unrolled; more loop)
        float4 v[3];
        float sc[3];
#pragma unroll
        for (int q = 0; q < 3; q++) {
            if (e0 + q < e1) {
                sc[q] = __ldg(a.lc_sim + e0 + q);
                v[q] = wide_ld(a.aup, __ldg(a.lc_row + e0 + q), jq);
            }
        }
        acc = make_float4(sc[0] * v[0].x, sc[0] * v[0].y, sc[0] * v[0].z, sc[0] * v[0].w);
#pragma unroll
        for (int q = 1; q < 3; q++) {
            if (e0 + q < e1) {
                acc.x += sc[q] * v[q].x;
                acc.y += sc[q] * v[q].y;
                acc.z += sc[q] * v[q].z;
                acc.w += sc[q] * v[q].w;
            }
        }
        for (int e = e0 + 3; e < e1; e++) {
            const float s3 = __ldg(a.lc_sim + e);
            const float4 w3 = wide_ld(a.aup, __ldg(a.lc_row + e), jq);
            acc.x += s3 * w3.x;
            acc.y += s3 * w3.y;
            acc.z += s3 * w3.z;
            acc.w += s3 * w3.w;
        }
    }
    const float4 L = __ldg(a.pl + node);
    const int j = 4 * jq;
    float4 e;
    e.x = j < a.m ? wide_cost(a, L, node, col, a.x0 + j) : kWidePad;
    e.y = j + 1 < a.m ? wide_cost(a, L, node, col, a.x0 + j + 1) : kWidePad;
    e.z = j + 2 < a.m ? wide_cost(a, L, node, col, a.x0 + j + 2) : kWidePad;
    e.w = j + 3 < a.m ? wide_cost(a, L, node, col, a.x0 + j + 3) : kWidePad;
    if (e1 > e0) {
        e.x = e.x + acc.x;
        e.y = e.y + acc.y;
        e.z = e.z + acc.z;
        e.w = e.w + acc.w;
    }
    return e;
}

// up pass of one path segment [k0, k0 + cnt) (a whole short path when it has
// no next segment): x(k) = b(k) + s(k+1) x(k+1) from the tail, kGrp nodes at a
// time (their metadata and inputs loaded together, then the recurrence); the
// carry factor P'(k) = prod_{j = k+1 .. end} s(j) of a segment with a next one
__device__ __forceinline__ void wide_up_run(const WideArgs& a, int64_t k0, int cnt, bool has_next, bool store_p,
                                            int jq, bool act, int lane) {
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    float s_after = has_next ? fabsf(__ldg(a.lsimf + k0 + cnt)) : 0.0f;  // s of the node after the group
    float p = s_after;                                                     // P' of the group's last node
    for (int hi = cnt; hi > 0; hi -= kGrp) {
        const int lo = max(0, hi - kGrp), gn = hi - lo;
        // lane u < gn: metadata of position k0 + lo + u
        int32_t nd = 0, cl = 0, e0 = 0, e1 = 0;
        float sf = 0.0f;
        if (lane < gn) {
            const int64_t k = k0 + lo + lane;
            const int4 mt = __ldg(a.lmeta + k);
            nd = mt.x;
            cl = mt.z;
            e0 = __ldg(a.lc_start + k);
            e1 = __ldg(a.lc_start + k + 1);
            sf = fabsf(__ldg(a.lsimf + k));
        }
        float4 b[kGrp];
#pragma unroll
        for (int u = 0; u < kGrp; u++) {
            const int32_t n_u = __shfl_sync(0xffffffffu, nd, u);
            const int c_u = __shfl_sync(0xffffffffu, cl, u);
            const int a_u = __shfl_sync(0xffffffffu, e0, u);
            const int b_u = __shfl_sync(0xffffffffu, e1, u);
            if (u < gn && act) b[u] = wide_b(a, n_u, c_u, a_u, b_u, jq);
        }
#pragma unroll
        for (int u = kGrp - 1; u >= 0; u--) {
            if (u >= gn) continue;
            const float s_next = u + 1 < gn ? __shfl_sync(0xffffffffu, sf, (u + 1) & 31) : s_after;
            const int64_t k = k0 + lo + u;
            if (act) {
                if (lo + u == cnt - 1) {
                    x = b[u];
                } else {
                    x.x = b[u].x + s_next * x.x;
                    x.y = b[u].y + s_next * x.y;
                    x.z = b[u].z + s_next * x.z;
                    x.w = b[u].w + s_next * x.w;
                }
                wide_row(a, k)[jq] = x;
            }
            if (store_p) {
                if (lane == 0) a.pprod[k] = p;
                p *= __shfl_sync(0xffffffffu, sf, u);  // P'(k - 1) = s(k) P'(k)
            }
        }
        s_after = __shfl_sync(0xffffffffu, sf, 0);
    }
}

// [short paths of the phase] + [segments of the phase]: one warp per (item, slice)
__global__ void __launch_bounds__(kWideThreads) k_wide_up(WideArgs a) {
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t item = wid / a.slices;
    const int g = (int)(wid - item * a.slices);
    const int jq = g * 32 + lane;
    const bool act = jq < a.mq;
    if (item < a.ns) {
        const int4 in = __ldg(a.sinfo + a.s0 + item);
        wide_up_run(a, in.x, in.y, false, false, jq, act, lane);
    } else if (item < a.ns + a.ng) {
        const SegDesc d = a.seg[a.g0 + item - a.ns];
        wide_up_run(a, d.a, d.cnt, d.s + 1 < d.nseg, g == 0, jq, act, lane);
    }
}

// Up carries of the phase's long paths (one warp per (head segment, slice)):
// X_in(S) = A_up(first node of S+1) = x_loc + P' X_in(S+1), from the tail;
// then the head row becomes final (the parent's light-children sum reads it).
constexpr int kCarryAhead = 16;
__global__ void __launch_bounds__(kWideThreads) k_wide_up_carry(WideArgs a) {
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t si = wid / a.slices;
    if (si >= a.ng) return;
    const int g = (int)(wid - si * a.slices);
    const int jq = g * 32 + lane;
    const bool act = jq < a.mq;
    const int64_t gs = a.g0 + si;
    const SegDesc d0 = a.seg[gs];
    if (d0.s != 0) return;  // head segments only
    const int nseg = d0.nseg;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 X = z;
    if (act) a.xin[(gs + nseg - 1) * a.mq + jq] = z;
    // S = nseg-1 .. 1, loads prefetched kCarryAhead segments ahead
    for (int S0 = nseg - 1; S0 >= 1; S0 -= kCarryAhead) {
        float4 xa[kCarryAhead];
        float pa[kCarryAhead];
#pragma unroll
        for (int u = 0; u < kCarryAhead; u++) {
            const int S = S0 - u;
            if (S >= 1 && act) {
                const SegDesc& dS = a.seg[gs + S];
                xa[u] = wide_row(a, dS.a)[jq];
                pa[u] = a.pprod[dS.a];
            }
        }
#pragma unroll
        for (int u = 0; u < kCarryAhead; u++) {
            const int S = S0 - u;
            if (S >= 1 && act) {
                X.x = xa[u].x + pa[u] * X.x;
                X.y = xa[u].y + pa[u] * X.y;
                X.z = xa[u].z + pa[u] * X.z;
                X.w = xa[u].w + pa[u] * X.w;
                a.xin[(gs + S - 1) * a.mq + jq] = X;
            }
        }
    }
    if (act) {
        float4* r = wide_row(a, d0.a) + jq;
        const float p = a.pprod[d0.a];
        float4 v = *r;
        v.x += p * X.x;
        v.y += p * X.y;
        v.z += p * X.z;
        v.w += p * X.w;
        *r = v;
    }
}

// A_up of the kGrp positions [k0 + lo, k0 + lo + gn) of segment d (nullptr:
// a short path, rows final): x_loc + P' X_in except at the path head, whose
// row the up carry already made final.  Lane u < gn returns (node id,
// similarity word) of position lo + u.
__device__ __forceinline__ void wide_load_grp(const WideArgs& a, const SegDesc* d, int64_t k0, int lo, int gn,
                                              float4 X, int jq, bool act, int lane, float4 (&u)[kGrp],
                                              int32_t& nd, float& sf) {
    nd = 0;
    sf = 0.0f;
    float pp = 0.0f;
    if (lane < gn) {
        const int64_t k = k0 + lo + lane;
        nd = __ldg(&a.lmeta[k].x);
        sf = __ldg(a.lsimf + k);
        if (d) pp = (d->s == 0 && lo + lane == 0) ? 0.0f : __ldg(a.pprod + k);
    }
#pragma unroll
    for (int v = 0; v < kGrp; v++) {
        const float p = __shfl_sync(0xffffffffu, pp, v);
        if (v < gn && act) {
            u[v] = wide_ld(a.aup, (k0 + lo + v) * (int64_t)a.mp, jq);
            if (d) {
                u[v].x += p * X.x;
                u[v].y += p * X.y;
                u[v].z += p * X.z;
                u[v].w += p * X.w;
            }
        }
    }
}

// down local pass of the phase's segments (Y_in = 0): segment maps
__global__ void __launch_bounds__(kWideThreads) k_wide_down_local(WideArgs a) {
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t si = wid / a.slices;
    if (si >= a.ng) return;
    const int g = (int)(wid - si * a.slices);
    const int jq = g * 32 + lane;
    const bool act = jq < a.mq;
    const int64_t gs = a.g0 + si;
    const SegDesc d = a.seg[gs];
    if (d.s + 1 >= d.nseg) return;  // the last segment's map is never used
    const float4 X = act ? a.xin[gs * a.mq + jq] : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    float Q = 1.0f;
    const bool root = d.s == 0 && d.prow < 0;
    for (int lo = 0; lo < d.cnt; lo += kGrp) {
        const int gn = min(kGrp, d.cnt - lo);
        float4 u[kGrp];
        int32_t nd;
        float sf;
        wide_load_grp(a, &d, d.a, lo, gn, X, jq, act, lane, u, nd, sf);
#pragma unroll
        for (int v = 0; v < kGrp; v++) {
            if (v >= gn) break;
            const float sv = __shfl_sync(0xffffffffu, sf, v);
            const float s = (root && lo + v == 0) ? 0.0f : fabsf(sv);
            Q *= s;
            if (act) {
                const float w = 1.0f - s * s;
                y.x = s * y.x + w * u[v].x;
                y.y = s * y.y + w * u[v].y;
                y.z = s * y.z + w * u[v].z;
                y.w = s * y.w + w * u[v].w;
            }
        }
    }
    if (act) a.yloc[gs * a.mq + jq] = y;
    if (lane == 0 && g == 0) a.qend[gs] = Q;
}

// down carries (head segments): Y_in(0) = A(parent) (0 at a root),
// Y_in(S+1) = y_loc(S) + Q(S) Y_in(S)
__global__ void __launch_bounds__(kWideThreads) k_wide_down_carry(WideArgs a) {
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t si = wid / a.slices;
    if (si >= a.ng) return;
    const int g = (int)(wid - si * a.slices);
    const int jq = g * 32 + lane;
    const bool act = jq < a.mq;
    const int64_t gs = a.g0 + si;
    const SegDesc d0 = a.seg[gs];
    if (d0.s != 0 || !act) return;
    float4 Y = d0.prow >= 0 ? reinterpret_cast<const float4*>(a.aup + d0.prow)[jq] : make_float4(0.f, 0.f, 0.f, 0.f);
    const int nseg = d0.nseg;
    for (int S0 = 0; S0 < nseg; S0 += kCarryAhead) {
        float4 yl[kCarryAhead];
        float q[kCarryAhead];
#pragma unroll
        for (int u = 0; u < kCarryAhead; u++) {
            const int S = S0 + u;
            if (S + 1 < nseg) {
                yl[u] = a.yloc[(gs + S) * a.mq + jq];
                q[u] = a.qend[gs + S];
            }
        }
#pragma unroll
        for (int u = 0; u < kCarryAhead; u++) {
            const int S = S0 + u;
            if (S < nseg) {
                a.yin[(gs + S) * a.mq + jq] = Y;
                if (S + 1 < nseg) {
                    Y.x = yl[u].x + q[u] * Y.x;
                    Y.y = yl[u].y + q[u] * Y.y;
                    Y.z = yl[u].z + q[u] * Y.z;
                    Y.w = yl[u].w + q[u] * Y.w;
                }
            }
        }
    }
}

__device__ __forceinline__ uint32_t wide_ord(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// first minimum of this warp's 128 lanes of node `node` folded into its key
__device__ __forceinline__ void wide_argmin(const WideArgs& a, float4 y, int jq, bool act, int32_t node) {
    float best = __int_as_float(0x7f800000);
    int bj = 0x7fffffff;
    if (act) {
        const int j = 4 * jq;
        if (y.x < best) { best = y.x; bj = j; }
        if (y.y < best) { best = y.y; bj = j + 1; }
        if (y.z < best) { best = y.z; bj = j + 2; }
        if (y.w < best) { best = y.w; bj = j + 3; }
    }
    uint32_t ob = bj == 0x7fffffff ? 0xffffffffu : wide_ord(best);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const uint32_t o2 = __shfl_xor_sync(0xffffffffu, ob, off);
        const int j2 = __shfl_xor_sync(0xffffffffu, bj, off);
        if (o2 < ob || (o2 == ob && j2 < bj)) {
            ob = o2;
            bj = j2;
        }
    }
    if ((threadIdx.x & 31) == 0 && bj != 0x7fffffff)
        atomicMin(a.keys + node, ((unsigned long long)ob << 32) | (uint32_t)(a.x0 + bj));
}

// down pass of a run of positions [k0, k0 + cnt) entering with Y: A = s A(prev)
// + (1 - s^2) A_up, first argmin per node, A stored where light children read it
__device__ __forceinline__ void wide_down_run(const WideArgs& a, const SegDesc* d, int64_t k0, int cnt, bool root_head,
                                              float4 y, float4 X, int jq, bool act, int lane) {
    for (int lo = 0; lo < cnt; lo += kGrp) {
        const int gn = min(kGrp, cnt - lo);
        float4 u[kGrp];
        int32_t nd;
        float sf;
        wide_load_grp(a, d, k0, lo, gn, X, jq, act, lane, u, nd, sf);
#pragma unroll
        for (int v = 0; v < kGrp; v++) {
            if (v >= gn) break;
            const float sv = __shfl_sync(0xffffffffu, sf, v);
            const int32_t node = __shfl_sync(0xffffffffu, nd, v);
            const float s = (root_head && lo + v == 0) ? 0.0f : fabsf(sv);
            if (act) {
                const float w = 1.0f - s * s;
                y.x = s * y.x + w * u[v].x;
                y.y = s * y.y + w * u[v].y;
                y.z = s * y.z + w * u[v].z;
                y.w = s * y.w + w * u[v].w;
                if (__float_as_uint(sv) >> 31) wide_row(a, k0 + lo + v)[jq] = y;  // light children read A
            }
            wide_argmin(a, y, jq, act, node);
        }
    }
}

__global__ void __launch_bounds__(kWideThreads) k_wide_down(WideArgs a) {
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t item = wid / a.slices;
    const int g = (int)(wid - item * a.slices);
    const int jq = g * 32 + lane;
    const bool act = jq < a.mq;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    if (item < a.ns) {
        const int4 in = __ldg(a.sinfo + a.s0 + item);
        const longlong2 rw = __ldg(a.srows + a.s0 + item);
        const float4 y = (rw.y >= 0 && act) ? wide_ld(a.aup, rw.y, jq) : z;
        wide_down_run(a, nullptr, in.x, in.y, rw.y < 0, y, z, jq, act, lane);
    } else if (item < a.ns + a.ng) {
        const int64_t gs = a.g0 + item - a.ns;
        const SegDesc d = a.seg[gs];
        float4 y = z, X = z;
        if (act) {
            X = a.xin[gs * a.mq + jq];
            if (d.s > 0) y = a.yin[gs * a.mq + jq];
            else if (d.prow >= 0) y = wide_ld(a.aup, d.prow, jq);
        }
        wide_down_run(a, &d, d.a, d.cnt, d.s == 0 && d.prow < 0, y, X, jq, act, lane);
    }
}

unsigned wide_grid(int64_t items, int slices) {
    const int64_t threads = items * slices * 32;
    return (unsigned)((threads + kWideThreads - 1) / kWideThreads);
}

}  // namespace

int wide_min_lanes() {
    static const int v = [] {
        const char* e = getenv("HDP_WIDE_MIN");  // tuning / A-B switch: 0 disables the wide path
        return e ? atoi(e) : 0;  // off by default: measured slower than aggregate.cu at C5
    }();
    return v;
}

int wide_aggregate(hdp_forest* f, const float* packed_l, const float* packed_r, int c, float alpha, float tau_c,
                   float tau_g, unsigned long long* keys, cudaStream_t st) {
    WideArgs a;
    a.lmeta = f->lmeta.get();
    a.lsimf = f->lsimf.get();
    a.lc_start = f->lc_start.get();
    a.lc_row = f->lc_row.get();
    a.lc_sim = f->lc_sim.get();
    a.sinfo = f->short_info.get();
    a.srows = f->short_rows.get();
    a.seg = f->seg_desc.get();
    a.pl = (const float4*)packed_l;
    a.pr = (const float4*)packed_r;
    a.m = f->max_m;
    a.mp = (f->max_m + 3) & ~3;
    a.mq = a.mp / 4;
    a.slices = (a.mq + 31) / 32;
    a.x0 = f->range_x0;
    a.c = c;
    a.alpha = alpha;
    a.tc = tau_c;
    a.tg = tau_g;
    a.border = (1.0f - alpha) * tau_c + alpha * tau_g;
    a.keys = keys;
    const int64_t nseg = f->n_segs;
    DevBuf<float> aup, pprod, qend;
    DevBuf<float4> xin, yloc, yin;
    HDP_TRY(aup.alloc(f->n * (int64_t)a.mp + 4, st));
    HDP_TRY(pprod.alloc(f->n + 1, st));
    HDP_TRY(qend.alloc(nseg + 1, st));
    HDP_TRY(xin.alloc((nseg + 1) * a.mq, st));
    HDP_TRY(yloc.alloc((nseg + 1) * a.mq, st));
    HDP_TRY(yin.alloc((nseg + 1) * a.mq, st));
    a.aup = aup.get();
    a.pprod = pprod.get();
    a.qend = qend.get();
    a.xin = xin.get();
    a.yloc = yloc.get();
    a.yin = yin.get();
    HDP_CHECK_CUDA(cudaMemsetAsync(keys, 0xff, sizeof(unsigned long long) * f->n, st));
    const int nph = (int)f->n_phases;
    auto set_phase = [&](int r) {
        a.s0 = f->short_off[r];
        a.ns = f->short_off[r + 1] - a.s0;
        a.g0 = f->seg_off[r];
        a.ng = f->seg_off[r + 1] - a.g0;
    };
    for (int r = nph - 1; r >= 0; r--) {
        set_phase(r);
        if (a.ns + a.ng > 0) {
            k_wide_up<<<wide_grid(a.ns + a.ng, a.slices), kWideThreads, 0, st>>>(a);
            note_launch();
        }
        if (a.ng > 0) {
            k_wide_up_carry<<<wide_grid(a.ng, a.slices), kWideThreads, 0, st>>>(a);
            note_launch();
        }
    }
    HDP_CHECK_LAUNCH();
    for (int r = 0; r < nph; r++) {
        set_phase(r);
        if (a.ng > 0) {
            k_wide_down_local<<<wide_grid(a.ng, a.slices), kWideThreads, 0, st>>>(a);
            note_launch();
            k_wide_down_carry<<<wide_grid(a.ng, a.slices), kWideThreads, 0, st>>>(a);
            note_launch();
        }
        if (a.ns + a.ng > 0) {
            k_wide_down<<<wide_grid(a.ns + a.ng, a.slices), kWideThreads, 0, st>>>(a);
            note_launch();
        }
    }
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

}  // namespace hdp
