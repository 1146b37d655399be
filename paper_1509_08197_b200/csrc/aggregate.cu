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
// its nodes share the tree's lane count m).  Per phase:
//   up   : k_ecompute   b(v) = E(v), all nodes of the phase in parallel (E
//                       recomputed from the packed image planes)
//          k_light      b(v) += sum_{light c} s_c A_up(c) for light parents
//          k_seg_up     A_up(v) = b(v) + s_h A_up(h) along paths > kShortPath
//                       nodes, cut into kSeg-node segments, one warp per
//                       (segment, 32 lanes): the segment is staged into shared
//                       memory with cp.async, a local pass yields its carry
//                       map (scalar product P, local value), carries are
//                       chained tail -> head by decoupled look-back (warps take
//                       segments by ticket, so a warp only waits on earlier
//                       tickets), and a second pass from shared memory writes
//                       the results
//          k_scan_up_short  register-resident walk of paths <= kShortPath
//   down : k_seg_down   the same for A (head -> tail), fused with the per-node
//                       first argmin (transpose butterfly, 31 shuffles / 32 nodes)
//          k_down_short short paths
// A is written back in place only where a light child will read it.
#include <cuda_runtime.h>

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
    unsigned long long* carry;  // per (segment, lane): (epoch << 32 | f32 bits), the
                                // epoch tag doubles as the readiness flag
    unsigned epoch_up, epoch_down;
    int* tickets;        // per (phase, pass, group)
    int groups;  // 32-lane groups per node when sub == 32
    int sub;     // lanes per item for the packed mappings (power of 2 <= 32)
    int sub_shift;
    int atomic_keys;
    int store_all;  // store A for every node (volume requested), not only light parents
    int max_m;
    int qsub, qsub_shift;  // chunk kernels: float4 lanes per path (power of 2 <= 32)
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
constexpr int kETile = 64;
__global__ void __launch_bounds__(256) k_ecost_pix(AggArgs a, const int32_t* __restrict__ lpos,
                                                   int d_hi, int use_smem) {
    extern __shared__ float4 win[];
    const int64_t base = (int64_t)blockIdx.x * a.w;  // node id of column 0 of this image row
    const int c0 = (int)blockIdx.y * kETile;
    const int lo = max(0, c0 - d_hi), hi = min(a.w, c0 + kETile);
    if (use_smem)
        for (int i = threadIdx.x; i < hi - lo; i += blockDim.x) win[i] = __ldg(a.pr + base + lo + i);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int per = 32 >> a.sub_shift;  // nodes per warp pass
    const int sl = lane & (a.sub - 1);
    for (int q = (threadIdx.x >> 5) * per + (lane >> a.sub_shift); q < kETile;
         q += (blockDim.x >> 5) * per) {
        const int col = c0 + q;
        if (col >= a.w) break;
        const int64_t node = base + col;
        const int kk = __ldg(lpos + node);
        const int4 mt = __ldg(a.lmeta + kk);
        float* out = a.aup + __ldg(a.rowoff + kk);
        const float4 L = __ldg(a.pl + node);
        const int mp = (mt.w + 3) & ~3;
        for (int j = sl; j < mp; j += a.sub) {
            if (j >= mt.w) {  // row padding
                out[j] = kPadCost;
                continue;
            }
            const int d = lane_disp(a, mt.y, j);
            float e = a.border;
            if (col - d >= 0) {
                const float4 R = use_smem ? win[col - d - lo] : __ldg(a.pr + node - d);
                float color;
                if (a.c == 3)
                    color = (fabsf(L.x - R.x) + fabsf(L.y - R.y) + fabsf(L.z - R.z)) * (1.0f / 3.0f);
                else
                    color = fabsf(L.x - R.x);
                e = (1.0f - a.alpha) * fminf(a.tc, color) + a.alpha * fminf(a.tg, fabsf(L.w - R.w));
            }
            out[j] = e;
        }
    }
}

// b(v) += sum_{light children c} s_c A_up(c) for the phase's light parents
// (children in ascending id order, their A_up final since the deeper phase).
// PU parents per thread; the first child of each is gathered up front.
__global__ void __launch_bounds__(256) k_light(AggArgs a, int64_t p0, int64_t np) {
    Slot s = slot_of(a);
    int32_t k[4], c0[4], c1[4];
    int m[4];
    bool ok[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
        int64_t it = s.item * 4 + u;
        ok[u] = it < np;
        k[u] = ok[u] ? a.lp_list[p0 + it] : 0;
        m[u] = a.lmeta[k[u]].w;
        c0[u] = a.lc_start[k[u]];
        c1[u] = a.lc_start[k[u] + 1];
        ok[u] = ok[u] && s.j < m[u];
    }
    float first[4], bv[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
        first[u] = ok[u] ? a.lc_sim[c0[u]] * a.aup[a.lc_row[c0[u]] + s.j] : 0.0f;
        bv[u] = ok[u] ? a.aup[a.rowoff[k[u]] + s.j] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
        if (!ok[u]) continue;
        float x = first[u];
        for (int32_t q = c0[u] + 1; q < c1[u]; q++) x += a.lc_sim[q] * a.aup[a.lc_row[q] + s.j];
        a.aup[a.rowoff[k[u]] + s.j] = bv[u] + x;
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

// ---------------------------------------------------------------- segments

struct SegCtx {
    int32_t start, len, m, doff, mp;
    int64_t row0, prow;
    int32_t a, b;    // segment node range [a, b) (layout positions)
    int s, nseg;
    int64_t gseg;    // global segment index
};

__device__ __forceinline__ SegCtx seg_ctx(const AggArgs& a, int64_t gseg) {
    int2 st = a.seg_tab[gseg];
    int4 info = a.pinfo[st.x];
    longlong2 rows = a.prows[st.x];
    SegCtx c;
    c.start = info.x;
    c.len = info.y;
    c.m = info.z;
    c.mp = (info.z + 3) & ~3;
    c.doff = info.w;
    c.row0 = rows.x;
    c.prow = rows.y;
    c.s = st.y;
    c.nseg = (c.len + kSeg - 1) / kSeg;
    c.a = c.start + c.s * kSeg;
    c.b = min(c.start + c.len, c.a + kSeg);
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

// Up pass over one segment (tail -> head).  Segments are taken by ticket in
// reverse table order, so a path's tail segment comes first; the carry is
// X_a = x_loc(a) + P * X_b with P = prod s_{a+1..b}.
__global__ void __launch_bounds__(128) k_seg_up(AggArgs a, int64_t g0, int64_t ng, int* ctr) {
    __shared__ float buf[4][kSeg][32];
    __shared__ float ssim[4][kSeg + 1];
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int g = (int)blockIdx.y;
    int t = warp_ticket(ctr + g);
    if (t >= ng) return;
    SegCtx c = seg_ctx(a, g0 + ng - 1 - t);
    if (g * 32 >= c.m) return;
    int j = g * 32 + lane;
    bool act = j < c.m;
    int cnt = c.b - c.a;
    const float* base = a.aup + c.row0 + (int64_t)(c.a - c.start) * c.mp + j;
    for (int i = 0; i < cnt; i++) cp_async4(&buf[warp][i][lane], base + (int64_t)i * c.mp, act);
    cp_commit();
    bool has_next = c.b < c.start + c.len;  // a segment toward the tail exists
    for (int i = lane; i <= cnt; i += 32) {
        int p = c.a + i;
        ssim[warp][i] = (i < cnt || has_next) ? fabsf(a.lsimf[p]) : 0.0f;
    }
    cp_wait_all();
    __syncwarp();
    // local pass with X_b = 0: x_loc(a) and P = prod_{t=a+1..b} s_t
    float x = 0.0f, P = 1.0f;
    for (int i = cnt - 1; i >= 0; i--) {
        float sn = ssim[warp][i + 1];  // s of the node after i (0 past the tail)
        x = buf[warp][i][lane] + sn * x;
        P *= sn;
    }
    float Xb = 0.0f;
    if (has_next && act) Xb = get_carry(a.carry + (c.gseg + 1) * a.max_m + j, a.epoch_up);
    if (act && c.s > 0) put_carry(a.carry + c.gseg * a.max_m + j, a.epoch_up, x + P * Xb);
    // final pass: exact recurrence from the true X_b
    x = Xb;
    float* out = a.aup + c.row0 + (int64_t)(c.a - c.start) * c.mp + j;
    for (int i = cnt - 1; i >= 0; i--) {
        x = buf[warp][i][lane] + ssim[warp][i + 1] * x;
        if (act) out[(int64_t)i * c.mp] = x;
    }
}

// warp transpose butterfly: lane l ends with the minimum key of node l
__device__ __forceinline__ unsigned long long warp_min_per_node(unsigned long long (&key)[32],
                                                                int lane) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        bool up_half = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; i++) {
            unsigned long long send = up_half ? key[i] : key[i + o];
            unsigned long long keep = up_half ? key[i + o] : key[i];
            unsigned long long recv = __shfl_xor_sync(0xffffffffu, send, o);
            key[i] = recv < keep ? recv : keep;
        }
    }
    return key[0];
}

// First argmin of (cost, d) over the lanes of one item: `width` lanes
// (power of two, aligned) or the full warp.  32-bit shuffle min on the
// order-preserving cost, then the lowest lane holding it (lanes are in
// ascending disparity order) supplies d.  Every lane gets the packed key.
__device__ __forceinline__ unsigned long long group_argmin(bool act, float y, int d, int width,
                                                           int lane) {
    uint32_t o = act ? ord_f32(y) : 0xffffffffu;
    uint32_t mn = o;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        uint32_t t = __shfl_xor_sync(0xffffffffu, mn, off);
        if (off < width) mn = min(mn, t);
    }
    unsigned gmask = width == 32 ? 0xffffffffu : ((1u << width) - 1u) << (lane & ~(width - 1));
    unsigned eq = __ballot_sync(0xffffffffu, o == mn) & gmask;
    int dmin = __shfl_sync(0xffffffffu, d, __ffs(eq) - 1);
    return ((unsigned long long)mn << 32) | (uint32_t)dmin;
}

__device__ __forceinline__ void store_key(const AggArgs& a, int32_t node, unsigned long long k) {
    if (!a.keys) return;
    if (a.atomic_keys)
        atomicMin(&a.keys[node], k);
    else
        a.keys[node] = k;
}

// Down pass over one segment (head -> tail).  The carry is
// Y_end = y_loc(b-1) + Q * Y_in with Q = prod_{t=a..b-1} s_t; the head of a
// root path uses s = 0 so that A(root) = A_up(root).  The first argmin of
// each node over this warp's 32 lanes is folded into the node's key with a
// 64-bit min (several lane groups per node) or stored (one group); A is
// written back only where a light child will read it.
__global__ void __launch_bounds__(128) k_seg_down(AggArgs a, int64_t g0, int64_t ng, int* ctr) {
    __shared__ float buf[4][kSeg][32];
    __shared__ float ssim[4][kSeg];
    __shared__ int32_t snode[4][kSeg];
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int g = (int)blockIdx.y;
    int t = warp_ticket(ctr + g);
    if (t >= ng) return;
    SegCtx c = seg_ctx(a, g0 + t);
    if (g * 32 >= c.m) return;
    int j = g * 32 + lane;
    bool act = j < c.m;
    int cnt = c.b - c.a;
    float* rows = a.aup + c.row0 + (int64_t)(c.a - c.start) * c.mp + j;
    for (int i = 0; i < cnt; i++) cp_async4(&buf[warp][i][lane], rows + (int64_t)i * c.mp, act);
    cp_commit();
    unsigned long long lmask = 0;  // bit i: node a+i has light children
    for (int i0 = 0; i0 < kSeg; i0 += 32) {
        int i = i0 + lane;
        float f = i < cnt ? a.lsimf[c.a + i] : 0.0f;
        if (i < cnt) snode[warp][i] = a.lmeta[c.a + i].x;
        float sv = fabsf(f);
        if (c.a + i == c.start && c.prow < 0) sv = 0.0f;  // root: A = A_up
        if (i < cnt) ssim[warp][i] = sv;
        unsigned b = __ballot_sync(0xffffffffu, i < cnt && (__float_as_uint(f) >> 31));
        lmask |= (unsigned long long)b << i0;
    }
    if (a.store_all) lmask = ~0ull;
    const int d = act ? lane_disp(a, c.doff, j) : 0;
    cp_wait_all();
    __syncwarp();
    // local pass with Y_in = 0: y_loc(b-1) and Q = prod_{t=a..b-1} s_t
    float yl = 0.0f, Q = 1.0f;
    for (int i = 0; i < cnt; i++) {
        float sv = ssim[warp][i];
        yl = sv * yl + (1.0f - sv * sv) * buf[warp][i][lane];
        Q *= sv;
    }
    float Yin = 0.0f;
    if (c.s == 0) {
        if (c.prow >= 0 && act) Yin = a.aup[c.prow + j];  // A(parent), stored in place
    } else if (act) {
        Yin = get_carry(a.carry + (c.gseg - 1) * a.max_m + j, a.epoch_down);
    }
    // publish the tail-end carry before the final pass
    if (act && c.s + 1 < c.nseg) put_carry(a.carry + c.gseg * a.max_m + j, a.epoch_down, yl + Q * Yin);
    float y = Yin;
    for (int i = 0; i < cnt; i++) {
        float sv = ssim[warp][i];
        y = sv * y + (1.0f - sv * sv) * buf[warp][i][lane];
        if (act && ((lmask >> i) & 1ull)) rows[(int64_t)i * c.mp] = y;
        unsigned long long key = group_argmin(act, y, d, 32, lane);
        if (lane == 0 && a.keys) {
            if (a.atomic_keys)
                atomicMin(&a.keys[snode[warp][i]], key);
            else
                a.keys[snode[warp][i]] = key;
        }
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
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

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
                                               unsigned long long* bar) {
    ChunkSm s = carve<UP>(d, sm4);
    const int tid = threadIdx.x, nt = blockDim.x;
    if (tid == 0) mbar_init(bar, 1);
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
    mbar_wait(bar, 0);
    __syncthreads();
    return s;
}

// Up pass: tail -> head, A_up(q) = (E(q) + sum_light s_c A_up(c)) + s_{q+1} A_up(q+1)
// (the operation order of k_light + k_scan_up_short).  One thread per
// (path, float4 column); changed rows are stored, a lone leaf row (A_up = E)
// is left alone.
__global__ void __launch_bounds__(kChunkThreads) k_up_chunk(AggArgs a, const ChunkDesc* __restrict__ descs,
                                                            int64_t cbase) {
    extern __shared__ float4 sm4[];
    const ChunkDesc d = descs[cbase + blockIdx.x];
    if (d.np == 0) return;
    __shared__ unsigned long long bar;
    const ChunkSm s = stage_chunk<true>(a, d, sm4, &bar);
    const float4* own4 = reinterpret_cast<const float4*>(s.own);
    const float4* aux4 = reinterpret_cast<const float4*>(s.aux);
    // with a uniform row width the (path, column) split is a multiply-high;
    // otherwise each path takes a 32-column stride of threads
    const int mqu = d.mqu;
    const int items = mqu > 0 ? d.np * mqu : d.np << a.qsub_shift;
    for (int t = threadIdx.x; t < items; t += blockDim.x) {
        int pi, jq;
        if (mqu > 0) {
            pi = (int)__umulhi((unsigned)t, d.inv);
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
}

// Down pass fused with the first argmin: head -> tail,
// A(q) = s_q A(q - 1) + (1 - s_q^2) A_up(q) with A(-1) = A(parent) (s = 0 at a
// root), one thread per (path, float4 column), A kept in shared memory and
// stored globally only where a light child will read it; then one thread
// per node scans its row for the first minimum (aggregation.py:249).
__global__ void __launch_bounds__(kChunkThreads) k_down_chunk(AggArgs a, const ChunkDesc* __restrict__ descs,
                                                              int64_t cbase) {
    extern __shared__ float4 sm4[];
    const ChunkDesc d = descs[cbase + blockIdx.x];
    if (d.np == 0) return;
    __shared__ unsigned long long bar;
    const ChunkSm s = stage_chunk<false>(a, d, sm4, &bar);
    float4* own4 = reinterpret_cast<float4*>(s.own);
    const float4* aux4 = reinterpret_cast<const float4*>(s.aux);
    const int mqu = d.mqu;
    const int items = mqu > 0 ? d.np * mqu : d.np << a.qsub_shift;
    for (int t = threadIdx.x; t < items; t += blockDim.x) {
        int pi, jq;
        if (mqu > 0) {
            pi = (int)__umulhi((unsigned)t, d.inv);
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
    for (int i = threadIdx.x; i < d.nk; i += blockDim.x) {
        const int4 mt = s.meta[i];
        const int mq = (mt.w + 3) >> 2;
        const float4* row = reinterpret_cast<const float4*>(s.own + (s.nrow[i] - d.a0));
        // the minimum (padding lanes hold kPadCost and never win), then the
        // first lane holding it
        float best = row[0].x;
        for (int jq = 0; jq < mq; jq++) {
            const float4 y = row[jq];
            best = fminf(best, fminf(fminf(y.x, y.y), fminf(y.z, y.w)));
        }
        int bj = 0;
        for (int jq = 0; jq < mq; jq++) {
            const float4 y = row[jq];
            if (y.x == best) { bj = 4 * jq; break; }
            if (y.y == best) { bj = 4 * jq + 1; break; }
            if (y.z == best) { bj = 4 * jq + 2; break; }
            if (y.w == best) { bj = 4 * jq + 3; break; }
        }
        if (a.keys) a.keys[mt.x] = ((unsigned long long)ord_f32(best) << 32) | (uint32_t)lane_disp(a, mt.y, bj);
    }
}

// First argmin per layout position (aggregation.py:249: np.argmin, smallest
// disparity on ties).  Rows are read in layout order (streaming); with sub
// < 32 several short rows share a warp, otherwise one warp scans a row.
__global__ void __launch_bounds__(256) k_wta(AggArgs a, int64_t n) {
    Slot s = slot_of(a);
    int lane = threadIdx.x & 31;
    bool valid = s.item < n;
    int4 mt = valid ? a.lmeta[s.item] : make_int4(0, 0, 0, 0);
    int64_t row = valid ? a.rowoff[s.item] : 0;
    uint32_t best = 0xffffffffu;
    int bj = 0x7fffffff;
    int width = a.sub < 32 ? a.sub : 32;
    int step = width;
    // sub == 32: lane j0 scans j0, j0+32, ... ; keep the first minimum
    for (int jj = (a.sub < 32 ? s.j : lane); valid && jj < mt.w; jj += step) {
        uint32_t o = ord_f32(a.aup[row + jj]);
        if (o < best) {
            best = o;
            bj = jj;
        }
    }
    uint32_t mn = best;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        uint32_t t = __shfl_xor_sync(0xffffffffu, mn, off);
        if (off < width) mn = min(mn, t);
    }
    int jm = (best == mn) ? bj : 0x7fffffff;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        int t = __shfl_xor_sync(0xffffffffu, jm, off);
        if (off < width) jm = min(jm, t);
    }
    if (valid && (lane & (width - 1)) == 0 && a.keys && jm != 0x7fffffff)
        a.keys[mt.x] = ((unsigned long long)mn << 32) | (uint32_t)lane_disp(a, mt.y, jm);
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

__global__ void k_keys_init(int64_t n, unsigned long long* keys) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = ~0ull;
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

extern "C" int hdp_aggregate_wta(hdp_forest* f, const float* packed_l, const float* packed_r,
                                 int h, int w, int c, float alpha, float tau_c, float tau_g,
                                 const float* cost_rows, int32_t* disp, float* min_cost,
                                 uint64_t* keys, float* volume, void* stream) {
    HDP_REQUIRE(f != nullptr && f->lanes_set, HDP_ERR_CONFIG, "forest lanes not set");
    HDP_REQUIRE(cost_rows || (packed_l && packed_r && h > 0 && w > 0), HDP_ERR_CONFIG,
                "need either cost rows or image planes");
    HDP_REQUIRE(cost_rows || (int64_t)h * w < ((int64_t)1 << 31), HDP_ERR_CONFIG, "image too large");
    cudaStream_t st = (cudaStream_t)stream;
    AggArgs a;
    a.lmeta = f->lmeta.get();
    a.lsimf = f->lsimf.get();
    a.lc_start = f->lc_start.get();
    a.lc_row = f->lc_row.get();
    a.lc_sim = f->lc_sim.get();
    a.pinfo = nullptr;
    a.prows = nullptr;
    a.seg_tab = f->seg_tab.get();
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
    a.sub = f->max_m <= 16 ? std::max(4, pow2_at_least(f->max_m)) : 32;  // >= one padded row
    a.sub_shift = 0;
    while ((1 << a.sub_shift) < a.sub) a.sub_shift++;
    {
        const int mq = (f->max_m + 3) >> 2;
        a.qsub = mq <= 16 ? pow2_at_least(mq) : 32;
        a.qsub_shift = 0;
        while ((1 << a.qsub_shift) < a.qsub) a.qsub_shift++;
    }
    DevBuf<float> aup;
    DevBuf<unsigned long long> carry;
    DevBuf<int> tickets;
    HDP_TRY(aup.alloc(f->total_rows + 32, st));
    a.aup = aup.get();
    const int64_t nseg = f->n_segs;
    HDP_TRY(carry.alloc(nseg * a.max_m + 1, st));
    HDP_TRY(tickets.alloc(2 * f->n_phases * a.groups + 1, st));
    HDP_CHECK_CUDA(cudaMemsetAsync(tickets.get(), 0,
                                   sizeof(int) * (2 * f->n_phases * a.groups + 1), st));
    // fresh epochs per call: stale words in recycled pool memory never match
    static std::atomic<unsigned> g_epoch{1};
    unsigned ep = g_epoch.fetch_add(2);
    if (ep == 0u || ep + 1 == 0u) ep = g_epoch.fetch_add(2);
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
    a.atomic_keys = (f->n_segs > 0 && a.groups > 1) ? 1 : 0;
    if (a.atomic_keys) HDP_CHECK_CUDA(cudaMemsetAsync(kp, 0xff, sizeof(unsigned long long) * f->n, st));
    a.store_all = volume != nullptr;
    if (!cost_rows && (f->geom_w != a.w || f->geom_np != a.npix)) {
        k_fill_cols<<<grid_for(f->n, 256), 256, 0, st>>>(f->n, f->lmeta.get(), a.npix, a.w); note_launch();
        f->geom_w = a.w;
        f->geom_np = a.npix;
    }

    AggArgs lg = a;  // segment kernels: one warp per (segment, 32 lanes)
    lg.sub = 32;
    lg.pinfo = f->long_info.get();
    lg.prows = f->long_rows.get();
    AggArgs sh = a;
    sh.pinfo = f->short_info.get();
    sh.prows = f->short_rows.get();
    if (cost_rows) {
        k_ecompute<<<packed_grid(a, f->n, BU, 256), 256, 0, st>>>(a, 0, f->n); note_launch();
    } else {
        HDP_REQUIRE(f->n % a.w == 0, HDP_ERR_CONFIG, "node count is not a whole number of image rows");
        int64_t rows = f->n / a.w;
        HDP_REQUIRE(rows < ((int64_t)1 << 31), HDP_ERR_CONFIG, "too many image rows");
        size_t smem = (size_t)(kETile + f->max_d) * sizeof(float4);
        int use = smem <= 48 * 1024;
        dim3 g((unsigned)rows, (unsigned)((a.w + kETile - 1) / kETile));
        k_ecost_pix<<<g, 256, use ? smem : 0, st>>>(a, f->lpos.get(), f->max_d, use); note_launch();
    }
    const bool chunks = f->chunks_ok != 0;
    const size_t csmem = (size_t)((f->chunk_words + 3) & ~3ll) * sizeof(float);
    sh.lc_rowoff = f->lc_rowoff.get();
    sh.auxd = f->auxd.get();
    if (chunks && csmem > 48 * 1024) {
        HDP_CHECK_CUDA(cudaFuncSetAttribute(k_up_chunk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
        HDP_CHECK_CUDA(cudaFuncSetAttribute(k_down_chunk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
    }
    for (int64_t r = f->n_phases - 1; r >= 0; r--) {
        // light parents on short paths are handled inside k_up_chunk
        int64_t p0 = chunks ? f->lp_mid[r] : f->lp_off[r], np = f->lp_off[r + 1] - p0;
        if (np > 0) {
            k_light<<<packed_grid(a, (np + 3) / 4, 1, 256), 256, 0, st>>>(a, p0, np); note_launch();
        }
        int64_t g0 = f->seg_off[r], ng = f->seg_off[r + 1] - g0;
        if (ng > 0) {
            k_seg_up<<<dim3(grid_for(ng * 32, 128), lg.groups), 128, 0, st>>>(
                lg, g0, ng, a.tickets + (2 * r) * a.groups); note_launch();
        }
        int64_t s0 = f->short_off[r], ns = f->short_off[r + 1] - s0;
        int64_t c0 = f->chunk_off[r], nc = f->chunk_off[r + 1] - c0;
        if (chunks && nc > 0) {
            k_up_chunk<<<(unsigned)nc, kChunkThreads, csmem, st>>>(sh, f->chunk_desc.get(), c0); note_launch();
        } else if (!chunks && ns > 0) {
            k_scan_up_short<<<grid_for(ns * sh.sub, 256), 256, 0, st>>>(sh, s0, ns); note_launch();
        }
    }
    HDP_CHECK_LAUNCH();
    for (int64_t r = 0; r < f->n_phases; r++) {
        int64_t g0 = f->seg_off[r], ng = f->seg_off[r + 1] - g0;
        if (ng > 0) {
            k_seg_down<<<dim3(grid_for(ng * 32, 128), lg.groups), 128, 0, st>>>(
                lg, g0, ng, a.tickets + (2 * r + 1) * a.groups); note_launch();
        }
        int64_t s0 = f->short_off[r], ns = f->short_off[r + 1] - s0;
        int64_t c0 = f->chunk_off[r], nc = f->chunk_off[r + 1] - c0;
        if (chunks && nc > 0) {
            k_down_chunk<<<(unsigned)nc, kChunkThreads, csmem, st>>>(sh, f->chunk_desc.get(), c0); note_launch();
        } else if (!chunks && ns > 0) {
            k_down_short<<<grid_for(ns * sh.sub, 256), 256, 0, st>>>(sh, s0, ns); note_launch();
        }
    }
    HDP_CHECK_LAUNCH();
    if (volume) {
        k_volume_copy<<<packed_grid(a, f->n, 1, 256), 256, 0, st>>>(a, f->n); note_launch();
    }
    if (disp || min_cost) {
        k_keys_finish<<<grid_for(f->n, 256), 256, 0, st>>>(f->n, kp, disp, min_cost); note_launch();
    }
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}
