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
    int max_m;
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
        ok[u] = ok[u] && s.j < mt[u].w;
    }
    float v[BU];
#pragma unroll
    for (int u = 0; u < BU; u++) {
        int d = ok[u] ? lane_disp(a, mt[u].y, j[u]) : 0;
        v[u] = ok[u] ? raw_cost(a, mt[u].x, mt[u].z, d, j[u]) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < BU; u++)
        if (ok[u]) a.aup[row[u] + j[u]] = v[u];
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

// A_up along short paths (2..kShortPath nodes), one thread per (PU paths,
// lane), values in registers.
__global__ void __launch_bounds__(256) k_scan_up_short(AggArgs a, int64_t s0, int64_t ns) {
    Slot s = slot_of(a);
    for (int u = 0; u < 4; u++) {
        int64_t it = s.item * 4 + u;
        if (it >= ns) return;
        int4 info = a.pinfo[s0 + it];
        int len = info.y, m = info.z;
        if (len < 2 || s.j >= m) continue;
        int64_t row0 = a.prows[s0 + it].x;
        float b[kShortPath], sim[kShortPath];
#pragma unroll
        for (int q = 0; q < kShortPath; q++) {
            b[q] = q < len ? a.aup[row0 + (int64_t)q * m + s.j] : 0.0f;
            sim[q] = q < len ? fabsf(a.lsimf[info.x + q]) : 0.0f;
        }
        float x = 0.0f;
#pragma unroll
        for (int q = kShortPath - 1; q >= 0; q--) {
            if (q < len) {
                float sn = (q + 1 < len) ? sim[q + 1] : 0.0f;
                x = b[q] + sn * x;
                a.aup[row0 + (int64_t)q * m + s.j] = x;
            }
        }
    }
}

// ---------------------------------------------------------------- segments

struct SegCtx {
    int32_t start, len, m, doff;
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
    const float* base = a.aup + c.row0 + (int64_t)(c.a - c.start) * c.m + j;
    for (int i = 0; i < cnt; i++) cp_async4(&buf[warp][i][lane], base + (int64_t)i * c.m, act);
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
    float* out = a.aup + c.row0 + (int64_t)(c.a - c.start) * c.m + j;
    for (int i = cnt - 1; i >= 0; i--) {
        x = buf[warp][i][lane] + ssim[warp][i + 1] * x;
        if (act) out[(int64_t)i * c.m] = x;
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
// root path uses s = 0 so that A(root) = A_up(root).  A is stored in place
// for every node; the argmin runs afterwards in k_wta.
__global__ void __launch_bounds__(128) k_seg_down(AggArgs a, int64_t g0, int64_t ng, int* ctr) {
    __shared__ float buf[4][kSeg][32];
    __shared__ float ssim[4][kSeg];
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int g = (int)blockIdx.y;
    int t = warp_ticket(ctr + g);
    if (t >= ng) return;
    SegCtx c = seg_ctx(a, g0 + t);
    if (g * 32 >= c.m) return;
    int j = g * 32 + lane;
    bool act = j < c.m;
    int cnt = c.b - c.a;
    float* rows = a.aup + c.row0 + (int64_t)(c.a - c.start) * c.m + j;
    for (int i = 0; i < cnt; i++) cp_async4(&buf[warp][i][lane], rows + (int64_t)i * c.m, act);
    cp_commit();
    for (int i = lane; i < cnt; i += 32) {
        float sv = fabsf(a.lsimf[c.a + i]);
        if (c.a + i == c.start && c.prow < 0) sv = 0.0f;  // root: A = A_up
        ssim[warp][i] = sv;
    }
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
        if (act) rows[(int64_t)i * c.m] = y;
    }
}

// Short paths (1..kShortPath nodes): A = s A(parent) + (1 - s^2) A_up head ->
// tail, stored in place.  Each thread takes 4 consecutive paths and issues
// the first-node loads of all of them up front (most have a single node).
__global__ void __launch_bounds__(256) k_down_short(AggArgs a, int64_t s0, int64_t ns) {
    Slot s = slot_of(a);
    int4 info[4];
    longlong2 rows[4];
    bool act[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
        int64_t it = s.item * 4 + u;
        bool valid = it < ns;
        info[u] = valid ? a.pinfo[s0 + it] : make_int4(0, 0, 0, 0);
        rows[u] = valid ? a.prows[s0 + it] : make_longlong2(0, -1);
        act[u] = valid && s.j < info[u].z;
    }
    float u0[4], y0[4], s0v[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
        s0v[u] = act[u] ? fabsf(a.lsimf[info[u].x]) : 0.0f;
        u0[u] = act[u] ? a.aup[rows[u].x + s.j] : 0.0f;
        y0[u] = (act[u] && rows[u].y >= 0) ? a.aup[rows[u].y + s.j] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
        if (!act[u]) continue;
        int m = info[u].z;
        float* row = a.aup + rows[u].x + s.j;
        float y = rows[u].y < 0 ? u0[u] : s0v[u] * y0[u] + (1.0f - s0v[u] * s0v[u]) * u0[u];
        row[0] = y;
        for (int q = 1; q < info[u].y; q++) {
            float sv = fabsf(a.lsimf[info[u].x + q]);
            float* rq = row + (int64_t)q * m;
            y = sv * y + (1.0f - sv * sv) * rq[0];
            rq[0] = y;
        }
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
    int m = (int)(a.rowoff[k + 1] - row);
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
    a.sub = f->max_m <= 16 ? pow2_at_least(f->max_m) : 32;
    a.sub_shift = 0;
    while ((1 << a.sub_shift) < a.sub) a.sub_shift++;
    DevBuf<float> aup;
    DevBuf<unsigned long long> carry;
    DevBuf<int> tickets;
    HDP_TRY(aup.alloc(f->total_entries + 32, st));
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
    a.atomic_keys = 0;  // k_wta writes each key once
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
    for (int64_t r = f->n_phases - 1; r >= 0; r--) {
        int64_t k0 = f->phase_node[r], nk = f->phase_node[r + 1] - k0;
        if (nk > 0) {
            k_ecompute<<<packed_grid(a, nk, BU, 256), 256, 0, st>>>(a, k0, nk); note_launch();
        }
        int64_t p0 = f->lp_off[r], np = f->lp_off[r + 1] - p0;
        if (np > 0) {
            k_light<<<packed_grid(a, (np + 3) / 4, 1, 256), 256, 0, st>>>(a, p0, np); note_launch();
        }
        int64_t g0 = f->seg_off[r], ng = f->seg_off[r + 1] - g0;
        if (ng > 0) {
            k_seg_up<<<dim3(grid_for(ng * 32, 128), lg.groups), 128, 0, st>>>(
                lg, g0, ng, a.tickets + (2 * r) * a.groups); note_launch();
        }
        int64_t s0 = f->short_off[r], ns = f->short_off[r + 1] - s0;
        if (ns > 0) {
            k_scan_up_short<<<packed_grid(sh, (ns + 3) / 4, 1, 256), 256, 0, st>>>(sh, s0, ns); note_launch();
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
        if (ns > 0) {
            k_down_short<<<packed_grid(sh, (ns + 3) / 4, 1, 256), 256, 0, st>>>(sh, s0, ns); note_launch();
        }
    }
    HDP_CHECK_LAUNCH();
    {
        AggArgs wa = a;  // one warp (sub == 32) or one sub-group per row
        wa.groups = 1;
        k_wta<<<packed_grid(wa, f->n, 1, 256), 256, 0, st>>>(wa, f->n); note_launch();
    }
    if (volume) {
        k_volume_copy<<<packed_grid(a, f->n, 1, 256), 256, 0, st>>>(a, f->n); note_launch();
    }
    if (disp || min_cost) {
        k_keys_finish<<<grid_for(f->n, 256), 256, 0, st>>>(f->n, kp, disp, min_cost); note_launch();
    }
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}
