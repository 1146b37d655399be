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
// every heavy path contiguous, rows of one path contiguous because all its
// nodes share the tree's lane count m).  Per phase:
//   up   : k_bcompute   b(v) = E(v) + sum_{light c} s_c A_up(c) for all nodes of
//                       the phase in parallel (E recomputed from the images)
//          k_scan_up    A_up(v) = b(v) + s_h A_up(h) along every path of length
//                       >= 2: one warp per (path, 32 lanes), chunks of 32 nodes
//                       staged with cp.async (double buffered) so the
//                       recurrence runs from shared memory at FMA latency
//   down : k_down_long  the same walk head -> tail, plus the per-node argmin
//                       (transpose butterfly, 31 shuffles per 32 nodes)
//          k_down_short single-node paths, fully parallel
// A is written back in place only where a light child will read it.
#include <cuda_runtime.h>

#include "forest.cuh"
#include "prims.cuh"

namespace hdp {

struct AggArgs {
    const int32_t* lnode;
    const float* lsim;
    const int32_t* lc_start;
    const int32_t* lc_list;
    const int32_t* p_start;
    const int32_t* p_len;
    const int32_t* p_par;
    const int32_t* p_tree;
    const int32_t* tree_id;
    const int32_t* t_m;
    const int32_t* t_doff;
    const int32_t* dlist;
    const int64_t* rowoff;
    const int64_t* nodeoff;
    const int32_t* paths;  // long or short path list of the launch
    const float4* pl;
    const float4* pr;
    const float* cost_rows;
    int32_t npix;  // pixels per pair
    int32_t w;
    int c;
    float alpha, tc, tg, border;
    float* aup;
    float* volume;
    unsigned long long* keys;
    int groups;  // 32-lane groups per node when sub == 32
    int sub;     // lanes per item for the packed mappings (power of 2 <= 32)
    int atomic_keys;
};

__device__ __forceinline__ float raw_cost(const AggArgs& a, int32_t node, int d, int j, int m) {
    if (a.cost_rows) return a.cost_rows[a.nodeoff[node] + j];  // pixel-major ragged rows
    int32_t p = node % a.npix;
    int32_t col = p % a.w;
    if (col - d < 0) return a.border;
    float4 L = a.pl[node];
    float4 R = a.pr[node - d];
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
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Thread -> (item, lane j): with sub < 32 several items share a warp (sub
// lanes each, aligned); otherwise one item spans `groups` warps.
struct Slot {
    int64_t item;
    int j;
};
__device__ __forceinline__ Slot slot_of(const AggArgs& a) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    Slot s;
    if (a.sub < 32) {
        s.item = t / a.sub;
        s.j = (int)(t % a.sub);
    } else {
        int64_t w = t >> 5;
        s.item = w / a.groups;
        s.j = (int)(w % a.groups) * 32 + (int)(t & 31);
    }
    return s;
}

// b(v) = E(v) + sum_{light children c} s_c A_up(c), every node of a phase.
__global__ void __launch_bounds__(256) k_bcompute(AggArgs a, int64_t k0, int64_t nk) {
    Slot s = slot_of(a);
    if (s.item >= nk) return;
    int64_t k = k0 + s.item;
    int64_t row = a.rowoff[k];
    int m = (int)(a.rowoff[k + 1] - row);
    if (s.j >= m) return;
    int32_t node = a.lnode[k];
    int d = a.dlist[a.t_doff[a.tree_id[node]] + s.j];
    float v = raw_cost(a, node, d, s.j, m);
    int32_t c0 = a.lc_start[k], c1 = a.lc_start[k + 1];
    for (int32_t q = c0; q < c1; q++) {
        int32_t ck = a.lc_list[q];
        v += a.lsim[ck] * a.aup[a.rowoff[ck] + s.j];
    }
    a.aup[row + s.j] = v;
}

constexpr int CH = 32;  // nodes per staged chunk

// A_up along paths of length >= 2, tail -> head, in place over b.
__global__ void __launch_bounds__(128) k_scan_up(AggArgs a, int64_t l0, int64_t nl) {
    __shared__ float buf[4][2][CH][32];
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t li = wid / a.groups;
    int g = (int)(wid % a.groups);
    if (li >= nl) return;
    int32_t pi = a.paths[l0 + li];
    int32_t start = a.p_start[pi], len = a.p_len[pi];
    int64_t row0 = a.rowoff[start];
    int m = (int)(a.rowoff[start + 1] - row0);
    if (g * 32 >= m) return;
    int j = g * 32 + lane;
    bool act = j < m;
    float* aup = a.aup;
    auto stage = [&](int bi, int32_t lo, int cnt) {
        for (int i = 0; i < cnt; i++)
            cp_async4(&buf[warp][bi][i][lane], aup + row0 + (int64_t)(lo + i - start) * m + j, act);
        cp_commit();
    };
    int32_t end = start + len;
    int32_t hi = end;
    int32_t lo = max(start, hi - CH);
    int bi = 0;
    stage(0, lo, hi - lo);
    float sim_l = (lane < hi - lo) ? a.lsim[lo + lane] : 0.0f;
    float x_prev = 0.0f, s_next = 0.0f;
    while (true) {
        int cnt = hi - lo;
        int32_t nhi = lo, nlo = max(start, lo - CH);
        bool more = nhi > start;
        float sim_n = 0.0f;
        if (more) {
            stage(bi ^ 1, nlo, nhi - nlo);
            sim_n = (lane < nhi - nlo) ? a.lsim[nlo + lane] : 0.0f;
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncwarp();
        for (int i = cnt - 1; i >= 0; i--) {
            float x = buf[warp][bi][i][lane] + s_next * x_prev;
            if (act) aup[row0 + (int64_t)(lo + i - start) * m + j] = x;
            x_prev = x;
            s_next = __shfl_sync(0xffffffffu, sim_l, i);
        }
        __syncwarp();
        if (!more) break;
        hi = nhi;
        lo = nlo;
        bi ^= 1;
        sim_l = sim_n;
    }
}

// warp transpose butterfly: lane l ends with the minimum key of node l
__device__ __forceinline__ unsigned long long warp_min_per_node(unsigned long long (&key)[CH],
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

// A along paths of length >= 2, head -> tail, fused with the argmin.
__global__ void __launch_bounds__(128) k_down_long(AggArgs a, int64_t l0, int64_t nl) {
    __shared__ float buf[4][2][CH][32];
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t li = wid / a.groups;
    int g = (int)(wid % a.groups);
    if (li >= nl) return;
    int32_t pi = a.paths[l0 + li];
    int32_t start = a.p_start[pi], len = a.p_len[pi];
    int64_t row0 = a.rowoff[start];
    int m = (int)(a.rowoff[start + 1] - row0);
    if (g * 32 >= m) return;
    int j = g * 32 + lane;
    bool act = j < m;
    int32_t node0 = a.lnode[start];
    int d = act ? a.dlist[a.t_doff[a.tree_id[node0]] + j] : 0;
    int32_t par = a.p_par[pi];
    float* aup = a.aup;
    float y = 0.0f;
    if (par >= 0 && act) y = aup[a.rowoff[par] + j];  // A(parent), stored in place
    auto stage = [&](int bi, int32_t lo, int cnt) {
        for (int i = 0; i < cnt; i++)
            cp_async4(&buf[warp][bi][i][lane], aup + row0 + (int64_t)(lo + i - start) * m + j, act);
        cp_commit();
    };
    auto meta = [&](int32_t lo, int cnt, float& sim, int32_t& node, unsigned& light) {
        bool in = lane < cnt;
        sim = in ? a.lsim[lo + lane] : 0.0f;
        node = in ? a.lnode[lo + lane] : 0;
        bool lt = in && a.lc_start[lo + lane + 1] > a.lc_start[lo + lane];
        light = __ballot_sync(0xffffffffu, lt);
    };
    int32_t end = start + len;
    int32_t lo = start, hi = min(end, start + CH);
    int bi = 0;
    stage(0, lo, hi - lo);
    float sim_l;
    int32_t node_l;
    unsigned light;
    meta(lo, hi - lo, sim_l, node_l, light);
    while (true) {
        int cnt = hi - lo;
        int32_t nlo = hi, nhi = min(end, hi + CH);
        bool more = nlo < end;
        float sim_n = 0.0f;
        int32_t node_n = 0;
        unsigned light_n = 0;
        if (more) {
            stage(bi ^ 1, nlo, nhi - nlo);
            meta(nlo, nhi - nlo, sim_n, node_n, light_n);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncwarp();
        unsigned long long key[CH];
#pragma unroll
        for (int i = 0; i < CH; i++) {
            float s = __shfl_sync(0xffffffffu, sim_l, i);
            if (i < cnt) {
                float u = buf[warp][bi][i][lane];
                if (par < 0 && lo + i == start)
                    y = u;
                else
                    y = s * y + (1.0f - s * s) * u;
                int64_t row = row0 + (int64_t)(lo + i - start) * m;
                if (act && (((light >> i) & 1u) || a.volume)) aup[row + j] = y;
                key[i] = act ? pack_key(y, d) : ~0ull;
            } else {
                key[i] = ~0ull;
            }
        }
        unsigned long long best = warp_min_per_node(key, lane);
        if (lane < cnt && a.keys) {
            if (a.atomic_keys)
                atomicMin(&a.keys[node_l], best);
            else
                a.keys[node_l] = best;
        }
        __syncwarp();
        if (!more) break;
        lo = nlo;
        hi = nhi;
        bi ^= 1;
        sim_l = sim_n;
        node_l = node_n;
        light = light_n;
    }
}

// Pixel-major copy of the final aggregated volume (parity / API use only):
// after the down pass every node's row holds A only where it was stored, so
// this is produced by a dedicated pass in volume mode (see hdp_aggregate_wta).
__global__ void __launch_bounds__(256) k_volume_copy(AggArgs a, int64_t n) {
    Slot s = slot_of(a);
    if (s.item >= n) return;
    int64_t k = s.item;
    int64_t row = a.rowoff[k];
    int m = (int)(a.rowoff[k + 1] - row);
    if (s.j >= m) return;
    a.volume[a.nodeoff[a.lnode[k]] + s.j] = a.aup[row + s.j];
}

// Single-node paths: A(v) = s A(parent) + (1 - s^2) A_up(v), then argmin.
__global__ void __launch_bounds__(256) k_down_short(AggArgs a, int64_t s0, int64_t ns) {
    Slot s = slot_of(a);
    int lane = threadIdx.x & 31;
    bool valid = s.item < ns;
    unsigned long long key = ~0ull;
    int32_t node = 0;
    if (valid) {
        int32_t pi = a.paths[s0 + s.item];
        int32_t k = a.p_start[pi];
        int64_t row = a.rowoff[k];
        int m = (int)(a.rowoff[k + 1] - row);
        node = a.lnode[k];
        if (s.j < m) {
            int d = a.dlist[a.t_doff[a.tree_id[node]] + s.j];
            float u = a.aup[row + s.j];
            int32_t par = a.p_par[pi];
            float y = u;
            if (par >= 0) {
                float sv = a.lsim[k];
                y = sv * a.aup[a.rowoff[par] + s.j] + (1.0f - sv * sv) * u;
            }
            if (a.lc_start[k + 1] > a.lc_start[k] || a.volume) a.aup[row + s.j] = y;
            key = pack_key(y, d);
        }
    }
    int width = a.sub < 32 ? a.sub : 32;
    for (int o = width >> 1; o >= 1; o >>= 1) {
        unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
        key = other < key ? other : key;
    }
    if (valid && (lane & (width - 1)) == 0 && a.keys) {
        if (a.atomic_keys)
            atomicMin(&a.keys[node], key);
        else
            a.keys[node] = key;
    }
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

static int64_t packed_threads(const AggArgs& a, int64_t items) {
    return a.sub < 32 ? items * a.sub : items * a.groups * 32;
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
    a.lnode = f->lnode.get();
    a.lsim = f->lsim.get();
    a.lc_start = f->lc_start.get();
    a.lc_list = f->lc_list.get();
    a.p_start = f->p_start.get();
    a.p_len = f->p_len.get();
    a.p_par = f->p_par.get();
    a.p_tree = f->p_tree.get();
    a.tree_id = f->tree_id.get();
    a.t_m = f->t_m.get();
    a.t_doff = f->t_doff.get();
    a.dlist = f->dlist.get();
    a.rowoff = f->rowoff.get();
    a.nodeoff = f->nodeoff.get();
    a.paths = nullptr;
    a.pl = (const float4*)packed_l;
    a.pr = (const float4*)packed_r;
    a.cost_rows = cost_rows;
    a.npix = (h > 0 && w > 0) ? h * w : 1;
    a.w = w > 0 ? w : 1;
    a.c = c;
    a.alpha = alpha;
    a.tc = tau_c;
    a.tg = tau_g;
    a.border = (1.0f - alpha) * tau_c + alpha * tau_g;
    a.volume = volume;
    a.groups = (f->max_m + 31) / 32;
    a.sub = f->max_m <= 16 ? pow2_at_least(f->max_m) : 32;
    DevBuf<float> aup;
    HDP_TRY(aup.alloc(f->total_entries + 32, st));
    a.aup = aup.get();
    DevBuf<unsigned long long> kbuf;
    unsigned long long* kp = (unsigned long long*)keys;
    if (!kp) {
        HDP_TRY(kbuf.alloc(f->n, st));
        kp = kbuf.get();
    }
    a.keys = kp;
    a.atomic_keys = a.groups > 1 ? 1 : 0;
    if (a.atomic_keys) k_keys_init<<<grid_for(f->n, 256), 256, 0, st>>>(f->n, kp); note_launch();

    AggArgs lg = a;  // long-path kernels: one warp per (path, 32 lanes)
    lg.sub = 32;
    lg.paths = f->long_paths.get();
    AggArgs sh = a;
    sh.paths = f->short_paths.get();
    for (int64_t r = f->n_phases - 1; r >= 0; r--) {
        int64_t k0 = f->phase_node[r], nk = f->phase_node[r + 1] - k0;
        if (nk > 0) k_bcompute<<<grid_for(packed_threads(a, nk), 256), 256, 0, st>>>(a, k0, nk); note_launch();
        int64_t l0 = f->long_off[r], nl = f->long_off[r + 1] - l0;
        if (nl > 0)
            k_scan_up<<<grid_for(nl * lg.groups * 32, 128), 128, 0, st>>>(lg, l0, nl); note_launch();
    }
    HDP_CHECK_LAUNCH();
    for (int64_t r = 0; r < f->n_phases; r++) {
        int64_t l0 = f->long_off[r], nl = f->long_off[r + 1] - l0;
        if (nl > 0)
            k_down_long<<<grid_for(nl * lg.groups * 32, 128), 128, 0, st>>>(lg, l0, nl); note_launch();
        int64_t s0 = f->short_off[r], ns = f->short_off[r + 1] - s0;
        if (ns > 0) k_down_short<<<grid_for(packed_threads(sh, ns), 256), 256, 0, st>>>(sh, s0, ns); note_launch();
    }
    HDP_CHECK_LAUNCH();
    if (volume) {
        AggArgs va = a;
        k_volume_copy<<<grid_for(packed_threads(va, f->n), 256), 256, 0, st>>>(va, f->n); note_launch();
    }
    if (disp || min_cost)
        k_keys_finish<<<grid_for(f->n, 256), 256, 0, st>>>(f->n, kp, disp, min_cost); note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}
