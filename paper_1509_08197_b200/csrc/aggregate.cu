// Two-pass tree aggregation fused with the matching cost and winner-takes-all.
//
// Replaces masked_cost_volume + aggregate_tree + winner_takes_all_with_cost
// (cost_volume.py:183-236, aggregation.py:158-256) and the baseline's
// streamed chunk loop (aggregation.py:311-326).
//
//   up:   A_up(v) = E(v) + sum_c s_c A_up(c)
//   down: A(root) = A_up(root);  A(v) = s_v A(parent) + (1 - s_v^2) A_up(v)
//
// Work is organised by the heavy-path layout built in forest.cu: phases are
// processed deepest-first (up) / shallowest-first (down), one launch per
// phase; one warp owns (heavy path, 32 consecutive disparity lanes) and walks
// the path in chunks of 32 nodes.  Per chunk every load is independent of
// the recurrence (32 nodes in flight), the recurrence itself is one FMA per
// node in registers, and the per-node argmin is a transpose butterfly across
// the warp (31 shuffles per 32 nodes).  The raw cost E is recomputed from
// the packed image planes, so HBM traffic is ~ A_up written once + read once.
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
    const int32_t* t_m;
    const int32_t* t_doff;
    const int32_t* dlist;
    const int64_t* rowoff;
    const int64_t* nodeoff;
    const float4* pl;
    const float4* pr;
    const float* cost_rows;
    int64_t npix;  // pixels per pair
    int w, c;
    float alpha, tc, tg, border;
    float* aup;
    float* volume;
    unsigned long long* keys;
    int groups;  // lane groups of 32 per path
};

__device__ __forceinline__ float raw_cost(const AggArgs& a, int32_t node, int d, int j, int m) {
    if (a.cost_rows) return a.cost_rows[(int64_t)node * m + j];
    int64_t p = node % a.npix;
    int col = (int)(p % a.w);
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

__global__ void __launch_bounds__(128) k_up(AggArgs a, int64_t p0, int64_t np) {
    int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    int64_t pi = wid / a.groups;
    int g = (int)(wid % a.groups);
    if (pi >= np) return;
    pi += p0;
    int32_t start = a.p_start[pi], len = a.p_len[pi];
    int32_t t = a.p_tree[pi];
    int m = a.t_m[t];
    if (g * 32 >= m) return;
    int j = g * 32 + lane;
    bool act = j < m;
    int d = act ? a.dlist[a.t_doff[t] + j] : 0;
    float x_prev = 0.0f, s_next = 0.0f;
    int32_t end = start + len;
    for (int32_t hi = end; hi > start; hi -= 32) {
        int32_t lo = max(start, hi - 32);
        int cnt = hi - lo;
        // per-node metadata, one node per lane
        int32_t k_l = lo + lane;
        int32_t node_l = 0, lcs_l = 0, lce_l = 0;
        float sim_l = 0.0f;
        int64_t row_l = 0;
        if (lane < cnt) {
            node_l = a.lnode[k_l];
            sim_l = a.lsim[k_l];
            lcs_l = a.lc_start[k_l];
            lce_l = a.lc_start[k_l + 1];
            row_l = a.rowoff[k_l];
        }
        float b[32];
#pragma unroll
        for (int i = 0; i < 32; i++) {
            if (i < cnt) {
                int32_t node = __shfl_sync(0xffffffffu, node_l, i);
                int32_t lcs = __shfl_sync(0xffffffffu, lcs_l, i);
                int32_t lce = __shfl_sync(0xffffffffu, lce_l, i);
                float v = act ? raw_cost(a, node, d, j, m) : 0.0f;
                for (int32_t q = lcs; q < lce; q++) {
                    int32_t ck = a.lc_list[q];
                    float sc = a.lsim[ck];
                    if (act) v += sc * a.aup[a.rowoff[ck] + j];
                }
                b[i] = v;
            }
        }
        // sequential recurrence, highest position first
#pragma unroll
        for (int i = 31; i >= 0; i--) {
            if (i < cnt) {
                float x = b[i] + s_next * x_prev;
                int64_t row = __shfl_sync(0xffffffffu, row_l, i);
                if (act) a.aup[row + j] = x;
                x_prev = x;
                s_next = __shfl_sync(0xffffffffu, sim_l, i);
            }
        }
    }
}

__global__ void __launch_bounds__(128) k_down(AggArgs a, int64_t p0, int64_t np) {
    int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    int64_t pi = wid / a.groups;
    int g = (int)(wid % a.groups);
    if (pi >= np) return;
    pi += p0;
    int32_t start = a.p_start[pi], len = a.p_len[pi];
    int32_t t = a.p_tree[pi];
    int m = a.t_m[t];
    if (g * 32 >= m) return;
    int j = g * 32 + lane;
    bool act = j < m;
    int d = act ? a.dlist[a.t_doff[t] + j] : 0;
    int32_t par = a.p_par[pi];
    float y = 0.0f;
    if (par >= 0 && act) y = a.aup[a.rowoff[par] + j];  // A(parent), stored in place
    bool root_path = par < 0;
    int32_t end = start + len;
    for (int32_t lo = start; lo < end; lo += 32) {
        int cnt = min(32, end - lo);
        int32_t k_l = lo + lane;
        int32_t node_l = 0;
        float sim_l = 0.0f;
        int64_t row_l = 0;
        bool light_l = false;
        if (lane < cnt) {
            node_l = a.lnode[k_l];
            sim_l = a.lsim[k_l];
            row_l = a.rowoff[k_l];
            light_l = a.lc_start[k_l + 1] > a.lc_start[k_l];
        }
        float u[32];
#pragma unroll
        for (int i = 0; i < 32; i++) {
            int64_t row = __shfl_sync(0xffffffffu, row_l, i);
            u[i] = (i < cnt && act) ? a.aup[row + j] : 0.0f;
        }
        unsigned long long key[32];
#pragma unroll
        for (int i = 0; i < 32; i++) {
            float s = __shfl_sync(0xffffffffu, sim_l, i);
            bool lt = __shfl_sync(0xffffffffu, light_l, i);
            int64_t row = __shfl_sync(0xffffffffu, row_l, i);
            int32_t node = __shfl_sync(0xffffffffu, node_l, i);
            if (i < cnt) {
                if (root_path && lo + i == start)
                    y = u[i];
                else
                    y = s * y + (1.0f - s * s) * u[i];
                if (act && lt) a.aup[row + j] = y;
                if (act && a.volume) a.volume[a.nodeoff[node] + j] = y;
                key[i] = act ? (((unsigned long long)ord_f32(y) << 32) | (uint32_t)d) : ~0ull;
            } else {
                key[i] = ~0ull;
            }
        }
        // transpose butterfly: afterwards lane l holds the min over lanes for node l
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
        if (lane < cnt && a.keys) {
            if (a.groups == 1)
                a.keys[node_l] = key[0];
            else
                atomicMin(&a.keys[node_l], key[0]);
        }
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

}  // namespace hdp

using namespace hdp;

extern "C" int hdp_aggregate_wta(hdp_forest* f, const float* packed_l, const float* packed_r,
                                 int h, int w, int c, float alpha, float tau_c, float tau_g,
                                 const float* cost_rows, int32_t* disp, float* min_cost,
                                 uint64_t* keys, float* volume, void* stream) {
    HDP_REQUIRE(f != nullptr && f->lanes_set, HDP_ERR_CONFIG, "forest lanes not set");
    HDP_REQUIRE(cost_rows || (packed_l && packed_r && h > 0 && w > 0), HDP_ERR_CONFIG,
                "need either cost rows or image planes");
    HDP_REQUIRE(cost_rows || (int64_t)h * w > 0, HDP_ERR_DATA, "empty image");
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
    a.t_m = f->t_m.get();
    a.t_doff = f->t_doff.get();
    a.dlist = f->dlist.get();
    a.rowoff = f->rowoff.get();
    a.nodeoff = f->nodeoff.get();
    a.pl = (const float4*)packed_l;
    a.pr = (const float4*)packed_r;
    a.cost_rows = cost_rows;
    a.npix = (int64_t)h * w;
    if (a.npix <= 0) a.npix = 1;
    a.w = w > 0 ? w : 1;
    a.c = c;
    a.alpha = alpha;
    a.tc = tau_c;
    a.tg = tau_g;
    a.border = (1.0f - alpha) * tau_c + alpha * tau_g;
    a.volume = volume;
    a.groups = (f->max_m + 31) / 32;
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
    if (a.groups > 1) k_keys_init<<<grid_for(f->n, 256), 256, 0, st>>>(f->n, kp);
    const int TPB = 128;
    for (int64_t r = f->n_phases - 1; r >= 0; r--) {
        int64_t p0 = f->phase_off[r], np = f->phase_off[r + 1] - p0;
        if (np == 0) continue;
        int64_t threads = np * a.groups * 32;
        k_up<<<grid_for(threads, TPB), TPB, 0, st>>>(a, p0, np);
    }
    HDP_CHECK_LAUNCH();
    for (int64_t r = 0; r < f->n_phases; r++) {
        int64_t p0 = f->phase_off[r], np = f->phase_off[r + 1] - p0;
        if (np == 0) continue;
        int64_t threads = np * a.groups * 32;
        k_down<<<grid_for(threads, TPB), TPB, 0, st>>>(a, p0, np);
    }
    HDP_CHECK_LAUNCH();
    if (disp || min_cost)
        k_keys_finish<<<grid_for(f->n, 256), 256, 0, st>>>(f->n, kp, disp, min_cost);
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}
