// Rooting a spanning forest and building its heavy-path layout, all on the
// device in O(log n) parallel rounds.
//
// Replaces _bfs_forest (spanning_forest.py:191-283).  The reference roots
// every tree at its lowest pixel id and walks BFS levels one by one; tree
// depth on these grids reaches thousands of levels, so a level-synchronous
// GPU walk would be latency bound.  Instead:
//   1. components -> root = min id per component, trees numbered by root id
//      (the reference's numbering);
//   2. Euler tour over the CSR adjacency, list-ranked by pointer jumping;
//      a tree edge is a parent link in the direction its tour arc comes
//      first; subtree size = half the tour span; depth and light depth come
//      from prefix sums over the tour;
//   3. heavy child = largest subtree (ties -> lower id), heavy paths by
//      pointer jumping, layout sorted by (light depth, path head, depth):
//      every heavy path is contiguous and every phase (light depth) a block.
// parent / depth / tree_id / subtree sizes are tree properties, identical to
// the reference's.  Only the node ORDER differs from BFS, which the
// reference uses as a layout (not a parity artifact).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "forest.cuh"
#include "prims.cuh"

namespace hdp {

int run_boruvka(int64_t n, int64_t m, const int32_t* eu, const int32_t* ev, const uint64_t* key,
                uint8_t* in_tree, int32_t* comp, int* rounds_out, cudaStream_t st, int grid_h = 0, int grid_w = 0);

// In-tree flags, plus a check that the edge list is sorted by (eu, ev) with
// eu < ev (grid edge lists are): then a stable sort of the arcs by source
// alone already leaves every adjacency list in ascending order.
__global__ void k_flag_edges(int64_t m, const uint8_t* __restrict__ in_tree, const int32_t* __restrict__ eu,
                             const int32_t* __restrict__ ev, int32_t* flags, int* unsorted) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool bad = false;
    if (e < m) {
        flags[e] = in_tree ? (in_tree[e] ? 1 : 0) : 1;
        const int32_t u = eu[e], v = ev[e];
        bad = u >= v;
        if (e + 1 < m) {
            const int32_t u2 = eu[e + 1], v2 = ev[e + 1];
            bad = bad || u > u2 || (u == u2 && v >= v2);
        }
    }
    if (__ballot_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0 && *(volatile int*)unsorted == 0) *unsorted = 1;
}

__global__ void k_edge_count(int64_t m, const int32_t* __restrict__ flags, const int32_t* __restrict__ pos,
                             int* out) {
    out[0] = pos[m - 1] + flags[m - 1];
}

__global__ void k_compact_edges(int64_t m, const int32_t* __restrict__ flags,
                                const int32_t* __restrict__ pos, const int32_t* __restrict__ eu,
                                const int32_t* __restrict__ ev, const float* __restrict__ ew,
                                int32_t* tu, int32_t* tv, float* tw, uint64_t* tkey) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m || !flags[e]) return;
    int32_t i = pos[e];
    tu[i] = eu[e];
    tv[i] = ev[e];
    tw[i] = ew ? ew[e] : 0.0f;
    tkey[i] = (uint64_t)i;
}

__global__ void k_fill_int(int64_t n, int32_t* a, int32_t v) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = v;
}

__global__ void k_min_root(int64_t n, const int32_t* __restrict__ comp, int32_t* minid, int32_t* csize) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool ok = v < n;
    int32_t c = ok ? comp[v] : -1;
    // lanes of a warp mostly share a component: one atomic per distinct label
    unsigned peers = __match_any_sync(0xffffffffu, c);
    int32_t mn = __reduce_min_sync(peers, ok ? (int32_t)v : INT_MAX);
    int leader = __ffs(peers) - 1;
    if (ok && (int)(threadIdx.x & 31) == leader) {
        atomicMin(&minid[c], mn);
        atomicAdd(&csize[c], __popc(peers));
    }
}

__global__ void k_root_flags(int64_t n, const int32_t* __restrict__ comp,
                             const int32_t* __restrict__ minid, const int32_t* __restrict__ csize,
                             int32_t* root, int32_t* is_root, int32_t* max_size) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int32_t sz = 0;
    if (v < n) {
        int32_t c = comp[v];
        int32_t r = minid[c];
        root[v] = r;
        is_root[v] = (r == v) ? 1 : 0;
        if (r == v) sz = csize[c];
    }
    sz = __reduce_max_sync(0xffffffffu, sz);
    if ((threadIdx.x & 31) == 0 && sz > 0) atomicMax(max_size, sz);
}

__global__ void k_tree_count(int64_t n, const int32_t* __restrict__ tindex, const int32_t* __restrict__ is_root,
                             int32_t* out) {
    out[0] = tindex[n - 1] + is_root[n - 1];
}

__global__ void k_tree_ids(int64_t n, const int32_t* __restrict__ root,
                           const int32_t* __restrict__ tindex, int32_t* tree_id) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) tree_id[v] = tindex[root[v]];
}

// CSR adjacency without a global sort: arcs are dropped into their source's
// slots (atomic cursor per source), then every source orders its few slots by
// destination (insertion sort; heap sort for the rare high-degree node).
__global__ void k_arc_degree(int64_t m, const int32_t* __restrict__ tu, const int32_t* __restrict__ tv,
                             int32_t* deg) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    atomicAdd(&deg[tu[e]], 1);
    atomicAdd(&deg[tv[e]], 1);
}

__global__ void k_arc_place(int64_t m, const int32_t* __restrict__ tu, const int32_t* __restrict__ tv,
                            const float* __restrict__ tw, const int32_t* __restrict__ adj_start,
                            int32_t* cur, int32_t* asrc, int32_t* adst, float* aw) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    const int32_t u = tu[e], v = tv[e];
    const float w = tw[e];
    const int32_t su = adj_start[u] + atomicAdd(&cur[u], 1);
    const int32_t sv = adj_start[v] + atomicAdd(&cur[v], 1);
    asrc[su] = u;
    adst[su] = v;
    aw[su] = w;
    asrc[sv] = v;
    adst[sv] = u;
    aw[sv] = w;
}

__device__ void adj_sift(int32_t* d, float* w, int root, int cnt) {
    for (;;) {
        int c = 2 * root + 1;
        if (c >= cnt) return;
        if (c + 1 < cnt && d[c + 1] > d[c]) c++;
        if (d[root] >= d[c]) return;
        int32_t td = d[root]; d[root] = d[c]; d[c] = td;
        float tw = w[root]; w[root] = w[c]; w[c] = tw;
        root = c;
    }
}

__global__ void k_arc_sort(int64_t n, const int32_t* __restrict__ adj_start, int32_t* adst, float* aw) {
    int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= n) return;
    const int32_t a = adj_start[x], cnt = adj_start[x + 1] - a;
    int32_t* d = adst + a;
    float* w = aw + a;
    if (cnt <= 4) {  // grid trees: at most 4 neighbours, sorted in registers
        int32_t kd[4];
        float kw[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            kd[i] = i < cnt ? d[i] : INT_MAX;
            kw[i] = i < cnt ? w[i] : 0.0f;
        }
#pragma unroll
        for (int i = 1; i < 4; i++)
#pragma unroll
            for (int j = i; j > 0; j--)
                if (kd[j - 1] > kd[j]) {
                    const int32_t td = kd[j - 1];
                    kd[j - 1] = kd[j];
                    kd[j] = td;
                    const float tw = kw[j - 1];
                    kw[j - 1] = kw[j];
                    kw[j] = tw;
                }
#pragma unroll
        for (int i = 0; i < 4; i++)
            if (i < cnt) {
                d[i] = kd[i];
                w[i] = kw[i];
            }
        return;
    }
    if (cnt <= 16) {
        for (int i = 1; i < cnt; i++) {
            const int32_t kd = d[i];
            const float kw = w[i];
            int j = i - 1;
            while (j >= 0 && d[j] > kd) {
                d[j + 1] = d[j];
                w[j + 1] = w[j];
                j--;
            }
            d[j + 1] = kd;
            w[j + 1] = kw;
        }
        return;
    }
    for (int r = cnt / 2 - 1; r >= 0; r--) adj_sift(d, w, r, cnt);
    for (int end = cnt - 1; end > 0; end--) {
        int32_t td = d[0]; d[0] = d[end]; d[end] = td;
        float tw = w[0]; w[0] = w[end]; w[end] = tw;
        adj_sift(d, w, 0, end);
    }
}

// twin arc (y -> x) of arc i = (x -> y): binary search in y's sorted list.
__device__ __forceinline__ int32_t find_arc(const int32_t* __restrict__ adj_start,
                                            const int32_t* __restrict__ adst, int32_t y,
                                            int32_t x) {
    int32_t lo = adj_start[y], hi = adj_start[y + 1] - 1;
    while (lo < hi) {
        int32_t mid = (lo + hi) >> 1;
        if (adst[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Euler-tour successor; the arc entering a root just before the tour would
// wrap around to the root's first arc ends the list (next = -1).
__global__ void k_tour_next(int64_t na, const int32_t* __restrict__ asrc,
                            const int32_t* __restrict__ adst, const int32_t* __restrict__ adj_start,
                            const int32_t* __restrict__ root, int32_t* twin, int32_t* next) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    int32_t x = asrc[i], y = adst[i];
    int32_t j = find_arc(adj_start, adst, y, x);
    twin[i] = j;
    int32_t s = adj_start[y], d = adj_start[y + 1] - s;
    int32_t nx = s + ((j - s + 1) % d);
    // wrapping past the last arc of the root back to its first arc ends the tour
    if (root[y] == y && nx == s) nx = -1;
    next[i] = nx;
}

// ---- ruling-set list ranking: rulers are every kRuler-th arc plus every list
// head; each ruler walks its sublist to the next ruler (owner, offset), the
// rulers alone are ranked by pointer jumping, and rank = ruler rank - offset.
#ifndef HDP_RULER
#define HDP_RULER 16
#endif
constexpr int kRuler = HDP_RULER;

__global__ void k_has_pred(int64_t na, const int32_t* __restrict__ next, uint8_t* hp) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < na && next[i] >= 0) hp[next[i]] = 1;
}

__global__ void k_ruler_flags(int64_t na, const uint8_t* __restrict__ hp, int32_t* flag) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < na) flag[i] = (i % kRuler == 0 || !hp[i]) ? 1 : 0;
    else if (i == na) flag[i] = 0;
}

__global__ void k_ruler_list(int64_t na, const int32_t* __restrict__ flag, const int32_t* __restrict__ rid,
                             int32_t* list) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < na && flag[i]) list[rid[i]] = (int32_t)i;
}

// one thread per ruler: walk to the next ruler (or the list's end)
__global__ void k_ruler_walk(int64_t na, const int32_t* __restrict__ rid, const int32_t* __restrict__ list,
                             const int32_t* __restrict__ flag, const int32_t* __restrict__ next, int32_t* owner,
                             int32_t* local, uint64_t* word) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rid[na]) return;
    int32_t cur = list[r], cnt = 0, nx;
    while (true) {
        owner[cur] = (int32_t)r;
        local[cur] = cnt++;
        nx = next[cur];
        if (nx < 0 || flag[nx]) break;
        cur = nx;
    }
    word[r] = ((uint64_t)(uint32_t)(nx < 0 ? -1 : rid[nx]) << 32) | (uint32_t)cnt;
}

__global__ void k_rank_jump_n(const int32_t* __restrict__ count, const uint64_t* __restrict__ in,
                              uint64_t* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= *count) return;
    const uint64_t w = in[i];
    const int32_t nx = (int32_t)(w >> 32);
    if (nx >= 0) {
        const uint64_t w2 = in[nx];
        out[i] = (w2 & 0xffffffff00000000ull) | (uint32_t)((uint32_t)w + (uint32_t)w2);
    } else {
        out[i] = w;
    }
}

// Asynchronous pointer jumping, all rounds in one launch.  A word is (next,
// sum over [self, next)) and is read and written as one 64-bit access, so a
// word read at any time is a valid jump: combining it with the word of its
// target, stale or fresh, gives another valid (shorter) jump.  Each thread
// jumps its own entry until it reaches the list end; no grid barrier, and
// threads started late find mostly-finished chains.
__device__ __forceinline__ uint64_t ld_word(const uint64_t* p) {
    uint64_t w;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    return w;
}
__device__ __forceinline__ void st_word(uint64_t* p, uint64_t w) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
// The grid is resident (at most the CTAs the GPU holds at once) and sweeps
// its entries one jump each until all are done: every chain then shortens
// like synchronous rounds (O(log length) sweeps).  A non-resident thread
// would find its successors not started yet and walk long chains hop by hop.
__global__ void k_rank_jump_async(const int32_t* __restrict__ count, uint64_t* word) {
    const int32_t nr = *count;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (;;) {
        bool more = false;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += stride) {
            uint64_t w = ld_word(word + i);
            const int32_t nx = (int32_t)(w >> 32);
            if (nx < 0) continue;
            const uint64_t w2 = ld_word(word + nx);
            w = (w2 & 0xffffffff00000000ull) | (uint32_t)((uint32_t)w + (uint32_t)w2);
            st_word(word + i, w);
            more = more || (int32_t)(w >> 32) >= 0;
        }
        if (!more) break;
    }
}

__global__ void k_rank_final(int64_t na, const int32_t* __restrict__ owner, const int32_t* __restrict__ local,
                             const uint64_t* __restrict__ rword, int32_t* rank) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < na) rank[i] = (int32_t)((uint32_t)rword[owner[i]] - (uint32_t)local[i]);
}

// Per tree: tour length L = rank of the root's first arc (0 for singletons).
__global__ void k_tour_len(int64_t n, const int32_t* __restrict__ adj_start,
                           const int32_t* __restrict__ root, const int32_t* __restrict__ tree_id,
                           const int32_t* __restrict__ rank, int32_t* tlen) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n || root[v] != v) return;
    int32_t s = adj_start[v], e = adj_start[v + 1];
    tlen[tree_id[v]] = (e > s) ? rank[s] : 0;
}

__global__ void k_tour_pos(int64_t na, const int32_t* __restrict__ asrc,
                           const int32_t* __restrict__ tree_id, const int32_t* __restrict__ tlen,
                           const int32_t* __restrict__ rank, int32_t* tpos) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < na) tpos[i] = tlen[tree_id[asrc[i]]] - rank[i];
}

// Parent links, subtree sizes and the +1/-1 tour steps for the depth scan.
__global__ void k_orient(int64_t na, const int32_t* __restrict__ asrc, const int32_t* __restrict__ adst,
                         const float* __restrict__ aw, const int32_t* __restrict__ twin,
                         const int32_t* __restrict__ tpos, const int32_t* __restrict__ tree_id,
                         const int32_t* __restrict__ toff, int32_t* parent, float* pweight,
                         int32_t* size, int32_t* down_arc, int32_t* steps) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    int32_t x = asrc[i], y = adst[i];
    int32_t j = twin[i];
    bool down = tpos[i] < tpos[j];
    int32_t t = tree_id[x];
    steps[toff[t] + tpos[i]] = down ? 1 : -1;
    if (down) {
        parent[y] = x;
        pweight[y] = aw[i];
        size[y] = (tpos[j] - tpos[i] + 1) / 2;
        down_arc[y] = toff[t] + tpos[i];
    }
}

__global__ void k_root_init(int64_t n, const int32_t* __restrict__ root,
                            const int32_t* __restrict__ tree_id, const int32_t* __restrict__ tlen,
                            int32_t* parent, float* pweight, int32_t* size, int32_t* depth,
                            int32_t* down_arc) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n || root[v] != v) return;
    parent[v] = (int32_t)v;
    pweight[v] = 0.0f;
    size[v] = tlen[tree_id[v]] / 2 + 1;
    depth[v] = 0;
    down_arc[v] = -1;
}

__global__ void k_depth_gather(int64_t n, const int32_t* __restrict__ down_arc,
                               const int32_t* __restrict__ scanned, int32_t* depth, int32_t* dmax) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int32_t d = 0;
    if (v < n) {
        int32_t a = down_arc[v];
        if (a >= 0) depth[v] = d = scanned[a];
    }
    d = __reduce_max_sync(0xffffffffu, d);
    if ((threadIdx.x & 31) == 0 && d > 0) atomicMax(dmax, d);
}

// heavy child: largest subtree among children, ties -> lower id (adjacency
// lists are ascending by id, so keep the first maximum).
__global__ void k_heavy(int64_t n, const int32_t* __restrict__ adj_start,
                        const int32_t* __restrict__ adst, const int32_t* __restrict__ parent,
                        const int32_t* __restrict__ size, int32_t* heavy) {
    int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= n) return;
    int32_t best = -1, bs = -1;
    for (int32_t k = adj_start[x]; k < adj_start[x + 1]; k++) {
        int32_t y = adst[k];
        if (parent[y] == x && y != x) {
            if (size[y] > bs) {
                bs = size[y];
                best = y;
            }
        }
    }
    heavy[x] = best;
}

// heavy-path heads: word = (heavy parent or self, distance)
// Heavy-path heads and distances by a ruling set.  Rulers: every path head
// (root or light child) and every heavy child at a depth divisible by kHpRuler.
// Each node walks up (< kHpRuler parent steps) to its nearest ruler; the
// non-head rulers, about n / kHpRuler of them, pointer-jump to their heads.
#ifndef HDP_HP_RULER
#define HDP_HP_RULER 16
#endif
constexpr int kHpRuler = HDP_HP_RULER;

// pr[v] = parent | ruler flag << 31
__global__ void k_hp_flags(int64_t n, const int32_t* __restrict__ parent, const int32_t* __restrict__ heavy,
                           const int32_t* __restrict__ depth, int32_t* pr) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int32_t p = parent[v];
    const bool on = (p != v) && heavy[p] == v;  // heavy child: not a head
    const bool ruler = !on || depth[v] % kHpRuler == 0;
    pr[v] = p | (ruler ? (int32_t)0x80000000 : 0);
}

__device__ __forceinline__ uint64_t hp_word(int32_t ptr, int32_t d) {
    return ((uint64_t)(uint32_t)ptr << 32) | (uint32_t)d;
}

// near[v] = (nearest ruler at or above v, steps); heads get the terminal word
// in both jump buffers, non-head rulers their next ruler up and a list slot
__global__ void k_hp_walk(int64_t n, const int32_t* __restrict__ pr, const int32_t* __restrict__ parent,
                          const int32_t* __restrict__ heavy, uint64_t* nearw, uint64_t* wa, uint64_t* wb,
                          int32_t* list, int32_t* cnt) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool listed = false;
    if (v < n) {
        int32_t x = pr[v];
        int32_t cur = (int32_t)v, s = 0;
        while (x >= 0) {  // not a ruler: one step up the heavy path
            cur = x;
            s++;
            x = pr[cur];
        }
        nearw[v] = hp_word(cur, s);
        const int32_t p = parent[v];
        const bool head = !((p != v) && heavy[p] == v);
        if (head) {
            wa[v] = wb[v] = hp_word((int32_t)v, 0);
        } else if (s == 0) {  // a non-head ruler: its next ruler up
            int32_t c = p, t = 1;
            int32_t y = pr[c];
            while (y >= 0) {
                c = y;
                t++;
                y = pr[c];
            }
            wa[v] = hp_word(c, t);
            listed = true;
        }
    }
    // warp-aggregated list append (order is irrelevant for pointer jumping)
    const unsigned m = __ballot_sync(0xffffffffu, listed);
    int base = 0;
    const int lane = threadIdx.x & 31;
    if (lane == 0 && m) base = atomicAdd(cnt, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (listed) list[base + __popc(m & ((1u << lane) - 1u))] = (int32_t)v;
}

// a chain of non-head rulers is at most max depth / kHpRuler + 1 long
__device__ __forceinline__ long long hp_chain(const int32_t* dmax) { return (long long)*dmax / kHpRuler + 1; }

// heavy-path ruler words, jumped asynchronously (see k_rank_jump_async); a
// head's word points at itself
__global__ void k_hp_jump_async(const int32_t* __restrict__ list, const int32_t* __restrict__ cnt, uint64_t* word) {
    const int32_t nl = *cnt;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (;;) {
        bool more = false;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += stride) {
            const int32_t v = list[i];
            const uint64_t w = ld_word(word + v);
            const int32_t h = (int32_t)(w >> 32);
            const uint64_t w2 = ld_word(word + h);
            const int32_t hh = (int32_t)(w2 >> 32);
            if (hh == h) continue;  // h is a head: done
            st_word(word + v, hp_word(hh, (int32_t)((uint32_t)w + (uint32_t)w2)));
            more = true;
        }
        if (!more) break;
    }
}

__global__ void k_hp_jump(const int32_t* __restrict__ list, const int32_t* __restrict__ cnt,
                          const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                          const int32_t* __restrict__ dmax, int r) {
    if ((1ll << r) >= hp_chain(dmax)) return;
    const int32_t nl = *cnt;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = list[i];
        const uint64_t w = in[v];
        const int32_t h = (int32_t)(w >> 32);
        const uint64_t w2 = in[h];
        const int32_t hh = (int32_t)(w2 >> 32);
        out[v] = hh != h ? hp_word(hh, (int32_t)((uint32_t)w + (uint32_t)w2)) : w;
    }
}

// the jumped words are in buffer a after an even number of executed rounds
__global__ void k_hp_unpack(int64_t n, const uint64_t* __restrict__ nearw, const uint64_t* __restrict__ a,
                            const uint64_t* __restrict__ b, const int32_t* __restrict__ dmax, int rounds,
                            int32_t* hp, int32_t* dist) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const long long ch = hp_chain(dmax);
    int done = 0;
    while (done < rounds && (1ll << done) < ch) done++;
    const uint64_t nw = nearw[v];
    const uint64_t w = ((done & 1) ? b : a)[(int32_t)(nw >> 32)];
    hp[v] = (int32_t)(w >> 32);
    dist[v] = (int32_t)((uint32_t)nw + (uint32_t)w);
}

// light-edge steps for the light-depth scan: entering / leaving a path head.
__global__ void k_light_steps(int64_t na, const int32_t* __restrict__ asrc,
                              const int32_t* __restrict__ adst, const int32_t* __restrict__ parent,
                              const int32_t* __restrict__ head, const int32_t* __restrict__ tpos,
                              const int32_t* __restrict__ tree_id, const int32_t* __restrict__ toff,
                              int32_t* steps) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    int32_t x = asrc[i], y = adst[i];
    int32_t pos = toff[tree_id[x]] + tpos[i];
    if (parent[y] == x) {
        steps[pos] = (head[y] == y) ? 1 : 0;  // down into y
    } else {
        steps[pos] = (head[x] == x) ? -1 : 0;  // up out of x
    }
}

// nodes per heavy path, stored at the head
__global__ void k_path_len(int64_t n, const int32_t* __restrict__ head,
                           const int32_t* __restrict__ dist, int32_t* plen) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // one atomic per (warp, path): neighbouring ids often share a heavy path
    const int32_t h = v < n ? head[v] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, h);
    const int32_t l = __reduce_max_sync(peers, v < n ? dist[v] + 1 : 0);
    if (v < n && (threadIdx.x & 31) == __ffs(peers) - 1) atomicMax(&plen[h], l);
}

// light depth of every node (scan of the light-edge tour steps)
__global__ void k_light_depth(int64_t n, const int32_t* __restrict__ down_arc, const int32_t* __restrict__ lscan,
                              int32_t* ld_out) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    int32_t a = down_arc[v];
    ld_out[v] = a >= 0 ? lscan[a] : 0;
}

__global__ void k_head_flags(int64_t n, const int32_t* __restrict__ head, int32_t* hf) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) hf[v] = head[v] == v ? 1 : 0;
    else if (v == n) hf[v] = 0;
}

// heads in ascending id with their layout class (light depth, long path)
__global__ void k_head_keys(int64_t n, const int32_t* __restrict__ hf, const int32_t* __restrict__ hpos,
                            const int32_t* __restrict__ ld, const int32_t* __restrict__ plen,
                            uint8_t* hkey, int32_t* hval) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n || !hf[v]) return;
    const int32_t i = hpos[v];
    // class within the phase: short paths of two or more nodes, then the lone
    // leaves (one-node paths: no work on the way up, so the up pass skips the
    // chunks that hold nothing else), then the long paths
    const int cls = plen[v] > kShortPath ? 2 : (plen[v] == 1 ? 1 : 0);
    hkey[i] = (uint8_t)((ld[v] << 2) | cls);
    hval[i] = (int32_t)v;
}

__global__ void k_head_lens(int64_t n, const int32_t* __restrict__ hpos, const int32_t* __restrict__ sorted,
                            const int32_t* __restrict__ plen, int32_t* slen, int32_t* hrank) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    const int32_t nh = hpos[n];
    if (i < nh) {
        const int32_t h = sorted[i];
        slen[i] = plen[h];
        hrank[h] = (int32_t)i;
    } else {
        slen[i] = 0;
    }
}

// layout position = first position of the node's path + distance from its head
__global__ void k_layout_place(int64_t n, const int32_t* __restrict__ head, const int32_t* __restrict__ dist,
                               const int32_t* __restrict__ hrank, const int32_t* __restrict__ pbase,
                               const float* __restrict__ pweight, float gamma, int32_t* lnode, int32_t* lpos,
                               float* lsim) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int32_t k = pbase[hrank[head[v]]] + dist[v];
    lnode[k] = (int32_t)v;
    lpos[v] = k;
    // RootedForest.similarities (spanning_forest.py:184-188) in float64,
    // rounded once to the f32 the aggregation runs in.
    lsim[k] = (float)exp(-(double)pweight[v] / ((double)gamma * 255.0));
}

__global__ void k_lp_flags(int64_t n, const int32_t* __restrict__ lc_start, int32_t* fl) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) fl[k] = lc_start[k + 1] > lc_start[k] ? 1 : 0;
    else if (k == n) fl[k] = 0;
}

__global__ void k_lp_fill(int64_t n, const int32_t* __restrict__ fl, const int32_t* __restrict__ ex,
                          int32_t* list) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n && fl[k]) list[ex[k]] = (int32_t)k;
}

__global__ void k_path_fill(int64_t n, const int32_t* __restrict__ flag,
                            const int32_t* __restrict__ pidx, int32_t* p_start) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n && flag[k]) p_start[pidx[k]] = (int32_t)k;
}

// light children of the node at layout position k, ascending id
// One thread per node id (not per layout position): the adjacency, parent
// and head reads of neighbouring threads are neighbouring (grid trees), only
// the count / the CSR start is gathered through lpos.
__global__ void k_lc_count(int64_t n, const int32_t* __restrict__ lpos,
                           const int32_t* __restrict__ adj_start, const int32_t* __restrict__ adst,
                           const int32_t* __restrict__ parent, const int32_t* __restrict__ head,
                           int32_t* cnt) {
    int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= n) return;
    int32_t c = 0;
    for (int32_t a = adj_start[x]; a < adj_start[x + 1]; a++) {
        int32_t y = adst[a];
        if (parent[y] == x && y != x && head[y] == y) c++;
    }
    cnt[lpos[x]] = c;
}

__global__ void k_lc_fill(int64_t n, const int32_t* __restrict__ lpos,
                          const int32_t* __restrict__ adj_start, const int32_t* __restrict__ adst,
                          const int32_t* __restrict__ parent, const int32_t* __restrict__ head,
                          const int32_t* __restrict__ lc_start, int32_t* lc_list) {
    int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= n) return;
    const int32_t a0 = adj_start[x], a1 = adj_start[x + 1];
    int32_t o = -1;
    for (int32_t a = a0; a < a1; a++) {
        int32_t y = adst[a];
        if (parent[y] == x && y != x && head[y] == y) {
            if (o < 0) o = lc_start[lpos[x]];
            lc_list[o++] = lpos[y];
        }
    }
}

// ---- lanes
__global__ void k_lanes_range(int64_t nt, int nx, int32_t* t_m, int32_t* t_doff) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    t_m[t] = nx;
    t_doff[t] = 0;
}

__global__ void k_iota(int64_t n, int32_t* a, int32_t x0) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = x0 + (int32_t)i;
}

// lanes per tree; the smallest count lands in *mn (an empty interval is an
// error, cost_volume.py:212-213)
__global__ void k_lanes_count(int64_t nt, const uint32_t* __restrict__ masks, int nw, int32_t* t_m, int32_t* mn) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int c = 0x7fffffff;
    if (t < nt) {
        c = 0;
        for (int i = 0; i < nw; i++) c += __popc(masks[t * nw + i]);
        t_m[t] = c;
    }
    c = __reduce_min_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c != 0x7fffffff) atomicMin(mn, c);
}

// per-node masks (valid at every node, e.g. hdp_hdpf's tree_masks) -> per tree,
// read at each tree's root
__global__ void k_tree_masks(int64_t n, const int32_t* __restrict__ root, const int32_t* __restrict__ tree_id,
                             const uint32_t* __restrict__ node_masks, int nw, uint32_t* out) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n || root[v] != v) return;
    const int64_t t = tree_id[v];
    for (int i = 0; i < nw; i++) out[t * nw + i] = node_masks[v * nw + i];
}

__global__ void k_lanes_fill(int64_t nt, const uint32_t* __restrict__ masks, int nw,
                             const int32_t* __restrict__ t_doff, int32_t* dlist) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    int32_t o = t_doff[t];
    for (int i = 0; i < nw; i++) {
        uint32_t word = masks[t * nw + i];
        while (word) {
            int b = __ffs(word) - 1;
            dlist[o++] = i * 32 + b;
            word &= word - 1;
        }
    }
}

__global__ void k_row_m(int64_t n, const int32_t* __restrict__ lnode,
                        const int32_t* __restrict__ tree_id, const int32_t* __restrict__ t_m,
                        int64_t* rm) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) rm[k] = (t_m[tree_id[lnode[k]]] + 3) & ~3;  // rows padded to 16 bytes
    if (k == n) rm[k] = 0;
}

__global__ void k_node_m(int64_t n, const int32_t* __restrict__ tree_id,
                         const int32_t* __restrict__ t_m, int64_t* nm) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) nm[v] = t_m[tree_id[v]];
}

// ---- device-count driven path/phase tables (steps 8-10): every count stays
// on the device until one summary read at the end of the build.
constexpr int kMaxPhases = 64;  // light depth <= log2(n) + 1
enum { C_NP = 0, C_NPH, C_NL, C_NSEG, C_NLC, C_NLP, C_MAXD, C_COUNT };
// per-phase table rows of the summary
enum { P_FIRST = 0, P_NODE, P_LONG, P_SHORT, P_SEG, P_SEND, P_LP, P_LPM, P_ROWS };

__global__ void k_path_flags_n(int64_t n, const int32_t* __restrict__ lnode,
                               const int32_t* __restrict__ head, int32_t* flag) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) {
        int32_t v = lnode[k];
        flag[k] = head[v] == v ? 1 : 0;
    } else if (k == n) {
        flag[k] = 0;
    }
}

// per path: length, parent position, tree, light depth, long flag; entries
// past the path count get is_long = 0 so that a scan over n + 1 is exact
__global__ void k_path_info_n(int64_t n, const int32_t* __restrict__ pidx, const int32_t* __restrict__ p_start,
                              const int32_t* __restrict__ lnode, const int32_t* __restrict__ parent,
                              const int32_t* __restrict__ lpos, const int32_t* __restrict__ tree_id,
                              const int32_t* __restrict__ ld, int32_t* p_len, int32_t* p_par,
                              int32_t* p_tree, int32_t* p_ld, int32_t* is_long) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    const int32_t np = pidx[n];
    if (i >= np) {
        is_long[i] = 0;
        return;
    }
    int32_t s = p_start[i];
    int32_t e = (i + 1 < np) ? p_start[i + 1] : (int32_t)n;
    int32_t h = lnode[s];
    p_len[i] = e - s;
    p_par[i] = parent[h] == h ? -1 : lpos[parent[h]];
    p_tree[i] = tree_id[h];
    p_ld[i] = ld[h];
    is_long[i] = (e - s) > kShortPath ? 1 : 0;
}

__global__ void k_path_counts(int64_t n, const int32_t* __restrict__ pidx, const int32_t* __restrict__ p_ld,
                              int32_t* cnt) {
    const int32_t np = pidx[n];
    cnt[C_NP] = np;
    cnt[C_NPH] = np > 0 ? p_ld[np - 1] + 1 : 0;
}

// first path of every phase (paths are phase-major)
__global__ void k_phase_bounds_n(int64_t n, const int32_t* __restrict__ cnt, const int32_t* __restrict__ p_ld,
                                 int32_t* first) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t np = cnt[C_NP], nph = cnt[C_NPH];
    if (i > np) return;
    int a = (i == 0) ? -1 : p_ld[i - 1];
    int b = (i == np) ? nph : p_ld[i];
    for (int r = a + 1; r <= b; r++) first[r] = (int32_t)i;
}

__global__ void k_split_paths_n(int64_t n, const int32_t* __restrict__ cnt, const int32_t* __restrict__ is_long,
                                const int32_t* __restrict__ lexcl, int32_t* long_paths, int32_t* short_paths) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cnt[C_NP]) return;
    int32_t l = lexcl[i];
    if (is_long[i]) long_paths[l] = (int32_t)i;
    else short_paths[i - l] = (int32_t)i;
}

// phase table rows FIRST, NODE, LONG, SHORT (r in [0, nph])
__global__ void k_phase_tab(int64_t n, int32_t* cnt, const int32_t* __restrict__ first,
                            const int32_t* __restrict__ p_start, const int32_t* __restrict__ lexcl, int32_t* ph) {
    const int32_t np = cnt[C_NP], nph = cnt[C_NPH];
    for (int r = threadIdx.x; r <= nph; r += blockDim.x) {
        int32_t fi = first[r];
        ph[P_FIRST * (kMaxPhases + 1) + r] = fi;
        ph[P_NODE * (kMaxPhases + 1) + r] = fi < np ? p_start[fi] : (int32_t)n;
        int32_t lo = lexcl[fi];
        ph[P_LONG * (kMaxPhases + 1) + r] = lo;
        ph[P_SHORT * (kMaxPhases + 1) + r] = fi - lo;
    }
    if (threadIdx.x == 0) cnt[C_NL] = lexcl[np];
}

// short-path block end of every phase (short paths come first in a phase)
__global__ void k_phase_send(int64_t n, const int32_t* __restrict__ cnt, const int32_t* __restrict__ short_paths,
                             const int32_t* __restrict__ p_start, const int32_t* __restrict__ p_len, int32_t* ph) {
    const int32_t nph = cnt[C_NPH];
    const int32_t* so = ph + P_SHORT * (kMaxPhases + 1);
    const int32_t* pn = ph + P_NODE * (kMaxPhases + 1);
    for (int r = threadIdx.x; r <= nph; r += blockDim.x) {
        int32_t e = (int32_t)n;
        if (r < nph) {
            if (so[r + 1] > so[r]) {
                int32_t p = short_paths[so[r + 1] - 1];
                e = p_start[p] + p_len[p];
            } else {
                e = pn[r];
            }
        }
        ph[P_SEND * (kMaxPhases + 1) + r] = e;
    }
}

__global__ void k_seg_count_n(int64_t n, const int32_t* __restrict__ cnt, const int32_t* __restrict__ long_paths,
                              const int32_t* __restrict__ p_len, int32_t* nseg) {
    int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l > n) return;
    nseg[l] = l < cnt[C_NL] ? (p_len[long_paths[l]] + kSeg - 1) / kSeg : 0;
}

__global__ void k_seg_fill_n(int64_t n, const int32_t* __restrict__ cnt, const int32_t* __restrict__ nseg,
                             const int32_t* __restrict__ soff, int2* seg_tab) {
    int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= cnt[C_NL]) return;
    int32_t o = soff[l];
    for (int s = 0; s < nseg[l]; s++) seg_tab[o + s] = make_int2((int)l, s);
}

// remaining rows (SEG, LP, LPM) and counts, then the packed summary
__global__ void k_forest_summary(int64_t n, int32_t* cnt, const int32_t* __restrict__ soff,
                                 const int32_t* __restrict__ lc_start, const int32_t* __restrict__ ex,
                                 int32_t* ph) {
    const int32_t nph = cnt[C_NPH];
    for (int r = threadIdx.x; r <= nph; r += blockDim.x) {
        ph[P_SEG * (kMaxPhases + 1) + r] = soff[ph[P_LONG * (kMaxPhases + 1) + r]];
        ph[P_LP * (kMaxPhases + 1) + r] = ex[ph[P_NODE * (kMaxPhases + 1) + r]];
        ph[P_LPM * (kMaxPhases + 1) + r] = ex[ph[P_SEND * (kMaxPhases + 1) + r]];
    }
    if (threadIdx.x == 0) {
        cnt[C_NSEG] = soff[cnt[C_NL]];
        cnt[C_NLC] = lc_start[n];
        cnt[C_NLP] = ex[n];
    }
}

}  // namespace hdp

using namespace hdp;

// CTAs of `block` threads for `items`, capped at what the GPU holds resident
// (the asynchronous jump kernels rely on all their threads running at once)
static unsigned resident_grid(int64_t items, int block) {
    static int cap = 0;
    if (cap == 0) {
        int dev = 0, nsm = 148, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&per, cudaDevAttrMaxThreadsPerMultiProcessor, dev);
        cap = nsm * std::max(1, per / block);
    }
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(grid_for(items, block), cap));
}

// pointer jumping without grid barriers (one launch); HDP_SYNC_JUMP=1: the
// round-synchronous launches (diagnostics / A-B)
static bool async_jump() {
    static const bool on = [] {
        const char* e = getenv("HDP_SYNC_JUMP");
        return !(e && e[0] == '1');
    }();
    return on;
}

static int forest_build(hdp_forest* f, int64_t m_in, const int32_t* eu, const int32_t* ev,
                        const float* ew, const uint8_t* in_tree, const int32_t* comp_in) {
    cudaStream_t st = f->st;
    const int64_t n = f->n;
    const int B = 256;

    Tracer tr(st);
    // ---- 1. tree edges
    DevBuf<int32_t> flags, fpos;
    HDP_TRY(flags.alloc(m_in + 1, st));
    HDP_TRY(fpos.alloc(m_in + 1, st));
    int64_t m = 0;
    // with a component labelling given, the tree-edge count is read together
    // with the tree count below (one host read less): buffers take the bound
    const bool defer_m = comp_in != nullptr;
    DevBuf<int> ecnt;  // (tree edges, unsorted flag)
    HDP_TRY(ecnt.alloc(2, st));
    HDP_CHECK_CUDA(cudaMemsetAsync(ecnt.get(), 0, 2 * sizeof(int), st));
    if (m_in > 0) {
        k_flag_edges<<<grid_for(m_in, B), B, 0, st>>>(m_in, in_tree, eu, ev, flags.get(), ecnt.get() + 1); note_launch();
        HDP_TRY(exclusive_sum(flags.get(), fpos.get(), m_in, st));
        k_edge_count<<<1, 1, 0, st>>>(m_in, flags.get(), fpos.get(), ecnt.get()); note_launch();
        if (!defer_m) {
            int hc[2] = {0, 0};
            HDP_TRY(to_host(hc, ecnt.get(), 2, st));
            m = hc[0];
            HDP_REQUIRE(m <= n - 1 || n == 0, HDP_ERR_DATA, "forest has %lld edges for %lld nodes (cycle)",
                        (long long)m, (long long)n);
        }
    }
    const int64_t mcap = defer_m ? m_in : m;  // rows of the compacted edge arrays
    DevBuf<int32_t> tu, tv;
    DevBuf<float> tw;
    DevBuf<uint64_t> tkey;
    HDP_TRY(tu.alloc(mcap + 1, st));
    HDP_TRY(tv.alloc(mcap + 1, st));
    HDP_TRY(tw.alloc(mcap + 1, st));
    HDP_TRY(tkey.alloc(mcap + 1, st));
    if (m_in > 0)
        k_compact_edges<<<grid_for(m_in, B), B, 0, st>>>(m_in, flags.get(), fpos.get(), eu, ev, ew,
                                                        tu.get(), tv.get(), tw.get(), tkey.get()); note_launch();
    flags.release();
    fpos.release();

    tr.mark("1 tree edges");
    // ---- 2. components, roots, tree numbering
    DevBuf<int32_t> comp;
    HDP_TRY(comp.alloc(n, st));
    if (comp_in) {
        HDP_CHECK_CUDA(cudaMemcpyAsync(comp.get(), comp_in, n * sizeof(int32_t),
                                       cudaMemcpyDeviceToDevice, st));
    } else {
        DevBuf<uint8_t> sel;
        HDP_TRY(sel.alloc(m + 1, st));
        HDP_TRY(run_boruvka(n, m, tu.get(), tv.get(), tkey.get(), sel.get(), comp.get(), nullptr, st));
    }
    tkey.release();
    DevBuf<int32_t> minid, is_root, tindex;
    HDP_TRY(minid.alloc(n, st));
    HDP_TRY(is_root.alloc(n, st));
    HDP_TRY(tindex.alloc(n, st));
    HDP_TRY(f->root.alloc(n, st));
    HDP_TRY(f->tree_id.alloc(n, st));
    int32_t max_tree = 1;  // nodes in the largest tree
    {
        DevBuf<int32_t> csize, cnt;  // cnt = (trees, largest tree, tree edges)
        HDP_TRY(csize.alloc(n, st));
        HDP_TRY(cnt.alloc(3, st));
        HDP_CHECK_CUDA(cudaMemsetAsync(csize.get(), 0, n * sizeof(int32_t), st));
        HDP_CHECK_CUDA(cudaMemsetAsync(cnt.get(), 0, 2 * sizeof(int32_t), st));
        HDP_CHECK_CUDA(cudaMemcpyAsync(cnt.get() + 2, ecnt.get(), sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        k_fill_int<<<grid_for(n, B), B, 0, st>>>(n, minid.get(), INT_MAX); note_launch();
        k_min_root<<<grid_for(n, B), B, 0, st>>>(n, comp.get(), minid.get(), csize.get()); note_launch();
        k_root_flags<<<grid_for(n, B), B, 0, st>>>(n, comp.get(), minid.get(), csize.get(), f->root.get(),
                                                  is_root.get(), cnt.get() + 1); note_launch();
        HDP_TRY(exclusive_sum(is_root.get(), tindex.get(), n, st));
        k_tree_count<<<1, 1, 0, st>>>(n, tindex.get(), is_root.get(), cnt.get()); note_launch();
        int32_t hc[3] = {0, 0, 0};
        HDP_TRY(to_host(hc, cnt.get(), 3, st));
        f->n_trees = hc[0];
        max_tree = hc[1] > 0 ? hc[1] : 1;
        if (defer_m) m = hc[2];
        // an acyclic edge set on n nodes with t components has exactly n - t
        // edges; a cycle, a self-loop or a repeated edge leaves more (the
        // Euler tour would then hold closed circuits that never terminate)
        HDP_REQUIRE(m == n - f->n_trees, HDP_ERR_DATA,
                    "edge set is not a forest: %lld edges, %lld nodes, %lld components (cycle, self-loop "
                    "or repeated edge)", (long long)m, (long long)n, (long long)f->n_trees);
    }
    k_tree_ids<<<grid_for(n, B), B, 0, st>>>(n, f->root.get(), tindex.get(), f->tree_id.get()); note_launch();
    HDP_CHECK_LAUNCH();
    comp.release();
    minid.release();
    tindex.release();

    tr.mark("2 components/roots");
    // ---- 3. CSR adjacency (arcs sorted by (src, dst))
    const int64_t na = 2 * m;
    DevBuf<float> aw2;
    DevBuf<int32_t> deg, adj_start, asrc, adst;
    HDP_TRY(aw2.alloc(na + 1, st));
    HDP_TRY(deg.alloc(n + 1, st));
    HDP_TRY(adj_start.alloc(n + 1, st));
    HDP_TRY(asrc.alloc(na + 1, st));
    HDP_TRY(adst.alloc(na + 1, st));
    HDP_CHECK_CUDA(cudaMemsetAsync(deg.get(), 0, (n + 1) * sizeof(int32_t), st));
    if (m > 0) {
        k_arc_degree<<<grid_for(m, B), B, 0, st>>>(m, tu.get(), tv.get(), deg.get()); note_launch();
    }
    HDP_TRY(exclusive_sum(deg.get(), adj_start.get(), n + 1, st));
    if (m > 0) {
        // deg doubles as the per-source cursor
        HDP_CHECK_CUDA(cudaMemsetAsync(deg.get(), 0, (n + 1) * sizeof(int32_t), st));
        k_arc_place<<<grid_for(m, B), B, 0, st>>>(m, tu.get(), tv.get(), tw.get(), adj_start.get(), deg.get(),
                                                 asrc.get(), adst.get(), aw2.get()); note_launch();
        k_arc_sort<<<grid_for(n, B), B, 0, st>>>(n, adj_start.get(), adst.get(), aw2.get()); note_launch();
    }
    tu.release();
    tv.release();
    tw.release();

    tr.mark("3 csr adjacency");
    // ---- 4. Euler tour + list ranking
    DevBuf<int32_t> twin, nxt, rank, tlen, toff, tpos;
    HDP_TRY(twin.alloc(na + 1, st));
    HDP_TRY(nxt.alloc(na + 1, st));
    HDP_TRY(rank.alloc(na + 1, st));
    HDP_TRY(tlen.alloc(f->n_trees + 1, st));
    HDP_TRY(toff.alloc(f->n_trees + 1, st));
    HDP_TRY(tpos.alloc(na + 1, st));
    HDP_CHECK_CUDA(cudaMemsetAsync(tlen.get(), 0, (f->n_trees + 1) * sizeof(int32_t), st));
    if (na > 0) {
        k_tour_next<<<grid_for(na, B), B, 0, st>>>(na, asrc.get(), adst.get(), adj_start.get(),
                                                  f->root.get(), twin.get(), nxt.get()); note_launch();
        // ruling-set ranking; rulers <= ceil(na / kRuler) + one head per tree
        const int64_t rmax = (na + kRuler - 1) / kRuler + f->n_trees + 1;
        DevBuf<uint8_t> hpred;
        DevBuf<int32_t> rflag, rid, rlist, owner, local;
        DevBuf<uint64_t> wa, wb;
        HDP_TRY(hpred.alloc(na, st));
        HDP_TRY(rflag.alloc(na + 1, st));
        HDP_TRY(rid.alloc(na + 1, st));
        HDP_TRY(rlist.alloc(rmax, st));
        HDP_TRY(owner.alloc(na, st));
        HDP_TRY(local.alloc(na, st));
        HDP_TRY(wa.alloc(rmax, st));
        HDP_TRY(wb.alloc(rmax, st));
        HDP_CHECK_CUDA(cudaMemsetAsync(hpred.get(), 0, na, st));
        k_has_pred<<<grid_for(na, B), B, 0, st>>>(na, nxt.get(), hpred.get()); note_launch();
        k_ruler_flags<<<grid_for(na + 1, B), B, 0, st>>>(na, hpred.get(), rflag.get()); note_launch();
        HDP_TRY(exclusive_sum(rflag.get(), rid.get(), na + 1, st));
        k_ruler_list<<<grid_for(na, B), B, 0, st>>>(na, rflag.get(), rid.get(), rlist.get()); note_launch();
        k_ruler_walk<<<grid_for(rmax, 128), 128, 0, st>>>(na, rid.get(), rlist.get(), rflag.get(), nxt.get(),
                                                          owner.get(), local.get(), wa.get()); note_launch();
        // the longest ruler chain is at most the largest tree's tour, 2 (size - 1) arcs
        const int rounds = ceil_log2(2 * (int64_t)max_tree);
        // asynchronous jumping pays while the ruler chains are short; one giant
        // tour (C5: 715k rulers in one chain) converges faster in synchronous rounds
        if (async_jump() && 2 * (int64_t)max_tree / kRuler <= (1 << 16)) {
            k_rank_jump_async<<<resident_grid(rmax, B), B, 0, st>>>(rid.get() + na, wa.get()); note_launch();
        } else {
            for (int r = 0; r < rounds; r++) {
                k_rank_jump_n<<<grid_for(rmax, B), B, 0, st>>>(rid.get() + na, wa.get(), wb.get()); note_launch();
                std::swap(wa.p, wb.p);
            }
        }
        k_rank_final<<<grid_for(na, B), B, 0, st>>>(na, owner.get(), local.get(), wa.get(), rank.get()); note_launch();
        HDP_CHECK_LAUNCH();
    }
    k_tour_len<<<grid_for(n, B), B, 0, st>>>(n, adj_start.get(), f->root.get(), f->tree_id.get(),
                                             rank.get(), tlen.get()); note_launch();
    HDP_TRY(exclusive_sum(tlen.get(), toff.get(), f->n_trees + 1, st));
    if (na > 0)
        k_tour_pos<<<grid_for(na, B), B, 0, st>>>(na, asrc.get(), f->tree_id.get(), tlen.get(),
                                                 rank.get(), tpos.get()); note_launch();
    nxt.release();
    rank.release();

    tr.mark("4 euler tour+ranking");
    // ---- 5. orientation, sizes, depth
    HDP_TRY(f->parent.alloc(n, st));
    HDP_TRY(f->pweight.alloc(n, st));
    HDP_TRY(f->size.alloc(n, st));
    HDP_TRY(f->depth.alloc(n, st));
    DevBuf<int32_t> down_arc, steps, scanned, dmax;
    HDP_TRY(dmax.alloc(1, st));
    HDP_CHECK_CUDA(cudaMemsetAsync(dmax.get(), 0, sizeof(int32_t), st));
    HDP_TRY(down_arc.alloc(n, st));
    HDP_TRY(steps.alloc(na + 1, st));
    HDP_TRY(scanned.alloc(na + 1, st));
    k_root_init<<<grid_for(n, B), B, 0, st>>>(n, f->root.get(), f->tree_id.get(), tlen.get(),
                                              f->parent.get(), f->pweight.get(), f->size.get(),
                                              f->depth.get(), down_arc.get()); note_launch();
    if (na > 0) {
        k_orient<<<grid_for(na, B), B, 0, st>>>(na, asrc.get(), adst.get(), aw2.get(), twin.get(),
                                               tpos.get(), f->tree_id.get(), toff.get(),
                                               f->parent.get(), f->pweight.get(), f->size.get(),
                                               down_arc.get(), steps.get()); note_launch();
        HDP_TRY(inclusive_sum(steps.get(), scanned.get(), na, st));
        k_depth_gather<<<grid_for(n, B), B, 0, st>>>(n, down_arc.get(), scanned.get(), f->depth.get(),
                                                     dmax.get()); note_launch();
    }
    HDP_CHECK_LAUNCH();
    aw2.release();
    twin.release();

    tr.mark("5 orient/depth");
    // ---- 6. heavy paths
    DevBuf<int32_t> heavy, hp, dist;
    HDP_TRY(heavy.alloc(n, st));
    HDP_TRY(hp.alloc(n, st));
    HDP_TRY(dist.alloc(n, st));
    k_heavy<<<grid_for(n, B), B, 0, st>>>(n, adj_start.get(), adst.get(), f->parent.get(),
                                          f->size.get(), heavy.get()); note_launch();
    {
        DevBuf<uint64_t> hw, hw2, nearw;
        DevBuf<int32_t> pr, hlist, hcnt;
        // ruler chains are at most (largest tree) / kHpRuler + 1 long
        const int rounds = ceil_log2((int64_t)max_tree / kHpRuler + 2);
        HDP_TRY(hw.alloc(n, st));
        HDP_TRY(hw2.alloc(n, st));
        HDP_TRY(nearw.alloc(n, st));
        HDP_TRY(pr.alloc(n, st));
        HDP_TRY(hlist.alloc(n, st));
        HDP_TRY(hcnt.alloc(1, st));
        HDP_CHECK_CUDA(cudaMemsetAsync(hcnt.get(), 0, sizeof(int32_t), st));
        k_hp_flags<<<grid_for(n, B), B, 0, st>>>(n, f->parent.get(), heavy.get(), f->depth.get(), pr.get()); note_launch();
        uint64_t* ba = hw.get();
        uint64_t* bb = hw2.get();
        k_hp_walk<<<grid_for(n, B), B, 0, st>>>(n, pr.get(), f->parent.get(), heavy.get(), nearw.get(), ba, bb,
                                                hlist.get(), hcnt.get()); note_launch();
        const int jg = (int)std::min<int64_t>(grid_for(n / kHpRuler + 1, B), 148 * 8);
        if (async_jump()) {
            k_hp_jump_async<<<resident_grid(n / kHpRuler + 1, B), B, 0, st>>>(hlist.get(), hcnt.get(), ba);
            note_launch();
            // zero rounds executed: the unpack reads buffer a
            k_hp_unpack<<<grid_for(n, B), B, 0, st>>>(n, nearw.get(), ba, bb, dmax.get(), 0, hp.get(), dist.get());
        } else {
            for (int r = 0; r < rounds; r++) {
                k_hp_jump<<<jg, B, 0, st>>>(hlist.get(), hcnt.get(), (r & 1) ? bb : ba, (r & 1) ? ba : bb, dmax.get(), r);
                note_launch();
            }
            k_hp_unpack<<<grid_for(n, B), B, 0, st>>>(n, nearw.get(), ba, bb, dmax.get(), rounds, hp.get(), dist.get());
        }
        note_launch();
    }
    HDP_CHECK_LAUNCH();
    heavy.release();
    int32_t* head = hp.get();

    tr.mark("6 heavy paths");
    // ---- 7. light depth (tour scan) and layout order
    DevBuf<int32_t> ld;
    HDP_TRY(ld.alloc(n, st));
    if (na > 0) {
        k_light_steps<<<grid_for(na, B), B, 0, st>>>(na, asrc.get(), adst.get(), f->parent.get(),
                                                    head, tpos.get(), f->tree_id.get(), toff.get(),
                                                    steps.get()); note_launch();
        HDP_TRY(inclusive_sum(steps.get(), scanned.get(), na, st));
    }
    // Layout order (light depth, long path, head id, distance from the head):
    // a stable 8-bit sort of the heads (already in id order) by (light depth,
    // long), a prefix sum of their path lengths, and every node lands at its
    // path's base + its distance from the head.
    HDP_TRY(f->lnode.alloc(n, st));
    HDP_TRY(f->lpos.alloc(n, st));
    HDP_TRY(f->lsim.alloc(n, st));
    k_light_depth<<<grid_for(n, B), B, 0, st>>>(n, down_arc.get(), scanned.get(), ld.get()); note_launch();
    {
        DevBuf<int32_t> plen, hf, hpos, hval, hsorted, slen, pbase, hrank;
        DevBuf<uint8_t> hkey, hkey2;
        HDP_TRY(plen.alloc(n, st));
        HDP_TRY(hf.alloc(n + 1, st));
        HDP_TRY(hpos.alloc(n + 1, st));
        HDP_TRY(hval.alloc(n, st));
        HDP_TRY(hsorted.alloc(n, st));
        HDP_TRY(slen.alloc(n + 1, st));
        HDP_TRY(pbase.alloc(n + 1, st));
        HDP_TRY(hrank.alloc(n, st));
        HDP_TRY(hkey.alloc(n, st));
        HDP_TRY(hkey2.alloc(n, st));
        HDP_CHECK_CUDA(cudaMemsetAsync(plen.get(), 0, n * sizeof(int32_t), st));
        HDP_CHECK_CUDA(cudaMemsetAsync(hkey.get(), 0xff, n, st));  // non-heads sort last
        k_path_len<<<grid_for(n, B), B, 0, st>>>(n, head, dist.get(), plen.get()); note_launch();
        k_head_flags<<<grid_for(n + 1, B), B, 0, st>>>(n, head, hf.get()); note_launch();
        HDP_TRY(exclusive_sum(hf.get(), hpos.get(), n + 1, st));
        k_head_keys<<<grid_for(n, B), B, 0, st>>>(n, hf.get(), hpos.get(), ld.get(), plen.get(), hkey.get(),
                                                  hval.get()); note_launch();
        HDP_TRY(sort_pairs(hkey.get(), hkey2.get(), hval.get(), hsorted.get(), n, 0, 8, st));
        k_head_lens<<<grid_for(n + 1, B), B, 0, st>>>(n, hpos.get(), hsorted.get(), plen.get(), slen.get(),
                                                      hrank.get()); note_launch();
        HDP_TRY(exclusive_sum(slen.get(), pbase.get(), n + 1, st));
        k_layout_place<<<grid_for(n, B), B, 0, st>>>(n, head, dist.get(), hrank.get(), pbase.get(),
                                                     f->pweight.get(), f->gamma, f->lnode.get(), f->lpos.get(),
                                                     f->lsim.get()); note_launch();
        HDP_CHECK_LAUNCH();
    }
    steps.release();
    scanned.release();
    tpos.release();
    toff.release();
    tlen.release();
    down_arc.release();
    asrc.release();

    tr.mark("7 layout sort");
    if (f->early.want) HDP_TRY(ecost_early(f));  // lpos is final: the raw cost starts beside steps 8+
    // ---- 8. paths and phases (sizes bounded by n; counts stay on the device)
    const int PH = kMaxPhases + 1;
    DevBuf<int32_t> dcnt;  // counters; f->dph holds the per-phase table
    HDP_TRY(dcnt.alloc(C_COUNT, st));
    HDP_TRY(f->dph.alloc(P_ROWS * PH, st));
    int32_t* dph = f->dph.get();
    HDP_CHECK_CUDA(cudaMemsetAsync(dcnt.get(), 0, C_COUNT * sizeof(int32_t), st));
    HDP_CHECK_CUDA(cudaMemsetAsync(dph, 0, P_ROWS * PH * sizeof(int32_t), st));
    HDP_TRY(reduce_max(f->depth.get(), dcnt.get() + C_MAXD, n, st));
    DevBuf<int32_t> pflag, pidx;
    HDP_TRY(pflag.alloc(n + 1, st));
    HDP_TRY(pidx.alloc(n + 1, st));
    k_path_flags_n<<<grid_for(n + 1, B), B, 0, st>>>(n, f->lnode.get(), head, pflag.get()); note_launch();
    HDP_TRY(exclusive_sum(pflag.get(), pidx.get(), n + 1, st));
    HDP_TRY(f->p_start.alloc(n + 1, st));
    HDP_TRY(f->p_len.alloc(n + 1, st));
    HDP_TRY(f->p_par.alloc(n + 1, st));
    HDP_TRY(f->p_tree.alloc(n + 1, st));
    k_path_fill<<<grid_for(n, B), B, 0, st>>>(n, pflag.get(), pidx.get(), f->p_start.get()); note_launch();
    DevBuf<int32_t> p_ld, is_long, lexcl, first;
    HDP_TRY(p_ld.alloc(n + 1, st));
    HDP_TRY(is_long.alloc(n + 1, st));
    HDP_TRY(lexcl.alloc(n + 1, st));
    HDP_TRY(first.alloc(PH, st));
    k_path_info_n<<<grid_for(n + 1, B), B, 0, st>>>(n, pidx.get(), f->p_start.get(), f->lnode.get(),
                                                    f->parent.get(), f->lpos.get(), f->tree_id.get(), ld.get(),
                                                    f->p_len.get(), f->p_par.get(), f->p_tree.get(), p_ld.get(),
                                                    is_long.get()); note_launch();
    k_path_counts<<<1, 1, 0, st>>>(n, pidx.get(), p_ld.get(), dcnt.get()); note_launch();
    k_phase_bounds_n<<<grid_for(n + 1, B), B, 0, st>>>(n, dcnt.get(), p_ld.get(), first.get()); note_launch();
    HDP_TRY(exclusive_sum(is_long.get(), lexcl.get(), n + 1, st));
    HDP_TRY(f->long_paths.alloc(n + 1, st));
    HDP_TRY(f->short_paths.alloc(n + 1, st));
    k_split_paths_n<<<grid_for(n, B), B, 0, st>>>(n, dcnt.get(), is_long.get(), lexcl.get(), f->long_paths.get(),
                                                  f->short_paths.get()); note_launch();
    k_phase_tab<<<1, 64, 0, st>>>(n, dcnt.get(), first.get(), f->p_start.get(), lexcl.get(), dph); note_launch();
    k_phase_send<<<1, 64, 0, st>>>(n, dcnt.get(), f->short_paths.get(), f->p_start.get(), f->p_len.get(),
                                   dph); note_launch();
    // segments of kSeg nodes over the long paths (head first), phase-major
    DevBuf<int32_t> nseg, soff;
    HDP_TRY(nseg.alloc(n + 1, st));
    HDP_TRY(soff.alloc(n + 1, st));
    k_seg_count_n<<<grid_for(n + 1, B), B, 0, st>>>(n, dcnt.get(), f->long_paths.get(), f->p_len.get(),
                                                    nseg.get()); note_launch();
    HDP_TRY(exclusive_sum(nseg.get(), soff.get(), n + 1, st));
    HDP_TRY(f->seg_tab.alloc(n + 1, st));
    k_seg_fill_n<<<grid_for(n, B), B, 0, st>>>(n, dcnt.get(), nseg.get(), soff.get(), f->seg_tab.get()); note_launch();
    HDP_CHECK_LAUNCH();
    pflag.release();
    pidx.release();
    p_ld.release();
    is_long.release();
    first.release();
    nseg.release();

    tr.mark("8 paths/phases");
    // ---- 9. light-children CSR in layout order
    DevBuf<int32_t> lcc;
    HDP_TRY(lcc.alloc(n + 1, st));
    HDP_TRY(f->lc_start.alloc(n + 1, st));
    HDP_CHECK_CUDA(cudaMemsetAsync(lcc.get(), 0, (n + 1) * sizeof(int32_t), st));
    k_lc_count<<<grid_for(n, B), B, 0, st>>>(n, f->lpos.get(), adj_start.get(), adst.get(),
                                             f->parent.get(), head, lcc.get()); note_launch();
    HDP_TRY(exclusive_sum(lcc.get(), f->lc_start.get(), n + 1, st));
    HDP_TRY(f->lc_list.alloc(n + 1, st));  // light children <= n - 1
    k_lc_fill<<<grid_for(n, B), B, 0, st>>>(n, f->lpos.get(), adj_start.get(), adst.get(),
                                            f->parent.get(), head, f->lc_start.get(), f->lc_list.get());
    note_launch();
    HDP_CHECK_LAUNCH();

    tr.mark("9 light children");
    // ---- 10. light parents (positions with light children), phase-major
    {
        DevBuf<int32_t> fl, ex;
        HDP_TRY(fl.alloc(n + 1, st));
        HDP_TRY(ex.alloc(n + 1, st));
        k_lp_flags<<<grid_for(n + 1, B), B, 0, st>>>(n, f->lc_start.get(), fl.get()); note_launch();
        HDP_TRY(exclusive_sum(fl.get(), ex.get(), n + 1, st));
        HDP_TRY(f->lp_list.alloc(n + 1, st));
        k_lp_fill<<<grid_for(n, B), B, 0, st>>>(n, fl.get(), ex.get(), f->lp_list.get()); note_launch();
        k_forest_summary<<<1, 64, 0, st>>>(n, dcnt.get(), soff.get(), f->lc_start.get(), ex.get(), dph); note_launch();
        HDP_CHECK_LAUNCH();
        // the one host read of steps 5-10: counts and the per-phase table
        std::vector<int32_t> hbuf(C_COUNT + P_ROWS * PH);
        HDP_CHECK_CUDA(cudaMemcpyAsync(hbuf.data(), dcnt.get(), C_COUNT * sizeof(int32_t),
                                       cudaMemcpyDeviceToHost, st));
        HDP_CHECK_CUDA(cudaMemcpyAsync(hbuf.data() + C_COUNT, dph, P_ROWS * PH * sizeof(int32_t),
                                       cudaMemcpyDeviceToHost, st));
        HDP_CHECK_CUDA(cudaStreamSynchronize(st));
        const int32_t* hc = hbuf.data();
        const int32_t* hp = hbuf.data() + C_COUNT;
        f->n_paths = hc[C_NP];
        f->n_phases = hc[C_NPH];
        f->max_depth = hc[C_MAXD];
        f->n_segs = hc[C_NSEG];
        f->n_lc = hc[C_NLC];
        HDP_REQUIRE(f->n_phases >= 1 && f->n_phases <= kMaxPhases, HDP_ERR_INTERNAL,
                    "light depth %lld out of range", (long long)f->n_phases);
        auto row = [&](int k, std::vector<int64_t>& out) {
            out.assign(f->n_phases + 1, 0);
            for (int64_t r = 0; r <= f->n_phases; r++) out[r] = hp[k * PH + r];
        };
        row(P_FIRST, f->phase_off);
        row(P_NODE, f->phase_node);
        row(P_LONG, f->long_off);
        row(P_SHORT, f->short_off);
        row(P_SEG, f->seg_off);
        row(P_SEND, f->short_end);
        row(P_LP, f->lp_off);
        row(P_LPM, f->lp_mid);
    }
    tr.mark("10 light parents");
    return HDP_OK;
}


namespace hdp {

__global__ void k_pos_meta(int64_t n, const int32_t* __restrict__ lnode,
                           const int32_t* __restrict__ tree_id, const int32_t* __restrict__ t_doff,
                           const float* __restrict__ lsim, const int32_t* __restrict__ lc_start,
                           const int32_t* __restrict__ t_m, int4* lmeta, float* lsimf) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    int32_t v = lnode[k];
    // (node, lane-table offset, image column (set per call), lane count m)
    lmeta[k] = make_int4(v, t_doff[tree_id[v]], -1, t_m[tree_id[v]]);
    float s = lsim[k];
    lsimf[k] = (lc_start[k + 1] > lc_start[k]) ? -s : s;  // sign bit: has light children
}

__global__ void k_lc_meta(int64_t nl, const int32_t* __restrict__ lc_list,
                          const int64_t* __restrict__ rowoff, const float* __restrict__ lsim,
                          int64_t* lc_row, float* lc_sim) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nl) return;
    int32_t ck = lc_list[q];
    lc_row[q] = rowoff[ck];
    lc_sim[q] = lsim[ck];
}

__global__ void k_path_meta(int64_t np, const int32_t* __restrict__ list,
                            const int32_t* __restrict__ p_start, const int32_t* __restrict__ p_len,
                            const int32_t* __restrict__ p_par, const int32_t* __restrict__ p_tree,
                            const int32_t* __restrict__ t_doff, const int32_t* __restrict__ t_m,
                            const int64_t* __restrict__ rowoff, int4* info, longlong2* rows) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    int32_t pi = list[i];
    int32_t s = p_start[pi];
    int64_t r0 = rowoff[s];
    int32_t m = t_m[p_tree[pi]];
    int32_t par = p_par[pi];
    info[i] = make_int4(s, p_len[pi], m, t_doff[p_tree[pi]]);
    rows[i] = make_longlong2(r0, par >= 0 ? rowoff[par] : -1);
}

// per short path: shared-memory weight (own rows, light-children rows, a
// parent row, per-node and per-entry metadata, path metadata) and the size
// of its parent row (0 at a root)
__global__ void k_chunk_weight(int64_t ns, const int4* __restrict__ sinfo,
                               const longlong2* __restrict__ srows,
                               const int32_t* __restrict__ lc_start, int64_t* wt, int64_t* pm) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > ns) return;
    if (i == ns) {
        wt[i] = 0;
        pm[i] = 0;
        return;
    }
    int4 in = sinfo[i];
    int64_t len = in.y, m = (in.z + 3) & ~3;
    int64_t nlc = lc_start[in.x + in.y] - lc_start[in.x];
    wt[i] = (len + nlc + 1) * m + 8 * len + 5 * nlc + 16;
    pm[i] = srows[i].y >= 0 ? m : 0;
}

// lane count of every light-child entry (parent and child share the tree)
__global__ void k_lc_m(int64_t nl, const int32_t* __restrict__ lc_list, const int4* __restrict__ lmeta,
                       int64_t* out) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q < nl) out[q] = (lmeta[lc_list[q]].w + 3) & ~3;
    else if (q == nl) out[q] = 0;
}

// chunk_first over the short paths: path i (phase r) starts chunk
// cbase[r] + ((W[i] - W[so[r]]) >> kChunkShift); every chunk id up to it that
// no earlier path claimed starts at i.
__global__ void k_chunk_fill(int64_t ns, int nph, const int32_t* __restrict__ so,
                             const int64_t* __restrict__ cbase, const int64_t* __restrict__ W,
                             int32_t* chunk_first) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ns) return;
    int lo = 0, hi = nph - 1;  // phase r with so[r] <= i < so[r+1]
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (so[mid] <= i) lo = mid;
        else hi = mid - 1;
    }
    const int r = lo;
    const int64_t w0 = W[so[r]];
    int64_t c = cbase[r] + ((W[i] - w0) >> kChunkShift);
    int64_t cp = (i == so[r]) ? cbase[r] - 1 : cbase[r] + ((W[i - 1] - w0) >> kChunkShift);
    for (int64_t q = cp + 1; q <= c; q++) chunk_first[q] = (int32_t)i;
    if (i == so[r + 1] - 1)
        for (int64_t q = c + 1; q < cbase[r + 1]; q++) chunk_first[q] = (int32_t)(i + 1);
}

// chunks per phase from the cumulative weights (one thread; <= 64 phases)
__global__ void k_chunk_plan(int nph, const int32_t* __restrict__ so, const int64_t* __restrict__ W,
                             int64_t* cbase, int32_t* chunk_first) {
    cbase[0] = 0;
    for (int r = 0; r < nph; r++)
        cbase[r + 1] = cbase[r] + ((W[so[r + 1]] - W[so[r]] + kChunkWords - 1) >> kChunkShift);
    chunk_first[cbase[nph]] = so[nph];
}

__global__ void k_chunk_desc(const int64_t* __restrict__ cbase, int nph, const int32_t* __restrict__ chunk_first,
                             const int4* __restrict__ sinfo, const longlong2* __restrict__ srows,
                             const int32_t* __restrict__ lc_start, const int64_t* __restrict__ lc_rowoff,
                             const int64_t* __restrict__ auxd, const int64_t* __restrict__ W,
                             ChunkDesc* desc, unsigned long long* max_words, int uniform) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = c < cbase[nph];
    unsigned long long words = 0;
    ChunkDesc d = {};
    int p0 = live ? chunk_first[c] : 0, p1 = live ? chunk_first[c + 1] : 0;
    d.p0 = p0;
    d.np = p1 - p0;
    if (p1 > p0) {
        int4 f = sinfo[p0], l = sinfo[p1 - 1];
        d.K0 = f.x;
        d.nk = l.x + l.y - f.x;
        d.L0 = lc_start[d.K0];
        d.nl = lc_start[d.K0 + d.nk] - d.L0;
        int64_t r0 = srows[p0].x, r1 = srows[p1 - 1].x + (int64_t)l.y * ((l.z + 3) & ~3);
        d.a0 = r0 & ~3ll;
        d.n4 = (int)((r1 - d.a0 + 3) >> 2);
        d.lcr0 = lc_rowoff[d.L0];
        d.naux_up = (int)(lc_rowoff[d.L0 + d.nl] - d.lcr0);
        d.auxd0 = auxd[p0];
        d.naux_dn = (int)(auxd[p1] - d.auxd0);
        int mq = (f.z + 3) >> 2;
        // range lanes: every row has the same width; otherwise the uniform
        // mapping only for chunks of few paths (a serial check per chunk)
        if (!uniform) {
            if (p1 - p0 > 64) mq = 0;
            for (int p = p0 + 1; p < p1 && mq > 0; p++)
                if (((sinfo[p].z + 3) >> 2) != mq) mq = 0;
        }
        d.mqu = mq;
        d.inv = mq > 1 ? (unsigned)((0x100000000ull + mq - 1) / mq) : 0u;
        words = (unsigned long long)(W[p1] - W[p0]);
        d.pad0 = (int)words;
    }
    if (live) desc[c] = d;
    // one atomic per warp (a same-address atomic per chunk serialised in L2)
    words = __reduce_max_sync(0xffffffffu, (unsigned)words);
    if ((threadIdx.x & 31) == 0 && words) atomicMax(max_words, words);
}

// chunk classes: big[c] = the chunk needs more than kChunkSmallWords;
// lone[c] = a small chunk of lone leaves only (one-node paths without light
// children: nothing to do on the way up)
__global__ void k_chunk_big_flags(int64_t nc, const ChunkDesc* __restrict__ desc, const int64_t* __restrict__ cbase,
                                  int nph, int32_t* big, int32_t* lone) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    if (c >= cbase[nph]) {  // past the chunk count (nc is its bound): no descriptor was written
        big[c] = 0;
        lone[c] = 0;
        return;
    }
    const ChunkDesc d = desc[c];
    const int b = d.pad0 + 64 > kChunkSmallWords ? 1 : 0;
    big[c] = b;
    lone[c] = (!b && d.np > 0 && d.nl == 0 && d.nk == d.np) ? 1 : 0;
}

// stable partition of every phase's chunks: small ones with work on the way
// up first, then the small lone-leaf chunks, then the big ones (bpos / lpos =
// exclusive scans of the flags); nbig[r] / nlone[r] = those chunks of phase r
__global__ void k_chunk_split(int64_t nc, int nph, const int64_t* __restrict__ cbase,
                              const int32_t* __restrict__ bpos, const int32_t* __restrict__ lpos,
                              const ChunkDesc* __restrict__ in, ChunkDesc* out, int64_t* nbig, int64_t* nlone) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < nph) {
        nbig[c] = bpos[cbase[c + 1]] - bpos[cbase[c]];
        nlone[c] = lpos[cbase[c + 1]] - lpos[cbase[c]];
    }
    if (c >= nc || c >= cbase[nph]) return;
    int lo = 0, hi = nph - 1;  // phase r with cbase[r] <= c < cbase[r + 1]
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (cbase[mid] <= c) lo = mid;
        else hi = mid - 1;
    }
    const int64_t b0 = bpos[cbase[lo]], nb = bpos[cbase[lo + 1]] - b0;
    const int64_t l0 = lpos[cbase[lo]], nl = lpos[cbase[lo + 1]] - l0;
    const int64_t n0 = cbase[lo + 1] - cbase[lo] - nb - nl;  // small chunks with work on the way up
    const int64_t lb = bpos[c] - b0, ll = lpos[c] - l0, ls = (c - cbase[lo]) - lb - ll;
    const bool isbig = bpos[c + 1] != bpos[c], islone = lpos[c + 1] != lpos[c];
    out[cbase[lo] + (isbig ? n0 + nl + lb : (islone ? n0 + ll : ls))] = in[c];
}
}  // namespace hdp

// chunk table of the short-path blocks (needs lmeta, lc rows and short_rows);
// one host read (chunks per phase, largest chunk)
namespace hdp {
__global__ void k_uniform_offsets(int64_t n, int m, int mp, int64_t* rowoff, int64_t* nodeoff) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    rowoff[i] = i * mp;
    if (nodeoff) nodeoff[i] = i * m;
}
}  // namespace hdp

static int build_chunks(hdp_forest* f) {
    cudaStream_t st = f->st;
    const int nph = (int)f->n_phases;
    const int64_t n = f->n, ns = f->short_off[nph], n_lc = f->n_lc;
    DevBuf<int64_t> wt, W, pm, lcm;
    HDP_TRY(wt.alloc(ns + 1, st));
    HDP_TRY(W.alloc(ns + 1, st));
    HDP_TRY(pm.alloc(ns + 1, st));
    HDP_TRY(f->auxd.alloc(ns + 2, st));
    HDP_TRY(lcm.alloc(n_lc + 1, st));
    HDP_TRY(f->lc_rowoff.alloc(n_lc + 2, st));
    k_chunk_weight<<<grid_for(ns + 1, 256), 256, 0, st>>>(ns, f->short_info.get(), f->short_rows.get(),
                                                          f->lc_start.get(), wt.get(), pm.get()); note_launch();
    HDP_TRY(exclusive_sum(wt.get(), W.get(), ns + 1, st));
    HDP_TRY(exclusive_sum(pm.get(), f->auxd.get(), ns + 1, st));
    if (f->range_x0 >= 0) {  // uniform rows: the light-child row offsets are multiples
        const int mpu = (f->max_m + 3) & ~3;
        k_uniform_offsets<<<grid_for(n_lc + 1, 256), 256, 0, st>>>(n_lc, f->max_m, mpu, f->lc_rowoff.get(), nullptr);
        note_launch();
    } else {
        k_lc_m<<<grid_for(n_lc + 1, 256), 256, 0, st>>>(n_lc, f->lc_list.get(), f->lmeta.get(), lcm.get());
        note_launch();
        HDP_TRY(exclusive_sum(lcm.get(), f->lc_rowoff.get(), n_lc + 1, st));
    }
    // chunk-count bound: every short path weighs at most (len + nlc + 1)(mp + 16)
    const int64_t mp = (f->max_m + 3) & ~3;
    const int64_t ncap = (((n + n_lc + ns) * (mp + 16)) >> kChunkShift) + nph + 2;
    const int32_t* so = f->dph.get() + P_SHORT * (kMaxPhases + 1);
    DevBuf<int64_t> cbase, hsum;  // hsum = (chunk bases..., largest chunk)
    DevBuf<unsigned long long> mx;
    HDP_TRY(cbase.alloc(nph + 1, st));
    HDP_TRY(mx.alloc(1, st));
    HDP_TRY(f->chunk_first.alloc(ncap + 1, st));
    HDP_TRY(f->chunk_desc.alloc(ncap + 1, st));
    HDP_CHECK_CUDA(cudaMemsetAsync(mx.get(), 0, sizeof(unsigned long long), st));
    k_chunk_plan<<<1, 1, 0, st>>>(nph, so, W.get(), cbase.get(), f->chunk_first.get()); note_launch();
    if (ns > 0)
        k_chunk_fill<<<grid_for(ns, 256), 256, 0, st>>>(ns, nph, so, cbase.get(), W.get(),
                                                        f->chunk_first.get()); note_launch();
    k_chunk_desc<<<grid_for(ncap, 256), 256, 0, st>>>(cbase.get(), nph, f->chunk_first.get(), f->short_info.get(),
                                                      f->short_rows.get(), f->lc_start.get(),
                                                      f->lc_rowoff.get(), f->auxd.get(), W.get(),
                                                      f->chunk_desc.get(), mx.get(), f->range_x0 >= 0 ? 1 : 0);
    note_launch();
    HDP_CHECK_LAUNCH();
    // size classes (k_chunk_split): the chunk count is only known on the
    // device, so the class passes run over the bound ncap
    DevBuf<int32_t> bflag, bpos, lflag, lpos;
    DevBuf<ChunkDesc> split;
    DevBuf<int64_t> nbig;  // nbig[0 .. nph), then nlone[0 .. nph)
    HDP_TRY(bflag.alloc(ncap + 1, st));
    HDP_TRY(bpos.alloc(ncap + 1, st));
    HDP_TRY(lflag.alloc(ncap + 1, st));
    HDP_TRY(lpos.alloc(ncap + 1, st));
    HDP_TRY(split.alloc(ncap + 1, st));
    HDP_TRY(nbig.alloc(2 * nph + 2, st));
    HDP_CHECK_CUDA(cudaMemsetAsync(bflag.get(), 0, sizeof(int32_t) * (ncap + 1), st));
    HDP_CHECK_CUDA(cudaMemsetAsync(lflag.get(), 0, sizeof(int32_t) * (ncap + 1), st));
    k_chunk_big_flags<<<grid_for(ncap, 256), 256, 0, st>>>(ncap, f->chunk_desc.get(), cbase.get(), nph, bflag.get(),
                                                           lflag.get());
    note_launch();
    HDP_TRY(exclusive_sum(bflag.get(), bpos.get(), ncap + 1, st));
    HDP_TRY(exclusive_sum(lflag.get(), lpos.get(), ncap + 1, st));
    k_chunk_split<<<grid_for(std::max<int64_t>(ncap, nph), 256), 256, 0, st>>>(
        ncap, nph, cbase.get(), bpos.get(), lpos.get(), f->chunk_desc.get(), split.get(), nbig.get(),
        nbig.get() + nph); note_launch();
    HDP_CHECK_LAUNCH();
    std::vector<int64_t> h(nph + 2), hb(2 * nph + 1);
    HDP_CHECK_CUDA(cudaMemcpyAsync(h.data(), cbase.get(), sizeof(int64_t) * (nph + 1), cudaMemcpyDeviceToHost, st));
    HDP_CHECK_CUDA(cudaMemcpyAsync(h.data() + nph + 1, mx.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    HDP_CHECK_CUDA(cudaMemcpyAsync(hb.data(), nbig.get(), sizeof(int64_t) * 2 * nph, cudaMemcpyDeviceToHost, st));
    HDP_CHECK_CUDA(cudaStreamSynchronize(st));
    f->chunk_desc = std::move(split);  // the partitioned table (chunks past the count are never read)
    f->chunk_big.assign(hb.begin(), hb.begin() + nph);
    f->chunk_lone.assign(hb.begin() + nph, hb.begin() + 2 * nph);
    HDP_REQUIRE(h[nph] <= ncap, HDP_ERR_INTERNAL, "chunk count %lld above its bound %lld", (long long)h[nph],
                (long long)ncap);
    f->chunk_off.assign(h.begin(), h.begin() + nph + 1);
    f->chunk_words = h[nph] > 0 ? h[nph + 1] + 64 : 0;
    if (getenv("HDP_CHUNK_STATS")) {  // diagnostics: chunk weight histogram
        std::vector<ChunkDesc> hd(h[nph]);
        std::vector<int64_t> hw(ns + 1);
        HDP_CHECK_CUDA(cudaMemcpyAsync(hd.data(), f->chunk_desc.get(), sizeof(ChunkDesc) * h[nph],
                                       cudaMemcpyDeviceToHost, st));
        HDP_CHECK_CUDA(cudaMemcpyAsync(hw.data(), W.get(), sizeof(int64_t) * (ns + 1), cudaMemcpyDeviceToHost, st));
        HDP_CHECK_CUDA(cudaStreamSynchronize(st));
        int64_t hist[12] = {0};
        double tot = 0;
        for (const ChunkDesc& d : hd) {
            const int64_t w = hw[d.p0 + d.np] - hw[d.p0];
            tot += (double)w;
            hist[std::min<int64_t>(11, w >> 11)]++;
        }
        fprintf(stderr, "[chunks] %lld chunks, mean %.0f words, max %lld; per 2K words:", (long long)h[nph],
                tot / std::max<int64_t>(1, h[nph]), (long long)h[nph + 1]);
        for (int i = 0; i < 12; i++) fprintf(stderr, " %lld", (long long)hist[i]);
        fprintf(stderr, "\n");
    }
    // rows of up to 32 float4 lanes: one lane group spans a row; wider rows
    // take the per-path kernels (lane groups across CTAs)
    f->chunks_ok = f->chunk_words <= kChunkMaxWords;
    {
        const char* e = getenv("HDP_NO_CHUNKS");  // A/B switch for diagnostics
        if (e && e[0] == '1') f->chunks_ok = 0;
    }
    return HDP_OK;
}

__global__ void k_lane_totals(int64_t n, const int64_t* __restrict__ nodeoff, const int64_t* __restrict__ rowoff,
                              const int32_t* __restrict__ mx, int64_t* out) {
    out[0] = nodeoff[n];
    out[1] = rowoff[n];
    out[2] = mx[0];
}

__global__ void k_seg_desc(int64_t n, const int2* __restrict__ seg_tab, const int4* __restrict__ info,
                           const longlong2* __restrict__ rows, const int32_t* __restrict__ lc_start,
                           SegDesc* out) {
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const int2 t = seg_tab[g];
    const int4 in = info[t.x];
    const longlong2 r = rows[t.x];
    SegDesc d;
    d.mp = (in.z + 3) & ~3;
    d.doff = in.w;
    d.s = t.y;
    d.nseg = (in.y + kSeg - 1) / kSeg;
    d.a = in.x + t.y * kSeg;
    const int b = min(in.x + in.y, d.a + kSeg);
    d.cnt = b - d.a;
    d.rowa = r.x + (long long)(d.a - in.x) * d.mp;
    d.prow = r.y;
    d.e0 = lc_start[d.a];
    d.e1 = lc_start[b];
    out[g] = d;
}

// uniform_m > 0: every tree has exactly that many lanes (totals known here)
static int lanes_finish(hdp_forest* f, int uniform_m) {
    cudaStream_t st = f->st;
    Tracer tr(st);
    const int B = 256;
    const int64_t n = f->n;
    HDP_TRY(f->rowoff.alloc(n + 1, st));
    HDP_TRY(f->nodeoff.alloc(n + 1, st));
    if (uniform_m > 0) {
        // every row is m lanes (padded to mp): the offsets are multiples
        k_uniform_offsets<<<grid_for(n + 1, B), B, 0, st>>>(n, uniform_m, (uniform_m + 3) & ~3, f->rowoff.get(),
                                                            f->nodeoff.get()); note_launch();
    } else {
        DevBuf<int64_t> rm, nm;
        HDP_TRY(rm.alloc(n + 1, st));
        HDP_TRY(nm.alloc(n + 1, st));
        k_row_m<<<grid_for(n + 1, B), B, 0, st>>>(n, f->lnode.get(), f->tree_id.get(), f->t_m.get(),
                                                  rm.get()); note_launch();
        HDP_TRY(exclusive_sum(rm.get(), f->rowoff.get(), n + 1, st));
        HDP_CHECK_CUDA(cudaMemsetAsync(nm.get() + n, 0, sizeof(int64_t), st));
        k_node_m<<<grid_for(n, B), B, 0, st>>>(n, f->tree_id.get(), f->t_m.get(), nm.get()); note_launch();
        HDP_TRY(exclusive_sum(nm.get(), f->nodeoff.get(), n + 1, st));
    }
    HDP_CHECK_LAUNCH();
    if (uniform_m > 0) {
        f->max_m = uniform_m;
        f->total_entries = n * (int64_t)uniform_m;
        f->total_rows = n * (int64_t)((uniform_m + 3) & ~3);
    } else {
        DevBuf<int32_t> mx;
        DevBuf<int64_t> tot;
        HDP_TRY(mx.alloc(1, st));
        HDP_TRY(tot.alloc(3, st));
        HDP_TRY(reduce_max(f->t_m.get(), mx.get(), f->n_trees, st));
        k_lane_totals<<<1, 1, 0, st>>>(n, f->nodeoff.get(), f->rowoff.get(), mx.get(), tot.get()); note_launch();
        int64_t ht[3] = {0, 0, 0};
        HDP_TRY(to_host(ht, tot.get(), 3, st));
        f->total_entries = ht[0];
        f->total_rows = ht[1];
        f->max_m = (int)ht[2];
    }
    // packed metadata for the aggregation kernels
    const int64_t n_lc = f->n_lc;
    HDP_TRY(f->lmeta.alloc(n, st));
    HDP_TRY(f->lsimf.alloc(n, st));
    HDP_TRY(f->lc_row.alloc(n_lc + 1, st));
    HDP_TRY(f->lc_sim.alloc(n_lc + 1, st));
    k_pos_meta<<<grid_for(n, B), B, 0, st>>>(n, f->lnode.get(), f->tree_id.get(), f->t_doff.get(),
                                            f->lsim.get(), f->lc_start.get(), f->t_m.get(),
                                            f->lmeta.get(),
                                            f->lsimf.get()); note_launch();
    if (n_lc > 0)
        k_lc_meta<<<grid_for(n_lc, B), B, 0, st>>>(n_lc, f->lc_list.get(), f->rowoff.get(),
                                                  f->lsim.get(), f->lc_row.get(), f->lc_sim.get()); note_launch();
    int64_t nl = f->long_off[f->n_phases], ns = f->short_off[f->n_phases];
    HDP_TRY(f->long_info.alloc(nl + 1, st));
    HDP_TRY(f->long_rows.alloc(nl + 1, st));
    HDP_TRY(f->short_info.alloc(ns + 1, st));
    HDP_TRY(f->short_rows.alloc(ns + 1, st));
    if (nl > 0)
        k_path_meta<<<grid_for(nl, B), B, 0, st>>>(nl, f->long_paths.get(), f->p_start.get(),
                                                  f->p_len.get(), f->p_par.get(), f->p_tree.get(),
                                                  f->t_doff.get(), f->t_m.get(), f->rowoff.get(),
                                                  f->long_info.get(), f->long_rows.get()); note_launch();
    if (ns > 0)
        k_path_meta<<<grid_for(ns, B), B, 0, st>>>(ns, f->short_paths.get(), f->p_start.get(),
                                                  f->p_len.get(), f->p_par.get(), f->p_tree.get(),
                                                  f->t_doff.get(), f->t_m.get(), f->rowoff.get(),
                                                  f->short_info.get(), f->short_rows.get()); note_launch();
    if (f->n_segs > 0) {
        HDP_TRY(f->seg_desc.alloc(f->n_segs, st));
        k_seg_desc<<<grid_for(f->n_segs, B), B, 0, st>>>(f->n_segs, f->seg_tab.get(), f->long_info.get(),
                                                        f->long_rows.get(), f->lc_start.get(),
                                                        f->seg_desc.get()); note_launch();
    }
    HDP_CHECK_LAUNCH();
    HDP_TRY(build_chunks(f));
    tr.mark("lanes finish");
    f->lanes_set = 1;
    f->geom_w = -1;
    return HDP_OK;
}

namespace hdp {
int forest_create_ex(int64_t n_nodes, int64_t n_edges, const int32_t* eu, const int32_t* ev, const float* ew,
                     const uint8_t* in_tree, const int32_t* comp, float gamma, const EarlyCost* req,
                     hdp_forest** out, void* stream) {
    HDP_REQUIRE(out != nullptr, HDP_ERR_CONFIG, "null output handle");
    HDP_REQUIRE(n_nodes >= 1 && n_nodes < ((int64_t)1 << 31) - 2, HDP_ERR_CONFIG,
                "node count %lld out of range", (long long)n_nodes);
    HDP_REQUIRE(n_edges >= 0 && 2 * n_edges < ((int64_t)1 << 31) - 2, HDP_ERR_CONFIG,
                "edge count %lld out of range", (long long)n_edges);
    HDP_REQUIRE(gamma > 0.0f, HDP_ERR_CONFIG, "gamma must be positive, got %g", (double)gamma);
    hdp_forest* f = new hdp_forest();
    f->st = (cudaStream_t)stream;
    f->n = n_nodes;
    f->gamma = gamma;
    if (req && req->want) {
        EarlyCost& e = f->early;
        e.want = 1;
        e.pl = req->pl; e.pr = req->pr;
        e.h = req->h; e.w = req->w; e.c = req->c; e.x0 = req->x0; e.nx = req->nx;
        e.alpha = req->alpha; e.tau_c = req->tau_c; e.tau_g = req->tau_g;
        e.side = req->side; e.layout_ev = req->layout_ev; e.done_ev = req->done_ev;
    }
    int s = forest_build(f, n_edges, eu, ev, ew, in_tree, comp);
    if (s != HDP_OK) {
        delete f;
        return s;
    }
    *out = f;
    return HDP_OK;
}
}  // namespace hdp

extern "C" {

int hdp_forest_create(int64_t n_nodes, int64_t n_edges, const int32_t* eu, const int32_t* ev,
                      const float* ew, const uint8_t* in_tree, const int32_t* comp, float gamma,
                      hdp_forest** out, void* stream) {
    return hdp::forest_create_ex(n_nodes, n_edges, eu, ev, ew, in_tree, comp, gamma, nullptr, out, stream);
}

int hdp_forest_stats(const hdp_forest* f, int64_t* n_trees, int64_t* n_paths, int64_t* n_phases,
                     int64_t* max_depth) {
    HDP_REQUIRE(f != nullptr, HDP_ERR_CONFIG, "null forest");
    if (n_trees) *n_trees = f->n_trees;
    if (n_paths) *n_paths = f->n_paths;
    if (n_phases) *n_phases = f->n_phases;
    if (max_depth) *max_depth = f->max_depth;
    return HDP_OK;
}

int hdp_forest_export(const hdp_forest* f, int32_t* parent, int32_t* depth, int32_t* tree_id,
                      int32_t* size, float* parent_weight, int32_t* root, void* stream) {
    HDP_REQUIRE(f != nullptr, HDP_ERR_CONFIG, "null forest");
    cudaStream_t st = (cudaStream_t)stream;
    size_t b = f->n * sizeof(int32_t);
    if (parent) HDP_CHECK_CUDA(cudaMemcpyAsync(parent, f->parent.get(), b, cudaMemcpyDeviceToDevice, st));
    if (depth) HDP_CHECK_CUDA(cudaMemcpyAsync(depth, f->depth.get(), b, cudaMemcpyDeviceToDevice, st));
    if (tree_id) HDP_CHECK_CUDA(cudaMemcpyAsync(tree_id, f->tree_id.get(), b, cudaMemcpyDeviceToDevice, st));
    if (size) HDP_CHECK_CUDA(cudaMemcpyAsync(size, f->size.get(), b, cudaMemcpyDeviceToDevice, st));
    if (root) HDP_CHECK_CUDA(cudaMemcpyAsync(root, f->root.get(), b, cudaMemcpyDeviceToDevice, st));
    if (parent_weight)
        HDP_CHECK_CUDA(cudaMemcpyAsync(parent_weight, f->pweight.get(), f->n * sizeof(float),
                                       cudaMemcpyDeviceToDevice, st));
    return HDP_OK;
}

int hdp_forest_set_lanes_nodes(hdp_forest* f, const uint32_t* node_masks, int nw, void* stream) {
    HDP_REQUIRE(f != nullptr, HDP_ERR_CONFIG, "null forest");
    HDP_REQUIRE(nw >= 1, HDP_ERR_CONFIG, "mask width must be >= 1 word");
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf<uint32_t> tm;
    HDP_TRY(tm.alloc((size_t)f->n_trees * nw + 1, st));
    k_tree_masks<<<grid_for(f->n, 256), 256, 0, st>>>(f->n, f->root.get(), f->tree_id.get(), node_masks, nw,
                                                      tm.get()); note_launch();
    return hdp_forest_set_lanes(f, tm.get(), nw, stream);
}

int hdp_forest_set_lanes_range(hdp_forest* f, int x0, int nx, void* stream) {
    HDP_REQUIRE(f != nullptr, HDP_ERR_CONFIG, "null forest");
    HDP_REQUIRE(nx >= 1 && x0 >= 0, HDP_ERR_CONFIG, "empty disparity range");
    f->st = (cudaStream_t)stream;
    cudaStream_t st = f->st;
    HDP_TRY(f->t_m.alloc(f->n_trees, st));
    HDP_TRY(f->t_doff.alloc(f->n_trees, st));
    HDP_TRY(f->dlist.alloc(nx, st));
    k_lanes_range<<<grid_for(f->n_trees, 256), 256, 0, st>>>(f->n_trees, nx, f->t_m.get(),
                                                             f->t_doff.get()); note_launch();
    k_iota<<<grid_for(nx, 256), 256, 0, st>>>(nx, f->dlist.get(), x0); note_launch();
    HDP_CHECK_LAUNCH();
    f->range_x0 = x0;
    f->max_d = x0 + nx - 1;
    return lanes_finish(f, nx);
}

int hdp_forest_set_lanes(hdp_forest* f, const uint32_t* tree_masks, int nw, void* stream) {
    HDP_REQUIRE(f != nullptr, HDP_ERR_CONFIG, "null forest");
    HDP_REQUIRE(nw >= 1, HDP_ERR_CONFIG, "mask width must be >= 1 word");
    f->st = (cudaStream_t)stream;
    cudaStream_t st = f->st;
    f->range_x0 = -1;
    f->max_d = 32 * nw - 1;
    HDP_TRY(f->t_m.alloc(f->n_trees, st));
    HDP_TRY(f->t_doff.alloc(f->n_trees + 1, st));
    DevBuf<int32_t> mn;  // (min lanes, last offset, last count)
    HDP_TRY(mn.alloc(3, st));
    const int32_t big = 0x7fffffff;
    HDP_CHECK_CUDA(cudaMemcpyAsync(mn.get(), &big, sizeof(int32_t), cudaMemcpyHostToDevice, st));
    k_lanes_count<<<grid_for(f->n_trees, 256), 256, 0, st>>>(f->n_trees, tree_masks, nw, f->t_m.get(), mn.get());
    note_launch();
    HDP_TRY(exclusive_sum(f->t_m.get(), f->t_doff.get(), f->n_trees, st));
    // one host read for the list size and the empty-interval check
    HDP_CHECK_CUDA(cudaMemcpyAsync(mn.get() + 1, f->t_doff.get() + f->n_trees - 1, sizeof(int32_t),
                                   cudaMemcpyDeviceToDevice, st));
    HDP_CHECK_CUDA(cudaMemcpyAsync(mn.get() + 2, f->t_m.get() + f->n_trees - 1, sizeof(int32_t),
                                   cudaMemcpyDeviceToDevice, st));
    int32_t h[3] = {0, 0, 0};
    HDP_TRY(to_host(h, mn.get(), 3, st));
    HDP_REQUIRE(h[0] >= 1, HDP_ERR_INTERNAL, "a tree has an empty disparity interval");
    HDP_TRY(f->dlist.alloc((size_t)h[1] + h[2] + 1, st));
    k_lanes_fill<<<grid_for(f->n_trees, 256), 256, 0, st>>>(f->n_trees, tree_masks, nw,
                                                            f->t_doff.get(), f->dlist.get()); note_launch();
    HDP_CHECK_LAUNCH();
    return lanes_finish(f, 0);
}

int hdp_forest_entries(hdp_forest* f, int64_t* total, int64_t* node_offsets, void* stream) {
    HDP_REQUIRE(f != nullptr && f->lanes_set, HDP_ERR_CONFIG, "forest lanes not set");
    if (total) *total = f->total_entries;
    if (node_offsets)
        HDP_CHECK_CUDA(cudaMemcpyAsync(node_offsets, f->nodeoff.get(), f->n * sizeof(int64_t),
                                       cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return HDP_OK;
}

void hdp_forest_destroy(hdp_forest* f) { delete f; }

}  // extern "C"

namespace hdp {
// per pair b: trees = tree_id of its first node .. next pair's first node;
// stored entries = node offsets over the pair's node range
__global__ void k_pair_stats(int batch, int64_t npp, int64_t n, int64_t n_trees, int64_t total,
                             const int32_t* __restrict__ tree_id,
                             const int64_t* __restrict__ nodeoff, int64_t* out) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    int64_t v0 = (int64_t)b * npp, v1 = v0 + npp;
    int64_t t0 = tree_id[v0], t1 = v1 < n ? tree_id[v1] : n_trees;
    int64_t e0 = nodeoff[v0], e1 = v1 < n ? nodeoff[v1] : total;
    out[b] = t1 - t0;
    out[batch + b] = e1 - e0;
}
}  // namespace hdp

extern "C" int hdp_forest_pair_stats_device(const hdp_forest* f, int batch, int64_t nodes_per_pair, int64_t* out,
                                            void* stream) {
    HDP_REQUIRE(f != nullptr && f->lanes_set, HDP_ERR_CONFIG, "forest lanes not set");
    HDP_REQUIRE(batch >= 1 && (int64_t)batch * nodes_per_pair == f->n, HDP_ERR_CONFIG,
                "batch x nodes_per_pair must equal the node count");
    k_pair_stats<<<grid_for(batch, 128), 128, 0, (cudaStream_t)stream>>>(batch, nodes_per_pair, f->n, f->n_trees,
                                                                        f->total_entries, f->tree_id.get(),
                                                                        f->nodeoff.get(), out); note_launch();
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

extern "C" int hdp_forest_pair_stats(const hdp_forest* f, int batch, int64_t nodes_per_pair,
                                     int64_t* n_trees, int64_t* stored, void* stream) {
    HDP_REQUIRE(f != nullptr && f->lanes_set, HDP_ERR_CONFIG, "forest lanes not set");
    HDP_REQUIRE(batch >= 1 && (int64_t)batch * nodes_per_pair == f->n, HDP_ERR_CONFIG,
                "batch x nodes_per_pair must equal the node count");
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf<int64_t> out;
    HDP_TRY(out.alloc(2 * batch, st));
    k_pair_stats<<<grid_for(batch, 128), 128, 0, st>>>(batch, nodes_per_pair, f->n, f->n_trees,
                                                       f->total_entries, f->tree_id.get(),
                                                       f->nodeoff.get(), out.get()); note_launch();
    HDP_CHECK_LAUNCH();
    std::vector<int64_t> h(2 * batch);
    HDP_TRY(to_host(h.data(), out.get(), 2 * batch, st));
    for (int b = 0; b < batch; b++) {
        if (n_trees) n_trees[b] = h[b];
        if (stored) stored[b] = h[batch + b];
    }
    return HDP_OK;
}
