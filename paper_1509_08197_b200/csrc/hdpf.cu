// Disparity-tree forest (HDPF) build, exact with the reference's sequential
// Kruskal-with-rules (hdp_forest.py:151-216), and the segment-tree variant.
//
// Rule 1 (pixel sets disjoint -> drop) is a static per-edge filter; the
// survivors are sorted per pair by the Kruskal key (weight, scan index).
// Rule 2 compares the LIVE tree sets of the two components at the moment the
// edge is reached, so the result depends on the order of merges; in general a
// plain connected-components / Boruvka formulation is not equivalent.  It is
// when no edge is "cross-pass" (k_hdpf_classify): then every tree keeps one
// pixel mask and the forest is the MSF of the equal-mask edges -- the fast
// path hdpf_run takes after one flag read.  The general kernel, k_grp,
// decides whole windows of 1023 edges per round, one CTA per
// pair: the window's live edges and the roots they touch form conflict groups
// (components in shared memory); groups touch disjoint trees, so each is
// walked independently by one thread in Kruskal order against shared-memory
// copies of its trees; merges are written back to the global union-find.
// k_grp<true> adds the segment-tree criterion w <= min(Int(A) + k/|A|,
// Int(B) + k/|B|) (hdp_segment_tree, tree kind "st").
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "prims.cuh"

namespace hdp {

int run_boruvka(int64_t n, int64_t m, const int32_t* eu, const int32_t* ev, const uint64_t* key,
                uint8_t* in_tree, int32_t* comp, int* rounds_out, cudaStream_t st, int grid_h, int grid_w);

__device__ __forceinline__ const uint32_t* pix_mask(const uint32_t* row_masks,
                                                   const int32_t* pixel_row, int32_t node,
                                                   int64_t npp, int n_rows, int nw) {
    int64_t b = node / npp;
    return row_masks + ((int64_t)b * n_rows + pixel_row[node]) * nw;
}

__global__ void k_rule1(int64_t m, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                        const uint64_t* __restrict__ key, const int32_t* __restrict__ pixel_row,
                        const uint32_t* __restrict__ row_masks, int64_t npp, int64_t epp,
                        int n_rows, int nw, int32_t* flag, uint64_t* skey, const int32_t* __restrict__ keep_v2,
                        int32_t* nonstd) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    int32_t a = eu[e], b = ev[e];
    bool meet = false;
    if (keep_v2) {  // mask-homogeneous: only the equal-mask edges can ever merge
        meet = keep_v2[e] != a;
    } else {
        const uint32_t* ma = pix_mask(row_masks, pixel_row, a, npp, n_rows, nw);
        const uint32_t* mb = pix_mask(row_masks, pixel_row, b, npp, n_rows, nw);
        for (int i = 0; i < nw; i++) meet |= (ma[i] & mb[i]) != 0;
    }
    flag[e] = meet ? 1 : 0;
    uint64_t k = key[e];
    uint64_t pair = (uint64_t)(e / epp);
    // keys whose low 24 bits are the edge's index in its pair (hdp_grid_edges,
    // rank keys) let the sort skip those bits: it is stable and its input is
    // in edge order
    if ((k & 0xffffffull) != (uint64_t)(e - (int64_t)pair * epp)) *nonstd = 1;
    // (pair, weight bits, scan index): weights are non-negative floats < 2^31
    skey[e] = (pair << 55) | ((k >> 32) << 24) | (k & 0xffffffull);
}

__global__ void k_select(int64_t m, const int32_t* __restrict__ flag,
                         const int32_t* __restrict__ pos, const uint64_t* __restrict__ skey,
                         uint64_t* okey, int32_t* oidx) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m || !flag[e]) return;
    okey[pos[e]] = skey[e];
    oidx[pos[e]] = (int32_t)e;
}

__global__ void k_seg_bounds(int64_t ms, const uint64_t* __restrict__ skey, int batch,
                             int32_t* seg) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > ms) return;
    int pb = (i == 0) ? -1 : (int)(skey[i - 1] >> 55);
    int pc = (i == ms) ? batch : (int)(skey[i] >> 55);
    for (int b = pb + 1; b <= pc; b++) seg[b] = (int32_t)i;
}

__global__ void k_uf_init(int64_t n, const int32_t* __restrict__ pixel_row,
                          const uint32_t* __restrict__ row_masks, int64_t npp, int n_rows, int nw,
                          int32_t* uf, int32_t* usz, uint32_t* tm) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    uf[v] = (int32_t)v;
    usz[v] = 1;
    const uint32_t* pm = pix_mask(row_masks, pixel_row, (int32_t)v, npp, n_rows, nw);
    for (int i = 0; i < nw; i++) tm[v * nw + i] = pm[i];
}

__device__ __forceinline__ int32_t uf_find(int32_t* uf, int32_t x) {
    while (true) {
        int32_t p = uf[x];
        if (p == x) return x;
        int32_t gp = uf[p];
        if (gp != p) uf[x] = gp;  // path halving (stores an ancestor: race-safe)
        x = gp;
    }
}

constexpr int DR_NW = 8;         // mask words per root staged in shared memory (d_max < 256)

// ---- whole-window rounds by conflict groups -------------------------------
//
// One CTA per stereo pair decides the NEXT GW edges of its sorted list in one
// round.  The window's live edges and the distinct roots they touch form a
// graph; its connected components ("groups") touch disjoint trees, so their
// sequential outcomes are independent.  Each group is walked by one thread in
// Kruskal order against shared-memory copies of its trees (local union-find,
// sizes, masks) -- exactly the reference's loop (hdp_forest.py:185-203)
// restricted to that group -- and the merges are written back to the global
// union-find.  Every round decides the whole window, so rounds = edges / GW.
constexpr int GW = 1024;          // window edges per round (= threads)
constexpr int GSLOTS = 2 * GW;    // distinct roots a window can touch
constexpr int GHASH = 4096;       // open-addressing table root -> slot

struct GrpSmem {
    int32_t e[GW], la[GW], lb[GW];    // per window position: edge, root slots
    int32_t ord[GW], grp[GW];         // next position of the same group (window order); group of each
    int32_t hkey[GHASH], hslot[GHASH];
    int32_t sroot[GSLOTS], gp[GSLOTS], mp[GSLOTS], sz[GSLOTS];
    uint32_t mask[GSLOTS * DR_NW];
    float wt[GW];                     // segment tree: window edge weights
    float sint[GSLOTS];               // segment tree: Int(T) of the slots' trees
    uint8_t dirty[GSLOTS];
    int nslots, changed;
};

__device__ __forceinline__ int grp_hash(int32_t k) {
    return (int)(((uint32_t)k * 2654435761u) >> 16) & (GHASH - 1);
}

__device__ __forceinline__ void grp_insert(GrpSmem& s, int32_t k) {
    int h = grp_hash(k);
    while (true) {
        const int32_t cur = atomicCAS(&s.hkey[h], -1, k);
        if (cur == -1 || cur == k) return;
        h = (h + 1) & (GHASH - 1);
    }
}

__device__ __forceinline__ int grp_lookup(const GrpSmem& s, int32_t k) {
    int h = grp_hash(k);
    while (s.hkey[h] != k) h = (h + 1) & (GHASH - 1);
    return s.hslot[h];
}

__device__ __forceinline__ int grp_find(int32_t* p, int x) {
    while (p[x] != x) {
        const int g = p[p[x]];
        p[x] = g;  // path halving: stores an ancestor (race-safe)
        x = g;
    }
    return x;
}

// read-only find for the sequential walk: no path-halving stores, so the two
// finds of an edge are independent loads (union by size keeps paths short)
__device__ __forceinline__ int grp_find_ro(const int32_t* p, int x) {
    int y = p[x];
    while (y != x) {
        x = y;
        y = p[x];
    }
    return x;
}

// FH (segment-tree pass 1): an edge that passes the rules merges two trees
// only when w <= min(Int(Ta) + k/|Ta|, Int(Tb) + k/|Tb|) (IEEE double, as
// oracle/hdp_oracle.c or_hdpf_st); Int(T) = the largest edge inside T, kept
// per root in `tint`.
// MASKS = false: every tree keeps a single set that never changes (the
// mask-homogeneous case, where the caller has already dropped every edge the
// rules reject; or one interval row for all pixels): no sets are staged,
// compared or merged.
constexpr int kFhDivTab = 256;  // fh_k / s for sizes below this, from a table
#ifndef HDP_GRP_MINB
#define HDP_GRP_MINB 1
#endif

template <bool FH, bool MASKS>
__global__ void __launch_bounds__(GW, HDP_GRP_MINB) k_grp(const int32_t* __restrict__ seg, const int32_t* __restrict__ order,
                                            const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                                            int32_t* uf, int32_t* usz, uint32_t* tm, int nw, double beta,
                                            uint8_t* in_tree, int* rounds_out, const float* __restrict__ ew,
                                            float* tint, double fh_k) {
    extern __shared__ unsigned long long g_dyn[];
    GrpSmem& s = *reinterpret_cast<GrpSmem*>(g_dyn);
    // rule 2 as an exact integer test: merge iff inter >= thr[uni], where thr[u]
    // is the least i with !(RN(i / u) < beta) (RN(i / u) is monotone in i)
    __shared__ int16_t thr[8 * 32 + 1];
    __shared__ double kdiv[FH ? kFhDivTab : 1];  // FH: RN(fh_k / s), the oracle's division
    const int b = blockIdx.x, tid = threadIdx.x;
    if (MASKS)
        for (int u = tid; u <= 32 * nw; u += GW) {
            int i = 0;
            if (u > 0)
                while (i <= u && __ddiv_rn((double)i, (double)u) < beta) i++;
            thr[u] = (int16_t)i;
        }
    if (FH)
        for (int i = tid; i < kFhDivTab; i += GW) kdiv[i] = i > 0 ? __ddiv_rn(fh_k, (double)i) : 0.0;
    auto fh_tau = [&](int sz) -> double { return sz < kFhDivTab ? kdiv[sz] : __ddiv_rn(fh_k, (double)sz); };
    int32_t head = seg[b];
    const int32_t end = seg[b + 1];
    int round = 0;
#ifdef HDP_DR_PROFILE
    long long g_ph[7] = {0, 0, 0, 0, 0, 0, 0}, g_t0 = clock64(), g_t1;
    int g_maxrun = 0;
#define G_TICK(k) do { __syncthreads(); g_t1 = clock64(); g_ph[k] += g_t1 - g_t0; g_t0 = g_t1; } while (0)
#else
#define G_TICK(k) do { } while (0)
#endif
    while (head < end) {
        const int w = min(GW - 1, end - head);
        // 1. roots of the window's edges
        for (int i = tid; i < GHASH; i += GW) s.hkey[i] = -1;
        if (tid == 0) s.nslots = 0;
        int32_t e = -1, ra = 0, rb = 0;
        bool live = false;
        if (tid < w) {
            e = order[head + tid];
            ra = uf_find(uf, eu[e]);
            rb = uf_find(uf, ev[e]);
            live = ra != rb;  // a cycle: rejected at once (hdp_forest.py:190-191)
        }
        __syncthreads();
        G_TICK(0);
        {
            // one insert per distinct root per warp (the largest tree's root is
            // touched by a large share of the window)
            const unsigned pa = __match_any_sync(0xffffffffu, live ? ra : -1);
            const unsigned pb = __match_any_sync(0xffffffffu, live ? rb : -1);
            const int lane = tid & 31;
            if (live && __ffs(pa) - 1 == lane) grp_insert(s, ra);
            if (live && __ffs(pb) - 1 == lane) grp_insert(s, rb);
        }
        __syncthreads();
        // 2. a slot per distinct root, holding the tree's current size and mask
        for (int h0 = 0; h0 < GHASH; h0 += GW) {
            const int h = h0 + tid;
            const int32_t k = s.hkey[h];
            // one atomic per warp for the slot numbers
            const unsigned occ = __ballot_sync(0xffffffffu, k >= 0);
            int base = 0;
            if ((tid & 31) == 0 && occ) base = atomicAdd(&s.nslots, __popc(occ));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (k >= 0) {
                const int sl = base + __popc(occ & ((1u << (tid & 31)) - 1u));
                s.hslot[h] = sl;
                s.sroot[sl] = k;
            }
        }
        __syncthreads();
        // the slots' tree state, every global load of the round issued together
        for (int sl = tid; sl < s.nslots; sl += GW) {
            const int32_t k = s.sroot[sl];
            s.gp[sl] = sl;
            s.mp[sl] = sl;
            s.dirty[sl] = 0;
            s.sz[sl] = usz[k];
            if (FH) s.sint[sl] = tint[k];
            if (MASKS)
                for (int i = 0; i < nw; i++) s.mask[sl * DR_NW + i] = tm[(int64_t)k * nw + i];
        }
        __syncthreads();
        int la = 0, lb = 0;
        if (live) {
            la = grp_lookup(s, ra);
            lb = grp_lookup(s, rb);
        }
        s.e[tid] = e;
        s.la[tid] = la;
        s.lb[tid] = lb;
        if (FH) s.wt[tid] = live ? ew[e] : 0.0f;
        G_TICK(1);
        // 3. groups = connected components of (slots, live edges)
        while (true) {
            if (tid == 0) s.changed = 0;
            __syncthreads();
            if (live) {
                const int ga = grp_find(s.gp, la), gb = grp_find(s.gp, lb);
                if (ga != gb) {
                    atomicMin(&s.gp[max(ga, gb)], min(ga, gb));
                    s.changed = 1;
                }
            }
            __syncthreads();
            if (!s.changed) break;
            __syncthreads();
        }
        G_TICK(2);
        // 4. per-group lists in window (Kruskal) order: ord[i] = the next window
        // position of i's group (-1 at the end).  Inside a warp the next
        // occurrence is the next higher peer lane; from a warp's last occurrence
        // the list continues in the next warp holding the group (a per-group
        // warp bitmask), at that warp's first lane of the group.  The group's
        // first occurrence walks it (no sort).
        uint32_t* wm = reinterpret_cast<uint32_t*>(s.hslot);  // the hash slots are no longer read
        for (int i = tid; i < GSLOTS; i += GW) wm[i] = 0u;
        const int g = live ? grp_find(s.gp, la) : -1;
        s.grp[tid] = g;
        __syncthreads();
        const int lane = tid & 31, warp = tid >> 5;
        const unsigned peers = __match_any_sync(0xffffffffu, g);
        const bool lowest = __ffs(peers) - 1 == lane;
        if (g >= 0 && lowest) atomicOr(&wm[g], 1u << warp);
        __syncthreads();
        bool walker = false;
        if (g >= 0) {
            const unsigned higher = peers & ~((2u << lane) - 1u);
            int nx = -1;
            const uint32_t m = wm[g];
            if (higher) {
                nx = warp * 32 + __ffs(higher) - 1;
            } else {
                const uint32_t later = warp == 31 ? 0u : (m & ~((2u << warp) - 1u));
                if (later) {
                    const int w2 = __ffs(later) - 1;
                    int j = 0;
                    while (s.grp[w2 * 32 + j] != g) j++;
                    nx = w2 * 32 + j;
                }
            }
            s.ord[tid] = nx;
            walker = lowest && warp == __ffs(m) - 1;
        }
        __syncthreads();
        G_TICK(3);
        // 5. the first occurrence of every group walks its list
        if (walker) {
            {
            int n_g = 0;
            // the next edge's indices are fetched while this one is decided
            int pos_n = tid;
            int la_n = s.la[pos_n], lb_n = s.lb[pos_n];
            // register copy of the last surviving root (runs mostly grow one
            // tree): its size and mask are read from / flushed to shared
            // memory only when the cached root changes
            int cr = -1, csz = 0;
            float ci = 0.0f;  // FH: Int of the cached root
            double ctx = 0.0;  // FH: its threshold Int + k / size
            uint32_t cm[DR_NW];
            while (pos_n >= 0) {
                n_g++;
                const int pos = pos_n, la_q = la_n, lb_q = lb_n;
                pos_n = s.ord[pos];
                if (pos_n >= 0) {
                    la_n = s.la[pos_n];
                    lb_n = s.lb[pos_n];
                }
                int x = grp_find_ro(s.mp, la_q), y = grp_find_ro(s.mp, lb_q);
                if (x == y) continue;  // joined earlier in this window: a cycle
                if (y == cr) {  // keep the cached root in x
                    y = x;
                    x = cr;
                }
                if (x != cr) {  // switch the cache to x
                    if (cr >= 0) {
                        s.sz[cr] = csz;
                        if (FH) s.sint[cr] = ci;
                        if (MASKS)
                            for (int i = 0; i < nw; i++) s.mask[cr * DR_NW + i] = cm[i];
                    }
                    cr = x;
                    csz = s.sz[x];
                    if (FH) {
                        ci = s.sint[x];
                        ctx = (double)ci + fh_tau(csz);
                    }
                    if (MASKS) {
#pragma unroll
                        for (int i = 0; i < DR_NW; i++) cm[i] = i < nw ? s.mask[x * DR_NW + i] : 0u;
                    }
                }
                uint32_t my[DR_NW];
                if (MASKS) {
                    int inter = 0, uni = 0;
#pragma unroll
                    for (int i = 0; i < DR_NW; i++) {
                        my[i] = i < nw ? s.mask[y * DR_NW + i] : 0u;
                        inter += __popc(cm[i] & my[i]);
                        uni += __popc(cm[i] | my[i]);
                    }
                    // rule 2 (hdp_forest.py:195) through the exact threshold table
                    if (inter < thr[uni]) continue;
                }
                const int ysz = s.sz[y];
                float nint = 0.0f;
                if (FH) {
                    const float wv = s.wt[pos];
                    const float iy = s.sint[y];
                    const double tx = ctx;  // (double)Int(x) + k / |x|, cached with the root
                    const double ty = (double)iy + fh_tau(ysz);
                    if (!((double)wv <= (tx < ty ? tx : ty))) continue;
                    const float mi = ci > iy ? ci : iy;
                    nint = wv > mi ? wv : mi;
                }
                s.dirty[x] = 1;
                s.dirty[y] = 1;
                in_tree[s.e[pos]] = 1;
                if (csz < ysz) {  // union by size, as dr_union: y survives
                    s.mp[x] = y;
                    s.sz[y] = csz + ysz;
                    if (FH) s.sint[y] = nint;
                    if (MASKS) {
#pragma unroll
                        for (int i = 0; i < DR_NW; i++)
                            if (i < nw) s.mask[y * DR_NW + i] = cm[i] | my[i];
                    }
                    cr = -1;  // x is absorbed: its cached state is not needed any more
                } else {
                    s.mp[y] = x;
                    csz += ysz;
                    if (FH) {
                        ci = nint;
                        ctx = (double)ci + fh_tau(csz);
                    }
                    if (MASKS) {
#pragma unroll
                        for (int i = 0; i < DR_NW; i++) cm[i] |= my[i];
                    }
                }
            }
            if (cr >= 0) {
                s.sz[cr] = csz;
                if (FH) s.sint[cr] = ci;
                if (MASKS)
                    for (int i = 0; i < nw; i++) s.mask[cr * DR_NW + i] = cm[i];
            }
#ifdef HDP_DR_PROFILE
            if (n_g > g_maxrun) g_maxrun = n_g;
#endif
            }
        }
        __syncthreads();
        G_TICK(4);
        // 6. write the merged trees back
        for (int sl = tid; sl < s.nslots; sl += GW) {
            if (!s.dirty[sl]) continue;
            const int r = grp_find(s.mp, sl);
            const int32_t k = s.sroot[sl];
            if (r != sl) {
                uf[k] = s.sroot[r];
            } else {
                usz[k] = s.sz[sl];
                if (FH) tint[k] = s.sint[sl];
                if (MASKS)
                    for (int i = 0; i < nw; i++) tm[(int64_t)k * nw + i] = s.mask[sl * DR_NW + i];
            }
        }
        __syncthreads();
        G_TICK(5);
        head += w;
        round++;
    }
    if (tid == 0) atomicMax(rounds_out, round);
#ifdef HDP_DR_PROFILE
    g_maxrun = __reduce_max_sync(0xffffffffu, g_maxrun);
    __shared__ int s_mr;
    if (tid == 0) s_mr = 0;
    __syncthreads();
    if ((tid & 31) == 0) atomicMax(&s_mr, g_maxrun);
    __syncthreads();
    if (tid == 0 && b == 0)
        printf("[grp] rounds %d cyc/round roots %.0f slots %.0f cc %.0f sort %.0f walk %.0f wb %.0f  max run %d\n",
               round, (double)g_ph[0] / round, (double)g_ph[1] / round, (double)g_ph[2] / round,
               (double)g_ph[3] / round, (double)g_ph[4] / round, (double)g_ph[5] / round, s_mr);
#endif
}

// segment-tree pass 2: keep the sorted edges whose endpoints are still in
// different trees after pass 1 (an edge inside a tree stays inside: trees
// only grow), order preserved
__global__ void k_live_edges(int64_t ms, const int32_t* __restrict__ order, const int32_t* __restrict__ eu,
                             const int32_t* __restrict__ ev, int32_t* uf, int32_t* flag) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ms) return;
    const int32_t e = order[i];
    flag[i] = uf_find(uf, eu[e]) != uf_find(uf, ev[e]) ? 1 : 0;
}

__global__ void k_compact_order(int64_t ms, const int32_t* __restrict__ order, const int32_t* __restrict__ flag,
                                const int32_t* __restrict__ pos, int32_t* out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < ms && flag[i]) out[pos[i]] = order[i];
}

__global__ void k_seg_remap(int batch, int64_t ms, const int32_t* __restrict__ seg, const int32_t* __restrict__ flag,
                            const int32_t* __restrict__ pos, int32_t* seg2) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > batch) return;
    const int32_t s0 = seg[b];
    seg2[b] = s0 < ms ? pos[s0] : (ms > 0 ? pos[ms - 1] + flag[ms - 1] : 0);
}

// Static classification for the mask-homogeneous fast path (hdpf_run).
// While every tree's set equals the pixel mask of each of its members, an
// edge reached between two trees is accepted iff the endpoints' masks are
// equal and non-empty (Jaccard 1 >= beta), and rejected otherwise -- unless
// the masks differ, intersect and still pass rule 2 (inter / union >= beta,
// the reference's float64 test): only such a "cross-pass" edge could ever
// merge two different sets.  With no cross-pass edge in a pair, induction over
// the Kruskal sequence keeps every tree homogeneous, so build_hdpf
// (hdp_forest.py:185-201) accepts exactly the edges plain Kruskal accepts on
// the equal-mask subgraph: its unique minimum spanning forest under the
// (weight, index) keys.  Edges outside that subgraph become self-loops (u, u),
// which Boruvka drops.
__global__ void k_hdpf_classify(int64_t m, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                                const int32_t* __restrict__ pixel_row, const uint32_t* __restrict__ row_masks,
                                int64_t npp, int64_t epp, int n_rows, int nw, double beta, int32_t* u2,
                                int32_t* v2, int* cross) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    const int32_t a = eu[e], b = ev[e];
    const int ra = pixel_row[a], rb = pixel_row[b];
    const int64_t pair = e / epp;
    const uint32_t* ma = row_masks + (pair * n_rows + ra) * nw;
    const uint32_t* mb = row_masks + (pair * n_rows + rb) * nw;
    bool eq = true;
    int inter = 0, uni = 0;
    for (int i = 0; i < nw; i++) {
        const uint32_t x = __ldg(ma + i), y = ra == rb ? x : __ldg(mb + i);
        eq = eq && x == y;
        inter += __popc(x & y);
        uni += __popc(x | y);
    }
    const bool keep = eq && inter > 0;
    if (!eq && inter > 0 && !(__ddiv_rn((double)inter, (double)uni) < beta)) atomicOr(cross + pair, 1);
    u2[e] = a;
    v2[e] = keep ? b : a;
}

// segment-tree pass 2 (homogeneous): an equal-mask edge (u2 != v2 after
// k_hdpf_classify) joins the pass-1 roots of its endpoints
__global__ void k_hdpf_relabel_roots(int64_t m, int32_t* uf, int32_t* u2, int32_t* v2) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    const int32_t a = u2[e], b = v2[e];
    if (a == b) return;
    const int32_t ra = uf_find(uf, a), rb = uf_find(uf, b);
    u2[e] = ra;
    v2[e] = ra == rb ? ra : rb;
}

__global__ void k_hdpf_link_final(int64_t m, int64_t n, const uint8_t* __restrict__ t2, uint8_t* in_tree,
                                  int32_t* uf, const int32_t* __restrict__ c2, int32_t* comp) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m && t2[i]) in_tree[i] = 1;
    if (i < n) comp[i] = c2[uf_find(uf, (int32_t)i)];
}

// tree sets of the homogeneous forest: every node's own pixel mask
__global__ void k_hdpf_node_masks(int64_t n, const int32_t* __restrict__ pixel_row,
                                  const uint32_t* __restrict__ row_masks, int64_t npp, int n_rows, int nw,
                                  uint32_t* tree_masks) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const uint32_t* pm = pix_mask(row_masks, pixel_row, (int32_t)v, npp, n_rows, nw);
    for (int i = 0; i < nw; i++) tree_masks[v * nw + i] = pm[i];
}

__global__ void k_uf_final(int64_t n, int32_t* uf, int nw, const uint32_t* __restrict__ tm,
                           int32_t* comp, uint32_t* tree_masks) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    int32_t r = (int32_t)v;
    while (uf[r] != r) r = uf[r];
    comp[v] = r;
    for (int i = 0; i < nw; i++) tree_masks[v * nw + i] = tm[(int64_t)r * nw + i];
}

}  // namespace hdp

using namespace hdp;

// build_hdpf on the device (see hdp_hdpf in the header).  st_k >= 0: the
// segment-tree variant, pass 1 with the FH criterion, then (link) pass 2 over
// the same sorted edges with the rules alone.
// One slice of at most kHdpfSlice pairs (edges [e0, e0 + nb * epp)): rule 1,
// the per-pair Kruskal sort, and the window rounds on the batch-wide
// union-find state (node ids are global over the batch).
constexpr int kHdpfSlice = 255;  // pairs per k_grp launch (9 pair bits in the sort key)

static int hdpf_slice(int nb, int64_t nodes_per_pair, int64_t edges_per_pair, const int32_t* eu, const int32_t* ev,
                      const uint64_t* key, const int32_t* pixel_row, const uint32_t* row_masks, int n_rows, int nw,
                      double beta, const float* ew, double st_k, bool link, uint8_t* in_tree, int32_t* uf,
                      int32_t* usz, uint32_t* tm, float* tint, int* rounds,
                      const int32_t* keep_v2, cudaStream_t st) {
    // no set ever changes: one interval row, or homogeneous trees over the
    // equal-mask edges (keep_v2)
    const bool masks = !(keep_v2 || n_rows == 1);
    bool std_keys = false;
    const int64_t m = (int64_t)nb * edges_per_pair;
    const int B = 256;
    DevBuf<int32_t> flag, pos, oidx, oidx2, seg, nonstd;
    DevBuf<uint64_t> skey, okey, okey2;
    HDP_TRY(nonstd.alloc(1, st));
    HDP_CHECK_CUDA(cudaMemsetAsync(nonstd.get(), 0, sizeof(int32_t), st));
    HDP_TRY(flag.alloc(m + 1, st));
    HDP_TRY(pos.alloc(m + 1, st));
    HDP_TRY(skey.alloc(m + 1, st));
    int64_t ms = 0;
    if (m > 0) {
        k_rule1<<<grid_for(m, B), B, 0, st>>>(m, eu, ev, key, pixel_row, row_masks, nodes_per_pair,
                                              edges_per_pair, n_rows, nw, flag.get(), skey.get(), keep_v2,
                                              nonstd.get());
        note_launch();
        HDP_TRY(exclusive_sum(flag.get(), pos.get(), m, st));
        int32_t a = 0, b2 = 0, ns = 0;
        HDP_CHECK_CUDA(cudaMemcpyAsync(&a, pos.get() + m - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        HDP_CHECK_CUDA(cudaMemcpyAsync(&b2, flag.get() + m - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        HDP_CHECK_CUDA(cudaMemcpyAsync(&ns, nonstd.get(), sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        HDP_CHECK_CUDA(cudaStreamSynchronize(st));
        ms = (int64_t)a + b2;
        std_keys = ns == 0;
    }
    HDP_TRY(okey.alloc(ms + 1, st));
    HDP_TRY(okey2.alloc(ms + 1, st));
    HDP_TRY(oidx.alloc(ms + 1, st));
    HDP_TRY(oidx2.alloc(ms + 1, st));
    HDP_TRY(seg.alloc(nb + 1, st));
    if (m > 0)
        k_select<<<grid_for(m, B), B, 0, st>>>(m, flag.get(), pos.get(), skey.get(), okey.get(),
                                               oidx.get()); note_launch();
    flag.release();
    pos.release();
    skey.release();
    {
        // (pair, weight, index) keys: with standard keys the index bits are
        // implied by the (stable) sort's input order, and only the pair bits
        // the slice uses are sorted
        int pb = 0;
        while ((1 << pb) < nb) pb++;
        HDP_TRY(sort_pairs(okey.get(), okey2.get(), oidx.get(), oidx2.get(), ms, std_keys ? 24 : 0, 55 + pb, st));
    }
    k_seg_bounds<<<grid_for(ms + 1, B), B, 0, st>>>(ms, okey2.get(), nb, seg.get()); note_launch();
    HDP_CHECK_LAUNCH();
    constexpr size_t g_smem = sizeof(GrpSmem);
    if (st_k >= 0.0) {
        auto kern = masks ? k_grp<true, true> : k_grp<true, false>;
        HDP_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g_smem));
        kern<<<nb, GW, g_smem, st>>>(seg.get(), oidx2.get(), eu, ev, uf, usz, tm, nw, beta, in_tree, rounds, ew, tint,
                                     st_k); note_launch();
    }
    const int32_t* order2 = oidx2.get();
    const int32_t* seg2p = seg.get();
    DevBuf<int32_t> lflag, lpos, oidx3, seg2;
    if (st_k >= 0.0 && link && ms > 0) {
        // pass 2 walks only the edges still between two trees
        HDP_TRY(lflag.alloc(ms + 1, st));
        HDP_TRY(lpos.alloc(ms + 1, st));
        HDP_TRY(oidx3.alloc(ms + 1, st));
        HDP_TRY(seg2.alloc(nb + 1, st));
        k_live_edges<<<grid_for(ms, B), B, 0, st>>>(ms, oidx2.get(), eu, ev, uf, lflag.get()); note_launch();
        HDP_TRY(exclusive_sum(lflag.get(), lpos.get(), ms, st));
        k_compact_order<<<grid_for(ms, B), B, 0, st>>>(ms, oidx2.get(), lflag.get(), lpos.get(), oidx3.get());
        note_launch();
        k_seg_remap<<<grid_for(nb + 1, B), B, 0, st>>>(nb, ms, seg.get(), lflag.get(), lpos.get(), seg2.get());
        note_launch();
        order2 = oidx3.get();
        seg2p = seg2.get();
    }
    if (st_k < 0.0 || link) {
        auto kern = masks ? k_grp<false, true> : k_grp<false, false>;
        HDP_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g_smem));
        kern<<<nb, GW, g_smem, st>>>(seg2p, order2, eu, ev, uf, usz, tm, nw, beta, in_tree, rounds, nullptr, nullptr,
                                     -1.0); note_launch();
    }
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}

// build_hdpf on the device (see hdp_hdpf in the header).  st_k >= 0: the
// segment-tree variant, pass 1 with the FH criterion, then (link) pass 2 over
// the same sorted edges with the rules alone.  Batches of any size: slices of
// kHdpfSlice pairs share the batch-wide union-find state.
static int hdpf_run(int batch, int64_t nodes_per_pair, int64_t edges_per_pair, const int32_t* eu, const int32_t* ev,
                    const uint64_t* key, const int32_t* pixel_row, const uint32_t* row_masks, int n_rows, int nw,
                    double beta, const float* ew, double st_k, bool link, uint8_t* in_tree, int32_t* comp,
                    uint32_t* tree_masks, int* rounds_out, cudaStream_t st) {
    HDP_REQUIRE(beta >= 0.0 && beta <= 1.0, HDP_ERR_CONFIG, "beta must be in [0, 1], got %g", beta);
    HDP_REQUIRE(batch >= 1, HDP_ERR_CONFIG, "batch must be >= 1");
    HDP_REQUIRE(edges_per_pair < (1 << 24), HDP_ERR_CONFIG, "too many edges per pair for HDPF keys");
    HDP_REQUIRE(nw >= 1 && n_rows >= 1, HDP_ERR_CONFIG, "empty interval table");
    HDP_REQUIRE(nw <= 8, HDP_ERR_CONFIG, "disparity range above 255 not supported by the HDPF kernel");
    HDP_REQUIRE(st_k < 0.0 || ew != nullptr, HDP_ERR_CONFIG, "the segment tree needs the edge weights");
    const int64_t n = (int64_t)batch * nodes_per_pair;
    const int64_t m = (int64_t)batch * edges_per_pair;
    const int B = 256;
    const char* fe = getenv("HDP_HDPF_FAST");  // diagnostics / tests: 0 = always the window kernel
    const bool fast_off = fe && fe[0] == '0';
    // mask-homogeneous fast path (k_hdpf_classify): exact whenever no pair has
    // a cross-pass edge, which one flag read decides.  Plain HDPF: the whole
    // forest is the MSF of the equal-mask subgraph.  Segment tree with rules
    // (link): pass 1 (FH) keeps the trees homogeneous too, so pass 2 is the MSF
    // of the equal-mask edges between pass-1 trees.
    DevBuf<int32_t> u2, v2;
    bool homog = false;
    if ((st_k < 0.0 || link) && !fast_off && m > 0) {
        DevBuf<int> cross;
        HDP_TRY(u2.alloc(m, st));
        HDP_TRY(v2.alloc(m, st));
        HDP_TRY(cross.alloc(batch, st));
        HDP_CHECK_CUDA(cudaMemsetAsync(cross.get(), 0, sizeof(int) * batch, st));
        k_hdpf_classify<<<grid_for(m, B), B, 0, st>>>(m, eu, ev, pixel_row, row_masks, nodes_per_pair,
                                                      edges_per_pair, n_rows, nw, beta, u2.get(), v2.get(),
                                                      cross.get()); note_launch();
        HDP_CHECK_LAUNCH();
        std::vector<int> cr(batch, 0);
        HDP_TRY(to_host(cr.data(), cross.get(), batch, st));
        homog = true;
        for (int x : cr) homog = homog && x == 0;
        if (homog && st_k < 0.0) {
            HDP_TRY(run_boruvka(n, m, u2.get(), v2.get(), key, in_tree, comp, rounds_out, st, 0, 0));
            k_hdpf_node_masks<<<grid_for(n, B), B, 0, st>>>(n, pixel_row, row_masks, nodes_per_pair, n_rows, nw,
                                                            tree_masks); note_launch();
            HDP_CHECK_LAUNCH();
            return HDP_OK;
        }
    }
    DevBuf<int32_t> uf, usz;
    DevBuf<uint32_t> tm;
    DevBuf<float> tint;
    DevBuf<int> rounds;
    if (m > 0) HDP_CHECK_CUDA(cudaMemsetAsync(in_tree, 0, m, st));
    HDP_TRY(uf.alloc(n, st));
    HDP_TRY(usz.alloc(n, st));
    HDP_TRY(tm.alloc(n * nw, st));
    HDP_TRY(rounds.alloc(1, st));
    HDP_CHECK_CUDA(cudaMemsetAsync(rounds.get(), 0, sizeof(int), st));
    k_uf_init<<<grid_for(n, B), B, 0, st>>>(n, pixel_row, row_masks, nodes_per_pair, n_rows, nw,
                                            uf.get(), usz.get(), tm.get()); note_launch();
    if (st_k >= 0.0) {
        HDP_TRY(tint.alloc(n, st));
        HDP_CHECK_CUDA(cudaMemsetAsync(tint.get(), 0, sizeof(float) * n, st));  // Int of a singleton: 0
    }
    HDP_CHECK_LAUNCH();
    for (int b0 = 0; b0 < batch; b0 += kHdpfSlice) {
        const int nb = std::min(kHdpfSlice, batch - b0);
        const int64_t e0 = (int64_t)b0 * edges_per_pair;
        HDP_TRY(hdpf_slice(nb, nodes_per_pair, edges_per_pair, eu + e0, ev + e0, key + e0, pixel_row, row_masks,
                           n_rows, nw, beta, ew ? ew + e0 : nullptr, st_k, link && !homog, in_tree + e0, uf.get(),
                           usz.get(), tm.get(), tint.get(), rounds.get(), homog ? v2.get() + e0 : nullptr,
                           st));
    }
    if (homog) {
        // segment tree, pass 2 on homogeneous pass-1 trees: Boruvka over the
        // equal-mask edges relabelled to their pass-1 roots (edges inside a
        // tree become self-loops), then comp = the linked component of the root
        DevBuf<int32_t> c2;
        DevBuf<uint8_t> t2;
        HDP_TRY(c2.alloc(n, st));
        HDP_TRY(t2.alloc(m, st));
        k_hdpf_relabel_roots<<<grid_for(m, B), B, 0, st>>>(m, uf.get(), u2.get(), v2.get()); note_launch();
        HDP_TRY(run_boruvka(n, m, u2.get(), v2.get(), key, t2.get(), c2.get(), nullptr, st, 0, 0));
        k_hdpf_link_final<<<grid_for(std::max(m, n), B), B, 0, st>>>(m, n, t2.get(), in_tree, uf.get(), c2.get(),
                                                                     comp); note_launch();
        k_hdpf_node_masks<<<grid_for(n, B), B, 0, st>>>(n, pixel_row, row_masks, nodes_per_pair, n_rows, nw,
                                                        tree_masks); note_launch();
    } else {
        k_uf_final<<<grid_for(n, B), B, 0, st>>>(n, uf.get(), nw, tm.get(), comp, tree_masks); note_launch();
    }
    HDP_CHECK_LAUNCH();
    if (rounds_out) HDP_TRY(to_host(rounds_out, rounds.get(), 1, st));
    return HDP_OK;
}

extern "C" int hdp_hdpf(int batch, int64_t nodes_per_pair, int64_t edges_per_pair,
                        const int32_t* eu, const int32_t* ev, const uint64_t* key,
                        const int32_t* pixel_row, const uint32_t* row_masks, int n_rows, int nw,
                        double beta, const float* ew, double st_k, uint8_t* in_tree, int32_t* comp,
                        uint32_t* tree_masks, int* rounds_out, void* stream) {
    return hdpf_run(batch, nodes_per_pair, edges_per_pair, eu, ev, key, pixel_row, row_masks, n_rows, nw, beta, ew,
                    st_k, true, in_tree, comp, tree_masks, rounds_out, (cudaStream_t)stream);
}

namespace hdp {
int run_boruvka(int64_t n, int64_t m, const int32_t* eu, const int32_t* ev, const uint64_t* key,
                uint8_t* in_tree, int32_t* comp, int* rounds_out, cudaStream_t st, int grid_h, int grid_w);

__global__ void k_relabel_edges(int64_t m, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                                const int32_t* __restrict__ comp, int32_t* u2, int32_t* v2) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    u2[e] = comp[eu[e]];
    v2[e] = comp[ev[e]];
}

__global__ void k_compose(int64_t n, const int32_t* __restrict__ c1, const int32_t* __restrict__ c2, int32_t* out) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) out[v] = c2[c1[v]];
}

__global__ void k_or_u8(int64_t m, const uint8_t* __restrict__ a, uint8_t* b) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < m) b[e] |= a[e];
}
}  // namespace hdp

extern "C" int hdp_segment_tree(int batch, int h, int w, const int32_t* eu, const int32_t* ev, const float* ew,
                                const uint64_t* key, double st_k, uint8_t* in_tree, int32_t* comp, int* rounds_out,
                                void* stream) {
    HDP_REQUIRE(st_k >= 0.0, HDP_ERR_CONFIG, "segment-tree k must be >= 0, got %g", st_k);
    HDP_REQUIRE(batch >= 1 && h >= 1 && w >= 1, HDP_ERR_CONFIG, "bad batch geometry");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t npp = (int64_t)h * w, epp = 2 * npp - h - w;
    const int64_t n = batch * npp, m = batch * epp;
    // pass 1: subtrees by the FH criterion (every pixel set full: the HDPF
    // rules always pass), one sequential walk per pair
    DevBuf<int32_t> rows, c1, u2, v2, c2;
    DevBuf<uint32_t> masks, tmask;
    DevBuf<uint8_t> t2;
    HDP_TRY(rows.alloc(n, st));
    HDP_TRY(c1.alloc(n, st));
    HDP_TRY(masks.alloc(batch, st));
    HDP_TRY(tmask.alloc(n, st));
    HDP_CHECK_CUDA(cudaMemsetAsync(rows.get(), 0, sizeof(int32_t) * n, st));
    HDP_CHECK_CUDA(cudaMemsetAsync(masks.get(), 0xff, sizeof(uint32_t) * batch, st));
    HDP_TRY(hdpf_run(batch, npp, epp, eu, ev, key, rows.get(), masks.get(), 1, 1, 0.0, ew, st_k, false, in_tree,
                     c1.get(), tmask.get(), rounds_out, st));
    // pass 2: link the subtrees = the MST of the subtree graph under the same
    // (weight, index) order (Boruvka on the relabelled edges; internal edges
    // are self-loops and drop out)
    HDP_TRY(u2.alloc(m + 1, st));
    HDP_TRY(v2.alloc(m + 1, st));
    HDP_TRY(c2.alloc(n, st));
    HDP_TRY(t2.alloc(m + 1, st));
    if (m > 0) {
        k_relabel_edges<<<grid_for(m, 256), 256, 0, st>>>(m, eu, ev, c1.get(), u2.get(), v2.get()); note_launch();
    }
    HDP_TRY(run_boruvka(n, m, u2.get(), v2.get(), key, t2.get(), c2.get(), nullptr, st, 0, 0));
    if (m > 0) {
        k_or_u8<<<grid_for(m, 256), 256, 0, st>>>(m, t2.get(), in_tree); note_launch();
    }
    if (comp) {  // a subtree's representative carries the linked component
        k_compose<<<grid_for(n, 256), 256, 0, st>>>(n, c1.get(), c2.get(), comp); note_launch();
    }
    HDP_CHECK_LAUNCH();
    return HDP_OK;
}
