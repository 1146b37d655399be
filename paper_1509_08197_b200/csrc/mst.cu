// Boruvka minimum spanning forest on unique 64-bit edge keys.
//
// Replaces the reference's Kruskal loop (spanning_forest.py:286-322 via
// hdp_forest.py:219-224 build_hdpf(beta=0)).  With keys (weight bits << 32 |
// scan index) the edge order is a total order equal to the reference's
// stable argsort (spanning_forest.py:96-107), the minimum spanning forest
// under a total order is unique, and Boruvka returns exactly that forest.
//
// Per round: every live edge offers its key to both endpoint components
// (atomicMin), the winning edge per component is identified, components hook
// along it (mutual pairs broken by the lower id), and components are
// relabelled by following hook chains.  Self-loops die.  HBM/L2-atomic bound.
#include <cuda_runtime.h>

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "prims.cuh"

namespace hdp {

__global__ void k_mst_init(int64_t n, int32_t* comp) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) comp[v] = (int32_t)v;
}

// Rounds are launched in batches without a host check in between; every
// kernel of round r first looks at the previous round's hook flag and does
// nothing once a round has made no hooks (the forest is final).
__device__ __forceinline__ bool converged(const int* prev) { return prev && *prev == 0; }

// `nodes` (optional): the representative list of the contracted phase; node
// kernels then run over it instead of 0..n-1.
__device__ __forceinline__ int64_t node_at(const int32_t* nodes, int64_t t) { return nodes ? nodes[t] : t; }

__global__ void k_mst_reset(int64_t n, unsigned long long* best, int32_t* win, const int* prev,
                            const int32_t* __restrict__ nodes) {
    if (converged(prev)) return;
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) {
        const int64_t v = node_at(nodes, t);
        best[v] = ~0ull;
        win[v] = -1;
    }
}

__global__ void k_mst_offer(int64_t m, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                            const uint64_t* __restrict__ key, const int32_t* __restrict__ comp,
                            uint8_t* __restrict__ alive, unsigned long long* best, const int* prev) {
    if (converged(prev)) return;
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m || !alive[e]) return;
    int32_t cu = comp[eu[e]], cv = comp[ev[e]];
    if (cu == cv) {
        alive[e] = 0;
        return;
    }
    unsigned long long k = key[e];
    if (k < best[cu]) atomicMin(&best[cu], k);
    if (k < best[cv]) atomicMin(&best[cv], k);
}

__global__ void k_mst_win(int64_t m, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                          const uint64_t* __restrict__ key, const int32_t* __restrict__ comp,
                          const uint8_t* __restrict__ alive, const unsigned long long* __restrict__ best,
                          int32_t* win, int32_t* wother, const int* prev) {
    if (converged(prev)) return;
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m || !alive[e]) return;
    int32_t cu = comp[eu[e]], cv = comp[ev[e]];
    unsigned long long k = key[e];
    // the winner also records the component across it (saves the hook two
    // dependent loads)
    if (best[cu] == k) {
        win[cu] = (int32_t)e;
        wother[cu] = cv;
    }
    if (best[cv] == k) {
        win[cv] = (int32_t)e;
        wother[cv] = cu;
    }
}

// Round 1 on a grid edge list (hdp_grid_edges' scan order): every component
// is one node, so a node's winning edge is the least key among its <= 4
// incident edges, gathered directly (no atomics, no pass over the edges).
__device__ __forceinline__ int64_t grid_right(int r, int col, int h, int w) {
    return r < h - 1 ? (int64_t)r * (2 * w - 1) + 2 * col : (int64_t)(h - 1) * (2 * w - 1) + col;
}
__device__ __forceinline__ int64_t grid_down(int r, int col, int w) {
    return (int64_t)r * (2 * w - 1) + 2 * col + (col < w - 1 ? 1 : 0);
}
__global__ void k_mst_grid_first(int64_t n, int h, int w, const uint64_t* __restrict__ key,
                                 unsigned long long* best_out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int64_t npp = (int64_t)h * w;
    const int64_t b = t / npp, p = t - b * npp;
    const int r = (int)(p / w), col = (int)(p - (int64_t)r * w);
    const int64_t eb = b * (2 * npp - h - w);
    unsigned long long best = ~0ull;
    int64_t be = -1, bo = -1;
    auto take = [&](int64_t e, int64_t other) {
        const unsigned long long k = key[eb + e];
        if (k < best) {
            best = k;
            be = eb + e;
            bo = other;
        }
    };
    if (col + 1 < w) take(grid_right(r, col, h, w), t + 1);
    if (r + 1 < h) take(grid_down(r, col, w), t + w);
    if (col > 0) take(grid_right(r, col - 1, h, w), t - 1);
    if (r > 0) take(grid_down(r - 1, col, w), t - w);
    (void)be;
    (void)bo;
    best_out[t] = best;
}

// Grid rounds: the low word of a grid key is the edge's index within its
// pair and a component never spans pairs, so the component's minimum key
// names its winning edge: (pair of v) * edges per pair + low word.  Hook
// without a separate winner pass.
__global__ void k_mst_hook_grid(int64_t n, int64_t npp, int64_t epp, const int32_t* __restrict__ eu,
                                const int32_t* __restrict__ ev, const int32_t* __restrict__ comp,
                                const unsigned long long* __restrict__ best, int32_t* __restrict__ link,
                                uint8_t* __restrict__ in_tree, int* __restrict__ hooks, const int* prev) {
    if (converged(prev)) return;
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool hooked = false;
    if (v < n && comp[v] == v) {
        const unsigned long long k = best[v];
        if (k == ~0ull) {
            link[v] = (int32_t)v;
        } else {
            const int64_t e = (v / npp) * epp + (int64_t)(uint32_t)k;
            const int32_t cu = comp[eu[e]], cv = comp[ev[e]];
            const int32_t other = cu == (int32_t)v ? cv : cu;
            in_tree[e] = 1;
            if (best[other] == k && v < other) {
                link[v] = (int32_t)v;  // mutual minimum: the lower id stays the root
            } else {
                link[v] = other;
                hooked = true;
            }
        }
    }
    if (__syncthreads_or(hooked) && threadIdx.x == 0 && *(volatile int*)hooks == 0) *hooks = 1;
}

// relabel by the hook chains and reset the next round's minima
__global__ void k_mst_relabel_reset(int64_t n, int32_t* __restrict__ comp, const int32_t* __restrict__ link,
                                    unsigned long long* __restrict__ best, const int* prev) {
    if (converged(prev)) return;
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    int32_t r = comp[v];
    while (link[r] != r) r = link[r];
    comp[v] = r;
    best[v] = ~0ull;
}

// eidx (optional): original edge index of each contracted edge
__global__ void k_mst_hook(int64_t n, const int32_t* __restrict__ wother,
                           const int32_t* __restrict__ comp, const int32_t* __restrict__ win,
                           int32_t* __restrict__ link, uint8_t* __restrict__ in_tree,
                           int* __restrict__ hooks, const int* prev, const int32_t* __restrict__ nodes,
                           const int32_t* __restrict__ eidx) {
    if (converged(prev)) return;
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool hooked = false;
    if (t < n) {
        const int64_t v = node_at(nodes, t);
        if (comp[v] == v) {  // representatives only
            int32_t e = win[v];
            if (e < 0) {
                link[v] = (int32_t)v;
            } else {
                const int32_t other = wother[v];
                in_tree[eidx ? eidx[e] : e] = 1;
                if (win[other] == e && v < other) {
                    link[v] = (int32_t)v;  // mutual minimum: the lower id stays the root
                } else {
                    link[v] = other;
                    hooked = true;
                }
            }
        }
    }
    // "another round is needed": one guarded flag write per block
    if (__syncthreads_or(hooked) && threadIdx.x == 0 && *(volatile int*)hooks == 0) *hooks = 1;
}

__global__ void k_mst_relabel(int64_t n, int32_t* __restrict__ comp, const int32_t* __restrict__ link,
                              const int* prev, const int32_t* __restrict__ nodes) {
    if (converged(prev)) return;
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int64_t v = node_at(nodes, t);
    int32_t r = comp[v];
    while (link[r] != r) r = link[r];
    comp[v] = r;
}

// ---- contraction between the two phases: edges between distinct components
// with endpoints relabelled to their representatives, and the representative
// list.  Counts land in cnt[0] (edges), cnt[1] (representatives).
__global__ void k_mst_cflags(int64_t m, int64_t n, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                             const int32_t* __restrict__ comp, int32_t* ef, int32_t* vf) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) ef[i] = comp[eu[i]] != comp[ev[i]] ? 1 : 0;
    else if (i == m) ef[i] = 0;
    if (i < n) vf[i] = comp[i] == i ? 1 : 0;
    else if (i == n) vf[i] = 0;
}

__global__ void k_mst_counts(int64_t m, int64_t n, const int32_t* __restrict__ epos, const int32_t* __restrict__ vpos,
                             int* cnt) {
    cnt[0] = epos[m];
    cnt[1] = vpos[n];
}

__global__ void k_mst_contract(int64_t m, int64_t n, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                               const uint64_t* __restrict__ key, const int32_t* __restrict__ comp,
                               const int32_t* __restrict__ ef, const int32_t* __restrict__ epos,
                               const int32_t* __restrict__ vf, const int32_t* __restrict__ vpos, int32_t* cu,
                               int32_t* cv, uint64_t* ckey, int32_t* cidx, int32_t* reps) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m && ef[i]) {
        const int32_t p = epos[i];
        cu[p] = comp[eu[i]];
        cv[p] = comp[ev[i]];
        // low word re-keyed to the contracted index: order-preserving (the
        // compaction keeps edge order, and keys are only compared within a
        // component, i.e. within one pair's run of the list), and the minimum
        // key of a component names its winning edge directly
        ckey[p] = (key[i] & 0xffffffff00000000ull) | (uint32_t)p;
        cidx[p] = (int32_t)i;
    }
    if (i < n && vf[i]) reps[vpos[i]] = (int32_t)i;
}

// The contracted phase in ONE cooperative launch: the rounds' steps are
// separated by grid-wide barriers instead of kernel boundaries, and the loop
// stops on the device at the first round without hooks (no host checks).
__global__ void __launch_bounds__(256) k_mst_coop(int64_t gm, int64_t gn, const int32_t* __restrict__ gu,
                                                  const int32_t* __restrict__ gv, const uint64_t* __restrict__ gk,
                                                  const int32_t* __restrict__ gidx, const int32_t* __restrict__ reps,
                                                  int32_t* comp, uint8_t* alive, unsigned long long* best,
                                                  int32_t* win, int32_t* wother, int32_t* link, uint8_t* in_tree,
                                                  int* flags, int max_rounds, int* rounds_out) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int64_t tid = (int64_t)grid.thread_rank(), nthr = (int64_t)grid.size();
    int r = 0;
    (void)win;
    (void)wother;
    for (int64_t t = tid; t < gn; t += nthr) best[reps[t]] = ~0ull;
    grid.sync();
    while (r < max_rounds) {
        for (int64_t e = tid; e < gm; e += nthr) {
            if (!alive[e]) continue;
            const int32_t cu = comp[gu[e]], cv = comp[gv[e]];
            if (cu == cv) {
                alive[e] = 0;
                continue;
            }
            const unsigned long long k = gk[e];
            if (k < best[cu]) atomicMin(&best[cu], k);
            if (k < best[cv]) atomicMin(&best[cv], k);
        }
        grid.sync();
        // hook: the component's minimum key carries its winning edge
        bool hooked = false;
        for (int64_t t = tid; t < gn; t += nthr) {
            const int32_t v = reps[t];
            if (comp[v] != v) continue;
            const unsigned long long k = best[v];
            if (k == ~0ull) {
                link[v] = v;
                continue;
            }
            const int32_t e = (int32_t)(uint32_t)k;
            const int32_t cu = comp[gu[e]], cv = comp[gv[e]];
            const int32_t other = cu == v ? cv : cu;
            in_tree[gidx[e]] = 1;
            if (best[other] == k && v < other) {
                link[v] = v;  // mutual minimum: the lower id stays the root
            } else {
                link[v] = other;
                hooked = true;
            }
        }
        if (__syncthreads_or(hooked) && threadIdx.x == 0 && *(volatile int*)(flags + r) == 0) flags[r] = 1;
        grid.sync();
        // relabel, and reset the next round's minima (hook, the last reader of
        // best, is behind the barrier above)
        for (int64_t t = tid; t < gn; t += nthr) {
            const int32_t v = reps[t];
            int32_t x = comp[v];
            while (link[x] != x) x = link[x];
            comp[v] = x;
            best[v] = ~0ull;
        }
        grid.sync();
        const bool more = *(volatile int*)(flags + r) != 0;
        r++;
        if (!more) break;  // round r - 1 made no hooks: the forest is final
    }
    if (tid == 0) *rounds_out = r;
}

// every node: its phase-1 representative's final root
__global__ void k_mst_final(int64_t n, int32_t* comp) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int32_t r = comp[v];
    if (r != v) comp[v] = comp[r];  // representatives (r == v) already hold their final root
}

// Shared driver, also used by the connected-component labelling of rooted
// forests (every edge key distinct).  Phase 1: kFull rounds over the whole
// graph (components grow ~3x per round, so most edges become internal);
// phase 2: the remaining rounds over the contracted graph (edges between
// distinct components, relabelled to representatives).
int run_boruvka(int64_t n, int64_t m, const int32_t* eu, const int32_t* ev, const uint64_t* key,
                uint8_t* in_tree, int32_t* comp, int* rounds_out, cudaStream_t st, int grid_h, int grid_w) {
    constexpr int kMaxRounds = 64, kBatch = 4;
    int kFull = 3;
    bool coop = true;  // the contracted phase as one cooperative launch
    {
        const char* e = getenv("HDP_MST_COOP");  // diagnostics: 0 = batched launches
        if (e && e[0] == '0') coop = false;
    }
    {
        const char* e = getenv("HDP_MST_FULL");  // diagnostics: full-graph rounds before contraction
        if (e && e[0] >= '1' && e[0] <= '9') kFull = e[0] == '1' ? kMaxRounds : e[0] - '0';
    }
    DevBuf<unsigned long long> best;
    DevBuf<int32_t> win, wother, link;
    DevBuf<uint8_t> alive;
    DevBuf<int> hooks;
    HDP_TRY(best.alloc(n, st));
    HDP_TRY(win.alloc(n, st));
    HDP_TRY(wother.alloc(n, st));
    HDP_TRY(link.alloc(n, st));
    HDP_TRY(alive.alloc(m > 0 ? m : 1, st));
    HDP_TRY(hooks.alloc(2 * kMaxRounds + 2, st));
    int* cnt = hooks.get() + 2 * kMaxRounds;  // contraction counts
    HDP_CHECK_CUDA(cudaMemsetAsync(hooks.get(), 0, sizeof(int) * (2 * kMaxRounds + 2), st));
    k_mst_init<<<grid_for(n, 256), 256, 0, st>>>(n, comp); note_launch();
    if (m > 0) {
        HDP_CHECK_CUDA(cudaMemsetAsync(alive.get(), 1, m, st));
        HDP_CHECK_CUDA(cudaMemsetAsync(in_tree, 0, m, st));
    }
    // current graph: full, later contracted
    const int32_t* gu = eu;
    const int32_t* gv = ev;
    const uint64_t* gk = key;
    const int32_t* gidx = nullptr;
    const int32_t* nodes = nullptr;
    int64_t gm = m, gn = n;
    DevBuf<int32_t> cu, cv, cidx, reps;
    DevBuf<uint64_t> ckey;
    int rounds = 0;
    bool contracted = false;
    Tracer tr(st);
    while (m > 0) {
        const int r0 = rounds;
        const int nb = contracted ? kBatch : std::min(kFull, kMaxRounds - rounds);  // first batch = full graph
        for (int r = r0; r < r0 + nb; r++) {
            const int* prev = r > 0 ? hooks.get() + r - 1 : nullptr;
            int* hk = hooks.get() + r;
            if (grid_h > 0 && !contracted) {
                // grid rounds: the first gathered per node, then offer -> hook (winner
                // from the key) -> relabel + reset
                const int64_t npp = (int64_t)grid_h * grid_w, epp = 2 * npp - grid_h - grid_w;
                if (r == 0) {
                    k_mst_grid_first<<<grid_for(gn, 256), 256, 0, st>>>(gn, grid_h, grid_w, gk, best.get());
                } else {
                    k_mst_offer<<<grid_for(gm, 256), 256, 0, st>>>(gm, gu, gv, gk, comp, alive.get(), best.get(),
                                                                   prev);
                }
                note_launch();
                k_mst_hook_grid<<<grid_for(gn, 256), 256, 0, st>>>(gn, npp, epp, gu, gv, comp, best.get(), link.get(),
                                                                   in_tree, hk, prev); note_launch();
                k_mst_relabel_reset<<<grid_for(gn, 256), 256, 0, st>>>(gn, comp, link.get(), best.get(), prev);
                note_launch();
                continue;
            }
            {
            k_mst_reset<<<grid_for(gn, 256), 256, 0, st>>>(gn, best.get(), win.get(), prev, nodes); note_launch();
            if (gm > 0) {
                k_mst_offer<<<grid_for(gm, 256), 256, 0, st>>>(gm, gu, gv, gk, comp, alive.get(), best.get(),
                                                               prev); note_launch();
                k_mst_win<<<grid_for(gm, 256), 256, 0, st>>>(gm, gu, gv, gk, comp, alive.get(), best.get(),
                                                             win.get(), wother.get(), prev); note_launch();
            }
            }
            k_mst_hook<<<grid_for(gn, 256), 256, 0, st>>>(gn, wother.get(), comp, win.get(), link.get(), in_tree, hk,
                                                         prev, nodes, gidx); note_launch();
            k_mst_relabel<<<grid_for(gn, 256), 256, 0, st>>>(gn, comp, link.get(), prev, nodes); note_launch();
        }
        DevBuf<int32_t> ef, epos, vf, vpos;
        if (!contracted) {
            // contraction counts ride along with the batch's hook flags
            HDP_TRY(ef.alloc(m + 1, st));
            HDP_TRY(epos.alloc(m + 1, st));
            HDP_TRY(vf.alloc(n + 1, st));
            HDP_TRY(vpos.alloc(n + 1, st));
            k_mst_cflags<<<grid_for(std::max(m, n) + 1, 256), 256, 0, st>>>(m, n, eu, ev, comp, ef.get(), vf.get()); note_launch();
            HDP_TRY(exclusive_sum(ef.get(), epos.get(), m + 1, st));
            HDP_TRY(exclusive_sum(vf.get(), vpos.get(), n + 1, st));
            k_mst_counts<<<1, 1, 0, st>>>(m, n, epos.get(), vpos.get(), cnt); note_launch();
        }
        HDP_CHECK_LAUNCH();
        std::vector<int> hb(std::max(nb, kBatch) + 2, 0);
        HDP_CHECK_CUDA(cudaMemcpyAsync(hb.data(), hooks.get() + r0, sizeof(int) * nb, cudaMemcpyDeviceToHost, st));
        if (!contracted) HDP_CHECK_CUDA(cudaMemcpyAsync(hb.data() + nb, cnt, sizeof(int) * 2, cudaMemcpyDeviceToHost, st));
        HDP_CHECK_CUDA(cudaStreamSynchronize(st));
        int k = 0;
        while (k < nb && hb[k] != 0) k++;
        if (k < nb) {  // round r0 + k made no hooks: it was the last
            rounds = r0 + k + 1;
            break;
        }
        rounds = r0 + nb;
        if (rounds >= kMaxRounds) {
            set_error("boruvka did not converge (duplicate keys?)");
            return HDP_ERR_INTERNAL;
        }
        if (!contracted) {
            const int64_t m2 = hb[nb], n2 = hb[nb + 1];
            HDP_TRY(cu.alloc(m2 + 1, st));
            HDP_TRY(cv.alloc(m2 + 1, st));
            HDP_TRY(ckey.alloc(m2 + 1, st));
            HDP_TRY(cidx.alloc(m2 + 1, st));
            HDP_TRY(reps.alloc(n2 + 1, st));
            k_mst_contract<<<grid_for(std::max(m, n), 256), 256, 0, st>>>(
                m, n, eu, ev, key, comp, ef.get(), epos.get(), vf.get(), vpos.get(), cu.get(), cv.get(), ckey.get(),
                cidx.get(), reps.get()); note_launch();
            if (m2 > 0) HDP_CHECK_CUDA(cudaMemsetAsync(alive.get(), 1, m2, st));
            gu = cu.get();
            gv = cv.get();
            gk = ckey.get();
            gidx = cidx.get();
            nodes = reps.get();
            gm = m2;
            gn = n2;
            contracted = true;
            if (coop) {
                int nb = 0, dev = 0, nsm = 0;
                HDP_CHECK_CUDA(cudaGetDevice(&dev));
                HDP_CHECK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
                HDP_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_mst_coop, 256, 0));
                {
                    // a grid barrier costs more with more CTAs: cap the grid
                    static const int cap = [] {
                        const char* e = getenv("HDP_MST_COOP_BPS");  // tuning: CTAs per SM
                        return e && *e ? atoi(e) : 0;
                    }();
                    if (cap > 0 && cap < nb) nb = cap;
                }
                int* fl = hooks.get() + kMaxRounds;  // per-round hook flags of this phase (zeroed)
                int* rc = hooks.get() + 2 * kMaxRounds - 1;
                int max_r = kMaxRounds - rounds - 1;
                int64_t gm_ = gm, gn_ = gn;
                uint8_t* al = alive.get();
                unsigned long long* bs = best.get();
                int32_t *wi = win.get(), *wo = wother.get(), *lk = link.get();
                int32_t* cp = comp;
                void* args[] = {(void*)&gm_, (void*)&gn_, (void*)&gu, (void*)&gv, (void*)&gk, (void*)&gidx,
                                (void*)&nodes, (void*)&cp, (void*)&al, (void*)&bs, (void*)&wi, (void*)&wo,
                                (void*)&lk, (void*)&in_tree, (void*)&fl, (void*)&max_r, (void*)&rc};
                HDP_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)k_mst_coop, dim3(nb * nsm), dim3(256), args,
                                                           0, st)); note_launch();
                // the round count and the convergence check (it can only fail on
                // duplicate keys; grid keys carry the unique edge index in the low
                // word) only when the caller asks for the rounds: no host read on
                // the pipeline path
                if (rounds_out) {
                    int hr = 0;
                    HDP_TRY(to_host(&hr, rc, 1, st));
                    rounds += hr;
                    if (hr >= max_r) {
                        set_error("boruvka did not converge (duplicate keys?)");
                        return HDP_ERR_INTERNAL;
                    }
                }
                break;
            }
        }
    }
    if (contracted) {
        k_mst_final<<<grid_for(n, 256), 256, 0, st>>>(n, comp); note_launch();
        HDP_CHECK_LAUNCH();
    }
    tr.mark("boruvka rounds");
    if (rounds_out) *rounds_out = rounds;
    return HDP_OK;
}

}  // namespace hdp

using namespace hdp;

extern "C" int hdp_mst(int64_t n_nodes, int64_t n_edges, const int32_t* eu, const int32_t* ev,
                       const uint64_t* key, uint8_t* in_tree, int32_t* comp, int* rounds_out,
                       void* stream) {
    HDP_REQUIRE(n_nodes >= 0 && n_nodes < ((int64_t)1 << 31), HDP_ERR_CONFIG, "bad node count");
    HDP_REQUIRE(n_edges >= 0 && n_edges < ((int64_t)1 << 31), HDP_ERR_CONFIG, "bad edge count");
    if (n_nodes == 0) return HDP_OK;
    return run_boruvka(n_nodes, n_edges, eu, ev, key, in_tree, comp, rounds_out,
                       (cudaStream_t)stream, 0, 0);
}

extern "C" int hdp_mst_grid(int batch, int h, int w, const int32_t* eu, const int32_t* ev, const uint64_t* key,
                            uint8_t* in_tree, int32_t* comp, int* rounds_out, void* stream) {
    HDP_REQUIRE(batch >= 1 && h >= 1 && w >= 1, HDP_ERR_CONFIG, "bad grid geometry");
    const int64_t n = (int64_t)batch * h * w, m = (int64_t)batch * (2 * (int64_t)h * w - h - w);
    HDP_REQUIRE(n < ((int64_t)1 << 31) && m < ((int64_t)1 << 31), HDP_ERR_CONFIG, "grid too large");
    return run_boruvka(n, m, eu, ev, key, in_tree, comp, rounds_out, (cudaStream_t)stream, h, w);
}
