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

#include "common.cuh"

namespace hdp {

__global__ void k_mst_init(int64_t n, int32_t* comp) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) comp[v] = (int32_t)v;
}

// Rounds are launched in batches without a host check in between; every
// kernel of round r first looks at the previous round's hook flag and does
// nothing once a round has made no hooks (the forest is final).
__device__ __forceinline__ bool converged(const int* prev) { return prev && *prev == 0; }

__global__ void k_mst_reset(int64_t n, unsigned long long* best, int32_t* win, const int* prev) {
    if (converged(prev)) return;
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) {
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
                          int32_t* win, const int* prev) {
    if (converged(prev)) return;
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m || !alive[e]) return;
    int32_t cu = comp[eu[e]], cv = comp[ev[e]];
    unsigned long long k = key[e];
    if (best[cu] == k) win[cu] = (int32_t)e;
    if (best[cv] == k) win[cv] = (int32_t)e;
}

__global__ void k_mst_hook(int64_t n, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                           const int32_t* __restrict__ comp, const int32_t* __restrict__ win,
                           int32_t* __restrict__ link, uint8_t* __restrict__ in_tree,
                           int* __restrict__ hooks, const int* prev) {
    if (converged(prev)) return;
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool hooked = false;
    if (v < n && comp[v] == v) {  // representatives only
        int32_t e = win[v];
        if (e < 0) {
            link[v] = (int32_t)v;
        } else {
            int32_t a = comp[eu[e]], b = comp[ev[e]];
            int32_t other = (a == v) ? b : a;
            in_tree[e] = 1;
            if (win[other] == e && v < other) {
                link[v] = (int32_t)v;  // mutual minimum: the lower id stays the root
            } else {
                link[v] = other;
                hooked = true;
            }
        }
    }
    // "another round is needed": one guarded flag write per block
    if (__syncthreads_or(hooked) && threadIdx.x == 0 && *(volatile int*)hooks == 0) *hooks = 1;
}

__global__ void k_mst_relabel(int64_t n, int32_t* __restrict__ comp, const int32_t* __restrict__ link,
                              const int* prev) {
    if (converged(prev)) return;
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    int32_t r = comp[v];
    while (link[r] != r) r = link[r];
    comp[v] = r;
}

// Shared driver, also used by the connected-component labelling of rooted
// forests (every edge key distinct).
int run_boruvka(int64_t n, int64_t m, const int32_t* eu, const int32_t* ev, const uint64_t* key,
                uint8_t* in_tree, int32_t* comp, int* rounds_out, cudaStream_t st) {
    DevBuf<unsigned long long> best;
    DevBuf<int32_t> win, link;
    DevBuf<uint8_t> alive;
    DevBuf<int> hooks;
    constexpr int kMaxRounds = 64, kBatch = 4;
    HDP_TRY(best.alloc(n, st));
    HDP_TRY(win.alloc(n, st));
    HDP_TRY(link.alloc(n, st));
    HDP_TRY(alive.alloc(m > 0 ? m : 1, st));
    HDP_TRY(hooks.alloc(kMaxRounds + kBatch, st));
    HDP_CHECK_CUDA(cudaMemsetAsync(hooks.get(), 0, sizeof(int) * (kMaxRounds + kBatch), st));
    k_mst_init<<<grid_for(n, 256), 256, 0, st>>>(n, comp); note_launch();
    if (m > 0) {
        HDP_CHECK_CUDA(cudaMemsetAsync(alive.get(), 1, m, st));
        HDP_CHECK_CUDA(cudaMemsetAsync(in_tree, 0, m, st));
    }
    int rounds = 0;
    Tracer tr(st);
    int hb[kBatch];
    while (m > 0) {
        // kBatch rounds per host check; hooks[r] = 1 iff round r hooked anything
        const int r0 = rounds;
        for (int r = r0; r < r0 + kBatch; r++) {
            const int* prev = r > 0 ? hooks.get() + r - 1 : nullptr;
            int* hk = hooks.get() + r;
            k_mst_reset<<<grid_for(n, 256), 256, 0, st>>>(n, best.get(), win.get(), prev); note_launch();
            k_mst_offer<<<grid_for(m, 256), 256, 0, st>>>(m, eu, ev, key, comp, alive.get(), best.get(), prev); note_launch();
            k_mst_win<<<grid_for(m, 256), 256, 0, st>>>(m, eu, ev, key, comp, alive.get(), best.get(),
                                                       win.get(), prev); note_launch();
            k_mst_hook<<<grid_for(n, 256), 256, 0, st>>>(n, eu, ev, comp, win.get(), link.get(),
                                                        in_tree, hk, prev); note_launch();
            k_mst_relabel<<<grid_for(n, 256), 256, 0, st>>>(n, comp, link.get(), prev); note_launch();
        }
        HDP_CHECK_LAUNCH();
        HDP_CHECK_CUDA(cudaMemcpyAsync(hb, hooks.get() + r0, sizeof(hb), cudaMemcpyDeviceToHost, st));
        HDP_CHECK_CUDA(cudaStreamSynchronize(st));
        int k = 0;
        while (k < kBatch && hb[k] != 0) k++;
        if (k < kBatch) {  // round r0 + k made no hooks: it was the last
            rounds = r0 + k + 1;
            break;
        }
        rounds = r0 + kBatch;
        if (rounds >= kMaxRounds) {
            set_error("boruvka did not converge (duplicate keys?)");
            return HDP_ERR_INTERNAL;
        }
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
                       (cudaStream_t)stream);
}
