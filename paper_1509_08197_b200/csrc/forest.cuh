// Device representation of a rooted spanning forest plus its heavy-path
// layout (the structure the aggregation passes scan).  See forest.cu.
#pragma once

#include <vector>

#include "common.cuh"

// Heavy paths of at most this many nodes are aggregated register-resident
// (one thread per (path, lane)); longer ones by a warp walking staged chunks.
#ifndef HDP_SHORT_PATH
#define HDP_SHORT_PATH 12
#endif
constexpr int kShortPath = HDP_SHORT_PATH;
// Long paths are cut into segments of kSeg nodes, one warp each, chained by
// decoupled look-back in the aggregation kernels.
#ifndef HDP_SEG
#define HDP_SEG 32
#endif
constexpr int kSeg = HDP_SEG;

namespace hdp {
// Short-path chunks: the short paths of a phase are cut into runs whose rows,
// light-children rows, parent rows and metadata fit in shared memory; chunk
// c of a phase holds the paths whose cumulative weight (4-byte words) falls
// in the c-th window of kChunkWords.
#ifndef HDP_CHUNK_SHIFT
#define HDP_CHUNK_SHIFT 13
#endif
constexpr int kChunkShift = HDP_CHUNK_SHIFT;
constexpr int kChunkWords = 1 << kChunkShift;
constexpr int kChunkMaxWords = 48 * 1024;  // 192 KB of shared memory per chunk
// Chunks are launched in two classes per phase: at most kChunkSmallWords
// (most of them; five CTAs per SM fit) and the rest with the largest chunk's
// shared memory.  The window scheme makes a chunk kChunkWords plus at most one
// path, so one size for all would cap residency by the rare heavy chunk.
#ifndef HDP_CHUNK_SMALL
#define HDP_CHUNK_SMALL (10 * 1024)
#endif
constexpr int kChunkSmallWords = HDP_CHUNK_SMALL;

struct alignas(16) ChunkDesc {
    int p0, np;        // short-path list range
    int K0, nk;        // layout positions of the chunk's nodes
    int L0, nl;        // light-child entries of those nodes
    int n4;            // float4 words of staged rows
    int naux_up, naux_dn;
    int mqu;           // float4 columns of every row when all paths share m, else 0
    unsigned inv;      // ceil(2^32 / mqu) for mqu > 1: t / mqu == umulhi(t, inv) for small t
    int pad0;
    long long a0;      // first staged row float (16-byte aligned)
    long long lcr0;    // lc_rowoff[L0]
    long long auxd0;   // auxd[p0]
    long long pad3;
};
// One long-path segment, everything its warp needs in one 48-byte record
// (built with the lanes): the aggregation kernels start staging after a
// single dependent load instead of a chain through the path tables.
struct alignas(16) SegDesc {
    long long rowa;    // row offset (floats) of the segment's first node
    long long prow;    // the path's parent row, -1 at a root path
    int a, cnt;        // first layout position, nodes (<= kSeg)
    int e0, e1;        // light-child entries of the segment's nodes
    int mp, doff;      // padded row width (floats), lane offset of the tree
    int s, nseg;       // segment index from the head, segments of the path
};
}  // namespace hdp

struct hdp_forest;
namespace hdp {
// Early raw cost (dense range lanes only, hdp_dense_pipeline): every row has
// the same width, so a node's row is its layout position times that width and
// the raw-cost pass only needs the layout order.  forest_build starts it on a
// side stream as soon as the layout is placed; it overlaps the rest of the
// build (paths, light children, chunks), and hdp_aggregate_wta then uses the
// filled rows instead of running its own pre-pass.
struct EarlyCost {
    int want = 0, done = 0;
    const float* pl = nullptr;  // packed left / right planes (float4 per pixel); the right one is
    const float* pr = nullptr;  // prepared on `side` before the request is handed over
    int h = 0, w = 0, c = 0, x0 = 0, nx = 0;
    float alpha = 0, tau_c = 0, tau_g = 0;
    cudaStream_t side = nullptr;
    cudaEvent_t layout_ev = nullptr, done_ev = nullptr;  // owned by the caller (per thread)
    DevBuf<float> rows;  // the row buffer (A_up), allocated on the forest's stream
    DevBuf<uint2> rec8;  // byte records of the two images (aggregate.cu k_pack_rec8)
    DevBuf<int> flag8;
};
int ecost_early(hdp_forest* f);  // aggregate.cu
// hdp_forest_create with an early raw-cost request (the request's plain fields are copied)
int forest_create_ex(int64_t n_nodes, int64_t n_edges, const int32_t* eu, const int32_t* ev, const float* ew,
                     const uint8_t* in_tree, const int32_t* comp, float gamma, const EarlyCost* req,
                     hdp_forest** out, void* stream);
}  // namespace hdp

struct hdp_forest {
    cudaStream_t st = nullptr;
    hdp::EarlyCost early;
    int64_t n = 0;         // nodes
    int64_t n_trees = 0;
    int64_t n_paths = 0;
    int64_t n_phases = 0;  // heavy-light phases = max light depth + 1
    int64_t max_depth = 0;
    float gamma = 0.1f;

    // per node id
    hdp::DevBuf<int32_t> parent, depth, tree_id, size, root, lpos;
    hdp::DevBuf<float> pweight;

    // per layout position k (phase-major, path-contiguous, head first)
    hdp::DevBuf<int32_t> lnode;     // node id at k
    hdp::DevBuf<int32_t> lp_list;   // positions with light children, phase-major
    std::vector<int64_t> lp_off;    // host: light parents of phase r = [lp_off[r], lp_off[r+1])
    hdp::DevBuf<float> lsim;        // exp(-w(parent)/(gamma*255)) of that node
    hdp::DevBuf<int32_t> lc_start;  // n+1, CSR over light children
    hdp::DevBuf<int32_t> lc_list;   // layout positions of light children

    // per heavy path (ordered by layout)
    hdp::DevBuf<int32_t> p_start, p_len, p_par, p_tree;
    std::vector<int64_t> phase_off;  // host: paths of phase r = [phase_off[r], phase_off[r+1])
    std::vector<int64_t> phase_node;  // host: layout positions of phase r = [phase_node[r], phase_node[r+1])
    // paths of length >= 2 (need a sequential scan) and single-node paths,
    // each list phase-major; host offsets per phase
    hdp::DevBuf<int32_t> long_paths, short_paths;
    std::vector<int64_t> long_off, short_off;
    std::vector<int64_t> short_end;  // host: short paths of phase r occupy positions [phase_node[r], short_end[r])
    std::vector<int64_t> lp_mid;     // host: light parents on long paths of phase r = [lp_mid[r], lp_off[r+1])
    hdp::DevBuf<int32_t> dph;        // device copy of the per-phase tables (forest.cu P_* rows)
    int64_t n_lc = 0;                // light-child entries
    hdp::DevBuf<int2> seg_tab;      // (long-path index, segment index from the head)
    hdp::DevBuf<hdp::SegDesc> seg_desc;  // per segment, built with the lanes
    std::vector<int64_t> seg_off;   // host: segments of phase r = [seg_off[r], seg_off[r+1])
    int64_t n_segs = 0;

    // disparity lanes per tree
    int lanes_set = 0;
    int max_m = 0;
    int max_d = 0;                 // upper bound on any lane's disparity
    hdp::DevBuf<int32_t> t_m, t_doff, dlist;
    hdp::DevBuf<int64_t> rowoff;   // layout order, n+1: row offsets (rows of ceil4(m) floats)
    hdp::DevBuf<int64_t> nodeoff;  // node-id order, n: pixel-major volume offsets
    int64_t total_entries = 0;     // sum of m over nodes (stored hypotheses)
    int64_t total_rows = 0;        // floats of the row layout (every row padded to a multiple of 4)
    int range_x0 = -1;             // >= 0: every tree's lanes are x0 + j

    // packed metadata for the aggregation kernels (built with the lanes):
    hdp::DevBuf<int4> lmeta;       // per layout position: (node, lane offset, column, m)
    int geom_w = -1, geom_np = -1; // image geometry the lmeta columns were filled for
    hdp::DevBuf<float> lsimf;      // per position: similarity, sign bit = has light children
    hdp::DevBuf<int64_t> lc_row;   // per light-child entry: row offset of the child
    hdp::DevBuf<float> lc_sim;     // per light-child entry: similarity of the child
    hdp::DevBuf<int4> long_info;   // long paths: (start, len, m, lane offset)
    hdp::DevBuf<longlong2> long_rows;   // (first row, parent's row or -1)
    hdp::DevBuf<int4> short_info;  // single-node paths: (position, m, lane offset, 0)
    hdp::DevBuf<longlong2> short_rows;
    // chunks of the short-path row block of every phase: chunk c holds the
    // short paths [chunk_first[c], chunk_first[c+1]) (indices into the short
    // list), those whose first row falls in the c-th kChunkRows-float window
    hdp::DevBuf<int32_t> chunk_first;
    hdp::DevBuf<hdp::ChunkDesc> chunk_desc;
    hdp::DevBuf<int64_t> lc_rowoff;  // per light-child entry: prefix of m (aux row offsets, up pass)
    hdp::DevBuf<int64_t> auxd;       // per short path: prefix of m over paths with a parent (down pass)
    std::vector<int64_t> chunk_off;  // host: chunks of phase r = [chunk_off[r], chunk_off[r+1])
    std::vector<int64_t> chunk_big;  // host: of those, the last chunk_big[r] exceed kChunkSmallWords
    std::vector<int64_t> chunk_lone; // host: the chunk_lone[r] small chunks before them hold lone leaves only
    int64_t chunk_words = 0;         // shared-memory words the largest chunk needs
    int chunks_ok = 0;               // chunks fit in shared memory

    // optional stage timing of hdp_aggregate_wta (hdp_forest_set_timing):
    // events at entry, after the raw-cost pass, at exit
    int timing = 0;
    cudaEvent_t tev[3] = {nullptr, nullptr, nullptr};
    ~hdp_forest() {
        for (auto& e : tev)
            if (e) cudaEventDestroy(e);
    }
};

namespace hdp {
}  // namespace hdp
