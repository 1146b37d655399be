// Device representation of a rooted spanning forest plus its heavy-path
// layout (the structure the aggregation passes scan).  See forest.cu.
#pragma once

#include <vector>

#include "common.cuh"

struct hdp_forest {
    cudaStream_t st = nullptr;
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

    // disparity lanes per tree
    int lanes_set = 0;
    int max_m = 0;
    hdp::DevBuf<int32_t> t_m, t_doff, dlist;
    hdp::DevBuf<int64_t> rowoff;   // layout order, n+1: hypothesis row offsets
    hdp::DevBuf<int64_t> nodeoff;  // node-id order, n: pixel-major volume offsets
    int64_t total_entries = 0;
};
