/*
 * hdp_stereo.h -- C ABI of the B200-native (sm_100a) HDP tree-stereo hot path.
 *
 * Plain pointers and sizes only.  Every device pointer is caller-owned CUDA
 * device memory; every entry point is stream-ordered on `stream` (a
 * cudaStream_t passed as void*, NULL = legacy default stream) and reentrant
 * per stream: scratch comes from the stream-ordered pool, there is no hidden
 * global mutable state (except the thread-local message behind
 * hdp_last_error).  Functions return an HDP_* status code, never abort.
 *
 * The reference (Python package `treestereo`, /root/reference/pkg/src/
 * treestereo/) has no FFI for this path; its public functions ARE the
 * interface.  Each entry point below names the reference function(s) it
 * replaces; the Python binding that maps them back onto those signatures is
 * paper_1509_08197_b200/ (see INTEGRATION.md).
 *
 * Layouts: a batch of B stereo pairs of identical geometry H x W x C
 * (C in {1,3}); node (pixel) ids are global: g = b*H*W + r*W + c.  Grid edge
 * ids are per pair, in the reference's scan order (right edge before down
 * edge, spanning_forest.py:61-93).
 */
#ifndef HDP_STEREO_H
#define HDP_STEREO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* Status codes: same numbering as the reference exit codes (errors.py:8-29). */
#define HDP_OK 0
#define HDP_ERR_CONFIG 2   /* -> ConfigError   */
#define HDP_ERR_DATA 3     /* -> DataError     */
#define HDP_ERR_INTERNAL 4 /* -> InternalError */
#define HDP_ERR_CUDA 5     /* CUDA runtime failure (-> InternalError)       */

#define HDP_ABI_VERSION 1

int hdp_abi_version(void);
/* Number of kernels this library has launched in the process (diagnostic). */
int64_t hdp_launch_count(void);
/* Message for the last non-OK status on the calling thread. */
const char *hdp_last_error(void);

/* ---------------------------------------------------------- images, pyramid */

/* uint8 -> float64 copy (RasterImage.data.astype(float64), aggregation.py:269). */
int hdp_u8_to_f64(const uint8_t *src, double *dst, int64_t n, void *stream);

/* S x S block mean over covered pixels, per pair (pyramid.py:62-75
 * block_mean; pyramid.py:78-113 build_pyramid calls it once per level).
 * src (B,H,W,C) f64 -> dst (B,ceil(H/S),ceil(W/S),C) f64, numpy's reduceat
 * summation order, so exact for the reference's inputs. */
int hdp_block_mean(const double *src, double *dst, int batch, int h, int w, int c, int s,
                   void *stream);

/* prepare_layer (cost_volume.py:62-69): unit = I/255, gray, row gradient.
 * Outputs (each nullable): unit (B,H,W,C) f64, gray (B,H,W) f64, grad
 * (B,H,W) f64 (all bit-identical to the reference) and packed (B,H,W,4) f32
 * = (u0,u1,u2,grad) for the fp32 matching cost. */
int hdp_prepare(const double *img, int batch, int h, int w, int c, double *unit, double *gray,
                double *grad, float *packed, void *stream);

/* prepare_layer's packed plane straight from uint8 (B,H,W,C): bit-identical
 * to hdp_u8_to_f64 followed by hdp_prepare (unit = RN(I/255) by table). */
int hdp_prepare_u8(const uint8_t *img, int batch, int h, int w, int c, float *packed, void *stream);
/* Stable ascending argsort of 64-bit keys (radix): perm[i] = index of the
 * i-th smallest key, ties in index order -- numpy argsort(kind="stable") on
 * the keys (mst_edge_order, spanning_forest.py:96-107, on weight-bit keys). */
int hdp_argsort_u64(const uint64_t *keys, int64_t n, int32_t *perm, void *stream);

/* cost_grid / cost_at_pixels (cost_volume.py:72-102) for the disparities
 * xs[0..nx): out (B*H*W, nx) f32, disparity innermost. */
int hdp_cost_volume(const float *packed_l, const float *packed_r, int batch, int h, int w, int c,
                    const int32_t *xs, int nx, float alpha, float tau_c, float tau_g, float *out,
                    void *stream);

/* ------------------------------------------------------------ edges + MST */

/* build_edge_list (spanning_forest.py:61-93) for a batch: per pair
 * E = 2HW-H-W edges in scan order.  eu/ev global node ids, ew = max channel
 * |difference| (f32; exact for uint8 inputs and S=2 pyramid levels), key =
 * (f32 bits of ew) << 32 | per-pair edge index  -- the (weight, index) order
 * of mst_edge_order's stable sort (spanning_forest.py:96-107). */
int hdp_grid_edges(const double *img, int batch, int h, int w, int c, int32_t *eu, int32_t *ev,
                   float *ew, uint64_t *key, void *stream);

/* hdp_grid_edges from uint8 (B,H,W,C): the same edges, weights and keys. */
int hdp_grid_edges_u8(const uint8_t *img, int batch, int h, int w, int c, int32_t *eu, int32_t *ev,
                      float *ew, uint64_t *key, void *stream);
/* The same edges' weights in float64 (EdgeList.weight, spanning_forest.py:
 * 33-49), for the host-facing API. */
int hdp_grid_edge_weights64(const double *img, int batch, int h, int w, int c, double *ew,
                            void *stream);

/* apply_median_prefilter (spanning_forest.py:342-347): 3x3 per-channel
 * median with reflected borders (scipy.ndimage mode "reflect"), uint8. */
int hdp_median3x3(const uint8_t *src, uint8_t *dst, int batch, int h, int w, int c, void *stream);

/* winner_takes_all_with_cost (aggregation.py:239-256) over an (n, m) float64
 * matrix whose unused entries hold +inf: arg[r] = the first (lowest-column)
 * minimum of row r, best[r] its value. */
int hdp_rows_first_argmin(const double *rows, int64_t n, int m, int32_t *arg, double *best,
                          void *stream);

/* masked_cost_volume's per-tree blocks (cost_volume.py:225-231) from a dense
 * (pixels, ncols) f32 cost grid: output row r = pixel node[r], columns
 * cols[cstart[r] .. cstart[r] + cnt[r]), as float64 at out + off[r]. */
int hdp_gather_ragged(const float *grid, int ncols, int64_t nrows, const int64_t *node,
                      const int64_t *off, const int32_t *cstart, const int32_t *cnt,
                      const int32_t *cols, double *out, void *stream);

/* build_forest(edges, "mst") edge selection (spanning_forest.py:286-322) as
 * Boruvka on unique 64-bit keys (the MST under a total order is unique, so it
 * equals stable-sort Kruskal's).  Works on any edge list (not only grids).
 * Outputs: in_tree[e] in {0,1}; comp[v] = a component representative. */
int hdp_mst(int64_t n_nodes, int64_t n_edges, const int32_t *eu, const int32_t *ev,
            const uint64_t *key, uint8_t *in_tree, int32_t *comp, int *rounds_out, void *stream);

/* hdp_mst for a grid edge list from hdp_grid_edges (B pairs of h x w, scan
 * order): the same forest; the first Boruvka round is gathered per node over
 * its <= 4 incident edges instead of atomics over all edges. */
int hdp_mst_grid(int batch, int h, int w, const int32_t *eu, const int32_t *ev, const uint64_t *key,
                 uint8_t *in_tree, int32_t *comp, int *rounds_out, void *stream);
/* --------------------------------------------------------------- HDP parts */

/* estimate_prior up to the histogram (hdp_model.py:425-470): sampled
 * windowed WTA in both directions, float64 bit-exact with the reference,
 * cross-check |dL - dR| <= max_offset.  counts (B, d_max+1) int64;
 * kept (B) int64 = number of surviving samples.  max_ctas > 0 caps the grid
 * (the kernel strides over the centres), leaving SM slots to other streams. */
int hdp_prior_counts(const double *unit_l, const double *grad_l, const double *unit_r,
                     const double *grad_r, int batch, int h, int w, int c, int d_max,
                     int stride, int window, int max_offset, double alpha, double tau_c,
                     double tau_g, int64_t *counts, int64_t *kept, int max_ctas, void *stream);

/* Self-check of the prior's correctly rounded division by a constant
 * (x / b as RN(q + (x - q b) RN(1/b)), q = RN(x RN(1/b))) against the IEEE
 * division __ddiv_rn, for b in {3, 49, 25} on n seeded inputs in [0, 4);
 * *mismatches (host) = number of differing quotients.  Synchronises. */
int hdp_check_exact_division(int64_t n, uint64_t seed, int64_t *mismatches, void *stream);

/* predict_intervals (hdp_model.py:498-525) for nrows rows of Bayes matrices
 * (rows x ncols f64, ncols <= 256): stable descending order, sequential
 * running mass, first P/(c+P) < delta stops; out masks (nrows, nw) u32
 * bitsets over the columns (pack of DisparityIntervalTable.masks()). */
int hdp_predict_masks(const double *bayes, int64_t nrows, int ncols, double delta, uint32_t *masks, int nw,
                      void *stream);
/* estimate_prior's histogram step (hdp_model.py:465-470) for B pairs:
 * priors[b, :] = (counts[b, :] + 1) / sum, the sum in numpy's add.reduce
 * order; kept[b] == 0 -> the uniform 1 / d1.  d1 <= 256. */
int hdp_priors_from_counts(const int64_t *counts, const int64_t *kept, int batch, int d1, double *priors,
                           void *stream);
/* bayes_child_given_parent (hdp_model.py:334-363) for B priors:
 * bayes[b, r, :] = cond[r, :] * priors[b, :] / row sum (numpy's add.reduce
 * order), a row without mass -> all 1 / cols (n_dead[b] counts them when
 * non-NULL; zero it first).  cond: (rows, cols) f64 (host-computed
 * conditional_parent_given_child), cols <= 256. */
int hdp_bayes(const double *cond, const double *priors, int batch, int rows, int cols, double *bayes,
              int32_t *n_dead, void *stream);
/* assign_pixel_intervals (hdp_forest.py:91-123): pixel_row[g] =
 * parent_disp[b, r/S, c/S]; DATA error if a parent disparity is outside
 * [0, n_rows). */
int hdp_assign_rows(const int32_t *parent_disp, int batch, int ph, int pw, int h, int w, int s,
                    int n_rows, int32_t *pixel_row, void *stream);

/* build_hdpf (hdp_forest.py:151-216): rule 1 (disjoint pixel sets drop the
 * edge), then Kruskal order (key) with rule 2 (Jaccard of the LIVE tree sets
 * >= beta, IEEE double division).  Exact fast path: when no edge of the batch
 * is "cross-pass" (endpoint masks differ, intersect and pass rule 2
 * statically), every tree keeps one pixel mask and the forest is the MSF of
 * the equal-mask edges (Boruvka).  Otherwise, decided exactly by whole-window
 * rounds: one CTA per pair takes the next 1023 edges of its sorted list,
 * splits their live edges into conflict groups (edges sharing a tree) and
 * walks every group in Kruskal order with one thread.  Keys: (weight or rank
 * bits << 32 | index of the edge in its pair); the low 24 bits break ties.
 * row_masks: (B, n_rows, nw) u32 bitsets;
 * pixel_row per node.  Outputs in_tree[e], comp[v] (representative),
 * tree_masks (n_nodes, nw): the final tree set, valid at every node.
 * st_k >= 0 builds the segment-tree variant (tree_kind "st", which the
 * reference does not implement -- parity unpinned): a first pass accepts an
 * edge only if also w <= min(Int(Ta) + st_k/|Ta|, Int(Tb) + st_k/|Tb|) (Int =
 * largest edge inside the tree, ew = the f32 edge weights), a second pass links
 * the subtrees with the rules alone.  st_k < 0 (ew may be NULL): the plain
 * build. */
int hdp_hdpf(int batch, int64_t nodes_per_pair, int64_t edges_per_pair, const int32_t *eu,
             const int32_t *ev, const uint64_t *key, const int32_t *pixel_row,
             const uint32_t *row_masks, int n_rows, int nw, double beta, const float *ew, double st_k,
             uint8_t *in_tree, int32_t *comp, uint32_t *tree_masks, int *rounds_out, void *stream);

/* Segment tree (tree_kind "st"; not in the reference, whose edge_order rejects
 * it, spanning_forest.py:115-120 -- the extension point it would plug into):
 * per pair, subtrees grown in Kruskal order under the criterion w <=
 * min(Int(Ta) + k/|Ta|, Int(Tb) + k/|Tb|), then linked into one spanning tree
 * by the MST of the subtree graph in the same (weight, index) order.  Grid
 * edges and keys of hdp_grid_edges; outputs in_tree[e] and a component
 * labelling comp[v] for hdp_forest_create. */
int hdp_segment_tree(int batch, int h, int w, const int32_t *eu, const int32_t *ev, const float *ew,
                     const uint64_t *key, double st_k, uint8_t *in_tree, int32_t *comp, int *rounds_out,
                     void *stream);

/* ------------------------------------------- rooted forest + aggregation */

typedef struct hdp_forest hdp_forest;

/* Root the forest given by the edges with in_tree set (all if NULL):
 * root = lowest node id per component, trees numbered by root id
 * (_bfs_forest, spanning_forest.py:191-283), parent / depth / subtree size
 * by Euler tour + list ranking, similarities exp(-w/(gamma*255))
 * (spanning_forest.py:184-188), and the heavy-path layout the aggregation
 * kernels scan.  comp (nullable) = any component labelling of the edges. */
int hdp_forest_create(int64_t n_nodes, int64_t n_edges, const int32_t *eu, const int32_t *ev,
                      const float *ew, const uint8_t *in_tree, const int32_t *comp, float gamma,
                      hdp_forest **out, void *stream);

/* Host-visible sizes (synchronises the creating stream once). */
int hdp_forest_stats(const hdp_forest *f, int64_t *n_trees, int64_t *n_paths, int64_t *n_phases,
                     int64_t *max_depth);

/* RootedForest fields (spanning_forest.py:146-188), nullable outputs:
 * parent (root: itself), depth, tree_id, subtree size, parent_weight (f32),
 * root id per node. */
int hdp_forest_export(const hdp_forest *f, int32_t *parent, int32_t *depth, int32_t *tree_id,
                      int32_t *size, float *parent_weight, int32_t *root, void *stream);

/* Per-tree disparity lanes.  set_lanes: tree_masks (n_trees, nw) u32
 * bitsets (DisparityForest.intervals, hdp_forest.py:126-148); set_lanes_range:
 * every tree gets x0 .. x0+nx-1 (dense baseline / a disparity slab). */
int hdp_forest_set_lanes(hdp_forest *f, const uint32_t *tree_masks, int nw, void *stream);
int hdp_forest_set_lanes_range(hdp_forest *f, int x0, int nx, void *stream);
/* set_lanes from per-node masks (n_nodes, nw) valid at every node (hdp_hdpf's
 * tree_masks): each tree's mask is read at its root. */
int hdp_forest_set_lanes_nodes(hdp_forest *f, const uint32_t *node_masks, int nw, void *stream);

/* Stored entries sum_p |interval(tree(p))| (hdp_forest.py:144-148) and,
 * optionally, the per-node offsets of the pixel-major volume layout. */
int hdp_forest_entries(hdp_forest *f, int64_t *total, int64_t *node_offsets, void *stream);

/* masked_cost_volume + aggregate_tree + winner_takes_all_with_cost
 * (cost_volume.py:183-236, aggregation.py:158-256, baseline fold
 * aggregation.py:311-326), fused: the raw cost is computed on the fly from
 * the packed planes of pair b = node / (h*w) (or read from cost_rows
 * pixel-major ragged rows f32 at the node offsets of hdp_forest_entries when
 * non-NULL: aggregate_forest / aggregate_tree, aggregation.py:182-236),
 * aggregated leaf->root and root->leaf along heavy paths, and reduced to the
 * first argmin per node.  Outputs (nullable): disp (int32), min_cost (f32),
 * keys (u64 = order-preserving f32 encoding << 32 | d: the u64 minimum is
 * the first argmin, so keys combine across disparity slabs with a min),
 * volume (f32, pixel-major at node_offsets). */
int hdp_aggregate_wta(hdp_forest *f, const float *packed_l, const float *packed_r, int h, int w,
                      int c, float alpha, float tau_c, float tau_g, const float *cost_rows,
                      int32_t *disp, float *min_cost, uint64_t *keys, float *volume,
                      void *stream);

/* Stage timing of hdp_aggregate_wta (PipelineResult.metrics["seconds"],
 * aggregation.py:401-416): when on, every call records device events at
 * entry, after the raw matching-cost pass and at exit; stage_ms waits for the
 * last call and returns its cost and aggregation (+ WTA) times in ms. */
int hdp_forest_set_timing(hdp_forest *f, int on);
int hdp_forest_stage_ms(const hdp_forest *f, float *cost_ms, float *aggregate_ms);

/* Per pair of a batch (nodes_per_pair consecutive node ids each): tree count
 * (LayerResult.n_trees) and stored entries (LayerResult.stored_entries,
 * aggregation.py:418-426); host output arrays of length batch. */
int hdp_forest_pair_stats(const hdp_forest *f, int batch, int64_t nodes_per_pair,
                          int64_t *n_trees, int64_t *stored, void *stream);
/* The same into a device array out[2 * batch] = (tree counts, stored
 * entries), stream-ordered, no host read. */
int hdp_forest_pair_stats_device(const hdp_forest *f, int batch, int64_t nodes_per_pair, int64_t *out,
                                 void *stream);

void hdp_forest_destroy(hdp_forest *f);

/* Disparity-slab keys (the C5 split): u64 = order-preserving
 * f32 cost << 32 | d, so the u64 minimum over slabs is the reference's first
 * argmin over the full range (strict '<' chunk fold, aggregation.py:320-326).
 * signed_order != 0 flips the top bit: int64 order == u64 order, for NCCL's
 * signed int64 MIN reduction.  pack: (disp, min_cost) -> keys; unpack: the
 * inverse, for keys combined across slabs. */
int hdp_keys_pack(const int32_t *disp, const float *min_cost, int64_t n, int signed_order,
                  uint64_t *keys, void *stream);
int hdp_keys_unpack(const uint64_t *keys, int64_t n, int signed_order, int32_t *disp,
                    float *min_cost, void *stream);

/* ------------------------------------------------------------ evaluation */

/* error_rate (evaluation.py:27-54) for a batch of B maps of npix pixels:
 * counts (B, n_thr + 1) int64 = per pair the number of evaluated pixels
 * (valid in both maps, not occluded; valid / occlusion masks are uint8,
 * nullable = all valid / none occluded) followed by, per threshold t, the
 * number of evaluated pixels with |pred - gt| >= t.  1 <= n_thr <= 8;
 * thresholds on the device. */
int hdp_error_counts(const int32_t *pred, const int32_t *gt, const uint8_t *pred_valid,
                     const uint8_t *gt_valid, const uint8_t *occlusion, int batch, int64_t npix,
                     const int32_t *thresholds, int n_thr, int64_t *counts, void *stream);

/* occlusion_from_gt (evaluation.py:57-76): occlusion (B,H,W) uint8 = a valid
 * left pixel whose match c - d is off the image, invalid in the right map, or
 * whose disparities differ by more than 1 (valid masks nullable). */
int hdp_occlusion_from_gt(const int32_t *gt_left, const int32_t *gt_right, const uint8_t *left_valid,
                          const uint8_t *right_valid, int batch, int h, int w, uint8_t *occlusion,
                          void *stream);

/* --------------------------------------------------------- whole pipeline */
/* Grow the library's stream-ordered memory pool to `bytes` once (one block
 * allocated and freed; the pool keeps its memory): later scratch allocations
 * up to that size never wait for the driver to map new physical memory in the
 * middle of a step.  Synchronises the stream. */
int hdp_pool_reserve(int64_t bytes, void *stream);

/* hdp_dense_pipeline option: start the raw-cost pass on a side stream as soon
 * as the tree's layout order is final, beside the rest of the build (dense
 * range lanes have uniform rows, so a node's row is known from its layout
 * position alone).  Returns the previous setting.  Off by default (measured
 * +1.5 % at C5); HDP_EARLY_COST=1 sets the default. */
int hdp_set_early_cost(int on);

/* run_baseline_pipeline (aggregation.py:263-358) for a batch of pairs in one
 * call: u8 -> f64, prepare_layer, build_edge_list, MST, rooted forest, lanes
 * [x0, x0+nx), fused cost + aggregation + first argmin.  left/right (B,H,W,C)
 * uint8 on the device; disp (B,H,W) int32, min_cost (B,H,W) f32; n_trees
 * (B, nullable) int64 = trees per pair.  The batch is cut into n_sub
 * sub-batches that run concurrently on their own streams (the tree build of
 * one overlaps the aggregation of another); the caller's stream waits for
 * all of them.  agg_ms (n_sub, nullable): device time of each sub-batch's
 * hdp_aggregate_wta call (synchronises the workers once at the end).
 * right_ready (a cudaEvent_t, nullable): the right image is read only after
 * this event (it is first needed after the tree build, so its host->device
 * copy can still be running on another stream while the trees are built). */
int hdp_dense_pipeline(const uint8_t *left, const uint8_t *right, int batch, int h, int w, int c,
                       int d_max, int x0, int nx, float alpha, float tau_c, float tau_g, float gamma,
                       int n_sub, int32_t *disp, float *min_cost, int64_t *n_trees, float *agg_ms,
                       void *right_ready, void *stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* HDP_STEREO_H */
