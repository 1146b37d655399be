"""The drop-in API (paper_1509_08197_b200.*) exercised the way the
reference's own test-suite exercises treestereo (pkg/tests/test_*.py), with
the fp32 tolerance of the north_star where the reference checks float64."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import cuda_available, golden

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

F32 = dict(rtol=1e-4, atol=1e-6)


# ------------------------------------------------------------- aggregation
def random_forest(rng, max_nodes=20):
    from paper_1509_08197_b200.spanning_forest import forest_from_edges

    n = int(rng.integers(2, max_nodes + 1))
    us, vs, ws = [], [], []
    for node in range(1, n):
        if rng.uniform() < 0.85:
            us.append(int(rng.integers(0, node)))
            vs.append(node)
            ws.append(float(rng.uniform(0.0, 255.0)))
    return forest_from_edges(n, np.array(us), np.array(vs), np.array(ws)), n, list(zip(us, vs, ws))


def brute_force_aggregate(n, edge_list, costs, gamma):
    adj = [[] for _ in range(n)]
    for u, v, w in edge_list:
        s = float(np.exp(-w / (gamma * 255.0)))
        adj[u].append((v, s))
        adj[v].append((u, s))
    out = np.zeros_like(costs)
    for src in range(n):
        prod = np.full(n, -1.0)
        prod[src] = 1.0
        stack = [src]
        while stack:
            cur = stack.pop()
            for nxt, s in adj[cur]:
                if prod[nxt] < 0:
                    prod[nxt] = prod[cur] * s
                    stack.append(nxt)
        reach = prod >= 0
        out[src] = (prod[reach, None] * costs[reach]).sum(axis=0)
    return out


@pytest.mark.parametrize("trial", range(25))
def test_two_pass_matches_brute_force(trial):
    from paper_1509_08197_b200.aggregation import aggregate_forest

    rng = np.random.default_rng(1000 + trial)
    forest, n, edge_list = random_forest(rng, max_nodes=60)
    m = int(rng.integers(1, 40))
    costs = rng.uniform(0.0, 1.0, size=(n, m))
    gamma = float(rng.uniform(0.01, 1.0))
    got = aggregate_forest(forest, costs, gamma)
    np.testing.assert_allclose(got, brute_force_aggregate(n, edge_list, costs, gamma), **F32)


def test_two_node_closed_form_and_singletons():
    from paper_1509_08197_b200.aggregation import aggregate_forest
    from paper_1509_08197_b200.spanning_forest import forest_from_edges

    f = forest_from_edges(2, np.array([0]), np.array([1]), np.array([51.0]))
    s = np.exp(-2.0)
    got = aggregate_forest(f, np.array([[1.0], [10.0]]), gamma=0.1)
    assert got[0, 0] == pytest.approx(1.0 + 10.0 * s, rel=1e-6)
    assert got[1, 0] == pytest.approx(10.0 + s, rel=1e-6)
    f3 = forest_from_edges(3, np.array([0]), np.array([1]), np.array([9.0]))
    assert aggregate_forest(f3, np.array([[2.0], [3.0], [7.0]]), 0.1)[2, 0] == 7.0


def test_trees_are_isolated():
    from paper_1509_08197_b200.aggregation import aggregate_forest
    from paper_1509_08197_b200.spanning_forest import forest_from_edges

    f = forest_from_edges(4, np.array([0, 2]), np.array([1, 3]), np.array([20.0, 30.0]))
    costs = np.array([[1.0], [2.0], [3.0], [4.0]])
    base = aggregate_forest(f, costs, gamma=0.3)
    bumped = costs.copy()
    bumped[2:] += 100.0
    moved = aggregate_forest(f, bumped, gamma=0.3)
    np.testing.assert_array_equal(base[:2], moved[:2])
    assert (moved[2:] != base[2:]).all()


def test_aggregate_forest_validates_shape():
    from paper_1509_08197_b200.aggregation import aggregate_forest
    from paper_1509_08197_b200.errors import ConfigError
    from paper_1509_08197_b200.spanning_forest import forest_from_edges

    f = forest_from_edges(2, np.array([0]), np.array([1]), np.array([1.0]))
    with pytest.raises(ConfigError):
        aggregate_forest(f, np.zeros((3, 1)))


def test_deep_chain_and_wide_star():
    """A 20k-node path (depth 20k, one heavy path) and a 5k-leaf star."""
    from paper_1509_08197_b200.aggregation import aggregate_forest
    from paper_1509_08197_b200.spanning_forest import forest_from_edges
    from oracle import oracle as O

    rng = np.random.default_rng(7)
    n = 20000
    u, v = np.arange(n - 1), np.arange(1, n)
    w = rng.uniform(0, 40, n - 1)
    costs = rng.uniform(0, 1, (n, 3))
    f = forest_from_edges(n, u, v, w)
    ref = O.aggregate_forest(O.bfs_forest(n, u, v, w), costs, 0.1)
    np.testing.assert_allclose(aggregate_forest(f, costs, 0.1), ref, **F32)
    n = 5001
    u, v = np.zeros(n - 1, np.int64), np.arange(1, n)
    w = rng.uniform(0, 255, n - 1)
    costs = rng.uniform(0, 1, (n, 2))
    f = forest_from_edges(n, u, v, w)
    ref = O.aggregate_forest(O.bfs_forest(n, u, v, w), costs, 0.1)
    np.testing.assert_allclose(aggregate_forest(f, costs, 0.1), ref, **F32)


def test_wta_tie_takes_smaller_disparity():
    from paper_1509_08197_b200.aggregation import winner_takes_all_with_cost
    from paper_1509_08197_b200.cost_volume import SparseCostVolume

    vol = SparseCostVolume(2, 1, 1, np.array([0, 1]), np.array([0, 2]), (np.array([0, 1]),),
                           [np.array([[0.5, 0.5], [0.3, 0.2]])], np.array([0, 1]), np.array([0, 0]))
    d, c = winner_takes_all_with_cost(vol)
    assert d.values.tolist() == [[0, 1]]
    assert c.tolist() == [[0.5, 0.2]]


# ------------------------------------------------------------ trees / edges
def random_layer(h, w, rng, channels=3):
    from paper_1509_08197_b200.pyramid import PyramidLayer

    return PyramidLayer(0, rng.integers(0, 256, size=(h, w, channels)).astype(np.float64), 4)


def test_edge_list_matches_reference_layout():
    from paper_1509_08197_b200.spanning_forest import build_edge_list

    g = golden("mst.npz")
    from paper_1509_08197_b200.pyramid import PyramidLayer

    for tag in ("int0", "int1", "dyadic", "int3", "int4"):
        e = build_edge_list(PyramidLayer(0, g[tag + "_in"], 4))
        np.testing.assert_array_equal(e.u, g[tag + "_u"])
        np.testing.assert_array_equal(e.v, g[tag + "_v"])
        np.testing.assert_array_equal(e.weight, g[tag + "_w"])


def test_mst_order_is_stable_sort():
    from paper_1509_08197_b200.spanning_forest import build_edge_list, mst_edge_order

    e = build_edge_list(random_layer(5, 7, np.random.default_rng(2)))
    expect = sorted(range(e.n_edges), key=lambda i: (e.weight[i], i))
    assert mst_edge_order(e).tolist() == expect


@pytest.mark.parametrize("trial", range(10))
def test_mst_weight_and_parents_match_reference(trial):
    from paper_1509_08197_b200.spanning_forest import (build_edge_list, build_forest,
                                                       forest_total_weight)
    from oracle import oracle as O

    rng = np.random.default_rng(100 + trial)
    layer = random_layer(int(rng.integers(2, 13)), int(rng.integers(2, 13)), rng)
    e = build_edge_list(layer)
    f = build_forest(e, "mst")
    ref = O.build_forest_mst(layer.intensities).base
    assert forest_total_weight(f) == float(ref.parent_weight.sum())
    np.testing.assert_array_equal(f.parent, ref.parent)
    np.testing.assert_array_equal(f.depth, ref.depth)


def test_forest_structure_invariants():
    from paper_1509_08197_b200.spanning_forest import build_edge_list, build_forest

    f = build_forest(build_edge_list(random_layer(6, 8, np.random.default_rng(5))), "mst")
    n = f.n_nodes
    assert f.n_trees == 1 and f.roots.tolist() == [0]
    assert np.array_equal(f.order[f.pos], np.arange(n))
    assert (np.diff(f.depth[f.order]) >= 0).all()
    for node in range(1, n):
        assert f.pos[f.parent[node]] < f.pos[node]
    for node in range(n):
        kids = f.children(node)
        assert kids.size < 2 or (np.diff(kids) > 0).all()
        assert all(f.parent[k] == node for k in kids.tolist())


def test_forest_from_edges_two_trees_and_similarity():
    from paper_1509_08197_b200.spanning_forest import forest_from_edges, forest_total_weight

    f = forest_from_edges(5, np.array([0, 1, 3]), np.array([1, 2, 4]), np.array([2.0, 1.0, 5.0]))
    assert f.n_trees == 2 and sorted(f.roots.tolist()) == [0, 3]
    assert forest_total_weight(f) == 8.0
    f2 = forest_from_edges(2, np.array([0]), np.array([1]), np.array([51.0]))
    assert f2.similarities(0.1)[1] == pytest.approx(np.exp(-51.0 / 25.5))


def test_rt_tree_is_seeded_and_matches_oracle():
    from paper_1509_08197_b200.spanning_forest import build_edge_list, build_forest

    g = golden("mst.npz")
    from paper_1509_08197_b200.pyramid import PyramidLayer

    e = build_edge_list(PyramidLayer(0, g["int1_in"], 4))
    f = build_forest(e, "rt", seed=3)
    np.testing.assert_array_equal(f.parent, g["int1_rt_parent"])


def test_median_prefilter_matches_scipy():
    scipy_nd = pytest.importorskip("scipy.ndimage")
    from paper_1509_08197_b200.raster_io import RasterImage
    from paper_1509_08197_b200.spanning_forest import apply_median_prefilter

    img = np.random.default_rng(3).integers(0, 256, size=(17, 23, 3), dtype=np.uint8)
    got = apply_median_prefilter(RasterImage(img)).data
    for c in range(3):
        np.testing.assert_array_equal(got[:, :, c],
                                      scipy_nd.median_filter(img[:, :, c], size=3, mode="reflect"))


# --------------------------------------------------------------- hdp forest
def _pim(rows, intervals, h, w, d):
    from paper_1509_08197_b200.hdp_forest import PixelIntervalMap

    ivs = tuple(np.array(sorted(iv), dtype=np.int64) for iv in intervals)
    masks = tuple(sum(1 << int(x) for x in iv) for iv in ivs)
    return PixelIntervalMap(h, w, d, np.asarray(rows, dtype=np.int64).ravel(), ivs, masks)


def _flat(h, w, d=7):
    from paper_1509_08197_b200.pyramid import PyramidLayer

    return PyramidLayer(0, np.zeros((h, w, 1)), d)


def test_hdpf_rules():
    from paper_1509_08197_b200.hdp_forest import build_hdpf
    from paper_1509_08197_b200.spanning_forest import build_edge_list

    e = build_edge_list(_flat(1, 2))
    assert build_hdpf(e, _pim([0, 1], [[0, 1], [4, 5]], 1, 2, 7), beta=0.0).n_trees == 2
    pim = _pim([0, 1], [[3, 4, 5], [4, 5, 6]], 1, 2, 7)
    assert build_hdpf(e, pim, beta=0.6).n_trees == 2
    merged = build_hdpf(e, pim, beta=0.5)
    assert merged.n_trees == 1 and merged.intervals[0].tolist() == [3, 4, 5, 6]
    e4 = build_edge_list(_flat(1, 4))
    f = build_hdpf(e4, _pim([0, 1, 1, 2], [[1, 2, 3], [2, 3, 4], [3, 4, 5]], 1, 4, 7), beta=0.5)
    assert f.n_trees == 2 and sorted(np.diff(f.base.tree_slices).tolist()) == [1, 3]


def test_hdpf_beta0_full_range_is_plain_forest_and_recompute():
    from paper_1509_08197_b200.hdp_forest import (build_hdpf, full_range_interval_map,
                                                  plain_disparity_forest,
                                                  recompute_tree_intervals)
    from paper_1509_08197_b200.spanning_forest import build_edge_list, build_forest
    from paper_1509_08197_b200.pyramid import PyramidLayer

    rng = np.random.default_rng(0)
    layer = PyramidLayer(0, rng.integers(0, 256, size=(7, 9, 3)).astype(np.float64), 5)
    e = build_edge_list(layer)
    plain = build_forest(e, "mst")
    via = build_hdpf(e, full_range_interval_map(7, 9, 5), beta=0.0)
    np.testing.assert_array_equal(via.base.parent, plain.parent)
    assert plain_disparity_forest(e, 5).total_search_entries() == 63 * 6
    rows = (np.arange(120) // 30) % 4
    layer2 = PyramidLayer(0, rng.integers(0, 256, size=(10, 12, 3)).astype(np.float64), 6)
    pim = _pim(rows, [[0, 1], [1, 2], [2, 3], [4, 5, 6]], 10, 12, 6)
    f = build_hdpf(build_edge_list(layer2), pim, beta=0.4)
    assert recompute_tree_intervals(f, pim) == f.masks


def test_hdpf_matches_reference_golden():
    from paper_1509_08197_b200.hdp_forest import build_hdpf
    from paper_1509_08197_b200.pyramid import PyramidLayer
    from paper_1509_08197_b200.spanning_forest import build_edge_list

    g = golden("hdpf.npz")
    for k in range(int(g["count"])):
        p = f"h{k}_"
        h, w = g[p + "in"].shape[:2]
        d = int(g[p + "d"])
        offs = np.concatenate(([0], np.cumsum(g[p + "tab_sizes"])))
        table = [g[p + "tab_flat"][offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]
        f = build_hdpf(build_edge_list(PyramidLayer(0, g[p + "in"], d)),
                       _pim(g[p + "rows"], table, h, w, d), beta=float(g[p + "beta"]))
        np.testing.assert_array_equal(f.base.parent, g[p + "parent"])
        np.testing.assert_array_equal(f.base.tree_id, g[p + "tree_id"])
        np.testing.assert_array_equal(np.concatenate(f.intervals), g[p + "iv_flat"])


# -------------------------------------------------------------------- cost
def test_cost_grid_matches_reference_golden():
    from paper_1509_08197_b200.cost_volume import CostParams, cost_at_pixels, cost_grid, prepare_layer
    from paper_1509_08197_b200.pyramid import PyramidLayer

    g = golden("cost.npz")
    L = prepare_layer(PyramidLayer(0, g["rgb_left"], 9))
    R = prepare_layer(PyramidLayer(0, g["rgb_right"], 9))
    np.testing.assert_array_equal(L.gray, g["rgb_gray"])
    for x in range(10):
        grid = cost_grid(L, R, x, CostParams())
        np.testing.assert_allclose(grid, g["rgb_cost"][x], rtol=1e-4, atol=1e-9)
        rows, cols = np.meshgrid(np.arange(20), np.arange(33), indexing="ij")
        np.testing.assert_array_equal(cost_at_pixels(L, R, x, rows.ravel(), cols.ravel(),
                                                     CostParams()), grid.ravel())


def test_raw_cost_border_and_zero():
    from paper_1509_08197_b200.cost_volume import CostParams, raw_cost
    from paper_1509_08197_b200.errors import ConfigError
    from paper_1509_08197_b200.pyramid import PyramidLayer

    rng = np.random.default_rng(2)
    L = PyramidLayer(0, rng.integers(0, 256, size=(3, 5, 3)).astype(np.float64), 4)
    R = PyramidLayer(0, rng.integers(0, 256, size=(3, 5, 3)).astype(np.float64), 4)
    assert raw_cost(L, R, (1, 2), 3) == pytest.approx(0.1 * 0.0275 + 0.9 * 0.0078, rel=1e-6)
    assert raw_cost(L, L, (2, 3), 0) == 0.0
    with pytest.raises(ConfigError):
        raw_cost(L, R, (0, 0), 5)


def test_masked_volume_and_aggregate_tree_match_oracle():
    from paper_1509_08197_b200.aggregation import aggregate_tree, winner_takes_all_with_cost
    from paper_1509_08197_b200.cost_volume import CostParams, masked_cost_volume
    from paper_1509_08197_b200.hdp_forest import build_hdpf
    from paper_1509_08197_b200.pyramid import PyramidLayer
    from paper_1509_08197_b200.spanning_forest import build_edge_list

    g = golden("hdpf.npz")
    p = "h1_"
    h, w = g[p + "in"].shape[:2]
    d = int(g[p + "d"])
    offs = np.concatenate(([0], np.cumsum(g[p + "tab_sizes"])))
    table = [g[p + "tab_flat"][offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]
    left = PyramidLayer(0, g[p + "in"], d)
    right = PyramidLayer(0, np.roll(g[p + "in"], -2, axis=1), d)
    f = build_hdpf(build_edge_list(left), _pim(g[p + "rows"], table, h, w, d), beta=0.6)
    vol = masked_cost_volume(left, right, f.base, f.intervals, CostParams())
    agg = aggregate_tree(vol, f, 0.1)
    disp, best = winner_takes_all_with_cost(agg)
    # oracle on the same forest: per-tree aggregation in float64
    from oracle import oracle as O

    of = O.build_hdpf(*O.build_edge_list(g[p + "in"]), h * w,
                      O.masks_from_rows(table, d)[g[p + "rows"]], d, 0.6)
    od, ob, o2 = O._layer_wta(g[p + "in"], right.intensities, d, of, 0.1)
    band = (o2 - ob) <= 1e-5 * np.abs(ob)
    assert not ((disp.values != od) & ~band).any()
    np.testing.assert_allclose(best, ob, rtol=1e-4, atol=1e-7)


# ---------------------------------------------------------------- prior
def test_estimate_prior_peaks_at_true_shift_and_fallback():
    from paper_1509_08197_b200.cost_volume import CostParams
    from paper_1509_08197_b200.hdp_model import estimate_prior
    from paper_1509_08197_b200.pyramid import PyramidLayer

    g = golden("prior.npz")
    prior = estimate_prior(PyramidLayer(0, g["shift_left"], 8), PyramidLayer(0, g["shift_right"], 8),
                           CostParams())
    np.testing.assert_array_equal(prior, g["shift_prior"])
    assert prior.argmax() == 3
    rng = np.random.default_rng(5)
    layer = PyramidLayer(0, rng.integers(0, 256, size=(20, 30, 1)).astype(np.float64), 6)
    np.testing.assert_allclose(estimate_prior(layer, layer, CostParams(), max_offset=-1), 1 / 7)


# ------------------------------------------------------------ pipelines
def test_baseline_pipeline_matches_golden_and_manual():
    from paper_1509_08197_b200.aggregation import AggregationParams, run_baseline_pipeline
    from paper_1509_08197_b200.raster_io import RasterImage, StereoPair
    from oracle import oracle as O

    g = golden("pipelines.npz")
    pair = StereoPair(RasterImage(g["c1_left"]), RasterImage(g["c1_right"]), 16)
    res = run_baseline_pipeline(pair, AggregationParams())
    ref = O.run_baseline(g["c1_left"], g["c1_right"], 16)
    band = (ref.second_cost - ref.min_cost) <= 1e-5 * np.abs(ref.min_cost)
    assert not ((res.disparity.values != g["c1_base_disp"]) & ~band).any()
    assert res.metrics["stored_entries"] == res.metrics["dense_entries"] == 96 * 128 * 17
    assert res.layers[0].n_trees == 1


def test_hdp_pipeline_api_hooks_and_metrics(gmm_text):
    from paper_1509_08197_b200.aggregation import AggregationParams, run_hdp_pipeline
    from paper_1509_08197_b200.errors import DataError
    from paper_1509_08197_b200.hdp_model import GmmModel
    from paper_1509_08197_b200.raster_io import RasterImage, StereoPair

    g = golden("pipelines.npz")
    model = GmmModel.parse(gmm_text)
    pair = StereoPair(RasterImage(g["c1_left"]), RasterImage(g["c1_right"]), 16)
    seen = []
    res = run_hdp_pipeline(pair, model, AggregationParams(levels=2),
                           on_forest=lambda lvl, f: seen.append((lvl, f.n_trees)))
    assert [s[0] for s in seen] == [2, 1, 0]
    lvl0 = next(lr for lr in res.layers if lr.level == 0)
    assert res.metrics["stored_entries"] == lvl0.stored_entries
    assert lvl0.stored_entries / res.metrics["dense_entries"] == pytest.approx(
        res.metrics["search_ratios"][0], abs=1e-12)
    assert seen[-1][1] == lvl0.n_trees == int(g["c1_hdp_l0_ntrees"])
    again = run_hdp_pipeline(pair, model, AggregationParams(levels=2))
    np.testing.assert_array_equal(res.disparity.values, again.disparity.values)
    with pytest.raises(DataError):
        run_hdp_pipeline(pair, model, AggregationParams(levels=6))


def test_constant_shift_scene_nearly_perfect(gmm_text):
    from paper_1509_08197_b200.aggregation import AggregationParams, run_hdp_pipeline
    from paper_1509_08197_b200.evaluation import error_rate
    from paper_1509_08197_b200.hdp_model import GmmModel
    from paper_1509_08197_b200.synthetic import SceneSpec, make_scene

    spec = SceneSpec(11, 96, 128, 16, 1, 0.0, 4.0, 1)
    sc = make_scene(spec, 0)
    res = run_hdp_pipeline(sc.pair, GmmModel.parse(gmm_text), AggregationParams(levels=2))
    assert error_rate(res.disparity, sc.gt_left, sc.occlusion, 1) <= 2.0


def test_slabs_combine_to_full_range():
    """C5 plan on one GPU: per-slab keys min-combined == full-range result."""
    import torch

    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.distributed import slab
    from paper_1509_08197_b200.synthetic import SceneSpec, make_scene

    sc = make_scene(SceneSpec(12, 50, 70, 40, 9, 0.4, 8.0, 1), 0)
    Ld = torch.from_numpy(sc.pair.left.data[None]).cuda()
    Rd = torch.from_numpy(sc.pair.right.data[None]).cuda()
    full = E.run_baseline_batch(Ld, Rd, 40, want_keys=True)
    comb = None
    for r in range(3):
        x0, nx = slab(40, r, 3)
        k = E.run_baseline_batch(Ld, Rd, 40, x0=x0, nx=nx, want_keys=True).extra["keys"]
        from paper_1509_08197_b200.distributed import keys_to_signed

        ks = keys_to_signed(k)
        comb = ks if comb is None else torch.minimum(comb, ks)
    disp, _ = E.keys_unpack(keys_to_signed(comb))
    np.testing.assert_array_equal(disp.cpu().numpy(), full.disparity.cpu().numpy().ravel())
    # keys packed from the one-call pipeline's (disparity, cost) slabs, in int64 order
    comb = None
    for r in range(3):
        x0, nx = slab(40, r, 3)
        o = E.run_baseline_fused(Ld, Rd, 40, x0=x0, nx=nx)
        ks = E.keys_pack(o.disparity, o.min_cost, signed_order=True)
        comb = ks if comb is None else torch.minimum(comb, ks)
    disp, mc = E.keys_unpack(comb, signed_order=True)
    np.testing.assert_array_equal(disp.cpu().numpy(), full.disparity.cpu().numpy().ravel())
    np.testing.assert_array_equal(mc.cpu().numpy(), full.min_cost.cpu().numpy().ravel())


def test_pipeline_metrics_seconds_filled(gmm_text):
    """PipelineResult.metrics["seconds"] carries every stage key of the
    reference (aggregation.py:347-357, :401-416), from device events."""
    from paper_1509_08197_b200.aggregation import AggregationParams, run_baseline_pipeline, run_hdp_pipeline
    from paper_1509_08197_b200.hdp_model import GmmModel
    from paper_1509_08197_b200.raster_io import RasterImage, StereoPair

    g = golden("pipelines.npz")
    pair = StereoPair(RasterImage(g["c1_left"]), RasterImage(g["c1_right"]), 16)
    base = run_baseline_pipeline(pair, AggregationParams())
    sec = base.metrics["seconds"]
    assert set(sec) == {"forest", "cost_aggregate", "total"}
    assert sec["forest"] > 0 and sec["cost_aggregate"] > 0 and sec["total"] >= sec["cost_aggregate"]
    res = run_hdp_pipeline(pair, GmmModel.parse(gmm_text), AggregationParams(levels=2))
    sec = res.metrics["seconds"]
    assert set(sec) == {"pyramid", "predict", "forest", "cost", "aggregate", "total"}
    for k in ("pyramid", "predict", "forest", "cost", "aggregate"):
        assert sec[k] > 0, k
    for lr in res.layers:
        assert set(lr.timings) == {"cost", "aggregate"} and lr.timings["cost"] > 0


@pytest.mark.parametrize("method", ["mst", "rt", "hdp+mst", "m+hdp+rt"])
def test_run_method_dispatch(method, gmm_text):
    """evaluation.run_method (evaluation.py:154-167): the label selects the
    pipeline, tree kind and prefilter; results equal the direct calls."""
    from paper_1509_08197_b200.aggregation import AggregationParams, run_baseline_pipeline, run_hdp_pipeline
    from paper_1509_08197_b200.errors import ConfigError
    from paper_1509_08197_b200.evaluation import parse_method, run_method
    from paper_1509_08197_b200.hdp_model import GmmModel

    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene

    sc = make_scene(CONFIGS[1], 2)
    model = GmmModel.parse(gmm_text)
    params = AggregationParams(levels=2, seed=4)
    median, hdp, tree = parse_method(method)
    got = run_method(sc.pair, method, params, model=model)
    if hdp:
        want = run_hdp_pipeline(sc.pair, model, params, tree_kind=tree, median_prefilter=median)
        with pytest.raises(ConfigError):
            run_method(sc.pair, method, params)  # HDP needs the offset model
    else:
        want = run_baseline_pipeline(sc.pair, params, tree_kind=tree, median_prefilter=median)
    np.testing.assert_array_equal(got.disparity.values, want.disparity.values)
    assert got.metrics["method"] == want.metrics["method"]
    assert got.metrics["tree"] == tree and got.metrics["hdp"] == hdp
    assert got.metrics["median_prefilter"] == median


def test_forest_from_edges_rejects_cycles():
    """An edge set with a cycle, a self-loop or a repeated edge is not a
    forest: DataError instead of a non-terminating Euler tour."""
    from paper_1509_08197_b200.errors import DataError
    from paper_1509_08197_b200.spanning_forest import forest_from_edges

    tri = (np.array([0, 1, 0]), np.array([1, 2, 2]), np.ones(3))
    loop = (np.array([0, 1]), np.array([1, 1]), np.ones(2))
    dup = (np.array([0, 0]), np.array([1, 1]), np.ones(2))
    for u, v, w in (tri, loop, dup):
        with pytest.raises(DataError):
            forest_from_edges(4, u, v, w)
    ok = forest_from_edges(4, np.array([0, 1]), np.array([1, 2]), np.ones(2))
    assert ok.n_trees == 2


def test_hdp_block_size_3_matches_oracle(gmm_text):
    """block_size 3 gives non-dyadic pyramid means: the levels above 0 are
    keyed on the float64 weight order, so their forests stay the reference's."""
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.hdp_model import GmmModel
    from paper_1509_08197_b200.synthetic import SceneSpec, make_scene
    from oracle import oracle as O

    import torch

    sc = make_scene(SceneSpec(13, 90, 120, 27, 10, 0.3, 8.0, 1), 0)
    L, R = sc.pair.left.data, sc.pair.right.data
    outs = E.run_hdp_batch(torch.from_numpy(L[None]).cuda(), torch.from_numpy(R[None]).cuda(), 27, GmmModel.parse(gmm_text), levels=2,
                           block_size=3, keep=True)
    teacher = {o.level: o.disparity[0].cpu().numpy() for o in outs}
    ref = O.run_hdp(L, R, 27, O.parse_gmm(gmm_text), levels=2, s=3, teacher=teacher, keep=True)
    for o, r in zip(outs, ref):
        assert int(o.n_trees[0]) == r.n_trees and int(o.stored_entries[0]) == r.stored_entries
        ex = {k: v.cpu().numpy() for k, v in o.forest.export().items()}
        np.testing.assert_array_equal(ex["parent"], r.forest.base.parent, f"level {o.level}")
        got = o.disparity[0].cpu().numpy()
        band = (r.second_cost - r.min_cost) <= 1e-5 * np.abs(r.min_cost)
        assert not ((got != r.disparity) & ~band).any(), f"level {o.level}"


def test_evaluation_on_device_matches_reference():
    """error_rate / occlusion_from_gt / evaluate_pair on the GPU equal the
    reference's outputs (golden, evaluation.py:27-124) exactly; the batched
    device scorer equals the per-pair one."""
    import torch

    from paper_1509_08197_b200.evaluation import (error_rate, error_rates_device, evaluate_pair,
                                                  occlusion_from_gt)
    from paper_1509_08197_b200.raster_io import DisparityMap

    g = golden("evaluation.npz")
    for k in range(int(g["count"])):
        p = f"e{k}_"
        L_ = DisparityMap(values=g[p + "gl"], valid=g[p + "vl"])
        R_ = DisparityMap(values=g[p + "gr"], valid=g[p + "vr"])
        P_ = DisparityMap(values=g[p + "pred"], valid=g[p + "pv"])
        occ = occlusion_from_gt(L_, R_)
        np.testing.assert_array_equal(occ, g[p + "occ"])
        for t in (1, 2, 3):
            assert error_rate(P_, L_, None, t) == float(g[p + f"err{t}"])
            assert error_rate(P_, L_, occ, t) == float(g[p + f"err{t}_occ"])
        rep = evaluate_pair("x", "mst", P_, L_, occ)
        assert rep.n_evaluated == int(g[p + "n_eval"])
        assert rep.err_ge_1 == float(g[p + "err1_occ"]) and rep.err_ge_2 == float(g[p + "err2_occ"])
    # batched, device-resident maps (all valid) == the per-pair host calls
    pred = np.stack([np.clip(g["e0_gl"] + d, 0, 30) for d in (0, 1, -2)]).astype(np.int32)
    gt = np.stack([g["e0_gl"]] * 3).astype(np.int32)
    occ = np.stack([g["e0_occ"]] * 3)
    got = error_rates_device(torch.from_numpy(pred).cuda(), torch.from_numpy(gt).cuda(),
                             torch.from_numpy(occ.astype(np.uint8)).cuda(), (1, 2))
    for b in range(3):
        ones = np.ones(gt[b].shape, bool)
        P_ = DisparityMap(values=pred[b], valid=ones)
        G_ = DisparityMap(values=gt[b], valid=ones)
        assert got[b, 0] == error_rate(P_, G_, occ[b], 1)
        assert got[b, 1] == error_rate(P_, G_, occ[b], 2)


def test_hdpf_batches_beyond_one_launch():
    """hdp_hdpf slices batches above 255 pairs (9 pair bits in the sort key)
    over several launches on one union-find: 260 small pairs equal their
    single-pair forests."""
    import torch

    from paper_1509_08197_b200 import engine as E

    rng = np.random.default_rng(5)
    b, h, w, d = 260, 6, 7, 7
    img = torch.from_numpy(rng.integers(0, 256, size=(b, h, w, 3)).astype(np.uint8)).cuda()
    il = E.to_f64(img)
    eu, ev, ew, key, nE = E.grid_edges(il)
    rows = torch.from_numpy(rng.integers(0, 4, size=b * h * w).astype(np.int32)).cuda()
    masks = torch.from_numpy(rng.integers(1, 255, size=(b, 4, 1)).astype(np.int32)).cuda()
    in_tree, comp, tm, _ = E.hdpf(b, h * w, nE, eu, ev, key, rows, masks, 0.5)
    for i in (0, 131, 255, 259):
        sl = slice(i * nE, (i + 1) * nE)
        one = E.hdpf(1, h * w, nE, eu[sl] - i * h * w, ev[sl] - i * h * w, key[sl],
                     rows[i * h * w:(i + 1) * h * w].contiguous(), masks[i:i + 1].contiguous(), 0.5)
        assert torch.equal(one[0], in_tree[sl])
