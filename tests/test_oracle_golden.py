"""Pin the CPU oracle (oracle/) against golden vectors produced by the real
reference package (tests/golden/make_golden.py).  CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O


def test_pyramid_levels_bit_exact():
    g = golden("pyramid.npz")
    layers = O.build_pyramid(g["image"], 40, 2, 3)
    for lvl, (I, d) in enumerate(layers):
        np.testing.assert_array_equal(I, g[f"level{lvl}"])
    np.testing.assert_array_equal(O.block_mean(g["bm3_in"], 3), g["bm3"])


@pytest.mark.parametrize("tag", ["rgb", "gray"])
def test_prepare_and_cost_grid_bit_exact(tag):
    g = golden("cost.npz")
    L, R = O.prepare_layer(g[tag + "_left"]), O.prepare_layer(g[tag + "_right"])
    np.testing.assert_array_equal(L.gray, g[tag + "_gray"])
    np.testing.assert_array_equal(L.grad, g[tag + "_grad"])
    cost = g[tag + "_cost"]
    for x in range(cost.shape[0]):
        np.testing.assert_array_equal(O.cost_grid(L, R, x), cost[x])


def test_prepare_dyadic_level_bit_exact():
    g = golden("cost.npz")
    P = O.prepare_layer(g["dyadic_in"])
    np.testing.assert_array_equal(P.gray, g["dyadic_gray"])
    np.testing.assert_array_equal(P.grad, g["dyadic_grad"])


MST_CASES = ["int0", "int1", "int2", "int3", "int4", "dyadic", "ties"]


@pytest.mark.parametrize("tag", MST_CASES)
def test_edges_order_and_forest_exact(tag):
    g = golden("mst.npz")
    u, v, w = O.build_edge_list(g[tag + "_in"])
    np.testing.assert_array_equal(u, g[tag + "_u"])
    np.testing.assert_array_equal(v, g[tag + "_v"])
    np.testing.assert_array_equal(w, g[tag + "_w"])
    order = O.mst_edge_order(w)
    np.testing.assert_array_equal(order, g[tag + "_edge_order"])
    h, wd = g[tag + "_in"].shape[:2]
    for kind in ("mst", "rt"):
        o = order if kind == "mst" else O.rt_edge_order(u.size, 3)
        f = O.build_hdpf(u, v, w, h * wd, O.full_masks(h * wd, 4), 4, 0.0, o).base
        p = f"{tag}_{kind}_"
        for key in ("parent", "parent_weight", "depth", "tree_id", "order", "tree_slices"):
            np.testing.assert_array_equal(getattr(f, key), g[p + key], err_msg=key)


def test_aggregate_forest_matches_reference():
    g = golden("aggregate.npz")
    for k in range(6):
        n = int(g[f"f{k}_n"])
        f = O.bfs_forest(n, g[f"f{k}_u"], g[f"f{k}_v"], g[f"f{k}_w"])
        np.testing.assert_array_equal(f.order, g[f"f{k}_order"])
        got = O.aggregate_forest(f, g[f"f{k}_costs"], float(g[f"f{k}_gamma"]))
        # same float64 evaluation order -> bit-identical up to exp() ulps
        np.testing.assert_allclose(got, g[f"f{k}_out"], rtol=1e-14, atol=0)


def test_prior_bit_exact():
    g = golden("prior.npz")
    counts, kept = O.prior_counts(g["shift_left"], g["shift_right"], 8)
    np.testing.assert_array_equal(O.prior_from_counts(counts, kept), g["shift_prior"])
    for lvl in (0, 1):
        d = int(g[f"c1_l{lvl}_dmax"])
        counts, kept = O.prior_counts(g[f"c1_l{lvl}_left"], g[f"c1_l{lvl}_right"], d)
        np.testing.assert_array_equal(O.prior_from_counts(counts, kept), g[f"c1_l{lvl}_prior"])


def test_tables_exact(gmm_text):
    g = golden("tables.npz")
    model = O.parse_gmm(gmm_text)
    for k in range(int(g["count"])):
        lvl = int(g[f"t{k}_level"])
        cond = O.conditional(model[lvl], int(g[f"t{k}_dc"]), int(g[f"t{k}_dp"]), 2)
        np.testing.assert_array_equal(cond, g[f"t{k}_cond"])
        bm = O.bayes(cond, g[f"t{k}_prior"])
        np.testing.assert_array_equal(bm, g[f"t{k}_bayes"])
        tab = O.predict_intervals(bm, float(g[f"t{k}_delta"]))
        np.testing.assert_array_equal([t.size for t in tab], g[f"t{k}_sizes"])
        np.testing.assert_array_equal(np.concatenate(tab), g[f"t{k}_flat"])


def _table(sizes, flat):
    offs = np.concatenate(([0], np.cumsum(sizes)))
    return [flat[offs[i]:offs[i + 1]] for i in range(len(sizes))]


def test_hdpf_exact():
    g = golden("hdpf.npz")
    for k in range(int(g["count"])):
        p = f"h{k}_"
        I = g[p + "in"]
        h, w = I.shape[:2]
        d = int(g[p + "d"])
        table = _table(g[p + "tab_sizes"], g[p + "tab_flat"])
        pix = O.masks_from_rows(table, d)[g[p + "rows"]]
        u, v, wt = O.build_edge_list(I)
        f = O.build_hdpf(u, v, wt, h * w, pix, d, float(g[p + "beta"]))
        np.testing.assert_array_equal(f.base.parent, g[p + "parent"])
        np.testing.assert_array_equal(f.base.tree_id, g[p + "tree_id"])
        np.testing.assert_array_equal(f.base.depth, g[p + "depth"])
        np.testing.assert_array_equal([iv.size for iv in f.intervals], g[p + "iv_sizes"])
        np.testing.assert_array_equal(np.concatenate(f.intervals), g[p + "iv_flat"])


def test_baseline_pipeline_c1():
    g = golden("pipelines.npz")
    out = O.run_baseline(g["c1_left"], g["c1_right"], 16)
    np.testing.assert_array_equal(out.disparity, g["c1_base_disp"])
    np.testing.assert_allclose(out.min_cost, g["c1_base_cost"], rtol=1e-12, atol=0)


def test_hdp_pipeline_c1(gmm_text):
    g = golden("pipelines.npz")
    model = O.parse_gmm(gmm_text)
    outs = O.run_hdp(g["c1_left"], g["c1_right"], 16, model, levels=2)
    assert [o.level for o in outs] == [2, 1, 0]
    for o in outs:
        p = f"c1_hdp_l{o.level}_"
        np.testing.assert_array_equal(o.disparity, g[p + "disp"])
        np.testing.assert_allclose(o.min_cost, g[p + "cost"], rtol=1e-12, atol=0)
        assert o.n_trees == int(g[p + "ntrees"])
        assert o.stored_entries == int(g[p + "stored"])
        assert o.search_ratio == float(g[p + "ratio"])


def test_hdp_pipeline_full_preset(gmm_text):
    g = golden("pipelines.npz")
    model = O.parse_gmm(gmm_text)
    outs = O.run_hdp(g["s2_left"], g["s2_right"], 24, model, levels=3, size_class="full")
    for o in outs:
        p = f"s2_hdp_l{o.level}_"
        np.testing.assert_array_equal(o.disparity, g[p + "disp"])
        np.testing.assert_allclose(o.min_cost, g[p + "cost"], rtol=1e-12, atol=0)
        assert o.n_trees == int(g[p + "ntrees"])
        assert o.stored_entries == int(g[p + "stored"])


def test_evaluation_matches_reference():
    """error_rate / occlusion_from_gt restatements vs the reference's outputs."""
    g = golden("evaluation.npz")
    for k in range(int(g["count"])):
        p = f"e{k}_"
        occ = O.occlusion_from_gt(g[p + "gl"], g[p + "vl"], g[p + "gr"], g[p + "vr"])
        np.testing.assert_array_equal(occ, g[p + "occ"])
        for t in (1, 2, 3):
            assert O.error_rate(g[p + "pred"], g[p + "pv"], g[p + "gl"], g[p + "vl"], None, t) == float(g[p + f"err{t}"])
            assert O.error_rate(g[p + "pred"], g[p + "pv"], g[p + "gl"], g[p + "vl"], occ, t) == float(
                g[p + f"err{t}_occ"])


def test_oracle_reduce_order_is_numpys():
    """The oracle's add.reduce order (or_np_sum: the prior's 49-value window
    mean, the prior histogram and Bayes row sums) against numpy itself."""
    import ctypes as C

    f = O.lib().or_np_sum
    f.restype = C.c_double
    f.argtypes = [C.c_void_p, C.c_int64]
    rng = np.random.default_rng(5)
    for n in (1, 3, 7, 8, 9, 49, 81, 121, 128, 129, 241, 300):
        a = rng.uniform(-1, 1, (64, n)) * rng.uniform(0, 1e3, (64, 1))
        want = a.sum(axis=-1)
        got = np.array([f(np.ascontiguousarray(r).ctypes.data, n) for r in a])
        np.testing.assert_array_equal(got, want, err_msg=f"n={n}")
