"""Generate golden vectors by running the REAL reference package.

Run once in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``treestereo`` read-only from /root/reference/pkg/src (with a
``sys.modules`` stub for matplotlib, which only the reference's CLI/figures
import) and writes small .npz fixtures next to this script.  Nothing on the GPU
box reads /root/reference: tests load only the committed fixtures.
"""

from __future__ import annotations

import os
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
_mpl = types.ModuleType("matplotlib")
_mpl.use = lambda *a, **k: None
sys.modules.setdefault("matplotlib", _mpl)
sys.modules.setdefault("matplotlib.pyplot", types.ModuleType("matplotlib.pyplot"))

from treestereo import aggregation as ref_agg  # noqa: E402
from treestereo import cost_volume as ref_cost  # noqa: E402
from treestereo import hdp_forest as ref_hf  # noqa: E402
from treestereo import hdp_model as ref_hm  # noqa: E402
from treestereo import pyramid as ref_pyr  # noqa: E402
from treestereo import spanning_forest as ref_sf  # noqa: E402
from treestereo.raster_io import RasterImage, StereoPair  # noqa: E402

from paper_1509_08197_b200.synthetic import CONFIGS, make_scene  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, sum(a.nbytes for a in arrays.values() if hasattr(a, "nbytes")), "bytes raw")


def ref_pair(left_u8, right_u8, d_max):
    return StereoPair(RasterImage(left_u8), RasterImage(right_u8), d_max)


def forest_arrays(prefix, f):
    return {
        prefix + "parent": f.parent, prefix + "parent_weight": f.parent_weight,
        prefix + "depth": f.depth, prefix + "tree_id": f.tree_id, prefix + "order": f.order,
        prefix + "tree_slices": f.tree_slices, prefix + "child_start": f.child_start,
        prefix + "child_list": f.child_list,
    }


def gen_pyramid():
    rng = np.random.default_rng(11)
    img = rng.integers(0, 256, size=(37, 53, 3), dtype=np.uint8)
    pyr = ref_pyr.build_pyramid(RasterImage(img), d_max=40, block_size=2, levels=3)
    vals = rng.uniform(0, 255, size=(9, 10, 3))
    out = {"image": img, "bm3": ref_pyr.block_mean(vals, 3), "bm3_in": vals}
    for layer in pyr:
        out[f"level{layer.level}"] = layer.intensities
    save("pyramid.npz", **out)


def gen_cost():
    rng = np.random.default_rng(12)
    out = {}
    for tag, (h, w, c, d) in {"rgb": (20, 33, 3, 9), "gray": (7, 12, 1, 4)}.items():
        li = rng.integers(0, 256, size=(h, w, c)).astype(np.float64)
        ri = rng.integers(0, 256, size=(h, w, c)).astype(np.float64)
        L = ref_pyr.PyramidLayer(0, li, d)
        R = ref_pyr.PyramidLayer(0, ri, d)
        pl, pr = ref_cost.prepare_layer(L), ref_cost.prepare_layer(R)
        out[tag + "_left"] = li
        out[tag + "_right"] = ri
        out[tag + "_gray"] = pl.gray
        out[tag + "_grad"] = pl.grad
        out[tag + "_cost"] = np.stack(
            [ref_cost.cost_grid(pl, pr, x, ref_cost.CostParams()) for x in range(d + 1)])
    # a dyadic pyramid level (level 2 of a random image): gray through BLAS
    img = rng.integers(0, 256, size=(40, 56, 3), dtype=np.uint8)
    lvl = ref_pyr.build_pyramid(RasterImage(img), d_max=16, levels=2)[2]
    pl = ref_cost.prepare_layer(lvl)
    out["dyadic_in"] = lvl.intensities
    out["dyadic_gray"] = pl.gray
    out["dyadic_grad"] = pl.grad
    save("cost.npz", **out)


def gen_mst():
    rng = np.random.default_rng(13)
    out = {}
    cases = []
    for k, (h, w) in enumerate([(6, 9), (17, 23), (31, 40), (1, 12), (12, 1)]):
        data = rng.integers(0, 256, size=(h, w, 3)).astype(np.float64)
        cases.append((f"int{k}", data))
    img = rng.integers(0, 256, size=(64, 80, 3), dtype=np.uint8)
    lvl = ref_pyr.build_pyramid(RasterImage(img), d_max=16, levels=2)[2]
    cases.append(("dyadic", lvl.intensities))
    # a low-contrast image: many equal weights, the tie-break matters
    flat = rng.integers(100, 103, size=(25, 30, 3)).astype(np.float64)
    cases.append(("ties", flat))
    for tag, data in cases:
        layer = ref_pyr.PyramidLayer(0, data, 4)
        edges = ref_sf.build_edge_list(layer)
        out[tag + "_in"] = data
        out[tag + "_u"], out[tag + "_v"], out[tag + "_w"] = edges.u, edges.v, edges.weight
        out[tag + "_edge_order"] = ref_sf.mst_edge_order(edges)
        out.update(forest_arrays(tag + "_mst_", ref_sf.build_forest(edges, "mst")))
        out.update(forest_arrays(tag + "_rt_", ref_sf.build_forest(edges, "rt", seed=3)))
    save("mst.npz", **out)


def gen_aggregate():
    rng = np.random.default_rng(14)
    out = {}
    for k in range(6):
        n = int(rng.integers(2, 40))
        us, vs, ws = [], [], []
        for node in range(1, n):
            if rng.uniform() < 0.85:
                us.append(int(rng.integers(0, node)))
                vs.append(node)
                ws.append(float(rng.uniform(0.0, 255.0)))
        u, v, w = np.array(us, np.int64), np.array(vs, np.int64), np.array(ws)
        f = ref_sf.forest_from_edges(n, u, v, w)
        m = int(rng.integers(1, 6))
        costs = rng.uniform(0.0, 1.0, size=(n, m))
        gamma = float(rng.uniform(0.05, 1.0))
        out[f"f{k}_n"] = np.array(n)
        out[f"f{k}_u"], out[f"f{k}_v"], out[f"f{k}_w"] = u, v, w
        out[f"f{k}_costs"] = costs
        out[f"f{k}_gamma"] = np.array(gamma)
        out[f"f{k}_out"] = ref_agg.aggregate_forest(f, costs, gamma)
        out.update(forest_arrays(f"f{k}_", f))
    save("aggregate.npz", **out)


def gen_prior():
    rng = np.random.default_rng(15)
    out = {}
    base = rng.integers(0, 256, size=(40, 60, 3)).astype(np.float64)
    right = np.roll(base, -3, axis=1)
    L = ref_pyr.PyramidLayer(0, base, 8)
    R = ref_pyr.PyramidLayer(0, right, 8)
    out["shift_left"], out["shift_right"] = base, right
    out["shift_prior"] = ref_hm.estimate_prior(L, R, ref_cost.CostParams())
    sc = make_scene(CONFIGS[1], 0)
    pyr = ref_pyr.build_pyramid_pair(sc.pair, 2, 2)
    for lvl in (0, 1):
        out[f"c1_l{lvl}_left"] = pyr.left[lvl].intensities
        out[f"c1_l{lvl}_right"] = pyr.right[lvl].intensities
        out[f"c1_l{lvl}_prior"] = ref_hm.estimate_prior(pyr.left[lvl], pyr.right[lvl])
        out[f"c1_l{lvl}_dmax"] = np.array(pyr.left[lvl].d_max)
    save("prior.npz", **out)


def gen_tables(model):
    rng = np.random.default_rng(16)
    out = {}
    k = 0
    for lvl, (dc, dp) in enumerate([(16, 8), (40, 20), (120, 60), (30, 15), (7, 3)]):
        mix = model.layers[lvl]
        cond = ref_hm.conditional_parent_given_child(mix, dc, dp, 2)
        prior = rng.dirichlet(np.full(dc + 1, 0.5))
        if k % 2:
            prior = np.full(dc + 1, 1.0 / (dc + 1))
        bay = ref_hm.bayes_child_given_parent(cond, prior)
        for delta in (0.004 * 2**lvl, 0.064 * 2**lvl):
            tab = ref_hm.predict_intervals(bay, delta)
            out[f"t{k}_level"] = np.array(lvl)
            out[f"t{k}_dc"], out[f"t{k}_dp"] = np.array(dc), np.array(dp)
            out[f"t{k}_prior"] = prior
            out[f"t{k}_delta"] = np.array(delta)
            out[f"t{k}_cond"] = cond.matrix
            out[f"t{k}_bayes"] = bay.matrix
            out[f"t{k}_sizes"] = tab.sizes()
            out[f"t{k}_flat"] = np.concatenate(tab.intervals)
            k += 1
    out["count"] = np.array(k)
    save("tables.npz", **out)


def gen_pipelines(model):
    out = {}
    sc = make_scene(CONFIGS[1], 0)
    out["c1_left"], out["c1_right"] = sc.pair.left.data, sc.pair.right.data
    base = ref_agg.run_baseline_pipeline(sc.pair, ref_agg.AggregationParams())
    out["c1_base_disp"] = base.disparity.values
    out["c1_base_cost"] = base.layers[0].min_cost
    forests = {}
    hdp = ref_agg.run_hdp_pipeline(sc.pair, model, ref_agg.AggregationParams(levels=2),
                                   on_forest=lambda lvl, f: forests.__setitem__(lvl, f))
    for lr in hdp.layers:
        p = f"c1_hdp_l{lr.level}_"
        out[p + "disp"] = lr.disparity.values
        out[p + "cost"] = lr.min_cost
        out[p + "ratio"] = np.array(lr.search_ratio)
        out[p + "ntrees"] = np.array(lr.n_trees)
        out[p + "stored"] = np.array(lr.stored_entries)
        f = forests[lr.level]
        out[p + "tree_id"] = f.base.tree_id
        out[p + "parent"] = f.base.parent
        out[p + "depth"] = f.base.depth
        out[p + "iv_sizes"] = np.array([iv.size for iv in f.intervals], np.int64)
        out[p + "iv_flat"] = np.concatenate(f.intervals)
    # a second, smaller scene with levels=3 and the full preset
    sc2 = make_scene(CONFIGS[2].__class__(9, 72, 100, 24, 12, 0.3, 8.0, 1), 0)
    out["s2_left"], out["s2_right"] = sc2.pair.left.data, sc2.pair.right.data
    hdp2 = ref_agg.run_hdp_pipeline(sc2.pair, model,
                                    ref_agg.AggregationParams(levels=3, size_class="full"))
    for lr in hdp2.layers:
        p = f"s2_hdp_l{lr.level}_"
        out[p + "disp"] = lr.disparity.values
        out[p + "cost"] = lr.min_cost
        out[p + "ratio"] = np.array(lr.search_ratio)
        out[p + "ntrees"] = np.array(lr.n_trees)
        out[p + "stored"] = np.array(lr.stored_entries)
    save("pipelines.npz", **out)


def gen_hdpf():
    """build_hdpf on hand-made interval maps with live-mask effects."""
    rng = np.random.default_rng(17)
    out = {}
    k = 0
    for h, w, d, beta in [(10, 12, 6, 0.4), (24, 31, 9, 0.6), (33, 20, 20, 0.95), (16, 16, 70, 0.5)]:
        data = rng.integers(0, 256, size=(h, w, 3)).astype(np.float64)
        layer = ref_pyr.PyramidLayer(0, data, d)
        edges = ref_sf.build_edge_list(layer)
        n_rows = max(2, d // 2)
        table = []
        for _ in range(n_rows):
            lo = int(rng.integers(0, d))
            size = int(rng.integers(1, 5))
            table.append(sorted(set(min(d, lo + t) for t in range(size))))
        ph, pw = -(-h // 2), -(-w // 2)
        prow = rng.integers(0, n_rows, size=(ph, pw))
        rows = prow[np.arange(h)[:, None] // 2, np.arange(w)[None, :] // 2].ravel()
        ivs = tuple(np.array(t, np.int64) for t in table)
        masks = tuple(sum(1 << x for x in t) for t in table)
        pim = ref_hf.PixelIntervalMap(h, w, d, rows.astype(np.int64), ivs, masks)
        f = ref_hf.build_hdpf(edges, pim, "mst", 0, beta)
        p = f"h{k}_"
        out[p + "in"] = data
        out[p + "rows"] = rows
        out[p + "tab_sizes"] = np.array([len(t) for t in table], np.int64)
        out[p + "tab_flat"] = np.concatenate([np.array(t, np.int64) for t in table])
        out[p + "d"], out[p + "beta"] = np.array(d), np.array(beta)
        out[p + "parent"], out[p + "tree_id"], out[p + "depth"] = f.base.parent, f.base.tree_id, f.base.depth
        out[p + "iv_sizes"] = np.array([iv.size for iv in f.intervals], np.int64)
        out[p + "iv_flat"] = np.concatenate(f.intervals)
        k += 1
    out["count"] = np.array(k)
    save("hdpf.npz", **out)


def gen_evaluation():
    """error_rate / occlusion_from_gt / evaluate_pair (evaluation.py:27-124)
    on random maps with validity holes and on a synthetic scene's ground truth."""
    from treestereo import evaluation as ref_ev
    from treestereo.raster_io import DisparityMap

    rng = np.random.default_rng(77)
    out = {}
    for k in range(4):
        h, w = int(rng.integers(20, 60)), int(rng.integers(20, 70))
        gl = rng.integers(0, 16, size=(h, w)).astype(np.int32)
        gr = np.clip(gl + rng.integers(-2, 3, size=(h, w)), 0, 15).astype(np.int32)
        vl = rng.uniform(size=(h, w)) < 0.85
        vr = rng.uniform(size=(h, w)) < 0.85
        pred = np.clip(gl + rng.integers(-4, 5, size=(h, w)), 0, 20).astype(np.int32)
        pv = rng.uniform(size=(h, w)) < 0.95
        L_ = DisparityMap(values=gl, valid=vl)
        R_ = DisparityMap(values=gr, valid=vr)
        P_ = DisparityMap(values=pred, valid=pv)
        occ = ref_ev.occlusion_from_gt(L_, R_)
        p = f"e{k}_"
        out.update({p + "gl": gl, p + "gr": gr, p + "vl": vl, p + "vr": vr, p + "pred": pred, p + "pv": pv,
                    p + "occ": occ})
        for t in (1, 2, 3):
            out[p + f"err{t}"] = np.array(ref_ev.error_rate(P_, L_, None, t))
            out[p + f"err{t}_occ"] = np.array(ref_ev.error_rate(P_, L_, occ, t))
        rep = ref_ev.evaluate_pair("x", "mst", P_, L_, occ)
        out[p + "n_eval"] = np.array(rep.n_evaluated)
    out["count"] = np.array(4)
    save("evaluation.npz", **out)


def main():
    if len(sys.argv) > 1:  # regenerate only the named fixtures: make_golden.py evaluation ...
        for name in sys.argv[1:]:
            globals()["gen_" + name]()
        return
    src = "/root/reference/pkg/src/treestereo/data/default.gmm"
    with open(src) as fh:
        text = fh.read()
    with open(os.path.join(HERE, "default.gmm"), "w") as fh:
        fh.write(text)
    model = ref_hm.GmmModel.parse(text)
    gen_pyramid()
    gen_cost()
    gen_mst()
    gen_aggregate()
    gen_prior()
    gen_tables(model)
    gen_hdpf()
    gen_pipelines(model)
    gen_evaluation()


if __name__ == "__main__":
    main()
