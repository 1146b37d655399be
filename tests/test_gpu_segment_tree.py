"""Segment tree (tree_kind "st").

The reference does NOT implement it (edge_order rejects "st",
spanning_forest.py:115-120; SPEC.md:14 names it an extension point), so these
tests check the GPU against the oracle's own restatement of the published
construction (oracle/hdp_oracle.c or_hdpf_st: subtrees grown in Kruskal order
under w <= min(Int(Ta) + k/|Ta|, Int(Tb) + k/|Tb|), then linked in the same
order) -- PARITY UNPINNED against the reference.  The GPU builds pass 1 with
the conflict-group kernel (k_grp<true>) and pass 2 with Boruvka on the subtree
graph (dense) or k_grp again (HDP levels); trees, intervals and counts must be
identical, disparities within the tie band.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import cuda_available
from test_gpu_pipeline import assert_cost_parity, assert_disp_parity, dev

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


def _forest_equal(ex, base, what):
    np.testing.assert_array_equal(ex["parent"], base.parent, what)
    np.testing.assert_array_equal(ex["depth"], base.depth, what)
    np.testing.assert_array_equal(ex["tree_id"], base.tree_id, what)


@pytest.mark.parametrize("cid,index", [(1, 0), (2, 2)])
def test_st_dense_tree_and_disparity(cid, index):
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene
    from oracle import oracle as O

    spec = CONFIGS[cid]
    sc = make_scene(spec, index)
    L, R = sc.pair.left.data, sc.pair.right.data
    out = E.run_baseline_batch(dev(L[None]), dev(R[None]), spec.d_max, tree_kind="st", keep_forest=True)
    ref = O.run_baseline(L, R, spec.d_max, tree_kind="st")
    ex = {k: v.cpu().numpy() for k, v in out.forest.export().items()}
    _forest_equal(ex, ref.forest.base, f"C{cid} ST tree")
    assert int(out.n_trees[0]) == ref.n_trees == 1
    got = out.disparity[0].cpu().numpy()
    assert_disp_parity(got, ref.disparity, ref.min_cost, ref.second_cost, f"C{cid} ST")
    same = got == ref.disparity
    assert_cost_parity(out.min_cost[0].cpu().numpy()[same], ref.min_cost[same], f"C{cid} ST costs")
    # a different tree from the MST (the criterion does change the tree)
    mst = O.build_forest_mst(np.asarray(L, np.float64)).base
    assert (mst.parent != ref.forest.base.parent).any()


def test_st_batch_matches_per_pair():
    """Pairs of a batch get exactly their own single-pair segment trees."""
    import torch

    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.synthetic import SceneSpec, make_scene

    spec = SceneSpec(7, 61, 83, 20, 10, 0.3, 8.0, 3)
    scenes = [make_scene(spec, i) for i in range(3)]
    L = np.stack([s.pair.left.data for s in scenes])
    R = np.stack([s.pair.right.data for s in scenes])
    out = E.run_baseline_batch(dev(L), dev(R), 20, tree_kind="st")
    for i in range(3):
        one = E.run_baseline_batch(dev(L[i:i + 1]), dev(R[i:i + 1]), 20, tree_kind="st")
        assert torch.equal(one.disparity[0], out.disparity[i])


def test_st_build_forest_api():
    """spanning_forest.build_forest(edges, "st") (the extension point) on an
    arbitrary edge list == the oracle's segment tree."""
    from paper_1509_08197_b200.pyramid import PyramidLayer
    from paper_1509_08197_b200.spanning_forest import build_edge_list, build_forest
    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene
    from oracle import oracle as O

    sc = make_scene(CONFIGS[1], 3)
    I = sc.pair.left.data.astype(np.float64)
    edges = build_edge_list(PyramidLayer(0, I, 16))
    f = build_forest(edges, "st")
    u, v, wt = O.build_edge_list(I)
    ref = O.build_hdpf(u, v, wt, I.shape[0] * I.shape[1], O.full_masks(I.shape[0] * I.shape[1], 0), 0, 0.0,
                       O.mst_edge_order(wt), O.ST_K).base
    np.testing.assert_array_equal(f.parent, ref.parent)
    np.testing.assert_array_equal(f.depth, ref.depth)


@pytest.mark.parametrize("cid,index,levels,size_class", [(1, 1, 2, "half"), (3, 28, 4, "half")])
def test_st_hdp_teacher_forced(cid, index, levels, size_class, gmm_text):
    """HDP over segment trees (configs C3/C4 name "segment tree + HDP"): the
    top level is the plain segment tree, finer levels the segment-tree HDPF;
    teacher-forced per level against the oracle, forests exact."""
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.aggregation import SIZE_CLASS_PRESETS
    from paper_1509_08197_b200.hdp_model import GmmModel
    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene
    from oracle import oracle as O

    spec = CONFIGS[cid]
    sc = make_scene(spec, index)
    L, R = sc.pair.left.data, sc.pair.right.data
    pre = SIZE_CLASS_PRESETS[size_class]
    outs = E.run_hdp_batch(dev(L[None]), dev(R[None]), spec.d_max, GmmModel.parse(gmm_text), levels=levels,
                           delta0=pre["delta0"], beta=pre["beta"], tree_kind="st", keep=True)
    teacher = {o.level: o.disparity[0].cpu().numpy() for o in outs}
    ref = O.run_hdp(L, R, spec.d_max, O.parse_gmm(gmm_text), levels=levels, size_class=size_class,
                    teacher=teacher, tree_kind="st", keep=True)
    for o, r in zip(outs, ref):
        ex = {k: v.cpu().numpy() for k, v in o.forest.export().items()}
        _forest_equal(ex, r.forest.base, f"level {o.level}")
        assert int(o.n_trees[0]) == r.n_trees and int(o.stored_entries[0]) == r.stored_entries
        got = o.disparity[0].cpu().numpy()
        assert_disp_parity(got, r.disparity, r.min_cost, r.second_cost, f"ST HDP level {o.level}")
