"""Full-size parity: the BASELINE configurations' own image sizes against the
CPU oracle.  At these sizes the aggregation runs every path of its layout
(multi-phase short-path chunks, long paths cut into many segments chained by
look-back, light children gathered on both), which the small fixtures of
test_gpu_pipeline.py only partly reach.  Same parity rule as there.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import cuda_available
from test_gpu_pipeline import assert_cost_parity, assert_disp_parity, dev

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


@pytest.mark.parametrize("cid", [2, 3])
def test_dense_fullsize_pair_matches_oracle(cid):
    """C2 (463x370, d 80) and C3 (695x555, d 120) scenes, dense MST, batched
    with a second pair so node ids and rows span two images."""
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.synthetic import CONFIGS, make_batch
    from oracle import oracle as O

    spec = CONFIGS[cid]
    scenes = make_batch(cid, 2)
    L = np.stack([s.pair.left.data for s in scenes])
    R = np.stack([s.pair.right.data for s in scenes])
    out = E.run_baseline_batch(dev(L), dev(R), spec.d_max)
    ref = O.run_baseline(L[0], R[0], spec.d_max)
    got = out.disparity[0].cpu().numpy()
    ties = assert_disp_parity(got, ref.disparity, ref.min_cost, ref.second_cost, f"C{cid} pair 0")
    same = got == ref.disparity
    assert_cost_parity(out.min_cost[0].cpu().numpy()[same], ref.min_cost[same], f"C{cid} costs")
    assert ties <= 1e-4 * got.size


def test_hdp_c2_size_teacher_forced(gmm_text):
    """C2-size pair through the 3-level HDP pipeline (half preset), each level
    against the oracle fed the GPU's coarser map."""
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.hdp_model import GmmModel
    from paper_1509_08197_b200.synthetic import CONFIGS, make_batch
    from oracle import oracle as O

    spec = CONFIGS[2]
    sc = make_batch(2, 1)[0]
    L, R = sc.pair.left.data, sc.pair.right.data
    model = GmmModel.parse(gmm_text)
    outs = E.run_hdp_batch(dev(L[None]), dev(R[None]), spec.d_max, model, levels=3)
    teacher = {o.level: o.disparity[0].cpu().numpy() for o in outs}
    ref = O.run_hdp(L, R, spec.d_max, O.parse_gmm(gmm_text), levels=3, teacher=teacher)
    for o, r in zip(outs, ref):
        assert o.level == r.level
        assert int(o.n_trees[0]) == r.n_trees, f"level {o.level} tree count"
        assert int(o.stored_entries[0]) == r.stored_entries, f"level {o.level} entries"
        got = o.disparity[0].cpu().numpy()
        assert_disp_parity(got, r.disparity, r.min_cost, r.second_cost, f"level {o.level}")


def test_dense_wide_rows_match_oracle():
    """C5-style rows (d_max 512, 513 lanes: wider than one 32-float4 column
    group) on a smaller image: the per-path short kernels and the segment
    scans with several column groups and 64-bit key minima."""
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.synthetic import SceneSpec, make_scene
    from oracle import oracle as O

    sc = make_scene(SceneSpec(5, 120, 720, 512, 24, 0.4, 8.0, 1), 0)
    L, R = sc.pair.left.data, sc.pair.right.data
    out = E.run_baseline_batch(dev(L[None]), dev(R[None]), 512)
    ref = O.run_baseline(L, R, 512)
    got = out.disparity[0].cpu().numpy()
    assert_disp_parity(got, ref.disparity, ref.min_cost, ref.second_cost, "d512")
    same = got == ref.disparity
    assert_cost_parity(out.min_cost[0].cpu().numpy()[same], ref.min_cost[same], "d512 costs")


def test_dense_giant_tree_matches_oracle():
    """One 600x1000 pair (600 k nodes, one tree): the Euler-tour ranking takes
    the synchronous rounds here (a single ruler chain above 64 k rulers, as at
    C5), the smaller configurations the asynchronous jumps."""
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.synthetic import SceneSpec, make_scene
    from oracle import oracle as O

    sc = make_scene(SceneSpec(5, 600, 1000, 12, 40, 0.3, 8.0, 1), 0)
    out = E.run_baseline_batch(dev(sc.pair.left.data[None]), dev(sc.pair.right.data[None]), 12)
    ref = O.run_baseline(sc.pair.left.data, sc.pair.right.data, 12)
    got = out.disparity[0].cpu().numpy()
    assert_disp_parity(got, ref.disparity, ref.min_cost, ref.second_cost, "giant tree")
    same = got == ref.disparity
    assert_cost_parity(out.min_cost[0].cpu().numpy()[same], ref.min_cost[same], "giant tree costs")
