"""Edge cases of the hot path against the oracle: gray (1-channel) pairs,
degenerate geometries (one row, one column, one pixel), the minimum disparity
range, a constant image (every edge weight tied: the MST is decided by the
edge index alone), HDP over random trees at the C2 size, and the API's
empty-batch / geometry errors.  Same parity rule as test_gpu_pipeline.py."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import cuda_available
from test_gpu_pipeline import assert_cost_parity, assert_disp_parity, dev

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


def _dense_vs_oracle(L, R, d, what, kind="mst"):
    from paper_1509_08197_b200 import engine as E
    from oracle import oracle as O

    out = E.run_baseline_batch(dev(L[None]), dev(R[None]), d, tree_kind=kind, keep_forest=True)
    ref = O.run_baseline(L, R, d, tree_kind=kind)
    got = out.disparity[0].cpu().numpy()
    assert_disp_parity(got, ref.disparity, ref.min_cost, ref.second_cost, what)
    same = got == ref.disparity
    assert_cost_parity(out.min_cost[0].cpu().numpy()[same], ref.min_cost[same], what)
    ex = {k: v.cpu().numpy() for k, v in out.forest.export().items()}
    np.testing.assert_array_equal(ex["parent"], ref.forest.base.parent, what)
    np.testing.assert_array_equal(ex["depth"], ref.forest.base.depth, what)
    return out, ref


@pytest.mark.parametrize("shape", [(1, 57), (43, 1), (1, 1), (2, 2), (3, 40)])
def test_degenerate_geometries(shape):
    rng = np.random.default_rng(sum(shape))
    h, w = shape
    L = rng.integers(0, 256, size=(h, w, 3)).astype(np.uint8)
    R = np.roll(L, -1, axis=1)
    _dense_vs_oracle(L, R, max(1, min(5, w - 1)), f"{h}x{w}")


def test_gray_pairs_dense_and_hdp(gmm_text):
    """1-channel images (RasterImage allows C in {1, 3}) through both pipelines."""
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.hdp_model import GmmModel
    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene
    from oracle import oracle as O

    sc = make_scene(CONFIGS[1], 4)
    L = sc.pair.left.data.mean(axis=2, keepdims=True).round().astype(np.uint8)
    R = sc.pair.right.data.mean(axis=2, keepdims=True).round().astype(np.uint8)
    _dense_vs_oracle(L, R, 16, "gray dense")
    outs = E.run_hdp_batch(dev(L[None]), dev(R[None]), 16, GmmModel.parse(gmm_text), levels=2)
    teacher = {o.level: o.disparity[0].cpu().numpy() for o in outs}
    ref = O.run_hdp(L, R, 16, O.parse_gmm(gmm_text), levels=2, teacher=teacher)
    for o, r in zip(outs, ref):
        assert int(o.n_trees[0]) == r.n_trees and int(o.stored_entries[0]) == r.stored_entries
        assert_disp_parity(o.disparity[0].cpu().numpy(), r.disparity, r.min_cost, r.second_cost,
                           f"gray HDP level {o.level}")


def test_minimum_disparity_range():
    from paper_1509_08197_b200.synthetic import SceneSpec, make_scene

    sc = make_scene(SceneSpec(15, 40, 60, 1, 5, 0.0, 8.0, 1), 0)
    _dense_vs_oracle(sc.pair.left.data, sc.pair.right.data, 1, "d_max 1")


@pytest.mark.parametrize("kind", ["mst", "st"])
def test_constant_image_ties(kind):
    """Every edge weight is 0: Kruskal's stable order is the edge index, which
    the device keys (weight bits << 32 | index) reproduce exactly."""
    L = np.full((37, 53, 3), 117, np.uint8)
    R = L.copy()
    R[:, :10] = 3
    _dense_vs_oracle(L, R, 9, f"constant image {kind}", kind)


def test_hdp_rt_c2_teacher_forced(gmm_text):
    """HDP over random spanning trees at the C2 size (3 levels)."""
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.hdp_model import GmmModel
    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene
    from oracle import oracle as O

    spec = CONFIGS[2]
    sc = make_scene(spec, 5)
    L, R = sc.pair.left.data, sc.pair.right.data
    outs = E.run_hdp_batch(dev(L[None]), dev(R[None]), spec.d_max, GmmModel.parse(gmm_text), levels=3,
                           tree_kind="rt", seed=11)
    teacher = {o.level: o.disparity[0].cpu().numpy() for o in outs}
    ref = O.run_hdp(L, R, spec.d_max, O.parse_gmm(gmm_text), levels=3, teacher=teacher, tree_kind="rt", seed=11)
    for o, r in zip(outs, ref):
        assert int(o.n_trees[0]) == r.n_trees and int(o.stored_entries[0]) == r.stored_entries
        assert_disp_parity(o.disparity[0].cpu().numpy(), r.disparity, r.min_cost, r.second_cost,
                           f"RT HDP level {o.level}")


def test_api_rejects_empty_and_mixed_batches():
    from paper_1509_08197_b200.aggregation import run_baseline_pipeline_batch
    from paper_1509_08197_b200.errors import DataError
    from paper_1509_08197_b200.synthetic import CONFIGS, SceneSpec, make_scene

    with pytest.raises(DataError):
        run_baseline_pipeline_batch([])
    a = make_scene(CONFIGS[1], 0).pair
    b = make_scene(SceneSpec(16, 40, 60, 16, 5, 0.0, 8.0, 1), 0).pair
    with pytest.raises(DataError):
        run_baseline_pipeline_batch([a, b])
