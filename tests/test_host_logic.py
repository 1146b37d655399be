"""Host-side logic of the drop-in (CPU only): the interval-table control
plane against the reference's golden tables, parameter validation, method
dispatch, the synthetic generator and the multi-GPU key packing."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O
from paper_1509_08197_b200 import engine as E
from paper_1509_08197_b200.aggregation import SIZE_CLASS_PRESETS, AggregationParams
from paper_1509_08197_b200.distributed import keys_to_signed, pack_keys_host, shard, slab
from paper_1509_08197_b200.errors import ConfigError, DataError
from paper_1509_08197_b200.evaluation import error_rate, parse_method
from paper_1509_08197_b200.hdp_model import (ConditionalMatrix, GmmModel, Mixture1D,
                                             bayes_child_given_parent,
                                             conditional_parent_given_child, predict_intervals)
from paper_1509_08197_b200.raster_io import DisparityMap, RasterImage, StereoPair
from paper_1509_08197_b200.synthetic import CONFIGS, SceneSpec, make_scene


def test_tables_match_reference_bit_exact(gmm_text):
    g = golden("tables.npz")
    model = GmmModel.parse(gmm_text)
    for k in range(int(g["count"])):
        lvl = int(g[f"t{k}_level"])
        cond = conditional_parent_given_child(model.layers[lvl], int(g[f"t{k}_dc"]),
                                              int(g[f"t{k}_dp"]), 2)
        np.testing.assert_array_equal(cond.matrix, g[f"t{k}_cond"])
        bm = bayes_child_given_parent(cond, g[f"t{k}_prior"])
        np.testing.assert_array_equal(bm.matrix, g[f"t{k}_bayes"])
        tab = predict_intervals(bm, float(g[f"t{k}_delta"]))
        np.testing.assert_array_equal(tab.sizes(), g[f"t{k}_sizes"])
        np.testing.assert_array_equal(np.concatenate(tab.intervals), g[f"t{k}_flat"])


def test_batched_tables_equal_per_pair(gmm_text):
    model = GmmModel.parse(gmm_text)
    rng = np.random.default_rng(3)
    cond = E.conditional_matrix(model.layers[0], 80, 40, 2)
    priors = rng.dirichlet(np.full(81, 0.3), size=5)
    priors[2] = 1.0 / 81
    bm, _ = E.bayes_batched(cond, priors)
    chosen = E.predict_masks(bm, 0.064)
    for i in range(5):
        ref = O.predict_intervals(O.bayes(O.conditional(
            (model.layers[0].weights, model.layers[0].means, model.layers[0].sigmas), 80, 40, 2),
            priors[i]), 0.064)
        got = [np.flatnonzero(r) for r in chosen[i]]
        assert all(np.array_equal(a, b) for a, b in zip(got, ref))


def test_predict_interval_hand_examples():
    row = ConditionalMatrix(np.array([[0.5, 0.3, 0.2]]), "child_given_parent")
    assert predict_intervals(row, 0.2).intervals[0].tolist() == [0, 1, 2]
    assert predict_intervals(row, 0.3).intervals[0].tolist() == [0, 1]
    assert predict_intervals(row, 0.9).intervals[0].tolist() == [0]
    tie = ConditionalMatrix(np.array([[0.25, 0.25, 0.5]]), "child_given_parent")
    assert predict_intervals(tie, 0.3).intervals[0].tolist() == [0, 2]
    with pytest.raises(ConfigError):
        predict_intervals(tie, 0.0)


def test_pack_masks_roundtrip():
    rng = np.random.default_rng(0)
    chosen = rng.uniform(size=(3, 7, 81)) < 0.2
    words = E.pack_masks(chosen)
    assert words.shape == (3, 7, 3)
    for b in range(3):
        for r in range(7):
            bits = [wi * 32 + k for wi in range(3) for k in range(32)
                    if (int(words[b, r, wi]) >> k) & 1]
            assert bits == np.flatnonzero(chosen[b, r]).tolist()


def test_gmm_parse_save_roundtrip(tmp_path, gmm_text):
    model = GmmModel.parse(gmm_text)
    assert model.n_layers == 5
    p = tmp_path / "m.gmm"
    model.save(p)
    again = GmmModel.load(p)
    for a, b in zip(model.layers, again.layers):
        np.testing.assert_array_equal(a.weights, b.weights)
        np.testing.assert_array_equal(a.sigmas, b.sigmas)
    with pytest.raises(DataError):
        GmmModel.parse("version 2\n")
    with pytest.raises(ConfigError):
        Mixture1D(np.ones(2), np.zeros(2), np.array([1.0, 0.0]))


def test_params_resolution_and_validation():
    r = AggregationParams().resolved()
    assert (r.delta0, r.beta) == (SIZE_CLASS_PRESETS["half"]["delta0"],
                                  SIZE_CLASS_PRESETS["half"]["beta"])
    assert (AggregationParams(size_class="full").resolved().delta0,) == (0.004,)
    for bad in (dict(size_class="tiny"), dict(beta=1.5), dict(gamma=0.0), dict(delta0=1.0)):
        with pytest.raises(ConfigError):
            AggregationParams(**bad).resolved()


def test_parse_method():
    assert parse_method("hdp+mst") == (False, True, "mst")
    assert parse_method("m+hdp+rt") == (True, True, "rt")
    assert parse_method("mst") == (False, False, "mst")
    # the segment tree: the extension the reference names but rejects
    assert parse_method("m+hdp+st") == (True, True, "st")
    with pytest.raises(ConfigError):
        parse_method("xt")


def test_boundary_types_validate():
    with pytest.raises(DataError):
        RasterImage(np.zeros((4, 4), np.uint8))
    img = RasterImage(np.zeros((4, 4, 3), np.uint8))
    with pytest.raises(ConfigError):
        StereoPair(img, img, 0)
    with pytest.raises(DataError):
        StereoPair(img, RasterImage(np.zeros((4, 5, 3), np.uint8)), 3)


def test_error_rate_validates_before_the_device():
    from paper_1509_08197_b200.errors import ConfigError, DataError
    from paper_1509_08197_b200.raster_io import DisparityMap

    a = DisparityMap(values=np.zeros((2, 3), np.int32), valid=np.ones((2, 3), bool))
    b = DisparityMap(values=np.zeros((3, 2), np.int32), valid=np.ones((3, 2), bool))
    with pytest.raises(DataError):
        error_rate(a, b)
    with pytest.raises(ConfigError):
        error_rate(a, a, threshold=0)


def test_synthetic_generator_is_seeded_and_consistent():
    spec = SceneSpec(9, 40, 64, 12, 6, 0.5, 8.0, 2)
    a, b = make_scene(spec, 0), make_scene(spec, 0)
    np.testing.assert_array_equal(a.pair.left.data, b.pair.left.data)
    np.testing.assert_array_equal(a.pair.right.data, b.pair.right.data)
    c = make_scene(spec, 1)
    assert not np.array_equal(a.pair.left.data, c.pair.left.data)
    d = a.gt_left.values
    assert d.min() >= 0 and d.max() <= spec.d_max
    # visible pixels are exact copies in the right view
    L, R = a.pair.left.data, a.pair.right.data
    rr, cc = np.nonzero(~a.occlusion)
    np.testing.assert_array_equal(L[rr, cc], R[rr, cc - d[rr, cc]])
    assert CONFIGS[2].height == 370 and CONFIGS[2].width == 463 and CONFIGS[2].d_max == 80


def test_shards_and_slabs_partition():
    for n, world in ((8, 3), (81, 4), (513, 8), (5, 8)):
        seen = [i for r in range(world) for i in shard(n, r, world)]
        assert seen == list(range(n))
    covered = []
    for r in range(4):
        x0, nx = slab(512, r, 4)
        covered += list(range(x0, x0 + nx))
    assert covered == list(range(513))


def test_key_packing_orders_like_first_argmin():
    rng = np.random.default_rng(5)
    cost = rng.uniform(0, 1, size=(200, 9)).astype(np.float32)
    cost[:, 4] = cost[:, 2]  # exact ties -> smaller d must win
    keys = pack_keys_host(cost, np.broadcast_to(np.arange(9), cost.shape))
    signed = keys_to_signed(keys)
    best = np.argmin(signed, axis=1)
    np.testing.assert_array_equal(best, np.argmin(cost, axis=1))
