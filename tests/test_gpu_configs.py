"""Parity on the BASELINE configurations' own pipelines at full size.

Every configuration's pipeline runs on the GPU against the CPU oracle
(oracle/, pinned to the reference by tests/test_oracle_golden.py):

* C2: every pair of the bench batch (dense MST), exact tree structure of the
  dense MST and of the level-0 HDP forest (parents, depths, tree ids, per-tree
  disparity sets), and a free-running HDP run;
* C3: HDP with 4 levels (half preset) on a plain pair and on the one pair of
  the 32 that carries a global brightness offset;
* C4: HDP with 5 levels, full preset (delta0 0.004, beta 0.95);
* C5: the dense full-range pipeline on the 2880x1988, d 512 pair, and the
  exact tree structure of its 5.7 M-node MST;
* HDP over random spanning trees (tree_kind "rt").

Parity rule (north_star): trees, interval sets, tree counts and
stored entries exact; disparities identical except where the two best float64
aggregated costs satisfy c2 - c1 <= 1e-5 * c1; fp32 costs within 1e-4 relative
(+1e-7 absolute).  HDP levels are compared teacher-forced (the oracle's level l
consumes the GPU's level l+1 map), which is what the reference's level loop
does with its own map (aggregation.py:439-467); the free-running comparison
additionally excuses pixels whose tree or interval differs because of an
excused flip upstream.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import cuda_available
from test_gpu_pipeline import TIE, assert_cost_parity, assert_disp_parity, dev

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


def _stack(scenes):
    return (np.stack([s.pair.left.data for s in scenes]),
            np.stack([s.pair.right.data for s in scenes]))


def _model(gmm_text):
    from paper_1509_08197_b200.hdp_model import GmmModel

    return GmmModel.parse(gmm_text)


def _bits(words: np.ndarray, d1: int) -> np.ndarray:
    """(k, nw) u32 or u64 little-endian bitsets -> (k, d1) bool."""
    w = np.ascontiguousarray(words)
    by = w.view(np.uint8).reshape(w.shape[0], -1)
    return np.unpackbits(by, axis=1, bitorder="little")[:, :d1].astype(bool)


def _gpu_forest(o):
    """(parent, depth, tree_id, per-tree bool sets or None) of a kept level."""
    ex = {k: v.cpu().numpy() for k, v in o.forest.export().items()}
    tm = o.extra.get("tree_masks")
    sets = None if tm is None else _bits(tm, o.d_max + 1)
    return ex, sets


def _check_teacher_forced(outs, ref, what):
    for o, r in zip(outs, ref):
        assert o.level == r.level
        assert int(o.n_trees[0]) == r.n_trees, f"{what} level {o.level}: tree count"
        assert int(o.stored_entries[0]) == r.stored_entries, f"{what} level {o.level}: entries"
        assert float(o.search_ratio[0]) == r.search_ratio, f"{what} level {o.level}: ratio"
        got = o.disparity[0].cpu().numpy()
        assert_disp_parity(got, r.disparity, r.min_cost, r.second_cost, f"{what} level {o.level}")
        same = got == r.disparity
        assert_cost_parity(o.min_cost[0].cpu().numpy()[same], r.min_cost[same],
                           f"{what} level {o.level} costs")


def _hdp_teacher_forced(cid, index, levels, size_class, gmm_text, tree_kind="mst"):
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.aggregation import SIZE_CLASS_PRESETS
    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene
    from oracle import oracle as O

    spec = CONFIGS[cid]
    sc = make_scene(spec, index)
    L, R = sc.pair.left.data, sc.pair.right.data
    pre = SIZE_CLASS_PRESETS[size_class]
    outs = E.run_hdp_batch(dev(L[None]), dev(R[None]), spec.d_max, _model(gmm_text),
                           levels=levels, delta0=pre["delta0"], beta=pre["beta"],
                           tree_kind=tree_kind, seed=3)
    teacher = {o.level: o.disparity[0].cpu().numpy() for o in outs}
    ref = O.run_hdp(L, R, spec.d_max, O.parse_gmm(gmm_text), levels=levels,
                    size_class=size_class, teacher=teacher, tree_kind=tree_kind, seed=3)
    _check_teacher_forced(outs, ref, f"C{cid}[{index}]")
    return outs, ref


# ------------------------------------------------------------------- C2
def test_c2_every_bench_pair_dense():
    """All 8 pairs of the bench batch (bench.py times exactly this batch)."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.synthetic import CONFIGS, make_batch
    from oracle import oracle as O

    spec = CONFIGS[2]
    L, R = _stack(make_batch(2))
    out = E.run_baseline_batch(dev(L), dev(R), spec.d_max)
    with ThreadPoolExecutor(8) as ex:
        refs = list(ex.map(lambda i: O.run_baseline(L[i], R[i], spec.d_max), range(len(L))))
    ties = 0
    for i, ref in enumerate(refs):
        got = out.disparity[i].cpu().numpy()
        ties += assert_disp_parity(got, ref.disparity, ref.min_cost, ref.second_cost, f"pair {i}")
        same = got == ref.disparity
        assert_cost_parity(out.min_cost[i].cpu().numpy()[same], ref.min_cost[same], f"pair {i}")
        assert int(out.n_trees[i]) == ref.n_trees == 1
    assert ties <= 1e-4 * L.shape[0] * spec.height * spec.width


def test_c2_dense_tree_exact():
    """The full-size dense MST (Boruvka, contracted cooperative rounds, Euler
    tour ranking all engaged) equals the reference's Kruskal + BFS tree."""
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene
    from oracle import oracle as O

    spec = CONFIGS[2]
    sc = make_scene(spec, 3)
    out = E.run_baseline_batch(dev(sc.pair.left.data[None]), dev(sc.pair.right.data[None]),
                               spec.d_max, keep_forest=True)
    ex = {k: v.cpu().numpy() for k, v in out.forest.export().items()}
    ref = O.build_forest_mst(np.asarray(sc.pair.left.data, np.float64)).base
    np.testing.assert_array_equal(ex["parent"], ref.parent)
    np.testing.assert_array_equal(ex["depth"], ref.depth)
    np.testing.assert_array_equal(ex["tree_id"], ref.tree_id)
    np.testing.assert_array_equal(ex["parent_weight"].astype(np.float64), ref.parent_weight)


def test_c2_hdp_forests_exact(gmm_text):
    """Teacher-forced 3-level HDP on a C2 pair: at every level the HDPF forest
    (parents, depths, tree ids) and every tree's disparity set are exactly the
    reference's (hdp_forest.py:151-216, spanning_forest.py:191-283)."""
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene
    from oracle import oracle as O

    spec = CONFIGS[2]
    sc = make_scene(spec, 1)
    L, R = sc.pair.left.data, sc.pair.right.data
    outs = E.run_hdp_batch(dev(L[None]), dev(R[None]), spec.d_max, _model(gmm_text), levels=3,
                           keep=True)
    teacher = {o.level: o.disparity[0].cpu().numpy() for o in outs}
    ref = O.run_hdp(L, R, spec.d_max, O.parse_gmm(gmm_text), levels=3, teacher=teacher,
                    keep=True)
    _check_teacher_forced(outs, ref, "C2 HDP")
    for o, r in zip(outs, ref):
        ex, sets = _gpu_forest(o)
        np.testing.assert_array_equal(ex["parent"], r.forest.base.parent, f"level {o.level}")
        np.testing.assert_array_equal(ex["depth"], r.forest.base.depth, f"level {o.level}")
        np.testing.assert_array_equal(ex["tree_id"], r.forest.base.tree_id, f"level {o.level}")
        want = _bits(r.forest.masks, o.d_max + 1)
        if sets is None:  # top level: plain forest, full range
            assert want.all()
        else:
            np.testing.assert_array_equal(sets, want, f"level {o.level} tree sets")


def _tree_fingerprint(parent_tree_id, n):
    """Per pixel: (tree size, sum of member ids, sum of squared ids) of its tree."""
    tid = parent_tree_id
    ids = np.arange(n, dtype=np.float64)
    k = tid.max() + 1
    size = np.bincount(tid, minlength=k)
    s1 = np.bincount(tid, ids, minlength=k)
    s2 = np.bincount(tid, ids * ids, minlength=k)
    return np.stack([size[tid], s1[tid], s2[tid]], axis=1)


def test_c2_hdp_free_running(gmm_text):
    """Free-running 3-level HDP on C2 pairs (each side consumes its own coarser
    map).  A disparity may differ only (a) inside the tie band, or (b) at a
    pixel whose tree or disparity set differs from the oracle's, which in turn
    can only come from an excused flip at a coarser level."""
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene
    from oracle import oracle as O

    spec = CONFIGS[2]
    cascade = []
    for index in (0, 6):
        sc = make_scene(spec, index)
        L, R = sc.pair.left.data, sc.pair.right.data
        outs = E.run_hdp_batch(dev(L[None]), dev(R[None]), spec.d_max, _model(gmm_text),
                               levels=3, keep=True)
        ref = O.run_hdp(L, R, spec.d_max, O.parse_gmm(gmm_text), levels=3, keep=True)
        upstream_flips = 0
        for o, r in zip(outs, ref):
            got = o.disparity[0].cpu().numpy().ravel()
            want = r.disparity.ravel()
            band = ((r.second_cost - r.min_cost) <= TIE * np.abs(r.min_cost)).ravel()
            ex, sets = _gpu_forest(o)
            n = got.size
            if sets is None:
                moved = np.zeros(n, bool)
            else:
                gset = sets[ex["tree_id"]]
                oset = _bits(r.forest.masks, o.d_max + 1)[r.forest.base.tree_id]
                moved = (gset != oset).any(axis=1)
                moved |= (_tree_fingerprint(ex["tree_id"], n)
                          != _tree_fingerprint(r.forest.base.tree_id, n)).any(axis=1)
            if upstream_flips == 0:
                assert not moved.any(), f"pair {index} level {o.level}: forest differs without a flip"
            bad = (got != want) & ~band & ~moved
            assert not bad.any(), f"pair {index} level {o.level}: {int(bad.sum())} unexcused"
            upstream_flips += int((got != want).sum())
            cascade.append(float(moved.mean()))
    assert max(cascade) < 0.2, cascade


# ------------------------------------------------------------------- C3
@pytest.mark.parametrize("index", [0, 28])  # pair 28 has a global right offset of -14
def test_c3_hdp_levels4_teacher_forced(index, gmm_text):
    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene

    if index == 28:
        assert make_scene(CONFIGS[3], 28).brightness_offset != 0
    _hdp_teacher_forced(3, index, 4, "half", gmm_text)


# ------------------------------------------------------------------- C4
def test_c4_hdp_levels5_full_preset_teacher_forced(gmm_text):
    outs, ref = _hdp_teacher_forced(4, 0, 5, "full", gmm_text)
    assert [o.level for o in outs] == [5, 4, 3, 2, 1, 0]
    assert ref[-1].search_ratio < 0.05  # the full preset prunes hard


# ------------------------------------------------------------------- C5
def test_c5_dense_fullsize():
    """The C5 pair (5.7 M px, one tree, 513 lanes) against the oracle's
    disparity-streamed baseline (float64, the reference's chunk fold)."""
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene
    from oracle import oracle as O

    spec = CONFIGS[5]
    sc = make_scene(spec, 0)
    L, R = sc.pair.left.data, sc.pair.right.data
    out = E.run_baseline_batch(dev(L[None]), dev(R[None]), spec.d_max, keep_forest=True)
    ex = {k: v.cpu().numpy() for k, v in out.forest.export().items()}
    got = out.disparity[0].cpu().numpy()
    cost = out.min_cost[0].cpu().numpy()
    del out
    ref = O.run_baseline_chunked(L, R, spec.d_max)
    base = ref.forest.base
    np.testing.assert_array_equal(ex["parent"], base.parent)
    np.testing.assert_array_equal(ex["depth"], base.depth)
    np.testing.assert_array_equal(ex["tree_id"], base.tree_id)
    ties = assert_disp_parity(got, ref.disparity, ref.min_cost, ref.second_cost, "C5")
    same = got == ref.disparity
    assert_cost_parity(cost[same], ref.min_cost[same], "C5 costs")
    assert ties <= 1e-4 * got.size


# ------------------------------------------------------------------ HDP + RT
def test_hdp_rt_teacher_forced(gmm_text):
    """HDP over random spanning trees (rt_edge_order, spanning_forest.py:110-112)
    at the C1 shape, each level teacher-forced."""
    _hdp_teacher_forced(1, 0, 2, "half", gmm_text, tree_kind="rt")
