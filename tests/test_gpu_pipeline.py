"""End-to-end GPU parity: baseline (dense MST) and HDP pipelines against the
reference golden run and the CPU oracle.

Parity rule (north_star): integer disparities identical except at
pixels whose two best float64 aggregated costs satisfy c2 - c1 <= 1e-5 * c1;
fp32 min costs within 1e-4 relative (+1e-7 absolute floor).  HDP levels are
compared teacher-forced: the oracle's level l consumes the GPU's level l+1 map.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import cuda_available, golden

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

TIE = 1e-5


def dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def assert_disp_parity(got, want, best, second, what=""):
    band = (second - best) <= TIE * np.abs(best)
    bad = (got != want) & ~band
    assert not bad.any(), f"{what}: {int(bad.sum())} disparity mismatches outside the tie band"
    return int(((got != want) & band).sum())


def assert_cost_parity(got, want, what=""):
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-7, err_msg=what)


def test_baseline_c1_matches_reference_and_oracle():
    from paper_1509_08197_b200 import engine as E
    from oracle import oracle as O

    g = golden("pipelines.npz")
    out = E.run_baseline_batch(dev(g["c1_left"][None]), dev(g["c1_right"][None]), 16)
    disp = out.disparity[0].cpu().numpy()
    cost = out.min_cost[0].cpu().numpy().astype(np.float64)
    ref = O.run_baseline(g["c1_left"], g["c1_right"], 16)
    np.testing.assert_array_equal(ref.disparity, g["c1_base_disp"])  # oracle pinned
    assert_disp_parity(disp, g["c1_base_disp"], ref.min_cost, ref.second_cost, "c1 baseline")
    same = disp == g["c1_base_disp"]
    assert_cost_parity(cost[same], g["c1_base_cost"][same], "c1 baseline min cost")
    assert out.n_trees[0] == 1 and out.stored_entries[0] == 96 * 128 * 17


@pytest.mark.parametrize("kind", ["mst", "rt"])
def test_baseline_batch_vs_oracle(kind):
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.synthetic import SceneSpec, make_scene
    from oracle import oracle as O

    spec = SceneSpec(7, 61, 83, 20, 10, 0.3, 8.0, 3)
    scenes = [make_scene(spec, i) for i in range(3)]
    L = np.stack([s.pair.left.data for s in scenes])
    R = np.stack([s.pair.right.data for s in scenes])
    out = E.run_baseline_batch(dev(L), dev(R), 20, tree_kind=kind, seed=5)
    for i in range(3):
        ref = O.run_baseline(L[i], R[i], 20, tree_kind=kind, seed=5)
        got = out.disparity[i].cpu().numpy()
        assert_disp_parity(got, ref.disparity, ref.min_cost, ref.second_cost, f"pair {i}")
        same = got == ref.disparity
        assert_cost_parity(out.min_cost[i].cpu().numpy()[same], ref.min_cost[same])


def test_hdp_c1_teacher_forced(gmm_text):
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.hdp_model import GmmModel
    from oracle import oracle as O

    g = golden("pipelines.npz")
    model = GmmModel.parse(gmm_text)
    outs = E.run_hdp_batch(dev(g["c1_left"][None]), dev(g["c1_right"][None]), 16, model, levels=2)
    assert [o.level for o in outs] == [2, 1, 0]
    teacher = {o.level: o.disparity[0].cpu().numpy() for o in outs}
    ref = O.run_hdp(g["c1_left"], g["c1_right"], 16, O.parse_gmm(gmm_text), levels=2,
                    teacher=teacher)
    for o, r in zip(outs, ref):
        assert o.level == r.level
        assert int(o.n_trees[0]) == r.n_trees, f"level {o.level} tree count"
        assert int(o.stored_entries[0]) == r.stored_entries, f"level {o.level} entries"
        assert float(o.search_ratio[0]) == r.search_ratio
        got = o.disparity[0].cpu().numpy()
        assert_disp_parity(got, r.disparity, r.min_cost, r.second_cost, f"level {o.level}")
    # free-running result vs the reference golden: same up to tie cascades
    final = outs[-1].disparity[0].cpu().numpy()
    assert (final != g["c1_hdp_l0_disp"]).mean() < 0.01


@pytest.mark.parametrize("n_sub", [1, 2, 3])
def test_dense_pipeline_one_call_matches_step_by_step(n_sub):
    """hdp_dense_pipeline (one library call, sub-batches on their own streams
    from the worker pool) returns exactly what the step-by-step engine path
    returns, for every split of the batch; per-pair tree counts too."""
    import torch

    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene

    spec = CONFIGS[2]
    scenes = [make_scene(spec, i) for i in range(3)]
    crop = (slice(0, 96), slice(0, 160))
    L = dev(np.stack([s.pair.left.data[crop] for s in scenes]))
    R = dev(np.stack([s.pair.right.data[crop] for s in scenes]))
    ref = E.run_baseline_batch(L, R, spec.d_max, stepwise=True)  # step-by-step path
    got = E.run_baseline_fused(L, R, spec.d_max, n_sub=n_sub)
    torch.cuda.synchronize()
    assert torch.equal(got.disparity, ref.disparity)
    assert torch.equal(got.min_cost, ref.min_cost)
    np.testing.assert_array_equal(got.n_trees, ref.n_trees)
    np.testing.assert_array_equal(got.stored_entries, ref.stored_entries)


def test_dense_pipeline_slab_lanes_match():
    """A disparity slab [x0, x0+nx) through the one-call pipeline equals the
    step-by-step slab (the multi-GPU split's per-rank call)."""
    import torch

    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene

    spec = CONFIGS[2]
    s = make_scene(spec, 5)
    L = dev(s.pair.left.data[None, :80, :120])
    R = dev(s.pair.right.data[None, :80, :120])
    ref = E.run_baseline_batch(L, R, spec.d_max, x0=17, nx=30, stepwise=True)
    got = E.run_baseline_fused(L, R, spec.d_max, x0=17, nx=30)
    torch.cuda.synchronize()
    assert torch.equal(got.disparity, ref.disparity)
    assert torch.equal(got.min_cost, ref.min_cost)


def test_host_entry_with_pinned_outputs():
    """run_baseline_host(out=pinned buffers) returns the same maps as the
    default (fresh arrays) path and fills the given buffers."""
    import torch

    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene

    spec = CONFIGS[2]
    scenes = [make_scene(spec, i) for i in range(2)]
    Lh = np.stack([s.pair.left.data[:64, :100] for s in scenes])
    Rh = np.stack([s.pair.right.data[:64, :100] for s in scenes])
    d0, c0 = E.run_baseline_host(Lh, Rh, spec.d_max)
    od = torch.empty(d0.shape, dtype=torch.int32).pin_memory()
    oc = torch.empty(c0.shape, dtype=torch.float32).pin_memory()
    d1, c1 = E.run_baseline_host(torch.from_numpy(Lh).pin_memory(), torch.from_numpy(Rh).pin_memory(),
                                 spec.d_max, out=(od, oc))
    np.testing.assert_array_equal(d1, d0)
    np.testing.assert_array_equal(c1, c0)
    np.testing.assert_array_equal(od.numpy(), d0)


def test_early_raw_cost_gives_identical_results():
    """hdp_set_early_cost(1): the raw-cost pass starts on a side stream once the
    layout order is final (forest.cuh EarlyCost) -- the same kernel into the
    same rows, so the maps must be bit-identical to the default path, for the
    full range, a disparity slab and a batch."""
    import torch

    from paper_1509_08197_b200 import _lib
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.synthetic import SceneSpec, make_scene

    lib = _lib.load()
    scs = [make_scene(SceneSpec(21, 170, 300, 140, 25, 0.3, 8.0, 1), i) for i in range(3)]  # rows of 144 floats: byte records
    L = dev(np.stack([s.pair.left.data for s in scs]))
    R = dev(np.stack([s.pair.right.data for s in scs]))
    prev = lib.hdp_set_early_cost(0)
    try:
        base = E.run_baseline_fused(L, R, 140)
        slab0 = E.run_baseline_fused(L[:1], R[:1], 140, x0=24, nx=30)
        assert lib.hdp_set_early_cost(1) == 0
        for _ in range(2):
            early = E.run_baseline_fused(L, R, 140)
            assert torch.equal(early.disparity, base.disparity)
            assert torch.equal(early.min_cost, base.min_cost)
        slab1 = E.run_baseline_fused(L[:1], R[:1], 140, x0=24, nx=30)
        assert torch.equal(slab1.disparity, slab0.disparity)
        assert torch.equal(slab1.min_cost, slab0.min_cost)
    finally:
        lib.hdp_set_early_cost(prev)


def test_byte_record_raw_cost_matches_oracle_and_f32_records():
    """Wide range-lane rows take the raw cost from 8-byte records (channel bytes
    + f32 gradient, aggregate.cu k_pack_rec8 / VABSDIFF4): parity with the
    oracle under the usual rule, and the gray (one-channel) variant too."""
    from oracle import oracle as O
    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.synthetic import SceneSpec, make_scene

    sc = make_scene(SceneSpec(22, 60, 200, 150, 12, 0.3, 8.0, 1), 0)
    for gray in (False, True):
        Lh, Rh = sc.pair.left.data, sc.pair.right.data
        if gray:
            Lh = np.ascontiguousarray(Lh[:, :, :1])
            Rh = np.ascontiguousarray(Rh[:, :, :1])
        got = E.run_baseline_fused(dev(Lh[None]), dev(Rh[None]), 150)
        ref = O.run_baseline(Lh, Rh, 150)
        assert_disp_parity(got.disparity[0].cpu().numpy(), ref.disparity, ref.min_cost, ref.second_cost,
                           f"byte records gray={gray}")
        assert_cost_parity(got.min_cost[0].cpu().numpy(), ref.min_cost, f"byte records gray={gray}")
