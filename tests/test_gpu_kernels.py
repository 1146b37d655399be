"""GPU parity of the individual kernels against the reference golden vectors
and the CPU oracle.  Run on a B200: pytest -m gpu."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import cuda_available, golden

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

COST_TOL = dict(rtol=1e-4, atol=1e-7)  # north_star: fp32 within 1e-4 rel (+ abs floor)


def dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_block_mean_bit_exact():
    from paper_1509_08197_b200 import engine as E

    g = golden("pyramid.npz")
    img = dev(g["image"][None])
    cur = E.to_f64(img)
    np.testing.assert_array_equal(cur[0].cpu().numpy(), g["level0"])
    for lvl in (1, 2, 3):
        cur = E.block_mean(cur, 2)
        np.testing.assert_array_equal(cur[0].cpu().numpy(), g[f"level{lvl}"])
    bm3 = E.block_mean(dev(g["bm3_in"][None]), 3)
    np.testing.assert_array_equal(bm3[0].cpu().numpy(), g["bm3"])


@pytest.mark.parametrize("tag", ["rgb", "gray"])
def test_prepare_bit_exact_and_cost_f32(tag):
    import torch

    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200 import _lib as L

    g = golden("cost.npz")
    il, ir = dev(g[tag + "_left"][None]), dev(g[tag + "_right"][None])
    unit, gray, grad, pl = E.prepare(il, True, True, True)
    _, _, _, pr = E.prepare(ir, False, True)
    np.testing.assert_array_equal(gray[0].cpu().numpy(), g[tag + "_gray"])
    np.testing.assert_array_equal(grad[0].cpu().numpy(), g[tag + "_grad"])
    cost = g[tag + "_cost"]
    nx = cost.shape[0]
    b, h, w, c = il.shape
    xs = torch.arange(nx, dtype=torch.int32, device="cuda")
    out = torch.empty((h * w, nx), dtype=torch.float32, device="cuda")
    L.call("hdp_cost_volume", L.ptr(pl), L.ptr(pr), 1, h, w, c, L.ptr(xs), nx, 0.9, 0.0275,
           0.0078, L.ptr(out), L.stream())
    got = out.cpu().numpy().T.reshape(nx, h, w)
    np.testing.assert_allclose(got, cost, **COST_TOL)


def test_prepare_dyadic_level_bit_exact():
    from paper_1509_08197_b200 import engine as E

    g = golden("cost.npz")
    _, gray, grad, _ = E.prepare(dev(g["dyadic_in"][None]), True, False, True)
    np.testing.assert_array_equal(gray[0].cpu().numpy(), g["dyadic_gray"])
    np.testing.assert_array_equal(grad[0].cpu().numpy(), g["dyadic_grad"])


MST_CASES = ["int0", "int1", "int2", "int3", "int4", "dyadic", "ties"]


@pytest.mark.parametrize("tag", MST_CASES)
@pytest.mark.parametrize("kind", ["mst", "rt"])
def test_tree_build_exact(tag, kind):
    from paper_1509_08197_b200 import engine as E

    g = golden("mst.npz")
    img = dev(g[tag + "_in"][None])
    h, w = img.shape[1:3]
    eu, ev, ew, key, nE = E.grid_edges(img)
    np.testing.assert_array_equal(eu.cpu().numpy(), g[tag + "_u"])
    np.testing.assert_array_equal(ev.cpu().numpy(), g[tag + "_v"])
    np.testing.assert_array_equal(ew.cpu().numpy().astype(np.float64), g[tag + "_w"])
    if kind == "rt":
        key = E.rt_keys(nE, 1, 3, img.device)
    in_tree, comp, _ = E.mst(h * w, eu, ev, key)
    f = E.DeviceForest(h * w, eu, ev, ew, in_tree, comp, 0.1)
    o = {k: v.cpu().numpy() for k, v in f.export().items()}
    p = f"{tag}_{kind}_"
    np.testing.assert_array_equal(o["parent"], g[p + "parent"])
    np.testing.assert_array_equal(o["depth"], g[p + "depth"])
    np.testing.assert_array_equal(o["tree_id"], g[p + "tree_id"])
    np.testing.assert_array_equal(o["parent_weight"].astype(np.float64), g[p + "parent_weight"])
    assert f.n_trees == len(g[p + "tree_slices"]) - 1


def test_aggregate_forest_cost_rows():
    import torch

    from paper_1509_08197_b200 import engine as E

    g = golden("aggregate.npz")
    for k in range(6):
        n = int(g[f"f{k}_n"])
        u, v, w = g[f"f{k}_u"], g[f"f{k}_v"], g[f"f{k}_w"]
        costs = g[f"f{k}_costs"]
        m = costs.shape[1]
        f = E.DeviceForest(n, dev(u.astype(np.int32)), dev(v.astype(np.int32)),
                           dev(w.astype(np.float32)), None, None, float(g[f"f{k}_gamma"]))
        o = f.export()
        np.testing.assert_array_equal(o["parent"].cpu().numpy(), g[f"f{k}_parent"])
        np.testing.assert_array_equal(o["depth"].cpu().numpy(), g[f"f{k}_depth"])
        f.set_lanes_range(0, m)
        rows = dev(costs.astype(np.float32))
        _, _, _, vol = f.aggregate(None, cost_rows=rows, want_volume=True)
        off = f.node_offsets().cpu().numpy()
        got = np.stack([vol.cpu().numpy()[off[i]:off[i] + m] for i in range(n)])
        np.testing.assert_allclose(got, g[f"f{k}_out"], **COST_TOL)


def test_prior_counts_match_reference():
    from paper_1509_08197_b200 import engine as E
    from oracle import oracle as O

    g = golden("prior.npz")
    cases = [("shift", 8)] + [(f"c1_l{l}", int(g[f"c1_l{l}_dmax"])) for l in (0, 1)]
    for tag, d in cases:
        il, ir = dev(g[tag + "_left"][None]), dev(g[tag + "_right"][None])
        ul, _, gl, _ = E.prepare(il, True, False)
        ur, _, gr, _ = E.prepare(ir, True, False)
        lev = E.Level(0, il.shape[1], il.shape[2], il.shape[3], d, il, ir, None, None, ul, gl, ur, gr)
        counts, kept = E.prior_counts(lev)
        counts, kept = counts.cpu().numpy(), kept.cpu().numpy()
        prior = E.priors_from_counts(counts, kept)[0]
        np.testing.assert_array_equal(prior, g[tag + "_prior"])
        oc, ok = O.prior_counts(g[tag + "_left"], g[tag + "_right"], d)
        np.testing.assert_array_equal(counts[0], oc)
        assert kept[0] == ok
        # a capped grid (the side-stream launches) strides over the centres
        c2, k2 = E.prior_counts(lev, max_ctas=3)
        np.testing.assert_array_equal(c2.cpu().numpy(), counts)
        np.testing.assert_array_equal(k2.cpu().numpy(), kept)


def _table(sizes, flat):
    offs = np.concatenate(([0], np.cumsum(sizes)))
    return [flat[offs[i]:offs[i + 1]] for i in range(len(sizes))]


@pytest.mark.parametrize("fast", ["1", "0"])
def test_hdpf_exact(fast, monkeypatch):
    """Golden build_hdpf forests, through the mask-homogeneous fast path where it
    applies (cases 0 and 2 have no cross-pass edge, 1 and 3 do and fall back to
    the window kernel) and with the window kernel forced (HDP_HDPF_FAST=0)."""
    import torch

    monkeypatch.setenv("HDP_HDPF_FAST", fast)

    from paper_1509_08197_b200 import engine as E
    from oracle import oracle as O

    g = golden("hdpf.npz")
    for k in range(int(g["count"])):
        p = f"h{k}_"
        I = g[p + "in"]
        h, w = I.shape[:2]
        d = int(g[p + "d"])
        table = _table(g[p + "tab_sizes"], g[p + "tab_flat"])
        chosen = np.zeros((1, len(table), d + 1), bool)
        for i, t in enumerate(table):
            chosen[0, i, t] = True
        row_masks = dev(E.pack_masks(chosen).view(np.int32))
        rows = dev(g[p + "rows"].astype(np.int32))
        img = dev(I[None])
        eu, ev, ew, key, nE = E.grid_edges(img)
        in_tree, comp, tm, rounds = E.hdpf(1, h * w, nE, eu, ev, key, rows, row_masks,
                                           float(g[p + "beta"]))
        f = E.DeviceForest(h * w, eu, ev, ew, in_tree, comp, 0.1)
        o = {kk: vv.cpu().numpy() for kk, vv in f.export().items()}
        np.testing.assert_array_equal(o["parent"], g[p + "parent"])
        np.testing.assert_array_equal(o["tree_id"], g[p + "tree_id"])
        np.testing.assert_array_equal(o["depth"], g[p + "depth"])
        roots = np.flatnonzero(o["root"] == np.arange(h * w))
        tm_h = tm.cpu().numpy().view(np.uint32)[roots]
        sizes = [int(sum(bin(x).count("1") for x in row)) for row in tm_h]
        np.testing.assert_array_equal(sizes, g[p + "iv_sizes"])
        flat = np.concatenate([[wi * 32 + b for wi, x in enumerate(row) for b in range(32)
                                if (int(x) >> b) & 1] for row in tm_h])
        np.testing.assert_array_equal(flat, g[p + "iv_flat"])


@pytest.mark.parametrize("c,shape", [(3, (2, 37, 53)), (1, (1, 20, 1)), (3, (1, 1, 9))])
def test_u8_prepare_and_edges_match_f64_path(c, shape):
    """hdp_prepare_u8 / hdp_grid_edges_u8 (the one-call pipeline's level 0)
    are bit-identical to u8 -> f64 -> hdp_prepare / hdp_grid_edges."""
    import torch

    from paper_1509_08197_b200 import _lib as L
    from paper_1509_08197_b200 import engine as E

    rng = np.random.default_rng(7)
    b, h, w = shape
    u8 = dev(rng.integers(0, 256, (b, h, w, c), dtype=np.uint8))
    _, _, _, packed = E.prepare(E.to_f64(u8), False)
    pk = torch.empty_like(packed)
    L.call("hdp_prepare_u8", L.ptr(u8), b, h, w, c, L.ptr(pk), L.stream())
    assert torch.equal(pk, packed)
    eu, ev, ew, key, n_e = E.grid_edges(E.to_f64(u8))
    if b * n_e:
        eu2, ev2, ew2, key2 = (torch.empty_like(x) for x in (eu, ev, ew, key))
        L.call("hdp_grid_edges_u8", L.ptr(u8), b, h, w, c, L.ptr(eu2), L.ptr(ev2), L.ptr(ew2), L.ptr(key2),
               L.stream())
        for x, y in ((eu, eu2), (ev, ev2), (ew, ew2), (key, key2)):
            assert torch.equal(x, y)


@pytest.mark.parametrize("cols,delta", [(81, 0.064), (17, 0.004), (241, 0.004), (2, 0.5), (33, 0.9)])
def test_predict_masks_device_matches_host(cols, delta):
    """hdp_predict_masks == pack_masks(predict_masks(...)) bit for bit, with
    heavy ties (quantised probabilities) and zero rows made uniform."""
    import torch

    from paper_1509_08197_b200 import engine as E

    rng = np.random.default_rng(cols)
    b, rows = 3, 23
    raw = np.floor(rng.random((b, rows, cols)) ** 4 * 16) / 16  # many exact ties and zeros
    raw[0, 0] = 0.0
    rs = raw.sum(-1, keepdims=True)
    bayes = np.where(rs > 0, raw / np.where(rs > 0, rs, 1), 1.0 / cols)
    want = E.pack_masks(E.predict_masks(bayes, delta)).view(np.int32)
    got = E.predict_masks_device(bayes, delta, torch.device("cuda")).cpu().numpy()
    np.testing.assert_array_equal(got, want)


def test_prior_division_is_ieee_exact():
    """The prior's division by a constant (Markstein: RN(q + r RN(1/b))) equals
    the IEEE quotient on 2^24 seeded inputs for b = 3, 49, 25."""
    import ctypes

    from paper_1509_08197_b200 import _lib as L

    L.device()
    bad = ctypes.c_int64(-1)
    L.call("hdp_check_exact_division", 1 << 24, 12345, ctypes.byref(bad), L.stream())
    assert bad.value == 0


@pytest.mark.parametrize("d_child,d_parent", [(80, 40), (240, 120), (12, 6), (5, 2)])
def test_device_bayes_matches_host(d_child, d_parent):
    """hdp_priors_from_counts + hdp_bayes (the HDP level loop's device path)
    == priors_from_counts + bayes_batched on the host, bit for bit, including
    a pair without kept samples and rows without mass."""
    import torch

    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.hdp_model import GmmModel

    with open(os.path.join(os.path.dirname(__file__), "golden", "default.gmm")) as fh:
        model = GmmModel.parse(fh.read())
    rng = np.random.default_rng(d_child)
    b = 5
    counts = rng.integers(0, 400, (b, d_child + 1)).astype(np.int64)
    counts[:, rng.integers(0, d_child + 1, d_child // 3)] = 0
    kept = counts.sum(axis=1).astype(np.int64)
    counts[1] = 0
    kept[1] = 0
    cond = E.conditional_matrix(model.layers[0], d_child, d_parent, 2)
    cond[cond.shape[0] // 2] = 0.0  # a parent row with no mass under any prior
    pri = E.priors_from_counts(counts, kept)
    bm, _ = E.bayes_batched(cond, pri)
    cd = torch.from_numpy(np.ascontiguousarray(cond)).cuda()
    got = E.bayes_device(torch.from_numpy(counts).cuda(), torch.from_numpy(kept).cuda(), cd)
    np.testing.assert_array_equal(got.cpu().numpy(), bm)


@pytest.mark.parametrize("cid,levels", [(2, 3), (4, 5)])
def test_prior_filter_equals_full_f64(cid, levels, monkeypatch):
    """The prior's f32 filter + f64 verification (default) gives the same
    histograms as evaluating every disparity in f64 (HDP_PRIOR_FILTER=0), on
    every pyramid level of a full-size pair of the configuration."""
    import torch

    from paper_1509_08197_b200 import engine as E
    from paper_1509_08197_b200.synthetic import CONFIGS, make_scene

    spec = CONFIGS[cid]
    sc = [make_scene(spec, i) for i in range(2)]
    L = torch.from_numpy(np.stack([s.pair.left.data for s in sc])).cuda()
    R = torch.from_numpy(np.stack([s.pair.right.data for s in sc])).cuda()
    lv = E.build_levels(L, R, spec.d_max, levels, 2, True)
    for lev in lv[:-1]:
        monkeypatch.setenv("HDP_PRIOR_FILTER", "1")
        c1, k1 = E.prior_counts(lev)
        monkeypatch.setenv("HDP_PRIOR_FILTER", "0")
        c0, k0 = E.prior_counts(lev)
        np.testing.assert_array_equal(c1.cpu().numpy(), c0.cpu().numpy())
        np.testing.assert_array_equal(k1.cpu().numpy(), k0.cpu().numpy())
