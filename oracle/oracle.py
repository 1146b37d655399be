"""CPU oracle for the HDP stereo hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline.  The product package (``paper_1509_08197_b200``) never
imports it; its CUDA path fails loudly when the extension is missing.

It restates the reference package ``treestereo`` (paths below are relative to
``/root/reference/pkg/src/treestereo/``) on top of the float64 C routines in
``hdp_oracle.c``; the small probability tables (A13-A15 of SURVEY.md §8a) are
restated with the same numpy operations the reference uses.  Parity of this
restatement is pinned against golden vectors produced by the real reference
(``tests/golden/make_golden.py``; checked by ``tests/test_oracle_golden.py``).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libhdp_oracle.so")
_lib = None

ALPHA, TAU_C, TAU_G = 0.9, 0.0275, 0.0078  # cost_volume.py:38-40
HALF = {"delta0": 0.064, "beta": 0.6}  # aggregation.py:70
FULL = {"delta0": 0.004, "beta": 0.95}  # aggregation.py:71

_i64 = C.POINTER(C.c_int64)
_f64 = C.POINTER(C.c_double)
_u64 = C.POINTER(C.c_uint64)


def build_lib() -> str:
    src = os.path.join(_HERE, "hdp_oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build_lib())
        i, i64, d, P = C.c_int, C.c_int64, C.c_double, C.c_void_p
        sig = {
            "or_block_mean": (None, [i, i, i, i, P, P]),
            "or_prepare": (None, [i, i, i, P, P, P, P]),
            "or_cost_grid": (None, [i, i, i, P, P, P, P, i, d, d, d, P]),
            "or_edge_list": (i64, [i, i, i, P, P, P, P]),
            "or_mst_order": (None, [i64, P, P]),
            "or_hdpf": (i64, [i64, i64, P, P, P, P, i, P, d, P, P, P, P, P]),
            "or_hdpf_st": (i64, [i64, i64, P, P, P, P, i, P, d, d, P, P, P, P, P]),
            "or_bfs_forest": (i64, [i64, i64, P, P, P, P, P, P, P, P, P]),
            "or_aggregate_forest": (None, [i64, i64, P, P, P, P, i64, P, P, P]),
            "or_np_sum": (d, [P, i64]),
            "or_windowed_wta": (None, [i, i, i, P, P, P, P, i64, P, P, i, i, i, d, d, d, P]),
            "or_layer_wta": (None, [i, i, i, P, P, P, P, d, d, d, i64, P, P, P, P, P, P, P, P,
                                    P, P, P, P, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


# ------------------------------------------------------------------ pyramid
def block_mean(values: np.ndarray, s: int) -> np.ndarray:
    """pyramid.py:62-75."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    if v.ndim == 2:
        v = v[:, :, None]
    h, w, c = v.shape
    out = np.empty(((h + s - 1) // s, (w + s - 1) // s, c))
    lib().or_block_mean(h, w, c, s, _p(v, _f64), _p(out, _f64))
    return out


def build_pyramid(image_u8: np.ndarray, d_max: int, s: int = 2, levels: int = 3):
    """pyramid.py:78-113 -> list of (intensities float64, d_max)."""
    layers = [(np.asarray(image_u8, dtype=np.float64), d_max)]
    for _ in range(levels):
        below, d = layers[-1]
        layers.append((block_mean(below, s), d // s))
    return layers


# ------------------------------------------------------------------ cost
@dataclass
class Prepared:
    unit: np.ndarray
    gray: np.ndarray
    grad: np.ndarray


def prepare_layer(intensities: np.ndarray) -> Prepared:
    """cost_volume.py:62-69."""
    I = np.ascontiguousarray(intensities, dtype=np.float64)
    h, w, c = I.shape
    unit = np.empty_like(I)
    gray = np.empty((h, w))
    grad = np.empty((h, w))
    lib().or_prepare(h, w, c, _p(I, _f64), _p(unit, _f64), _p(gray, _f64), _p(grad, _f64))
    return Prepared(unit, gray, grad)


def cost_grid(left: Prepared, right: Prepared, x: int,
              alpha=ALPHA, tc=TAU_C, tg=TAU_G) -> np.ndarray:
    """cost_volume.py:91-102."""
    h, w, c = left.unit.shape
    out = np.empty((h, w))
    lib().or_cost_grid(h, w, c, _p(left.unit, _f64), _p(left.grad, _f64),
                       _p(right.unit, _f64), _p(right.grad, _f64), int(x),
                       C.c_double(alpha), C.c_double(tc), C.c_double(tg), _p(out, _f64))
    return out


def dense_cost(left: Prepared, right: Prepared, d_max: int) -> np.ndarray:
    """(N, d_max+1) raw cost, rows by pixel id."""
    return np.stack([cost_grid(left, right, x).ravel() for x in range(d_max + 1)], axis=1)


# ------------------------------------------------------------------ trees
def build_edge_list(intensities: np.ndarray):
    """spanning_forest.py:61-93 -> (u, v, w)."""
    I = np.ascontiguousarray(intensities, dtype=np.float64)
    h, w, c = I.shape
    E = 2 * h * w - h - w
    u = np.empty(max(E, 0), np.int64)
    v = np.empty(max(E, 0), np.int64)
    wt = np.empty(max(E, 0))
    lib().or_edge_list(h, w, c, _p(I, _f64), _p(u, _i64), _p(v, _i64), _p(wt, _f64))
    return u, v, wt


def mst_edge_order(wt: np.ndarray) -> np.ndarray:
    """spanning_forest.py:96-107 (stable by weight)."""
    wt = np.ascontiguousarray(wt, dtype=np.float64)
    order = np.empty(wt.size, np.int64)
    lib().or_mst_order(wt.size, _p(wt, _f64), _p(order, _i64))
    return order


def rt_edge_order(n_edges: int, seed: int) -> np.ndarray:
    """spanning_forest.py:110-112."""
    return np.random.default_rng(seed).permutation(n_edges)


@dataclass
class Forest:
    """Mirror of RootedForest (spanning_forest.py:146-188)."""

    n_nodes: int
    parent: np.ndarray
    parent_weight: np.ndarray
    depth: np.ndarray
    tree_id: np.ndarray
    order: np.ndarray
    tree_slices: np.ndarray

    @property
    def n_trees(self) -> int:
        return len(self.tree_slices) - 1

    @property
    def roots(self):
        return self.order[self.tree_slices[:-1]]

    def similarities(self, gamma: float) -> np.ndarray:
        return np.exp(-self.parent_weight / (gamma * 255.0))


def bfs_forest(n, acc_u, acc_v, acc_w) -> Forest:
    """spanning_forest.py:191-283."""
    acc_u = np.ascontiguousarray(acc_u, np.int64)
    acc_v = np.ascontiguousarray(acc_v, np.int64)
    acc_w = np.ascontiguousarray(acc_w, np.float64)
    parent = np.empty(n, np.int64)
    pw = np.empty(n)
    depth = np.empty(n, np.int64)
    tid = np.empty(n, np.int64)
    order = np.empty(n, np.int64)
    slices = np.empty(n + 1, np.int64)
    nt = lib().or_bfs_forest(n, acc_u.size, _p(acc_u, _i64), _p(acc_v, _i64), _p(acc_w, _f64),
                             _p(parent, _i64), _p(pw, _f64), _p(depth, _i64), _p(tid, _i64),
                             _p(order, _i64), _p(slices, _i64))
    return Forest(n, parent, pw, depth, tid, order, slices[: nt + 1].copy())


def _words(d_max: int) -> int:
    return (d_max + 1 + 63) // 64


def masks_from_rows(row_sets, d_max: int) -> np.ndarray:
    """Table rows (sorted int arrays) -> (n_rows, nw) uint64 bitsets."""
    nw = _words(d_max)
    out = np.zeros((len(row_sets), nw), np.uint64)
    for i, s in enumerate(row_sets):
        for j in np.asarray(s).tolist():
            out[i, j // 64] |= np.uint64(1) << np.uint64(j % 64)
    return out


def mask_bits(words: np.ndarray) -> np.ndarray:
    bits = []
    for wi, word in enumerate(words.tolist()):
        while word:
            low = word & -word
            bits.append(wi * 64 + low.bit_length() - 1)
            word ^= low
    return np.array(bits, np.int64)


@dataclass
class DForest:
    """Mirror of DisparityForest (hdp_forest.py:126-148)."""

    base: Forest
    masks: np.ndarray  # (n_trees, nw) uint64
    intervals: list
    d_max: int
    accepted: tuple  # (u, v, w) in acceptance order

    @property
    def n_trees(self):
        return self.base.n_trees

    def search_ratio(self) -> float:
        sizes = np.array([iv.size for iv in self.intervals], dtype=np.float64)
        return float(sizes[self.base.tree_id].mean()) / (self.d_max + 1)

    def total_search_entries(self) -> int:
        sizes = np.array([iv.size for iv in self.intervals], dtype=np.int64)
        return int((sizes * np.diff(self.base.tree_slices)).sum())


ST_K = 1200.0  # segment-tree merge parameter k (paper_1509_08197_b200.spanning_forest.ST_K)


def build_hdpf(u, v, wt, n, pix_masks: np.ndarray, d_max: int, beta: float,
               order: np.ndarray | None = None, st_k: float | None = None) -> DForest:
    """hdp_forest.py:151-216 (pix_masks: (n, nw) uint64).  st_k: build the
    segment-tree variant (or_hdpf_st; no reference exists, parity unpinned)."""
    if order is None:
        order = mst_edge_order(wt)
    pix_masks = np.ascontiguousarray(pix_masks, np.uint64)
    nw = pix_masks.shape[1]
    E = u.size
    au = np.empty(max(n - 1, 1), np.int64)
    av = np.empty(max(n - 1, 1), np.int64)
    aw = np.empty(max(n - 1, 1))
    roots = np.empty(n, np.int64)
    rmask = np.empty((n, nw), np.uint64)
    order = np.ascontiguousarray(order, np.int64)
    u = np.ascontiguousarray(u, np.int64)
    v = np.ascontiguousarray(v, np.int64)
    wt = np.ascontiguousarray(wt, np.float64)
    if st_k is None:
        k = lib().or_hdpf(n, E, _p(u, _i64), _p(v, _i64), _p(wt, _f64), _p(order, _i64), nw,
                          _p(pix_masks, _u64), C.c_double(beta), _p(au, _i64), _p(av, _i64),
                          _p(aw, _f64), _p(roots, _i64), _p(rmask, _u64))
    else:
        k = lib().or_hdpf_st(n, E, _p(u, _i64), _p(v, _i64), _p(wt, _f64), _p(order, _i64), nw,
                             _p(pix_masks, _u64), C.c_double(beta), C.c_double(st_k), _p(au, _i64),
                             _p(av, _i64), _p(aw, _f64), _p(roots, _i64), _p(rmask, _u64))
    base = bfs_forest(n, au[:k], av[:k], aw[:k])
    tmasks = rmask[base.roots]
    intervals = [mask_bits(m) for m in tmasks]
    return DForest(base, tmasks, intervals, d_max, (au[:k].copy(), av[:k].copy(), aw[:k].copy()))


def full_masks(n: int, d_max: int) -> np.ndarray:
    row = masks_from_rows([np.arange(d_max + 1)], d_max)
    return np.repeat(row, n, axis=0)


def build_forest_mst(intensities, d_max: int = 1) -> DForest:
    """plain_disparity_forest (hdp_forest.py:219-224)."""
    u, v, wt = build_edge_list(intensities)
    h, w = intensities.shape[:2]
    return build_hdpf(u, v, wt, h * w, full_masks(h * w, d_max), d_max, 0.0)


# ------------------------------------------------------------ aggregation
def aggregate_forest(forest: Forest, costs: np.ndarray, gamma: float = 0.1) -> np.ndarray:
    """aggregation.py:216-236 (float64)."""
    costs = np.ascontiguousarray(costs, np.float64)
    if costs.ndim == 1:
        costs = costs[:, None]
    n, m = costs.shape
    sim = np.ascontiguousarray(forest.similarities(gamma))
    out = np.empty_like(costs)
    lib().or_aggregate_forest(n, m, _p(forest.parent, _i64), _p(forest.order, _i64),
                              _p(forest.depth, _i64), _p(forest.tree_slices, _i64),
                              forest.n_trees, _p(sim, _f64), _p(costs, _f64), _p(out, _f64))
    return out


def wta(values: np.ndarray, columns: np.ndarray):
    """aggregation.py:239-256 on one row block: first argmin."""
    j = np.argmin(values, axis=1)
    return columns[j], values[np.arange(values.shape[0]), j]


# ------------------------------------------------------------------ prior
def windowed_wta(src: Prepared, dst: Prepared, cr, cc, d_max, sign, window=7,
                 alpha=ALPHA, tc=TAU_C, tg=TAU_G) -> np.ndarray:
    h, w, c = src.unit.shape
    cr = np.ascontiguousarray(cr, np.int64)
    cc = np.ascontiguousarray(cc, np.int64)
    out = np.empty(cr.size, np.int64)
    lib().or_windowed_wta(h, w, c, _p(src.unit, _f64), _p(src.grad, _f64), _p(dst.unit, _f64),
                          _p(dst.grad, _f64), cr.size, _p(cr, _i64), _p(cc, _i64), d_max, sign,
                          window, C.c_double(alpha), C.c_double(tc), C.c_double(tg), _p(out, _i64))
    return out


def prior_counts(left_I, right_I, d_max, stride=5, window=7, max_offset=1):
    """hdp_model.py:425-470 up to the histogram: returns (counts, n_kept)."""
    L, R = prepare_layer(left_I), prepare_layer(right_I)
    h, w = L.gray.shape
    rs = np.arange(0, h, stride)
    cs = np.arange(0, w, stride)
    rc = (rs + np.minimum(rs + stride, h) - 1) // 2
    ccn = (cs + np.minimum(cs + stride, w) - 1) // 2
    rr, cc = np.meshgrid(rc, ccn, indexing="ij")
    rr, cc = rr.ravel(), cc.ravel()
    d_left = windowed_wta(L, R, rr, cc, d_max, -1, window)
    match = cc - d_left
    ok = match >= 0
    d_right = windowed_wta(R, L, rr[ok], match[ok], d_max, +1, window)
    stable = np.abs(d_left[ok] - d_right) <= max_offset
    kept = d_left[ok][stable]
    return np.bincount(kept, minlength=d_max + 1).astype(np.int64), int(kept.size)


def prior_from_counts(counts: np.ndarray, n_kept: int) -> np.ndarray:
    """hdp_model.py:465-470."""
    d1 = counts.size
    if n_kept == 0:
        return np.full(d1, 1.0 / d1)
    hist = counts.astype(np.float64) + 1.0
    return hist / hist.sum()


# ------------------------------------------------------------------ tables
def mixture_density(weights, means, sigmas, x):
    """hdp_model.py:67-72 (same numpy ops, incl. the BLAS matvec)."""
    x = np.asarray(x, dtype=np.float64)
    z = (x[..., None] - means) / sigmas
    comp = np.exp(-0.5 * z * z) / (sigmas * np.sqrt(2.0 * np.pi))
    return comp @ weights


def conditional(mix, d_child, d_parent, s):
    """hdp_model.py:320-331 -> matrix[i, j] = P(parent=i | child=j)."""
    i = np.arange(d_parent + 1)
    j = np.arange(d_child + 1)
    dens = mixture_density(*mix, i[:, None] - (j // s)[None, :])
    return dens / dens.sum(axis=0)


def bayes(cond, prior):
    """hdp_model.py:334-363."""
    joint = cond * np.asarray(prior, np.float64)[None, :]
    row_sum = joint.sum(axis=1, keepdims=True)
    dead = row_sum[:, 0] <= 0.0
    if np.any(dead):
        joint[dead] = 1.0
        row_sum = joint.sum(axis=1, keepdims=True)
    return joint / row_sum


def predict_intervals(bmat, delta):
    """hdp_model.py:498-525."""
    out = []
    for row in bmat:
        order = np.argsort(-row, kind="stable")
        chosen = [int(order[0])]
        c = float(row[order[0]])
        for j in order[1:].tolist():
            p = float(row[j])
            if p / (c + p) < delta:
                break
            chosen.append(j)
            c += p
        out.append(np.array(sorted(chosen), np.int64))
    return out


def parse_gmm(text: str):
    """Minimal reader for the .gmm format (hdp_model.py:105-147)."""
    rows = [ln.strip() for ln in text.splitlines() if ln.strip() and not ln.strip().startswith("#")]
    it = iter(rows)
    assert next(it) == "version 1"
    n = int(next(it).split()[1])
    layers = []
    for _ in range(n):
        next(it)
        next(it)
        pi = np.array([float(t) for t in next(it).split()[1:]])
        mu = np.array([float(t) for t in next(it).split()[1:]])
        sg = np.array([float(t) for t in next(it).split()[1:]])
        layers.append((pi, mu, sg))
    return layers


# --------------------------------------------------------------- pipelines
@dataclass
class LevelOut:
    level: int
    disparity: np.ndarray  # (H, W) int32
    min_cost: np.ndarray  # (H, W) float64
    second_cost: np.ndarray  # (H, W) float64: second-best aggregated cost (tie band)
    search_ratio: float
    n_trees: int
    stored_entries: int
    forest: DForest | None = None
    table: list | None = None
    counts: np.ndarray | None = None


def _layer_wta(left_I, right_I, d_max, forest: DForest, gamma, want_volume=False, prepared=None):
    """masked_cost_volume + aggregate_tree + WTA (cost_volume.py:183-236,
    aggregation.py:182-256), evaluated tree by tree on each tree's interval.
    Returns (disparity, best, second[, entries, ent_off])."""
    h, w = left_I.shape[:2]
    L, R = prepared if prepared is not None else (prepare_layer(left_I), prepare_layer(right_I))
    c = L.unit.shape[2]
    n = h * w
    base = forest.base
    sizes = np.array([iv.size for iv in forest.intervals], np.int64)
    iv_off = np.concatenate(([0], np.cumsum(sizes))).astype(np.int64)
    iv_vals = (np.concatenate(forest.intervals).astype(np.int64)
               if forest.intervals else np.zeros(0, np.int64))
    pos = np.empty(n, np.int64)
    pos[base.order] = np.arange(n)
    sim = np.ascontiguousarray(base.similarities(gamma))
    disp = np.zeros(n, np.int32)
    best = np.empty(n)
    second = np.empty(n)
    m_px = sizes[base.tree_id]
    ent_off = np.concatenate(([0], np.cumsum(m_px)[:-1])).astype(np.int64)
    vol = np.empty(int(m_px.sum())) if want_volume else None
    lib().or_layer_wta(h, w, c, _p(L.unit, _f64), _p(L.grad, _f64), _p(R.unit, _f64),
                       _p(R.grad, _f64), C.c_double(ALPHA), C.c_double(TAU_C),
                       C.c_double(TAU_G), base.n_trees, _p(base.tree_slices, _i64),
                       _p(base.order, _i64), _p(pos, _i64), _p(base.parent, _i64),
                       _p(base.depth, _i64), _p(sim, _f64), _p(iv_off, _i64), _p(iv_vals, _i64),
                       disp.ctypes.data_as(C.POINTER(C.c_int32)), _p(best, _f64),
                       _p(second, _f64), _p(ent_off, _i64),
                       _p(vol, _f64) if want_volume else None)
    out = (disp.reshape(h, w), best.reshape(h, w), second.reshape(h, w))
    if want_volume:
        out = out + (vol, ent_off)
    return out


def _order(wt, tree_kind, n_edges, seed):
    """edge_order (spanning_forest.py:115-120); "st" walks the MST order."""
    return rt_edge_order(n_edges, seed) if tree_kind == "rt" else mst_edge_order(wt)


def run_baseline(left_u8, right_u8, d_max, gamma=0.1, tree_kind="mst", seed=0, st_k=ST_K) -> LevelOut:
    """aggregation.py:274-358 (tree mst/rt; streaming is result-neutral)."""
    I_l = np.asarray(left_u8, np.float64)
    I_r = np.asarray(right_u8, np.float64)
    h, w = I_l.shape[:2]
    u, v, wt = build_edge_list(I_l)
    order = _order(wt, tree_kind, u.size, seed)
    forest = build_hdpf(u, v, wt, h * w, full_masks(h * w, d_max), d_max, 0.0, order,
                        st_k if tree_kind == "st" else None)
    d, c, c2 = _layer_wta(I_l, I_r, d_max, forest, gamma)
    return LevelOut(0, d, c, c2, 1.0, forest.n_trees, h * w * (d_max + 1), forest)


def merge_best(a, b):
    """Fold two (disparity, best, second) partial WTA results over disjoint
    disparity chunks, `a` holding the smaller disparities: strict `<` keeps
    `a` on exact ties (the global first argmin, aggregation.py:320-326);
    `second` stays the second-smallest aggregated cost over both chunks."""
    da, ba, sa = a
    db, bb, sb = b
    take_b = bb < ba
    d = np.where(take_b, db, da)
    best = np.where(take_b, bb, ba)
    second = np.where(take_b, np.minimum(ba, sb), np.minimum(sa, bb))
    return d, best, second


def _mem_budget(default=24 << 30) -> int:
    """Host bytes the chunked oracle may hold at once: 24 GiB or 40 % of the
    available memory, whichever is smaller."""
    try:
        with open("/proc/meminfo") as fh:
            for ln in fh:
                if ln.startswith("MemAvailable:"):
                    return int(min(default, 0.4 * int(ln.split()[1]) * 1024))
    except OSError:
        pass
    return default


def chunk_plan(n: int, d_max: int, threads: int, mem_budget: int | None = None):
    """Disparity chunk size of the streamed oracle: as many lanes per thread
    as the memory budget allows (up + down float64 passes, 16 B per lane and
    pixel), like the reference's STREAM_ENTRY_BUDGET streaming."""
    mem_budget = _mem_budget() if mem_budget is None else mem_budget
    return int(max(1, min(d_max + 1, mem_budget // max(1, threads * 16 * n))))


def run_baseline_chunked(left_u8, right_u8, d_max, gamma=0.1, chunk=None, threads=None,
                         forest=None, starts=None) -> LevelOut:
    """run_baseline for pairs whose full float64 volume does not fit in host
    memory (C5: 5.7 M px x 513 lanes): the reference's own disparity
    streaming (aggregation.py:311-326), chunks on a thread pool (the C
    routine releases the GIL), partial results folded by merge_best.  The
    tree is built once and both layers prepared once, as the reference does.
    `starts` restricts the run to the chunks beginning at those disparities
    (a timing sample)."""
    from concurrent.futures import ThreadPoolExecutor
    from dataclasses import replace

    I_l = np.asarray(left_u8, np.float64)
    I_r = np.asarray(right_u8, np.float64)
    h, w = I_l.shape[:2]
    n = h * w
    if forest is None:
        u, v, wt = build_edge_list(I_l)
        forest = build_hdpf(u, v, wt, n, full_masks(n, 0), 0, 0.0, mst_edge_order(wt))
    threads = threads or min(os.cpu_count() or 1, 64)
    chunk = chunk or chunk_plan(n, d_max, threads)
    if starts is None:
        starts = list(range(0, d_max + 1, chunk))
    prepared = (prepare_layer(I_l), prepare_layer(I_r))

    def one(x0):
        xs = np.arange(x0, min(x0 + chunk, d_max + 1), dtype=np.int64)
        f = replace(forest, intervals=[xs] * forest.n_trees, d_max=d_max)
        d, c, c2 = _layer_wta(I_l, I_r, d_max, f, gamma, prepared=prepared)
        return d.ravel(), c.ravel(), c2.ravel()

    with ThreadPoolExecutor(threads) as ex:
        parts = list(ex.map(one, starts))
    acc = parts[0]
    for p in parts[1:]:
        acc = merge_best(acc, p)
    d, c, c2 = acc
    return LevelOut(0, d.reshape(h, w).astype(np.int32), c.reshape(h, w), c2.reshape(h, w), 1.0,
                    forest.n_trees, n * (d_max + 1), forest)


def assign_rows(parent_disp: np.ndarray, ch: int, cw: int, s: int) -> np.ndarray:
    """hdp_forest.py:91-123 -> per-pixel table row."""
    rows = np.arange(ch) // s
    cols = np.arange(cw) // s
    return parent_disp[np.ix_(rows, cols)].astype(np.int64).ravel()


def run_hdp(left_u8, right_u8, d_max, model_layers, levels=3, size_class="half",
            gamma=0.1, s=2, delta0=None, beta=None, tree_kind="mst", seed=0, st_k=ST_K,
            teacher=None, keep=False):
    """aggregation.py:367-488.  `teacher`, if given, maps level -> the
    level's disparity map to hand to the next finer level instead of this
    oracle's own result (teacher forcing)."""
    preset = HALF if size_class == "half" else FULL
    delta0 = preset["delta0"] if delta0 is None else delta0
    beta = preset["beta"] if beta is None else beta
    pl = build_pyramid(left_u8, d_max, s, levels)
    pr = build_pyramid(right_u8, d_max, s, levels)
    outs = []
    top = levels
    I_l, dt = pl[top]
    h, w = I_l.shape[:2]
    u, v, wt = build_edge_list(I_l)
    stk = st_k if tree_kind == "st" else None
    order = _order(wt, tree_kind, u.size, seed)
    forest = build_hdpf(u, v, wt, h * w, full_masks(h * w, dt), dt, 0.0, order, stk)
    d, c, c2 = _layer_wta(I_l, pr[top][0], dt, forest, gamma)
    outs.append(LevelOut(top, d, c, c2, forest.search_ratio(), forest.n_trees,
                         forest.total_search_entries(), forest if keep else None))
    parent = d if teacher is None or top not in teacher else teacher[top]
    for level in range(top - 1, -1, -1):
        I_l, dc = pl[level]
        I_r = pr[level][0]
        dp = pl[level + 1][1]
        h, w = I_l.shape[:2]
        counts, kept = prior_counts(I_l, I_r, dc)
        prior = prior_from_counts(counts, kept)
        cond = conditional(model_layers[level], dc, dp, s)
        bm = bayes(cond, prior)
        table = predict_intervals(bm, delta0 * s**level)
        rows = assign_rows(parent, h, w, s)
        row_masks = masks_from_rows(table, dc)
        pix = row_masks[rows]
        u, v, wt = build_edge_list(I_l)
        order = _order(wt, tree_kind, u.size, seed)
        forest = build_hdpf(u, v, wt, h * w, pix, dc, beta, order, stk)
        d, c, c2 = _layer_wta(I_l, I_r, dc, forest, gamma)
        outs.append(LevelOut(level, d, c, c2, forest.search_ratio(), forest.n_trees,
                             forest.total_search_entries(), forest if keep else None,
                             table if keep else None, counts if keep else None))
        parent = d if teacher is None or level not in teacher else teacher[level]
    return outs


# --------------------------------------------------------------- evaluation
def error_rate(pred, pred_valid, gt, gt_valid, occlusion=None, threshold=1) -> float:
    """evaluation.py:27-54 (numpy restatement)."""
    evaluated = pred_valid & gt_valid
    if occlusion is not None:
        evaluated = evaluated & ~occlusion
    n = int(evaluated.sum())
    diff = np.abs(pred.astype(np.int64) - gt.astype(np.int64))
    return 100.0 * float((diff[evaluated] >= threshold).sum()) / n


def occlusion_from_gt(gl, gl_valid, gr, gr_valid) -> np.ndarray:
    """evaluation.py:57-76 (numpy restatement)."""
    h, w = gl.shape
    target = np.arange(w)[None, :] - gl
    inside = target >= 0
    safe = np.maximum(target, 0)
    rows = np.arange(h)[:, None]
    consistent = inside & gr_valid[rows, safe] & (np.abs(gl - gr[rows, safe]) <= 1)
    return gl_valid & ~consistent
