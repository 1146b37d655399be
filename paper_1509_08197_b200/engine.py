"""Device-resident, batched HDP stereo pipeline.

Torch tensors carry device memory and the current stream; all arithmetic is
in libhdpstereo.so (sm_100a) behind the C ABI (include/hdp_stereo.h).  Host
code here only sequences stages and builds the small probability tables
(A13-A15 of SURVEY.md §8a, <= 121x241 entries) with the reference's own numpy
formulas -- control plane, not a fallback.

Entry points:
  run_baseline_batch -- run_baseline_pipeline (aggregation.py:274-358) for B pairs
  run_hdp_batch      -- run_hdp_pipeline (aggregation.py:367-488) for B pairs
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .errors import ConfigError, DataError, InternalError

ALPHA, TAU_C, TAU_G = 0.9, 0.0275, 0.0078  # cost_volume.py:38-40
TREE_KINDS = ("mst", "rt", "st")
# Segment tree (tree_kind "st", absent from the reference): k of the subtree
# criterion w <= min(Int(Ta) + k/|Ta|, Int(Tb) + k/|Tb|), weights on 0..255.
ST_K = 1200.0


def _t():
    return L.torch_mod()


@dataclass(frozen=True)
class CostConsts:
    alpha: float = ALPHA
    tau_color: float = TAU_C
    tau_grad: float = TAU_G


# ------------------------------------------------------------------ levels
@dataclass
class Level:
    level: int
    h: int
    w: int
    c: int
    d_max: int
    img_l: object  # (B, h, w, c) f64
    img_r: object
    packed_l: object = None  # (B, h, w, 4) f32
    packed_r: object = None
    unit_l: object = None  # f64 planes for the exact prior
    grad_l: object = None
    unit_r: object = None
    grad_r: object = None


def to_f64(u8):
    torch = _t()
    out = torch.empty(u8.shape, dtype=torch.float64, device=u8.device)
    L.call("hdp_u8_to_f64", L.ptr(u8), L.ptr(out), u8.numel(), L.stream())
    return out


def block_mean(img, s: int):
    torch = _t()
    b, h, w, c = img.shape
    out = torch.empty((b, -(-h // s), -(-w // s), c), dtype=torch.float64, device=img.device)
    L.call("hdp_block_mean", L.ptr(img), L.ptr(out), b, h, w, c, s, L.stream())
    return out


def prepare(img, want_f64: bool, want_packed: bool = True, want_gray: bool = False):
    torch = _t()
    b, h, w, c = img.shape
    dev = img.device
    unit = torch.empty((b, h, w, c), dtype=torch.float64, device=dev) if want_f64 else None
    grad = torch.empty((b, h, w), dtype=torch.float64, device=dev) if want_f64 else None
    gray = torch.empty((b, h, w), dtype=torch.float64, device=dev) if want_gray else None
    packed = torch.empty((b, h, w, 4), dtype=torch.float32, device=dev) if want_packed else None
    L.call("hdp_prepare", L.ptr(img), b, h, w, c, L.ptr(unit), L.ptr(gray), L.ptr(grad),
           L.ptr(packed), L.stream())
    return unit, gray, grad, packed


def build_levels(left_u8, right_u8, d_max: int, levels: int, s: int, need_prior: bool):
    """pyramid.py:78-122 + prepare_layer per level (device)."""
    out = []
    il, ir = to_f64(left_u8), to_f64(right_u8)
    d = d_max
    for lvl in range(levels + 1):
        if lvl > 0:
            il, ir = block_mean(il, s), block_mean(ir, s)
            d = d // s
        b, h, w, c = il.shape
        prior = need_prior and lvl < levels
        ul, _, gl, pl = prepare(il, prior)
        ur, _, gr, pr = prepare(ir, prior)
        out.append(Level(lvl, h, w, c, d, il, ir, pl, pr, ul, gl, ur, gr))
    return out


# ------------------------------------------------------------------- edges
def grid_edges(img):
    torch = _t()
    b, h, w, c = img.shape
    E = 2 * h * w - h - w
    dev = img.device
    eu = torch.empty(b * E, dtype=torch.int32, device=dev)
    ev = torch.empty(b * E, dtype=torch.int32, device=dev)
    ew = torch.empty(b * E, dtype=torch.float32, device=dev)
    key = torch.empty(b * E, dtype=torch.int64, device=dev)
    if b * E > 0:
        L.call("hdp_grid_edges", L.ptr(img), b, h, w, c, L.ptr(eu), L.ptr(ev), L.ptr(ew),
               L.ptr(key), L.stream())
    return eu, ev, ew, key, E


def rt_keys(n_edges: int, batch: int, seed: int, device):
    """rt_edge_order (spanning_forest.py:110-112): the seeded numpy PCG64
    permutation defines the order; key = (rank << 32) | index."""
    torch = _t()
    perm = np.random.default_rng(seed).permutation(n_edges)
    rank = np.empty(n_edges, np.int64)
    rank[perm] = np.arange(n_edges, dtype=np.int64)
    key = (rank << 32) | np.arange(n_edges, dtype=np.int64)
    return torch.from_numpy(np.tile(key, batch)).to(device)


def mst(n_nodes: int, eu, ev, key):
    torch = _t()
    m = eu.numel()
    in_tree = torch.empty(max(m, 1), dtype=torch.uint8, device=eu.device)
    comp = torch.empty(n_nodes, dtype=torch.int32, device=eu.device)
    rounds = C.c_int(0)
    L.call("hdp_mst", n_nodes, m, L.ptr(eu), L.ptr(ev), L.ptr(key), L.ptr(in_tree), L.ptr(comp),
           C.byref(rounds), L.stream())
    return in_tree[:m], comp, rounds.value


def st_grid(batch: int, h: int, w: int, eu, ev, ew, key, st_k: float):
    """Segment tree per pair of a grid batch (hdp_segment_tree): subtrees
    under the FH criterion, then linked by the MST of the subtree graph."""
    torch = _t()
    m = eu.numel()
    in_tree = torch.empty(max(m, 1), dtype=torch.uint8, device=eu.device)
    comp = torch.empty(batch * h * w, dtype=torch.int32, device=eu.device)
    rounds = C.c_int(0)
    L.call("hdp_segment_tree", batch, h, w, L.ptr(eu), L.ptr(ev), L.ptr(ew), L.ptr(key), float(st_k),
           L.ptr(in_tree), L.ptr(comp), C.byref(rounds), L.stream())
    return in_tree[:m], comp, rounds.value


def plain_tree(tree_kind: str, batch: int, h: int, w: int, eu, ev, ew, key, st_k: float):
    """The plain spanning forest of a grid batch: MST / RT by Boruvka on the
    keys, segment tree by hdp_segment_tree."""
    if tree_kind == "st":
        return st_grid(batch, h, w, eu, ev, ew, key, st_k)
    return mst_grid(batch, h, w, eu, ev, key)


def mst_grid(batch: int, h: int, w: int, eu, ev, key):
    """mst() for a grid edge list of grid_edges (first Boruvka round gathered
    per node)."""
    torch = _t()
    m = eu.numel()
    in_tree = torch.empty(max(m, 1), dtype=torch.uint8, device=eu.device)
    comp = torch.empty(batch * h * w, dtype=torch.int32, device=eu.device)
    rounds = C.c_int(0)
    L.call("hdp_mst_grid", batch, h, w, L.ptr(eu), L.ptr(ev), L.ptr(key), L.ptr(in_tree), L.ptr(comp),
           C.byref(rounds), L.stream())
    return in_tree[:m], comp, rounds.value


# ------------------------------------------------------------------ forest
class DeviceForest:
    """Rooted forest + heavy-path layout owned by libhdpstereo (hdp_forest*)."""

    def __init__(self, n_nodes, eu, ev, ew, in_tree=None, comp=None, gamma: float = 0.1):
        self._h = C.c_void_p()
        self.n = int(n_nodes)
        L.call("hdp_forest_create", self.n, eu.numel(), L.ptr(eu), L.ptr(ev), L.ptr(ew),
               L.ptr(in_tree), L.ptr(comp), float(gamma), C.byref(self._h), L.stream())
        a, b, c, d = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        L.call("hdp_forest_stats", self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(d))
        self.n_trees, self.n_paths, self.n_phases, self.max_depth = a.value, b.value, c.value, d.value
        self.total_entries = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                L.load().hdp_forest_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._h = None

    def enable_timing(self):
        """Record device events around the cost and aggregation stages of
        every aggregate() call (hdp_forest_set_timing)."""
        L.call("hdp_forest_set_timing", self._h, 1)

    def stage_seconds(self) -> tuple[float, float]:
        """(cost, aggregate) seconds of the last aggregate() call; waits for it."""
        a, b = C.c_float(), C.c_float()
        L.call("hdp_forest_stage_ms", self._h, C.byref(a), C.byref(b))
        return a.value / 1e3, b.value / 1e3

    def export(self):
        torch = _t()
        dev = L.device()
        o = {k: torch.empty(self.n, dtype=torch.int32, device=dev)
             for k in ("parent", "depth", "tree_id", "size", "root")}
        o["parent_weight"] = torch.empty(self.n, dtype=torch.float32, device=dev)
        L.call("hdp_forest_export", self._h, L.ptr(o["parent"]), L.ptr(o["depth"]),
               L.ptr(o["tree_id"]), L.ptr(o["size"]), L.ptr(o["parent_weight"]),
               L.ptr(o["root"]), L.stream())
        return o

    def set_lanes_range(self, x0: int, nx: int):
        L.call("hdp_forest_set_lanes_range", self._h, int(x0), int(nx), L.stream())
        self._entries()

    def set_lanes_nodes(self, node_masks):
        """node_masks: (n, nw) int32/uint32 bitsets valid at every node (hdpf)."""
        L.call("hdp_forest_set_lanes_nodes", self._h, L.ptr(node_masks), node_masks.shape[1], L.stream())
        self._entries()

    def set_lanes(self, tree_masks):
        """tree_masks: (n_trees, nw) int32/uint32 bitsets on the device."""
        L.call("hdp_forest_set_lanes", self._h, L.ptr(tree_masks), tree_masks.shape[1], L.stream())
        self._entries()

    def _entries(self):
        t = C.c_int64()
        L.call("hdp_forest_entries", self._h, C.byref(t), None, L.stream())
        self.total_entries = t.value

    def node_offsets(self):
        torch = _t()
        off = torch.empty(self.n + 1, dtype=torch.int64, device=L.device())
        L.call("hdp_forest_entries", self._h, None, L.ptr(off), L.stream())
        off[self.n] = self.total_entries
        return off

    def aggregate(self, lev: Level | None = None, cost: CostConsts = CostConsts(),
                  cost_rows=None, want_volume=False, want_keys=False):
        """Fused cost + two-pass aggregation + WTA.  Returns
        (disp int32 (n), min_cost f32 (n), keys u64-as-int64 (n) | None,
        volume f32 (total_entries) | None)."""
        torch = _t()
        dev = L.device()
        disp = torch.empty(self.n, dtype=torch.int32, device=dev)
        mc = torch.empty(self.n, dtype=torch.float32, device=dev)
        keys = torch.empty(self.n, dtype=torch.int64, device=dev) if want_keys else None
        vol = (torch.empty(max(self.total_entries, 1), dtype=torch.float32, device=dev)
               if want_volume else None)
        if lev is not None:
            args = (L.ptr(lev.packed_l), L.ptr(lev.packed_r), lev.h, lev.w, lev.c)
        else:
            args = (None, None, 0, 0, 3)
        L.call("hdp_aggregate_wta", self._h, *args, cost.alpha, cost.tau_color, cost.tau_grad,
               L.ptr(cost_rows), L.ptr(disp), L.ptr(mc), L.ptr(keys), L.ptr(vol), L.stream())
        return disp, mc, keys, vol


def keys_unpack(keys, signed_order: bool = False):
    torch = _t()
    n = keys.numel()
    disp = torch.empty(n, dtype=torch.int32, device=keys.device)
    mc = torch.empty(n, dtype=torch.float32, device=keys.device)
    L.call("hdp_keys_unpack", L.ptr(keys), n, int(signed_order), L.ptr(disp), L.ptr(mc), L.stream())
    return disp, mc


def keys_pack(disp, min_cost, signed_order: bool = False):
    """(disparity, min cost) -> u64 slab keys (int64 tensor; signed_order:
    top bit flipped for an int64 MIN reduction)."""
    torch = _t()
    n = disp.numel()
    keys = torch.empty(n, dtype=torch.int64, device=disp.device)
    disp, min_cost = disp.contiguous(), min_cost.contiguous()  # referenced until the launch
    L.call("hdp_keys_pack", L.ptr(disp), L.ptr(min_cost), n, int(signed_order),
           L.ptr(keys), L.stream())
    return keys


# ------------------------------------------------------------------ tables
def nwords32(d_max: int) -> int:
    return (d_max + 1 + 31) // 32


def mixture_density(weights, means, sigmas, x):
    """Mixture1D.density (hdp_model.py:67-72), same numpy expression."""
    x = np.asarray(x, dtype=np.float64)
    z = (x[..., None] - means) / sigmas
    comp = np.exp(-0.5 * z * z) / (sigmas * np.sqrt(2.0 * np.pi))
    return comp @ weights


def conditional_matrix(mix, d_child, d_parent, s):
    """conditional_parent_given_child (hdp_model.py:320-331)."""
    from .errors import InternalError

    i = np.arange(d_parent + 1)
    j = np.arange(d_child + 1)
    dens = mixture_density(mix.weights, mix.means, mix.sigmas, i[:, None] - (j // s)[None, :])
    col_sum = dens.sum(axis=0)
    if np.any(col_sum <= 0):
        raise InternalError("conditional column vanished; mixture degenerated")
    return dens / col_sum


def bayes_batched(cond, priors):
    """bayes_child_given_parent (hdp_model.py:334-363) for B priors at once.
    Returns (matrix (B, rows, cols), number of dead rows per pair)."""
    joint = cond[None, :, :] * priors[:, None, :]
    row_sum = joint.sum(axis=2, keepdims=True)
    dead = row_sum[:, :, 0] <= 0.0
    n_dead = dead.sum(axis=1)
    if np.any(dead):
        joint[dead] = 1.0
        row_sum = joint.sum(axis=2, keepdims=True)
    return joint / row_sum, n_dead


def predict_masks(bayes, delta: float):
    """predict_intervals (hdp_model.py:498-525), vectorised but in the same
    arithmetic: descending stable order, running mass c accumulated left to
    right (np.cumsum is sequential), stop at the first P/(c+P) < delta.
    Returns chosen (B, rows, cols) bool over disparities."""
    order = np.argsort(-bayes, axis=-1, kind="stable")
    p = np.take_along_axis(bayes, order, axis=-1)
    csum = np.cumsum(p, axis=-1)
    ratio = p[..., 1:] / (csum[..., :-1] + p[..., 1:])
    fail = ratio < delta
    first_fail = np.where(fail.any(axis=-1), fail.argmax(axis=-1), fail.shape[-1])
    k = first_fail + 1  # number of chosen candidates
    ranks = np.arange(bayes.shape[-1])
    chosen_sorted = ranks[None, None, :] < k[..., None]
    chosen = np.zeros_like(chosen_sorted)
    np.put_along_axis(chosen, order, chosen_sorted, axis=-1)
    return chosen


_COND_CACHE: dict = {}


def conditional_device(mix, d_child: int, d_parent: int, s: int, device):
    """conditional_matrix on the host (numpy's exp and column sums), cached on
    the device per (mixture, sizes): it depends only on the model."""
    torch = _t()
    key = (id(mix), d_child, d_parent, s, device.index if hasattr(device, "index") else device)
    hit = _COND_CACHE.get(key)
    if hit is not None and hit[0] is mix:
        return hit[1]
    cond = conditional_matrix(mix, d_child, d_parent, s)
    t = torch.from_numpy(np.ascontiguousarray(cond, dtype=np.float64)).to(device)
    _COND_CACHE[key] = (mix, t)
    return t


def bayes_device(counts, kept, cond_d):
    """priors_from_counts + bayes_batched on the device (hdp_priors_from_counts,
    hdp_bayes; numpy's summation order): no host round trip between the
    prior's counts and the interval masks.  Returns (B, rows, cols) f64."""
    torch = _t()
    b, d1 = counts.shape
    rows, cols = cond_d.shape
    if cols != d1:
        raise InternalError(f"conditional matrix has {cols} columns, prior has {d1}")
    pri = torch.empty((b, d1), dtype=torch.float64, device=counts.device)
    L.call("hdp_priors_from_counts", L.ptr(counts.contiguous()), L.ptr(kept.contiguous()), b, d1, L.ptr(pri),
           L.stream())
    bm = torch.empty((b, rows, cols), dtype=torch.float64, device=counts.device)
    L.call("hdp_bayes", L.ptr(cond_d), L.ptr(pri), b, rows, cols, L.ptr(bm), None, L.stream())
    return bm


def predict_masks_device(bayes, delta: float, device):
    """predict_masks + pack_masks on the device (hdp_predict_masks): (B, rows,
    cols) f64 Bayes matrices (host numpy or a device tensor) -> (B, rows, nw)
    int32-viewed u32 bitsets on `device`, bit-identical to the host functions."""
    torch = _t()
    b, rows, cols = bayes.shape
    nw = (cols + 31) // 32
    if isinstance(bayes, np.ndarray):
        bd = torch.from_numpy(np.ascontiguousarray(bayes, dtype=np.float64)).to(device, non_blocking=True)
    else:
        bd = bayes.contiguous()
    out = torch.empty((b, rows, nw), dtype=torch.int32, device=device)
    L.call("hdp_predict_masks", L.ptr(bd), b * rows, cols, float(delta), L.ptr(out), nw, L.stream())
    return out


def pack_masks(chosen) -> np.ndarray:
    """(…, d+1) bool -> (…, nw) uint32 bitsets."""
    d1 = chosen.shape[-1]
    nw = (d1 + 31) // 32
    pad = np.zeros(chosen.shape[:-1] + (nw * 32,), bool)
    pad[..., :d1] = chosen
    bits = pad.reshape(chosen.shape[:-1] + (nw, 32)).astype(np.uint64)
    weights = (np.uint64(1) << np.arange(32, dtype=np.uint64))
    return (bits * weights).sum(axis=-1).astype(np.uint32)


# CTAs of the early (side-stream) prior launches; 0 = one warp per centre, uncapped
PRIOR_SIDE_CTAS = int(os.environ.get("HDP_PRIOR_SIDE_CTAS", "0"))
_PRIOR_EARLY_ENV = os.environ.get("HDP_PRIOR_EARLY", "")
# diagnostics only (never set by bench.py or the tests): reuse the first step's prior counts, to
# measure how much of an HDP step the sampled prior leaves exposed
_DIAG_PRIOR_CACHE = os.environ.get("HDP_DIAG_PRIOR_CACHE", "0") == "1"
_DIAG_PRIORS: dict = {}
PRIOR_SIDE = os.environ.get("HDP_PRIOR_SIDE", "1") != "0"  # diagnostics: 0 = priors inline on the level stream
PRIOR_EARLY = _PRIOR_EARLY_ENV == "1"


def prior_counts(lev: Level, stride=5, window=7, max_offset=1, cost: CostConsts = CostConsts(),
                 max_ctas: int = 0):
    torch = _t()
    b = lev.img_l.shape[0]
    dev = lev.img_l.device
    counts = torch.empty((b, lev.d_max + 1), dtype=torch.int64, device=dev)
    kept = torch.empty(b, dtype=torch.int64, device=dev)
    L.call("hdp_prior_counts", L.ptr(lev.unit_l), L.ptr(lev.grad_l), L.ptr(lev.unit_r),
           L.ptr(lev.grad_r), b, lev.h, lev.w, lev.c, lev.d_max, stride, window, max_offset,
           cost.alpha, cost.tau_color, cost.tau_grad, L.ptr(counts), L.ptr(kept), int(max_ctas), L.stream())
    return counts, kept


def priors_from_counts(counts: np.ndarray, kept: np.ndarray) -> np.ndarray:
    """hdp_model.py:465-470 per pair."""
    b, d1 = counts.shape
    out = np.empty((b, d1))
    for i in range(b):
        if kept[i] == 0:
            out[i] = np.full(d1, 1.0 / d1)
        else:
            hist = counts[i].astype(np.float64) + 1.0
            out[i] = hist / hist.sum()
    return out


def assign_rows(parent_disp, h: int, w: int, s: int, n_rows: int):
    torch = _t()
    b, ph, pw = parent_disp.shape
    rows = torch.empty(b * h * w, dtype=torch.int32, device=parent_disp.device)
    L.call("hdp_assign_rows", L.ptr(parent_disp), b, ph, pw, h, w, s, n_rows, L.ptr(rows),
           L.stream())
    return rows


def hdpf(batch, npp, epp, eu, ev, key, pixel_row, row_masks, beta: float, ew=None, st_k: float = -1.0):
    """build_hdpf for a batch (hdp_hdpf); st_k >= 0: the segment-tree variant."""
    torch = _t()
    dev = eu.device
    n = batch * npp
    nw = row_masks.shape[-1]
    n_rows = row_masks.shape[1]
    in_tree = torch.empty(max(eu.numel(), 1), dtype=torch.uint8, device=dev)
    comp = torch.empty(n, dtype=torch.int32, device=dev)
    tmasks = torch.empty((n, nw), dtype=torch.int32, device=dev)
    rounds = C.c_int(0)
    L.call("hdp_hdpf", batch, npp, epp, L.ptr(eu), L.ptr(ev), L.ptr(key), L.ptr(pixel_row),
           L.ptr(row_masks), n_rows, nw, float(beta), L.ptr(ew), float(st_k), L.ptr(in_tree), L.ptr(comp),
           L.ptr(tmasks), C.byref(rounds), L.stream())
    return in_tree[: eu.numel()], comp, tmasks, rounds.value


# --------------------------------------------------------------- pipelines
class _Lazy:
    """A LevelOut statistic still on the device (hdp_forest_pair_stats_device):
    read back on first access, so the level loop never waits for it."""

    def __init__(self, dev, batch: int, npp: int, d_max: int, which: int):
        self.dev, self.batch, self.npp, self.d_max, self.which = dev, batch, npp, d_max, which

    def get(self):
        h = self.dev.cpu().numpy()
        nt, st = h[: self.batch].copy(), h[self.batch:].copy()
        if self.which == 0:
            return nt
        if self.which == 1:
            return st
        return np.array([float(v) / self.npp / (self.d_max + 1) for v in st])


@dataclass
class LevelOut:
    level: int
    h: int
    w: int
    d_max: int
    disparity: object  # (B, h, w) int32 device
    min_cost: object  # (B, h, w) f32 device
    n_trees: np.ndarray  # (B,)
    stored_entries: np.ndarray  # (B,)
    search_ratio: np.ndarray  # (B,) float
    timings: dict = field(default_factory=dict)
    forest: object = None
    extra: dict = field(default_factory=dict)

    def __getattribute__(self, name):
        v = object.__getattribute__(self, name)
        if isinstance(v, _Lazy):
            v = v.get()
            object.__setattr__(self, name, v)
        return v


def _per_pair_stats_lazy(f: DeviceForest, batch: int, npp: int, d_max: int):
    """(n_trees, stored_entries, search_ratio) as _Lazy device-backed values."""
    torch = _t()
    dev = torch.empty(2 * batch, dtype=torch.int64, device=L.device())
    L.call("hdp_forest_pair_stats_device", f._h, batch, npp, L.ptr(dev), L.stream())
    return tuple(_Lazy(dev, batch, npp, d_max, k) for k in range(3))


def _per_pair_stats(f: DeviceForest, batch: int, npp: int, d_max: int):
    ntrees = np.zeros(batch, np.int64)
    stored = np.zeros(batch, np.int64)
    L.call("hdp_forest_pair_stats", f._h, batch, npp, ntrees.ctypes.data, stored.ctypes.data,
           L.stream())
    # DisparityForest.search_ratio: mean interval size over pixels / (d+1)
    ratio = np.array([float(s) / npp / (d_max + 1) for s in stored])
    return ntrees, stored, ratio


class _Clock:
    """Stage timers from CUDA events recorded on the current stream: no
    synchronisation inside the pipeline (the stages keep overlapping the side
    streams); durations are resolved once the caller has the results."""

    def __init__(self, on: bool):
        self.on = on
        self.marks: list = []
        self.forests: list = []  # forests whose aggregate() stages were timed
        self.acc: dict = {}
        self.last = self._record() if on else None

    @staticmethod
    def _record():
        ev = L.torch_mod().cuda.Event(enable_timing=True)
        ev.record()
        return ev

    def lap(self, key, t0=None):
        """Charge the time since the previous mark to `key`."""
        if not self.on:
            return None
        ev = self._record()
        self.marks.append((key, self.last, ev))
        self.last = ev
        return None

    def add(self, key, seconds: float):
        self.acc[key] = self.acc.get(key, 0.0) + seconds

    def resolve(self) -> dict:
        for key, a, b in self.marks:
            if key.startswith("_"):
                continue
            b.synchronize()
            self.add(key, a.elapsed_time(b) / 1e3)
        for f in self.forests:
            c, a = f.stage_seconds()
            self.add("cost", c)
            self.add("aggregate", a)
        self.marks, self.forests = [], []
        return self.acc


def _forest_layer(lev: Level, eu, ev, ew, in_tree, comp, gamma, cost, masks=None,
                  x0=0, nx=None, want_volume=False, want_keys=False, clock=None, probe=None):
    f = DeviceForest(lev.img_l.shape[0] * lev.h * lev.w, eu, ev, ew, in_tree, comp, gamma)
    if masks is None:
        f.set_lanes_range(x0, lev.d_max + 1 if nx is None else nx)
    else:
        f.set_lanes(masks)
    disp, mc, keys, vol = _aggregate_timed(f, lev, cost, clock, probe, want_volume=want_volume,
                                           want_keys=want_keys)
    return f, disp, mc, keys, vol


def _aggregate_timed(f: DeviceForest, lev: Level, cost, clock=None, probe=None, **kw):
    """f.aggregate with the stage clock: the tree build up to here is charged
    to "forest"; the cost and aggregation stages come from the library's own
    events (resolved later by clock.resolve)."""
    if clock is not None and clock.on:
        clock.lap("forest")
        f.enable_timing()
    if probe is not None:  # CUDA events around the fused aggregation (bench roofline)
        ev0 = _t().cuda.Event(enable_timing=True)
        ev1 = _t().cuda.Event(enable_timing=True)
        ev0.record()
    out = f.aggregate(lev, cost, **kw)
    if probe is not None:
        ev1.record()
        probe.append((ev0, ev1, f.total_entries, f.n))
    if clock is not None and clock.on:
        clock.lap("_cost_aggregate")
        clock.forests.append(f)
    return out



# ---- scratch pool sizing
# The library's scratch comes from the stream-ordered CUDA pool.  A pool that
# grows piecemeal goes back to the driver for physical memory in the middle of
# steps whenever the streams' interleaving asks for a block it cannot carve from
# what it holds (C4 at 64 pairs: one step in ten took 0.5-2 s instead of 0.35 s).
# Sizing it once for the workload (one block allocated and freed,
# hdp_pool_reserve; the pool keeps its memory) removes those stalls: every
# later allocation is carved from memory the process already owns.
# HDP_POOL_RESERVE=0 disables; HDP_POOL_RESERVE_GB=<n> fixes the size.
_POOL_RESERVED: dict = {}
_POOL_ON = os.environ.get("HDP_POOL_RESERVE", "1") != "0"
_POOL_FIXED_GB = float(os.environ.get("HDP_POOL_RESERVE_GB", "0") or 0)


def reserve_pool(nbytes: int) -> None:
    """Grow the scratch pool of the current device to at least `nbytes` (once
    per size: a later, smaller request is a no-op)."""
    if not _POOL_ON:
        return
    torch = _t()
    dev = torch.cuda.current_device()
    if _POOL_FIXED_GB > 0:
        nbytes = int(_POOL_FIXED_GB * 2**30)
    have = _POOL_RESERVED.get(dev, 0)
    if nbytes <= have:
        return
    free, _total = torch.cuda.mem_get_info(dev)
    nbytes = int(min(nbytes, 0.6 * (free + have)))  # never more than 60 % of what is available
    if nbytes <= have:
        return
    L.call("hdp_pool_reserve", int(nbytes), L.stream())
    _POOL_RESERVED[dev] = nbytes


def _dense_scratch_bytes(b, h, w, lanes):
    """Upper estimate of the dense pipeline's scratch: the row buffer (4 bytes
    per hypothesis, rows padded to 4 lanes), keys / records / planes and the
    forest's tables (~450 bytes per pixel measured at C5 and C2)."""
    return int(b * h * w * (4 * ((lanes + 3) & ~3) + 600))


def _hdp_scratch_bytes(b, h, w):
    """Upper estimate of the HDP level loop's scratch (measured: 197 bytes per
    pixel at C4 with 64 pairs, the prior's record sets included) x 2."""
    return int(b * h * w * 400)

# sub-batches of the one-call dense pipeline (hdp_dense_pipeline): the tree
# build of one overlaps the aggregation of another
DENSE_SUB_BATCHES = int(os.environ.get("HDP_DENSE_SUB", "1"))


def run_baseline_fused(left_u8, right_u8, d_max: int, gamma: float = 0.1,
                       cost: CostConsts = CostConsts(), x0: int = 0, nx: int | None = None,
                       n_sub: int | None = None, agg_ms=None, right_ready=None,
                       timing: bool = False) -> LevelOut:
    """run_baseline_batch for plain MST trees in ONE library call
    (hdp_dense_pipeline): the batch runs as concurrent sub-batches on their own
    streams.  agg_ms: optional list that receives each sub-batch's aggregation
    time (ms, device events).  timing: fill LevelOut.timings with the
    reference's stage keys ("forest", "cost_aggregate") from device events."""
    torch = _t()
    if d_max < 1:
        raise ConfigError(f"d_max must be >= 1, got {d_max}")
    b, h, w, c = left_u8.shape
    nx = d_max + 1 if nx is None else nx
    reserve_pool(_dense_scratch_bytes(b, h, w, nx))
    n_sub = DENSE_SUB_BATCHES if n_sub is None else n_sub
    n_sub = max(1, min(n_sub, b))
    dev = left_u8.device
    disp = torch.empty(b * h * w, dtype=torch.int32, device=dev)
    mc = torch.empty(b * h * w, dtype=torch.float32, device=dev)
    ntrees = np.zeros(b, np.int64)
    want_ms = agg_ms is not None or timing
    ams = np.zeros(n_sub, np.float32) if want_ms else None
    if timing:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
    left_u8, right_u8 = left_u8.contiguous(), right_u8.contiguous()  # referenced until the launch
    L.call("hdp_dense_pipeline", L.ptr(left_u8), L.ptr(right_u8), b, h, w, c,
           d_max, x0, nx, cost.alpha, cost.tau_color, cost.tau_grad, gamma, n_sub, L.ptr(disp), L.ptr(mc),
           ntrees.ctypes.data, ams.ctypes.data if ams is not None else None,
           right_ready.cuda_event if right_ready is not None else None, L.stream())
    timings = {}
    if timing:
        e1.record()
        e1.synchronize()
        total = e0.elapsed_time(e1) / 1e3
        agg = float(ams.max()) / 1e3
        timings = {"forest": max(0.0, total - agg), "cost_aggregate": agg}
    if agg_ms is not None:
        agg_ms.extend(float(x) for x in ams)
    stored = np.full(b, h * w * nx, np.int64)
    ratio = np.array([float(s) / (h * w) / (d_max + 1) for s in stored])
    return LevelOut(0, h, w, d_max, disp.view(b, h, w), mc.view(b, h, w), ntrees, stored, ratio,
                    timings, None)


def level_keys(img, E: int, level: int, block_size: int, key):
    """Kruskal keys of a pyramid level's grid edges.  hdp_grid_edges keys on
    the f32 weight bits, exact for uint8 images and every S=2 level (dyadic
    block means).  Other block sizes give non-dyadic means whose
    f32 weights can merge distinct float64 weights: those levels are keyed on
    the stable rank of the float64 weights (mst_edge_order's order,
    spanning_forest.py:96-107) instead."""
    if level == 0 or block_size == 2:
        return key
    torch = _t()
    b, h, w, c = img.shape
    dev = img.device
    w64 = torch.empty(b * E, dtype=torch.float64, device=dev)
    L.call("hdp_grid_edge_weights64", L.ptr(img), b, h, w, c, L.ptr(w64), L.stream())
    bits = w64.view(torch.int64)  # monotone for non-negative weights
    idx = torch.arange(E, dtype=torch.int64, device=dev)
    out = torch.empty(b * E, dtype=torch.int64, device=dev)
    perm = torch.empty(E, dtype=torch.int32, device=dev)
    rank = torch.empty(E, dtype=torch.int64, device=dev)
    for i in range(b):
        L.call("hdp_argsort_u64", L.ptr(bits[i * E:(i + 1) * E]), E, L.ptr(perm), L.stream())
        rank[perm.long()] = idx
        out[i * E:(i + 1) * E] = (rank << 32) | idx
    return out


def run_baseline_batch(left_u8, right_u8, d_max: int, gamma: float = 0.1,
                       cost: CostConsts = CostConsts(), tree_kind: str = "mst", seed: int = 0,
                       x0: int = 0, nx: int | None = None, want_volume=False, want_keys=False,
                       keep_forest=False, timing=False, probe=None, stepwise=False,
                       st_k: float = ST_K) -> LevelOut:
    """Full-range aggregation over one MST per pair (aggregation.py:274-358).
    left/right: (B, H, W, C) uint8 device tensors.  [x0, x0+nx) restricts the
    disparity lanes (a slab of the multi-GPU split); default full range.
    MST runs without extra outputs take the one-call pipeline; `stepwise`
    forces the stage-by-stage path (same results, used to test the former)."""
    if tree_kind not in TREE_KINDS:
        raise ConfigError(f"unknown tree kind {tree_kind!r} (want 'mst', 'rt' or 'st')")
    if d_max < 1:
        raise ConfigError(f"d_max must be >= 1, got {d_max}")
    if (tree_kind == "mst" and DENSE_SUB_BATCHES > 0 and not stepwise
            and not (want_volume or want_keys or keep_forest or probe is not None)):
        return run_baseline_fused(left_u8, right_u8, d_max, gamma, cost, x0, nx, timing=timing)
    clock = _Clock(timing)
    b, h, w, c = left_u8.shape
    reserve_pool(_dense_scratch_bytes(b, h, w, d_max + 1 if nx is None else nx) + b * h * w * 200)
    il, ir = to_f64(left_u8), to_f64(right_u8)
    _, _, _, pl = prepare(il, False)
    _, _, _, pr = prepare(ir, False)
    lev = Level(0, h, w, c, d_max, il, ir, pl, pr)
    eu, ev, ew, key, E = grid_edges(il)
    if tree_kind == "rt":
        key = rt_keys(E, b, seed, il.device)
    in_tree, comp, _ = plain_tree(tree_kind, b, h, w, eu, ev, ew, key, st_k)
    f, disp, mc, keys, vol = _forest_layer(lev, eu, ev, ew, in_tree, comp, gamma, cost, None, x0,
                                           nx, want_volume, want_keys, clock, probe)
    ntrees, stored, ratio = _per_pair_stats(f, b, h * w, d_max)
    acc = clock.resolve() if timing else {}
    timings = ({"forest": acc.get("forest", 0.0),
                "cost_aggregate": acc.get("cost", 0.0) + acc.get("aggregate", 0.0)}
               if timing else {})
    out = LevelOut(0, h, w, d_max, disp.view(b, h, w), mc.view(b, h, w), ntrees, stored, ratio,
                   timings, f if keep_forest else None)
    out.extra["keys"] = keys
    out.extra["volume"] = vol
    return out


def run_hdp_batch(left_u8, right_u8, d_max: int, model, levels: int = 3, block_size: int = 2,
                  gamma: float = 0.1, delta0: float = 0.064, beta: float = 0.6,
                  cost: CostConsts = CostConsts(), tree_kind: str = "mst", seed: int = 0,
                  teacher: dict | None = None, keep=False, want_volume=False, timing=False,
                  on_level=None, st_k: float = ST_K) -> list[LevelOut]:
    """Coarse-to-fine HDP matching for B pairs (aggregation.py:367-488).

    `model` exposes .layers[l] with .weights/.means/.sigmas (GmmModel).
    `teacher`: optional {level: (B, h_l, w_l) int32 device map} handed to the
    next finer level instead of this level's own result (teacher forcing).
    timing: per-level stage times from device events (LevelOut.timings keys
    "pyramid" (top level only), "predict", "forest", "cost", "aggregate")."""
    torch = _t()
    if tree_kind not in TREE_KINDS:
        raise ConfigError(f"unknown tree kind {tree_kind!r} (want 'mst', 'rt' or 'st')")
    if len(model.layers) < levels:
        raise DataError(f"model covers {len(model.layers)} level transitions, run needs {levels}")
    if d_max // block_size**levels < 1:
        raise ConfigError(f"d_max={d_max} collapses to {d_max // block_size**levels} after "
                          f"{levels} levels of /{block_size}; reduce levels or block_size")
    # The sampled priors of all levels depend only on that level's images:
    # they run on a side stream from the start, beside the coarser levels'
    # tree builds (HDPF keeps one SM per pair busy), while the level loop
    # runs on a high-priority stream so the block scheduler serves it first.
    reserve_pool(_hdp_scratch_bytes(left_u8.shape[0], left_u8.shape[1], left_u8.shape[2]))
    caller = torch.cuda.current_stream()
    pri, hi = _hdp_streams()
    pri.wait_stream(caller)
    hi.wait_stream(caller)
    with torch.cuda.stream(hi):
        outs = _run_hdp_levels(left_u8, right_u8, d_max, model, levels, block_size, gamma, delta0,
                               beta, cost, tree_kind, seed, teacher, keep, want_volume, timing,
                               on_level, prior_stream=pri if PRIOR_SIDE else None, st_k=st_k)
    caller.wait_stream(hi)
    for o in outs:
        o.disparity.record_stream(caller)
        o.min_cost.record_stream(caller)
        if o.extra.get("volume") is not None:
            o.extra["volume"].record_stream(caller)
        clk = o.extra.pop("clock", None)
        if clk is not None:
            o.timings = dict(clk.resolve())
    return outs


_HDP_STREAMS: dict = {}


def _hdp_streams():
    """(prior stream, high-priority level stream) per device."""
    torch = _t()
    dev = torch.cuda.current_device()
    if dev not in _HDP_STREAMS:
        _HDP_STREAMS[dev] = (torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev, priority=-1))
    return _HDP_STREAMS[dev]


def _run_hdp_levels(left_u8, right_u8, d_max, model, levels, block_size, gamma, delta0, beta, cost,
                    tree_kind, seed, teacher, keep, want_volume, timing, on_level, prior_stream=None,
                    st_k: float = ST_K):
    torch = _t()
    clock = _Clock(timing)
    b = left_u8.shape[0]
    lv = build_levels(left_u8, right_u8, d_max, levels, block_size, True)
    clock.lap("pyramid")
    outs: list[LevelOut] = []
    early = {}

    def launch_prior(level):
        # the prior of `level` on the side stream, started once everything
        # queued so far on the level stream has run: called right after the
        # coarser level's forest (the window kernel of the segment tree needs
        # whole SMs, which a running prior grid would keep busy), so it
        # overlaps that level's tree build and aggregation
        if prior_stream is None or level < 0:
            return
        if _DIAG_PRIOR_CACHE and (level, lv[level].h, lv[level].w, b) in _DIAG_PRIORS:
            c_, k_ = _DIAG_PRIORS[(level, lv[level].h, lv[level].w, b)]
            ev_ = torch.cuda.Event()
            ev_.record(torch.cuda.current_stream())
            early[level] = (c_, k_, ev_)
            return
        prior_stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(prior_stream):
            c_, k_ = prior_counts(lv[level], cost=cost, max_ctas=PRIOR_SIDE_CTAS)
            ev_ = torch.cuda.Event()
            ev_.record(prior_stream)
            early[level] = (c_, k_, ev_)
            if _DIAG_PRIOR_CACHE:
                _DIAG_PRIORS[(level, lv[level].h, lv[level].w, b)] = (c_, k_)

    def finish(lev, f, disp, mc, vol, clk):
        ntrees, stored, ratio = _per_pair_stats_lazy(f, b, lev.h * lev.w, lev.d_max)
        o = LevelOut(lev.level, lev.h, lev.w, lev.d_max, disp.view(b, lev.h, lev.w),
                     mc.view(b, lev.h, lev.w), ntrees, stored, ratio, {},
                     f if keep else None)
        o.extra["volume"] = vol
        if timing:
            o.extra["clock"] = clk
        outs.append(o)
        return o

    top = lv[levels]
    eu, ev, ew, key, E = grid_edges(top.img_l)
    if tree_kind == "rt":
        key = rt_keys(E, b, seed, top.img_l.device)
    else:
        key = level_keys(top.img_l, E, levels, block_size, key)
    # every prior at once before the top level (HDP_PRIOR_EARLY=0: each level's
    # prior after the coarser level's forest -- measured equal at C4, 4 %
    # slower at C3 once the pool stopped inserting cross-stream waits)
    prior_first = PRIOR_EARLY or _PRIOR_EARLY_ENV == ""
    if prior_first:
        for level in range(levels - 1, -1, -1):
            launch_prior(level)
    in_tree, comp, _ = plain_tree(tree_kind, b, top.h, top.w, eu, ev, ew, key, st_k)
    if not prior_first:
        launch_prior(levels - 1)
    f, disp, mc, _, vol = _forest_layer(top, eu, ev, ew, in_tree, comp, gamma, cost, None,
                                        want_volume=want_volume, clock=clock)
    o = finish(top, f, disp, mc, vol, clock)
    if on_level is not None:
        on_level(o)
    parent = o.disparity if teacher is None or levels not in teacher else teacher[levels]
    for level in range(levels - 1, -1, -1):
        lev = lv[level]
        lclock = _Clock(timing)
        if level in early:
            counts, kept, ev = early[level]
            torch.cuda.current_stream().wait_event(ev)
        else:
            counts, kept = prior_counts(lev, cost=cost)
        # prior -> Bayes -> interval masks stay on the device (no host read)
        cond_d = conditional_device(model.layers[level], lev.d_max, lv[level + 1].d_max, block_size,
                                    lev.img_l.device)
        bm = bayes_device(counts, kept, cond_d)
        row_masks = predict_masks_device(bm, delta0 * block_size**level, lev.img_l.device)
        counts_h = kept_h = chosen = None
        if keep:
            counts_h, kept_h = counts.cpu().numpy(), kept.cpu().numpy()
            chosen = predict_masks(bm.cpu().numpy(), delta0 * block_size**level)
        rows = assign_rows(parent.contiguous(), lev.h, lev.w, block_size, bm.shape[1])
        lclock.lap("predict")
        eu, ev, ew, key, E = grid_edges(lev.img_l)
        if tree_kind == "rt":
            key = rt_keys(E, b, seed, lev.img_l.device)
        else:
            key = level_keys(lev.img_l, E, level, block_size, key)
        in_tree, comp, tmasks, rounds = hdpf(b, lev.h * lev.w, E, eu, ev, key, rows,
                                             row_masks.contiguous(), beta, ew=ew,
                                             st_k=st_k if tree_kind == "st" else -1.0)
        if not prior_first:
            launch_prior(level - 1)
        fo = DeviceForest(b * lev.h * lev.w, eu, ev, ew, in_tree, comp, gamma)
        fo.set_lanes_nodes(tmasks.contiguous())
        disp, mc, _, vol = _aggregate_timed(fo, lev, cost, lclock, want_volume=want_volume)
        o = finish(lev, fo, disp, mc, vol, lclock)
        o.extra.update(counts=counts_h, kept=kept_h, chosen=chosen if keep else None,
                       dr_rounds=rounds,
                       tree_masks=(_tree_masks_host(fo, tmasks) if keep else None))
        if on_level is not None:
            on_level(o)
        parent = o.disparity if teacher is None or level not in teacher else teacher[level]
    return outs


_SIDE: dict = {}


def _side_stream():
    torch = _t()
    dev = torch.cuda.current_device()
    if dev not in _SIDE:
        _SIDE[dev] = torch.cuda.Stream(device=dev)
    return _SIDE[dev]


def _tree_masks_host(fo: DeviceForest, tmasks):
    """Per-tree masks (trees numbered by root id) on the host (keep=True)."""
    torch = _t()
    roots = fo.export()["root"]
    ar = torch.arange(fo.n, device=roots.device, dtype=torch.int32)
    root_ids = torch.nonzero(roots == ar).flatten()
    return tmasks[root_ids].cpu().numpy().view(np.uint32)


_STAGE: dict = {}
_STAGER = []


STAGE_THREADS = int(os.environ.get("HDP_STAGE_THREADS", "4"))


def _stager():
    if not _STAGER:
        from concurrent.futures import ThreadPoolExecutor

        _STAGER.append(ThreadPoolExecutor(max(2, STAGE_THREADS), thread_name_prefix="hdp-stage"))
    return _STAGER[0]


def _stack_into(images, out: np.ndarray, pool, parts: int):
    """np.stack(images, out=out) as `parts` row blocks copied on the pool's
    threads (numpy releases the GIL while copying): one host thread copies
    ~10 GB/s, so a C5 eye (17 MB) alone takes ~2 ms."""
    b, h = out.shape[0], out.shape[1]
    rows = max(1, -(-b * h // max(1, parts)))
    jobs = []
    for r0 in range(0, b * h, rows):
        r1 = min(b * h, r0 + rows)
        for i in range(r0 // h, (r1 - 1) // h + 1):
            a0, a1 = max(r0, i * h) - i * h, min(r1, (i + 1) * h) - i * h
            jobs.append(pool.submit(np.copyto, out[i, a0:a1], np.asarray(images[i])[a0:a1]))
    return jobs


def stage_pairs(lefts, rights):
    """Host -> device for a list of same-shape (H, W, C) uint8 images per eye:
    the images are stacked straight into cached pinned buffers and copied
    asynchronously, the left eye on the current stream, the right eye on a
    side stream (the dense pipeline first reads it after the tree build).
    Returns (left (B,H,W,C), right, right_ready event): the caller makes its
    stream wait for right_ready before reading the right eye (or hands it to
    hdp_dense_pipeline, which waits only where the right eye is first read)."""
    torch = _t()
    dev = L.device()
    shape = (len(lefts),) + tuple(np.shape(lefts[0]))
    key = (dev.index, shape)
    st = _STAGE.get(key)
    if st is None:
        st = [torch.empty(shape, dtype=torch.uint8).pin_memory(),
              torch.empty(shape, dtype=torch.uint8).pin_memory(), None]
        _STAGE[key] = st
    pl, pr, last = st
    if last is not None:  # the previous call's copies out of these buffers are done
        last.synchronize()
    # both eyes are stacked in row blocks on the staging threads (left blocks
    # first); the left eye's copy starts as soon as its blocks are in
    pool = _stager()
    parts = max(1, STAGE_THREADS) if pl.numel() >= (8 << 20) else 1
    lj = _stack_into(lefts, pl.numpy(), pool, parts)
    rj = _stack_into(rights, pr.numpy(), pool, parts)
    for j in lj:
        j.result()
    ld = pl.to(dev, non_blocking=True)
    side = _side_stream()
    side.wait_stream(torch.cuda.current_stream())
    for j in rj:
        j.result()
    with torch.cuda.stream(side):
        rd = pr.to(dev, non_blocking=True)
        ready = torch.cuda.Event()
        ready.record(side)
    rd.record_stream(torch.cuda.current_stream())
    done = torch.cuda.Event()
    done.record()
    st[2] = _Both(done, ready)
    return ld, rd, ready


class _Both:
    def __init__(self, *events):
        self.events = events

    def synchronize(self):
        for e in self.events:
            e.synchronize()


def run_baseline_host(left_u8: np.ndarray, right_u8: np.ndarray, d_max: int, out=None, **kw):
    """Host-buffer entry point: (B, H, W, C) uint8 numpy (pinned if the caller
    wants async copies) -> (disparity (B, H, W) int32, min_cost (B, H, W)
    float32) numpy.  The copies in both directions are part of the call.
    out: optional (disparity, min_cost) host tensors / arrays to fill (pinned:
    the device->host copies then run as DMA on the stream, one synchronise)."""
    torch = _t()
    dev = L.device()
    lt = torch.from_numpy(left_u8) if isinstance(left_u8, np.ndarray) else left_u8
    rt = torch.from_numpy(right_u8) if isinstance(right_u8, np.ndarray) else right_u8
    ld = lt.to(dev, non_blocking=True)
    if not kw and DENSE_SUB_BATCHES > 0:
        # the right image is first read after the tree build: copy it on a side
        # stream while the left one's trees are built
        side = _side_stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            rd = rt.to(dev, non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(side)
        rd.record_stream(torch.cuda.current_stream())
        res = run_baseline_fused(ld, rd, d_max, right_ready=ready)
    else:
        rd = rt.to(dev, non_blocking=True)
        res = run_baseline_batch(ld, rd, d_max, **kw)
    if out is None:
        return res.disparity.cpu().numpy(), res.min_cost.cpu().numpy()
    od, oc = (torch.from_numpy(o) if isinstance(o, np.ndarray) else o for o in out)
    od.copy_(res.disparity, non_blocking=True)
    oc.copy_(res.min_cost, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return od.numpy(), oc.numpy()


def run_hdp_host(left_u8, right_u8, d_max: int, model, **kw):
    """Host-buffer HDP entry point -> finest-level disparity (B, H, W) int32."""
    torch = _t()
    dev = L.device()
    lt = torch.from_numpy(left_u8) if isinstance(left_u8, np.ndarray) else left_u8
    rt = torch.from_numpy(right_u8) if isinstance(right_u8, np.ndarray) else right_u8
    outs = run_hdp_batch(lt.to(dev, non_blocking=True), rt.to(dev, non_blocking=True), d_max,
                         model, **kw)
    return outs[-1].disparity.cpu().numpy()
