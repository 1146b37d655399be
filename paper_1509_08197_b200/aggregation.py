"""Tree cost aggregation and the two pipelines (drop-in for
treestereo.aggregation).

run_baseline_pipeline / run_hdp_pipeline keep the reference signatures
(aggregation.py:274-281, :367-375) and return the same PipelineResult /
LayerResult objects; the work runs device-resident in libhdpstereo.so
(engine.py).  Batched variants take a list of same-geometry pairs and run them
in one pass.  Costs and aggregation are fp32 (north_star); disparities match
the reference except at near-ties (c2 - c1 <= 1e-5 c1)."""

from __future__ import annotations

import time
from dataclasses import dataclass, replace

import numpy as np

from . import _lib as L
from . import engine as E
from .cost_volume import CostParams, SparseCostVolume
from .errors import ConfigError, DataError, InternalError
from .hdp_forest import DisparityForest, disparity_forest_from_device
from .hdp_model import GmmModel
from .raster_io import DisparityMap, RasterImage, StereoPair
from .spanning_forest import RootedForest, apply_median_prefilter

SIZE_CLASS_PRESETS = {
    "half": {"delta0": 0.064, "beta": 0.6},
    "full": {"delta0": 0.004, "beta": 0.95},
}

# The reference streams the disparity axis in chunks of this many float64
# entries (aggregation.py:74).  The fused GPU pass never materialises the
# raw cost volume, so the constant is kept only for API compatibility.
STREAM_ENTRY_BUDGET = 16_000_000


@dataclass(frozen=True)
class AggregationParams:
    """aggregation.py:77-109."""

    gamma: float = 0.1
    size_class: str = "half"
    block_size: int = 2
    levels: int = 3
    delta0: float | None = None
    beta: float | None = None
    seed: int = 0

    def resolved(self) -> "AggregationParams":
        if self.size_class not in SIZE_CLASS_PRESETS:
            raise ConfigError(f"unknown size class {self.size_class!r} "
                              f"(want one of {sorted(SIZE_CLASS_PRESETS)})")
        preset = SIZE_CLASS_PRESETS[self.size_class]
        out = replace(self,
                      delta0=self.delta0 if self.delta0 is not None else preset["delta0"],
                      beta=self.beta if self.beta is not None else preset["beta"])
        if not 0.0 < out.delta0 < 1.0:
            raise ConfigError(f"delta0 must be in (0, 1), got {out.delta0}")
        if not 0.0 < out.beta <= 1.0:
            raise ConfigError(f"beta must be in (0, 1], got {out.beta}")
        if out.gamma <= 0:
            raise ConfigError(f"gamma must be positive, got {out.gamma}")
        if out.block_size < 2 or out.levels < 1:
            raise ConfigError("block_size must be >= 2 and levels >= 1")
        return out


@dataclass
class LayerResult:
    level: int
    disparity: DisparityMap
    min_cost: np.ndarray
    search_ratio: float
    n_trees: int
    stored_entries: int
    timings: dict[str, float]


@dataclass
class PipelineResult:
    disparity: DisparityMap
    layers: list[LayerResult]
    metrics: dict


# ------------------------------------------------------------- filters
def _device_forest_of(forest: RootedForest, gamma: float) -> "E.DeviceForest":
    torch = E._t()
    dev = L.device()
    n = forest.n_nodes
    nodes = np.flatnonzero(forest.parent != np.arange(n))
    u = torch.from_numpy(forest.parent[nodes].astype(np.int32)).to(dev)
    v = torch.from_numpy(nodes.astype(np.int32)).to(dev)
    w = torch.from_numpy(forest.parent_weight[nodes].astype(np.float32)).to(dev)
    return E.DeviceForest(n, u, v, w, None, None, gamma)


def aggregate_forest(forest: RootedForest, costs: np.ndarray, gamma: float = 0.1) -> np.ndarray:
    """aggregation.py:216-236: two-pass filter of a dense (n, m) matrix (fp32
    on the GPU)."""
    costs = np.asarray(costs, dtype=np.float64)
    if costs.ndim == 1:
        costs = costs[:, None]
    if costs.shape[0] != forest.n_nodes:
        raise ConfigError("cost row count must equal the node count")
    if gamma <= 0:
        raise ConfigError(f"gamma must be positive, got {gamma}")
    n, m = costs.shape
    if m == 0:
        return costs.copy()
    torch = E._t()
    f = _device_forest_of(forest, gamma)
    f.set_lanes_range(0, m)
    rows = torch.from_numpy(np.ascontiguousarray(costs, np.float32).ravel()).to(L.device())
    _, _, _, vol = f.aggregate(None, cost_rows=rows, want_volume=True)
    return vol[: n * m].cpu().numpy().astype(np.float64).reshape(n, m)


def aggregate_tree(volume: SparseCostVolume, forest: DisparityForest,
                   gamma: float = 0.1) -> SparseCostVolume:
    """aggregation.py:182-213 on the GPU (ragged per-tree intervals)."""
    base = forest.base
    if volume.node_order is not base.order and not np.array_equal(volume.node_order, base.order):
        raise InternalError("cost volume and forest disagree on node order")
    if len(volume.intervals) != forest.n_trees:
        raise InternalError("cost volume and forest disagree on tree count")
    for t in range(forest.n_trees):
        if not np.array_equal(volume.intervals[t], forest.intervals[t]):
            raise InternalError(f"tree {t} interval mismatch between volume and forest")
    torch = E._t()
    dev = L.device()
    f = _device_forest_of(base, gamma)
    nw = max(1, (forest.d_max + 1 + 31) // 32)
    words = np.zeros((forest.n_trees, nw), np.uint32)
    for t, m in enumerate(forest.masks):
        for k in range(nw):
            words[t, k] = (m >> (32 * k)) & 0xFFFFFFFF
    f.set_lanes(torch.from_numpy(words.view(np.int32)).to(dev))
    off = f.node_offsets().cpu().numpy()
    flat = np.empty(int(off[-1]), np.float32)
    for t in range(forest.n_trees):
        nodes = base.order[base.tree_slices[t]:base.tree_slices[t + 1]]
        blk = volume.costs[t]
        idx = off[nodes][:, None] + np.arange(blk.shape[1])[None, :]
        flat[idx] = blk
    _, _, _, vol = f.aggregate(None, cost_rows=torch.from_numpy(flat).to(dev), want_volume=True)
    out = vol[: flat.size].cpu().numpy().astype(np.float64)
    costs = []
    for t in range(forest.n_trees):
        nodes = base.order[base.tree_slices[t]:base.tree_slices[t + 1]]
        m = volume.costs[t].shape[1]
        costs.append(out[off[nodes][:, None] + np.arange(m)[None, :]])
    return SparseCostVolume(volume.width, volume.height, volume.d_max, volume.node_order,
                            volume.tree_slices, volume.intervals, costs, volume.pos,
                            volume.tree_of)


def winner_takes_all_with_cost(volume: SparseCostVolume) -> tuple[DisparityMap, np.ndarray]:
    """aggregation.py:239-256: first argmin per pixel (on the device)."""
    torch = E._t()
    n = volume.width * volume.height
    max_m = max((c.shape[1] for c in volume.costs), default=1)
    pad = np.full((n, max_m), np.inf)
    cols = np.zeros((n, max_m), np.int64)
    for t in range(volume.n_trees):
        nodes = volume.node_order[volume.tree_slices[t]:volume.tree_slices[t + 1]]
        blk = volume.costs[t]
        pad[nodes, : blk.shape[1]] = blk
        cols[nodes, : blk.shape[1]] = volume.intervals[t]
    dp = torch.from_numpy(pad).to(L.device())
    j = torch.empty(n, dtype=torch.int32, device=dp.device)
    bd = torch.empty(n, dtype=torch.float64, device=dp.device)
    L.call("hdp_rows_first_argmin", L.ptr(dp), n, int(max_m), L.ptr(j), L.ptr(bd), L.stream())
    best = bd.cpu().numpy()
    jn = j.cpu().numpy().astype(np.int64)
    values = cols[np.arange(n), jn].astype(np.int32)
    disp = DisparityMap(values=values.reshape(volume.height, volume.width),
                        valid=np.ones((volume.height, volume.width), dtype=bool))
    return disp, best.reshape(volume.height, volume.width)


def winner_takes_all(volume: SparseCostVolume) -> DisparityMap:
    return winner_takes_all_with_cost(volume)[0]


# ------------------------------------------------------------ pipelines
def _stack_pairs(pairs: list[StereoPair], median_prefilter: bool, defer_right: bool = False):
    """Host pairs -> device (B,H,W,C) uint8 batches through pinned staging
    (engine.stage_pairs).  With defer_right the right eye's copy may still be
    in flight: the returned event must be waited on before it is read."""
    if not pairs:
        raise DataError("empty batch")
    shape, d = pairs[0].left.data.shape, pairs[0].d_max
    for p in pairs:
        if p.left.data.shape != shape or p.d_max != d:
            raise DataError("batched pairs must share geometry and d_max")
    torch = E._t()
    Ld, Rd, ready = E.stage_pairs([p.left.data for p in pairs], [p.right.data for p in pairs])
    if median_prefilter or not defer_right:
        torch.cuda.current_stream().wait_event(ready)
        ready = None
    if median_prefilter:
        b, h, w, c = Ld.shape
        Lm, Rm = torch.empty_like(Ld), torch.empty_like(Rd)
        L.call("hdp_median3x3", L.ptr(Ld), L.ptr(Lm), b, h, w, c, L.stream())
        L.call("hdp_median3x3", L.ptr(Rd), L.ptr(Rm), b, h, w, c, L.stream())
        Ld, Rd = Lm, Rm
    return Ld, Rd, d, ready


def _dmap(a: np.ndarray) -> DisparityMap:
    return DisparityMap(values=a.astype(np.int32, copy=False), valid=np.ones(a.shape, dtype=bool))


def _to_host(*tensors):
    """Device results -> fresh host numpy arrays: min costs widened to float64
    (the reference's dtype) on the device, then one asynchronous DMA per
    tensor into page-locked memory from torch's caching host allocator (no
    page faults on the hot path) and a single synchronise.  The arrays own
    their pinned blocks; the block returns to the cache when they are freed."""
    torch = E._t()
    outs = []
    for t in tensors:
        if t.dtype == torch.float32:
            t = t.to(torch.float64)
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        outs.append(h)
    torch.cuda.current_stream().synchronize()
    return [h.numpy() for h in outs]


def run_baseline_pipeline_batch(pairs: list[StereoPair], params: AggregationParams | None = None,
                                cost_params: CostParams | None = None, tree_kind: str = "mst",
                                median_prefilter: bool = False,
                                on_forest=None) -> list[PipelineResult]:
    """run_baseline_pipeline for several same-geometry pairs in one pass."""
    params = (params or AggregationParams()).resolved()
    cost_params = cost_params or CostParams()
    if tree_kind not in E.TREE_KINDS:
        raise ConfigError(f"unknown tree kind {tree_kind!r} (want 'mst', 'rt' or 'st')")
    t_start = time.perf_counter()
    fused = tree_kind == "mst" and on_forest is None
    Ld, Rd, d_max, ready = _stack_pairs(pairs, median_prefilter, defer_right=fused)
    # stage times come from device events (no synchronisation between stages);
    # plain MST batches take the one-call dense pipeline, which reads the right
    # eye only after the tree build (its copy overlaps the build)
    if fused:
        out = E.run_baseline_fused(Ld, Rd, d_max, params.gamma, cost_params.consts(),
                                   right_ready=ready, timing=True)
    else:
        out = E.run_baseline_batch(Ld, Rd, d_max, params.gamma, cost_params.consts(), tree_kind,
                                   params.seed, keep_forest=on_forest is not None, timing=True)
    disp, cost = _to_host(out.disparity, out.min_cost)
    total = time.perf_counter() - t_start
    b, h, w = disp.shape
    if on_forest is not None:
        if b != 1:
            raise ConfigError("on_forest is supported for single-pair calls")
        words = np.full((out.forest.n_trees, (d_max + 1 + 31) // 32), 0xFFFFFFFF, np.uint32)
        rem = (d_max + 1) % 32
        if rem:
            words[:, -1] = (1 << rem) - 1
        on_forest(0, disparity_forest_from_device(out.forest, words, d_max))
    res = []
    for i in range(b):
        dm = _dmap(disp[i])
        t_forest = out.timings.get("forest", 0.0)
        t_agg = out.timings.get("cost_aggregate", 0.0)
        layer = LayerResult(0, dm, cost[i], 1.0, int(out.n_trees[i]), h * w * (d_max + 1),
                            {"forest": t_forest, "cost_aggregate": t_agg})
        metrics = {"method": f"{tree_kind}-baseline", "tree": tree_kind, "hdp": False,
                   "median_prefilter": median_prefilter, "seed": params.seed,
                   "search_ratios": [1.0], "stored_entries": layer.stored_entries,
                   "dense_entries": h * w * (d_max + 1),
                   "seconds": {"forest": t_forest, "cost_aggregate": t_agg, "total": total}}
        res.append(PipelineResult(dm, [layer], metrics))
    return res


def run_baseline_pipeline(pair: StereoPair, params: AggregationParams | None = None,
                          cost_params: CostParams | None = None, tree_kind: str = "mst",
                          median_prefilter: bool = False, on_forest=None) -> PipelineResult:
    """aggregation.py:274-358."""
    return run_baseline_pipeline_batch([pair], params, cost_params, tree_kind, median_prefilter,
                                       on_forest)[0]


def run_hdp_pipeline_batch(pairs: list[StereoPair], model: GmmModel,
                           params: AggregationParams | None = None,
                           cost_params: CostParams | None = None, tree_kind: str = "mst",
                           median_prefilter: bool = False, on_forest=None) -> list[PipelineResult]:
    """run_hdp_pipeline for several same-geometry pairs in one pass."""
    params = (params or AggregationParams()).resolved()
    cost_params = cost_params or CostParams()
    if model.n_layers < params.levels:
        raise DataError(f"model covers {model.n_layers} level transitions, run needs "
                        f"{params.levels}")
    t_start = time.perf_counter()
    Ld, Rd, d_max, _ = _stack_pairs(pairs, median_prefilter)
    if on_forest is not None and len(pairs) != 1:
        raise ConfigError("on_forest is supported for single-pair calls")

    def hook(o):
        if on_forest is None:
            return
        if o.extra.get("tree_masks") is None:  # top level: full range
            nw = (o.d_max + 1 + 31) // 32
            words = np.full((o.forest.n_trees, nw), 0xFFFFFFFF, np.uint32)
            rem = (o.d_max + 1) % 32
            if rem:
                words[:, -1] = (1 << rem) - 1
        else:
            words = o.extra["tree_masks"]
        on_forest(o.level, disparity_forest_from_device(o.forest, words, o.d_max))

    # the prior side stream and the level stream keep overlapping; stage times
    # are device events resolved after the run (aggregation.py:401-416 keys)
    outs = E.run_hdp_batch(Ld, Rd, d_max, model, params.levels, params.block_size, params.gamma,
                           params.delta0, params.beta, cost_params.consts(), tree_kind,
                           params.seed, keep=on_forest is not None, timing=True, on_level=hook)
    b = len(pairs)
    host = _to_host(*[t for o in outs for t in (o.disparity, o.min_cost)])
    disps, costs = host[0::2], host[1::2]
    total = time.perf_counter() - t_start
    stage = {"pyramid": 0.0, "predict": 0.0, "forest": 0.0, "cost": 0.0, "aggregate": 0.0}
    for o in outs:
        for k in stage:
            stage[k] += o.timings.get(k, 0.0)
    stage["total"] = total
    h0, w0 = outs[-1].h, outs[-1].w
    res = []
    for i in range(b):
        layers = [LayerResult(o.level, _dmap(disps[k][i]), costs[k][i], float(o.search_ratio[i]),
                              int(o.n_trees[i]), int(o.stored_entries[i]),
                              {"cost": o.timings.get("cost", 0.0),
                               "aggregate": o.timings.get("aggregate", 0.0)})
                  for k, o in enumerate(outs)]
        by_level = sorted(layers, key=lambda lr: lr.level)
        metrics = {"method": f"hdp-{tree_kind}", "tree": tree_kind, "hdp": True,
                   "median_prefilter": median_prefilter, "seed": params.seed,
                   "delta0": params.delta0, "beta": params.beta, "levels": params.levels,
                   "block_size": params.block_size,
                   "search_ratios": [lr.search_ratio for lr in by_level],
                   "stored_entries": by_level[0].stored_entries,
                   "dense_entries": h0 * w0 * (d_max + 1), "seconds": dict(stage)}
        res.append(PipelineResult(layers[-1].disparity, layers, metrics))
    return res


def run_hdp_pipeline(pair: StereoPair, model: GmmModel, params: AggregationParams | None = None,
                     cost_params: CostParams | None = None, tree_kind: str = "mst",
                     median_prefilter: bool = False, on_forest=None) -> PipelineResult:
    """aggregation.py:367-488."""
    return run_hdp_pipeline_batch([pair], model, params, cost_params, tree_kind,
                                  median_prefilter, on_forest)[0]
