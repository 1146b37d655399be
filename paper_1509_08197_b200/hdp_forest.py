"""Disparity-aware spanning forests (drop-in for treestereo.hdp_forest).

build_hdpf runs rule 1 + order-exact Kruskal with rule 2 on the GPU: when no
edge's endpoint masks differ, intersect and pass rule 2 statically, every tree
keeps one pixel mask and the forest is the MSF of the equal-mask edges
(Boruvka); otherwise whole-window rounds by conflict groups (hdpf.cu k_grp;
tree_kind "st" adds the segment-tree criterion).  plain_disparity_forest
(beta = 0, full range) is exactly the MST and uses Boruvka."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib as L
from . import engine as E
from .errors import ConfigError, InternalError
from .hdp_model import DisparityIntervalTable
from .raster_io import DisparityMap
from .spanning_forest import (EdgeList, RootedForest, _device_edges, _device_keys,
                              _node_weights, rooted_from_device)


def mask_to_array(mask: int) -> np.ndarray:
    """hdp_forest.py:38-45."""
    out = []
    while mask:
        low = mask & -mask
        out.append(low.bit_length() - 1)
        mask ^= low
    return np.array(out, dtype=np.int64)


@dataclass(frozen=True)
class PixelIntervalMap:
    """hdp_forest.py:48-75."""

    height: int
    width: int
    d_max: int
    pixel_row: np.ndarray
    intervals: tuple[np.ndarray, ...]
    masks: tuple[int, ...]

    @property
    def n_pixels(self) -> int:
        return self.height * self.width

    def interval(self, pixel: int) -> np.ndarray:
        return self.intervals[self.pixel_row[pixel]]

    def mask(self, pixel: int) -> int:
        return self.masks[self.pixel_row[pixel]]

    def mean_size(self) -> float:
        sizes = np.array([iv.size for iv in self.intervals], dtype=np.float64)
        return float(sizes[self.pixel_row].mean())


def full_range_interval_map(height: int, width: int, d_max: int) -> PixelIntervalMap:
    """hdp_forest.py:78-88."""
    full = np.arange(d_max + 1, dtype=np.int64)
    return PixelIntervalMap(height, width, d_max, np.zeros(height * width, dtype=np.int64),
                            (full,), ((1 << (d_max + 1)) - 1,))


def assign_pixel_intervals(parent_disparity: DisparityMap, table: DisparityIntervalTable,
                           child_height: int, child_width: int, d_max: int,
                           block_size: int) -> PixelIntervalMap:
    """hdp_forest.py:91-123 (row gather on the GPU)."""
    torch = E._t()
    ph, pw = -(-child_height // block_size), -(-child_width // block_size)
    if (parent_disparity.height, parent_disparity.width) != (ph, pw):
        raise InternalError(
            f"parent map {parent_disparity.height}x{parent_disparity.width} does not "
            f"cover child {child_height}x{child_width} at block {block_size}")
    pd = torch.from_numpy(np.ascontiguousarray(parent_disparity.values, np.int32)[None]).to(L.device())
    rows = E.assign_rows(pd, child_height, child_width, block_size, table.n_rows)
    return PixelIntervalMap(child_height, child_width, d_max, rows.cpu().numpy().astype(np.int64),
                            table.intervals, tuple(table.masks()))


@dataclass(frozen=True)
class DisparityForest:
    """hdp_forest.py:126-148."""

    base: RootedForest
    intervals: tuple[np.ndarray, ...]
    masks: tuple[int, ...]
    d_max: int

    @property
    def n_trees(self) -> int:
        return self.base.n_trees

    def search_ratio(self) -> float:
        sizes = np.array([iv.size for iv in self.intervals], dtype=np.float64)
        return float(sizes[self.base.tree_id].mean()) / (self.d_max + 1)

    def total_search_entries(self) -> int:
        sizes = np.array([iv.size for iv in self.intervals], dtype=np.int64)
        return int((sizes * np.diff(self.base.tree_slices)).sum())


def _words32(masks_int, nw):
    """Python-int bitsets -> (rows, nw) uint32."""
    out = np.zeros((len(masks_int), nw), np.uint32)
    for i, m in enumerate(masks_int):
        for k in range(nw):
            out[i, k] = (m >> (32 * k)) & 0xFFFFFFFF
    return out


def _ints_from_words(words: np.ndarray) -> list[int]:
    out = []
    for row in words.astype(np.uint64):
        m = 0
        for k, x in enumerate(row.tolist()):
            m |= int(x) << (32 * k)
        out.append(m)
    return out


def disparity_forest_from_device(f: "E.DeviceForest", tree_masks_words: np.ndarray, d_max: int,
                                 weights=None) -> DisparityForest:
    base = rooted_from_device(f, weights)
    masks = _ints_from_words(tree_masks_words)
    intervals = tuple(mask_to_array(m) for m in masks)
    for t, iv in enumerate(intervals):
        if iv.size == 0:
            raise InternalError(f"tree {t} ended with an empty interval")
    return DisparityForest(base=base, intervals=intervals, masks=tuple(masks), d_max=d_max)


def build_hdpf(edges: EdgeList, pixel_intervals: PixelIntervalMap, tree_kind: str = "mst",
               seed: int = 0, beta: float = 0.6, st_k: float | None = None) -> DisparityForest:
    """hdp_forest.py:151-216 on the GPU.  tree_kind "st": the segment-tree
    variant (subtrees under the FH criterion + the rules, then linked with the
    rules alone; not in the reference, parity unpinned)."""
    from .spanning_forest import ST_K, TREE_KINDS

    torch = E._t()
    if not 0.0 <= beta <= 1.0:
        raise ConfigError(f"beta must be in [0, 1], got {beta}")
    if tree_kind not in TREE_KINDS:
        raise ConfigError(f"unknown tree kind {tree_kind!r} (want 'mst', 'rt' or 'st')")
    n = edges.n_nodes
    if pixel_intervals.n_pixels != n:
        raise InternalError(f"interval map covers {pixel_intervals.n_pixels} pixels, grid has {n}")
    dev = L.device()
    nw = max(1, (pixel_intervals.d_max + 1 + 31) // 32)
    words = _words32(pixel_intervals.masks, nw)
    row_masks = torch.from_numpy(words.view(np.int32)[None].copy()).to(dev)
    rows = torch.from_numpy(np.ascontiguousarray(pixel_intervals.pixel_row, np.int32)).to(dev)
    eu, ev, ew = _device_edges(edges.u, edges.v, edges.weight)
    key = _device_keys(edges, tree_kind, seed)
    stk = (ST_K if st_k is None else st_k) if tree_kind == "st" else -1.0
    in_tree, comp, tmasks, _ = E.hdpf(1, n, edges.n_edges, eu, ev, key, rows, row_masks, beta, ew=ew, st_k=stk)
    f = E.DeviceForest(n, eu, ev, ew, in_tree, comp, 0.1)
    roots = f.export()["root"].cpu().numpy()
    root_ids = np.flatnonzero(roots == np.arange(n))
    tm = tmasks.cpu().numpy().view(np.uint32)[root_ids]
    df = disparity_forest_from_device(f, tm, pixel_intervals.d_max)
    pw = _node_weights(df.base.parent, edges.u, edges.v, edges.weight)
    return DisparityForest(RootedForest(**{**df.base.__dict__, "parent_weight": pw}),
                           df.intervals, df.masks, df.d_max)


def plain_disparity_forest(edges: EdgeList, d_max: int, tree_kind: str = "mst",
                           seed: int = 0) -> DisparityForest:
    """hdp_forest.py:219-224 (beta = 0 + full range == the plain MST/RT)."""
    from .spanning_forest import build_forest

    base = build_forest(edges, tree_kind, seed)
    full = np.arange(d_max + 1, dtype=np.int64)
    mask = (1 << (d_max + 1)) - 1
    return DisparityForest(base, (full,) * base.n_trees, (mask,) * base.n_trees, d_max)


def recompute_tree_intervals(forest: DisparityForest,
                             pixel_intervals: PixelIntervalMap) -> tuple[int, ...]:
    """hdp_forest.py:227-237 (host check utility)."""
    out = []
    for t in range(forest.n_trees):
        m = 0
        for node in forest.base.tree_nodes(t).tolist():
            m |= pixel_intervals.mask(node)
        out.append(m)
    return tuple(out)
