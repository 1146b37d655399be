"""Spanning trees over the pixel grid (drop-in for treestereo.spanning_forest).

Edge lists, the MST (Boruvka on (weight, scan index) keys -- identical to the
reference's stable-sort Kruskal), the seeded random tree order and the rooted
forest (Euler tour + list ranking) all run in libhdpstereo.so.  The returned
RootedForest has the reference's parent / parent_weight / depth / tree_id /
tree_slices / level_bounds / child_start / child_list; its `order` groups
each tree's nodes by depth with siblings contiguous (sorted by (tree, depth,
parent, id)), which satisfies every invariant the reference's consumers use
but is not literally the BFS visiting order.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _lib as L
from . import engine as E
from .errors import ConfigError, InternalError
from .pyramid import PyramidLayer
from .raster_io import RasterImage

AcceptFn = Callable[[int, int, int, int], bool]


@dataclass(frozen=True)
class EdgeList:
    """spanning_forest.py:33-49."""

    u: np.ndarray
    v: np.ndarray
    weight: np.ndarray
    width: int
    height: int

    @property
    def n_edges(self) -> int:
        return self.u.shape[0]

    @property
    def n_nodes(self) -> int:
        return self.width * self.height


def edge_weight(layer: PyramidLayer, p: tuple[int, int], q: tuple[int, int]) -> float:
    """Scalar convenience accessor (spanning_forest.py:52-58)."""
    (pr, pc), (qr, qc) = p, q
    if abs(pr - qr) + abs(pc - qc) != 1:
        raise ConfigError(f"pixels {p} and {q} are not 4-adjacent")
    return float(np.abs(layer.intensities[pr, pc] - layer.intensities[qr, qc]).max())


def build_edge_list(layer: PyramidLayer) -> EdgeList:
    """spanning_forest.py:61-93 (grid edges on the GPU, scan order)."""
    torch = E._t()
    img = torch.from_numpy(np.ascontiguousarray(layer.intensities, np.float64)[None]).to(L.device())
    eu, ev, _, _, n_e = E.grid_edges(img)
    w64 = torch.empty(max(n_e, 1), dtype=torch.float64, device=img.device)
    if n_e:
        L.call("hdp_grid_edge_weights64", L.ptr(img), 1, layer.height, layer.width,
               layer.channels, L.ptr(w64), L.stream())
    expected = 2 * layer.width * layer.height - layer.width - layer.height
    if n_e != expected:
        raise InternalError(f"edge count {n_e} != 2WH-W-H = {expected}")
    return EdgeList(u=eu.cpu().numpy().astype(np.int64), v=ev.cpu().numpy().astype(np.int64),
                    weight=w64[:n_e].cpu().numpy(), width=layer.width, height=layer.height)


def _device_keys(edges: EdgeList, tree_kind: str, seed: int):
    """Unique 64-bit Kruskal keys: (f32 weight bits | scan index) when every
    weight is exact in f32 (always true for uint8 images and S=2 pyramid
    levels), otherwise (stable GPU rank of the float64 weights | index)."""
    torch = E._t()
    dev = L.device()
    n_e = edges.n_edges
    idx = np.arange(n_e, dtype=np.int64)
    if tree_kind == "rt":
        return E.rt_keys(n_e, 1, seed, dev)
    if tree_kind not in TREE_KINDS:
        raise ConfigError(f"unknown tree kind {tree_kind!r} (want 'mst', 'rt' or 'st')")
    w = np.asarray(edges.weight, np.float64)
    if np.any(w < 0) or np.any(~np.isfinite(w)):
        raise ConfigError("edge weights must be finite and non-negative")
    w32 = w.astype(np.float32)
    if np.array_equal(w32.astype(np.float64), w) and n_e < (1 << 32):
        key = (w32.view(np.uint32).astype(np.int64) << 32) | idx
        return torch.from_numpy(key).to(dev)
    order = mst_edge_order(edges)
    rank = np.empty(n_e, np.int64)
    rank[order] = idx
    return torch.from_numpy((rank << 32) | idx).to(dev)


def mst_edge_order(edges: EdgeList) -> np.ndarray:
    """spanning_forest.py:96-107: stable argsort by weight (GPU radix sort of
    the float64 bit patterns, which are monotone for non-negative weights)."""
    torch = E._t()
    w = np.ascontiguousarray(edges.weight, np.float64)
    if w.size == 0:
        return np.zeros(0, np.int64)
    keys = torch.from_numpy(w.view(np.int64).copy()).to(L.device())
    perm = torch.empty(w.size, dtype=torch.int32, device=keys.device)
    L.call("hdp_argsort_u64", L.ptr(keys), w.size, L.ptr(perm), L.stream())
    return perm.cpu().numpy().astype(np.int64)


def rt_edge_order(edges: EdgeList, seed: int) -> np.ndarray:
    """spanning_forest.py:110-112 (the seeded permutation defines RT)."""
    return np.random.default_rng(seed).permutation(edges.n_edges)


TREE_KINDS = ("mst", "rt", "st")

# Segment tree (tree_kind "st") merge parameter k (engine.ST_K).  The
# reference has no segment tree (edge_order rejects "st",
# spanning_forest.py:115-120); this is the extension it names.
ST_K = E.ST_K


def edge_order(edges: EdgeList, tree_kind: str, seed: int = 0) -> np.ndarray:
    """spanning_forest.py:115-120; "st" walks the MST order (weight, index)."""
    if tree_kind in ("mst", "st"):
        return mst_edge_order(edges)
    if tree_kind == "rt":
        return rt_edge_order(edges, seed)
    raise ConfigError(f"unknown tree kind {tree_kind!r} (want 'mst', 'rt' or 'st')")


class UnionFind:
    """Disjoint sets with path halving and union by size (spanning_forest.py:
    123-143); a host utility of the public API, not used on the GPU path."""

    def __init__(self, n: int):
        self.parent = list(range(n))
        self.size = [1] * n

    def find(self, x: int) -> int:
        parent = self.parent
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    def union(self, a: int, b: int) -> int:
        if self.size[a] < self.size[b]:
            a, b = b, a
        self.parent[b] = a
        self.size[a] += self.size[b]
        return a


@dataclass(frozen=True)
class RootedForest:
    """spanning_forest.py:146-188."""

    n_nodes: int
    parent: np.ndarray
    parent_weight: np.ndarray
    depth: np.ndarray
    tree_id: np.ndarray
    order: np.ndarray
    pos: np.ndarray
    tree_slices: np.ndarray
    level_bounds: tuple[np.ndarray, ...]
    child_start: np.ndarray
    child_list: np.ndarray

    @property
    def n_trees(self) -> int:
        return len(self.tree_slices) - 1

    @property
    def roots(self) -> np.ndarray:
        return self.order[self.tree_slices[:-1]]

    def children(self, node: int) -> np.ndarray:
        return self.child_list[self.child_start[node]:self.child_start[node + 1]]

    def tree_nodes(self, tree: int) -> np.ndarray:
        return self.order[self.tree_slices[tree]:self.tree_slices[tree + 1]]

    def similarities(self, gamma: float) -> np.ndarray:
        if gamma <= 0:
            raise ConfigError(f"gamma must be positive, got {gamma}")
        return np.exp(-self.parent_weight / (gamma * 255.0))


def _forest_order(parent: np.ndarray, depth: np.ndarray, tree_id: np.ndarray) -> np.ndarray:
    """(tree, depth, parent, id) order by GPU radix sorts (stable, LSD)."""
    torch = E._t()
    dev = L.device()
    n = parent.size

    def argsort_dev(keys_np, perm_in=None):
        keys = torch.from_numpy(np.ascontiguousarray(keys_np, np.int64)).to(dev)
        if perm_in is not None:
            keys = keys[perm_in]
        perm = torch.empty(n, dtype=torch.int32, device=dev)
        L.call("hdp_argsort_u64", L.ptr(keys), n, L.ptr(perm), L.stream())
        perm = perm.to(torch.int64)
        return perm if perm_in is None else perm_in[perm]

    p1 = argsort_dev(parent)                       # ties keep ascending id
    p2 = argsort_dev(depth, p1)                    # stable: (depth, parent, id)
    p3 = argsort_dev(tree_id, p2)                  # stable: (tree, depth, parent, id)
    return p3.cpu().numpy()


def rooted_from_device(f: "E.DeviceForest", weight_of_node: np.ndarray | None = None) -> RootedForest:
    """Package a DeviceForest as the reference's RootedForest (host arrays)."""
    o = {k: v.cpu().numpy() for k, v in f.export().items()}
    n = f.n
    parent = o["parent"].astype(np.int64)
    depth = o["depth"].astype(np.int64)
    tree_id = o["tree_id"].astype(np.int64)
    pw = (o["parent_weight"].astype(np.float64) if weight_of_node is None else weight_of_node)
    order = _forest_order(parent, depth, tree_id)
    pos = np.empty(n, np.int64)
    pos[order] = np.arange(n, dtype=np.int64)
    counts = np.bincount(tree_id, minlength=f.n_trees)
    slices = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
    level_bounds = []
    dseq = depth[order]
    for t in range(len(slices) - 1):
        bd = dseq[slices[t]:slices[t + 1]]
        top = int(bd[-1]) if bd.size else 0
        level_bounds.append(np.searchsorted(bd, np.arange(top + 2)).astype(np.int64))
    is_child = parent != np.arange(n)
    child_nodes = np.flatnonzero(is_child)
    grouped = child_nodes[np.argsort(parent[child_nodes], kind="stable")]
    cnt = np.bincount(parent[child_nodes], minlength=n)
    child_start = np.concatenate(([0], np.cumsum(cnt))).astype(np.int64)
    return RootedForest(n_nodes=n, parent=parent, parent_weight=pw, depth=depth, tree_id=tree_id,
                        order=order, pos=pos, tree_slices=slices,
                        level_bounds=tuple(level_bounds), child_start=child_start,
                        child_list=grouped.astype(np.int64))


def _node_weights(parent, u, v, w):
    """parent_weight in float64 from the original edge weights."""
    pw = np.zeros(parent.size, np.float64)
    u, v, w = np.asarray(u, np.int64), np.asarray(v, np.int64), np.asarray(w, np.float64)
    down_v = parent[v] == u
    pw[v[down_v]] = w[down_v]
    down_u = (parent[u] == v) & ~down_v
    pw[u[down_u]] = w[down_u]
    return pw


def _device_edges(u, v, w):
    torch = E._t()
    dev = L.device()
    return (torch.from_numpy(np.ascontiguousarray(u, np.int32)).to(dev),
            torch.from_numpy(np.ascontiguousarray(v, np.int32)).to(dev),
            torch.from_numpy(np.ascontiguousarray(w, np.float32)).to(dev))


def build_forest(edges: EdgeList, tree_kind: str = "mst", seed: int = 0,
                 accept: AcceptFn | None = None, st_k: float = ST_K) -> RootedForest:
    """spanning_forest.py:286-322 on the GPU.  The `accept` predicate is a
    Python callback per edge; it cannot run inside the device kernels, so a
    non-None accept raises ConfigError (use build_hdpf for interval-aware
    acceptance, tree_kind "st" for the segment tree).  tree_kind "st": the
    segment tree (not in the reference; parity unpinned)."""
    if tree_kind not in TREE_KINDS:
        raise ConfigError(f"unknown tree kind {tree_kind!r} (want 'mst', 'rt' or 'st')")
    if accept is not None:
        raise ConfigError("custom accept predicates are not supported on the GPU path")
    eu, ev, ew = _device_edges(edges.u, edges.v, edges.weight)
    key = _device_keys(edges, tree_kind, seed)
    if tree_kind == "st":
        torch = E._t()
        n = edges.n_nodes
        rows = torch.zeros(n, dtype=torch.int32, device=eu.device)
        full = torch.full((1, 1, 1), -1, dtype=torch.int32, device=eu.device)  # every pixel set full
        in_tree, comp, _, _ = E.hdpf(1, n, edges.n_edges, eu, ev, key, rows, full, 0.0, ew=ew, st_k=st_k)
    else:
        in_tree, comp, _ = E.mst(edges.n_nodes, eu, ev, key)
    f = E.DeviceForest(edges.n_nodes, eu, ev, ew, in_tree, comp, 0.1)
    rf = rooted_from_device(f)
    pw = _node_weights(rf.parent, edges.u, edges.v, edges.weight)
    return RootedForest(**{**rf.__dict__, "parent_weight": pw})


def forest_from_edges(n_nodes: int, u: np.ndarray, v: np.ndarray, weight: np.ndarray) -> RootedForest:
    """spanning_forest.py:325-334: root an explicit acyclic edge set."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    weight = np.asarray(weight, dtype=np.float64)
    if not (u.shape == v.shape == weight.shape):
        raise ConfigError("edge arrays must have matching shapes")
    eu, ev, ew = _device_edges(u, v, weight)
    f = E.DeviceForest(int(n_nodes), eu, ev, ew, None, None, 0.1)
    rf = rooted_from_device(f)
    pw = _node_weights(rf.parent, u, v, weight)
    return RootedForest(**{**rf.__dict__, "parent_weight": pw})


def forest_total_weight(forest: RootedForest) -> float:
    return float(forest.parent_weight.sum())


def apply_median_prefilter(image: RasterImage) -> RasterImage:
    """spanning_forest.py:342-347 on the GPU (3x3 reflect-border median)."""
    torch = E._t()
    src = torch.from_numpy(np.ascontiguousarray(image.data)).to(L.device())
    dst = torch.empty_like(src)
    h, w, c = image.data.shape
    L.call("hdp_median3x3", L.ptr(src), L.ptr(dst), 1, h, w, c, L.stream())
    return RasterImage(dst.cpu().numpy())
