"""Disparity prediction across pyramid levels (drop-in for treestereo.hdp_model).

Hot-path pieces: the sampled prior (estimate_prior, float64 bit-exact GPU
kernel) and the per-level interval table.  The table (<= 121 x 241 entries)
is assembled on the host with the reference's numpy formulas: it is control
data for the GPU forest build, and the reference's own BLAS/exp calls are the
only bit-identical route.  GMM training (coarsen_ground_truth,
train_mixture, train_gmm) is offline tooling, out of scope.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import engine as E
from .cost_volume import CostParams
from .errors import ConfigError, DataError, InternalError
from .pyramid import PyramidLayer

logger = logging.getLogger(__name__)

SIGMA_FLOOR = 0.25


@dataclass(frozen=True)
class Mixture1D:
    """1-D Gaussian mixture (hdp_model.py:47-72)."""

    weights: np.ndarray
    means: np.ndarray
    sigmas: np.ndarray
    loglik_history: tuple[float, ...] = field(default=(), compare=False)

    def __post_init__(self) -> None:
        k = self.weights.shape[0]
        if self.means.shape != (k,) or self.sigmas.shape != (k,):
            raise ConfigError("mixture parameter arrays disagree in length")
        if np.any(self.sigmas <= 0):
            raise ConfigError("mixture sigmas must be positive")

    @property
    def n_components(self) -> int:
        return self.weights.shape[0]

    def density(self, x: np.ndarray) -> np.ndarray:
        return E.mixture_density(self.weights, self.means, self.sigmas, x)


@dataclass(frozen=True)
class GmmModel:
    """One offset mixture per level transition (hdp_model.py:75-147)."""

    layers: tuple[Mixture1D, ...]

    @property
    def n_layers(self) -> int:
        return len(self.layers)

    def save(self, path: str | Path, comments: tuple[str, ...] = ()) -> None:
        lines = ["# offset mixture model: one 1-D GMM per pyramid level transition"]
        lines += [f"# {c}" for c in comments]
        lines += ["version 1", f"layers {self.n_layers}"]
        for idx, mix in enumerate(self.layers):
            lines += [f"layer {idx}", f"components {mix.n_components}",
                      "pi " + " ".join(repr(float(w)) for w in mix.weights),
                      "mu " + " ".join(repr(float(m)) for m in mix.means),
                      "sigma " + " ".join(repr(float(s)) for s in mix.sigmas)]
        Path(path).write_text("\n".join(lines) + "\n")

    @classmethod
    def load(cls, path: str | Path) -> "GmmModel":
        try:
            text = Path(path).read_text()
        except OSError as exc:
            raise DataError(f"cannot read model {path}: {exc}") from exc
        return cls.parse(text, source=str(path))

    @classmethod
    def parse(cls, text: str, source: str = "<string>") -> "GmmModel":
        rows = [ln.strip() for ln in text.splitlines()
                if ln.strip() and not ln.lstrip().startswith("#")]
        it = iter(rows)

        def fail(msg):
            return DataError(f"{source}: malformed model file: {msg}")

        def take(prefix):
            try:
                line = next(it)
            except StopIteration:
                raise fail(f"missing '{prefix}' line") from None
            if not line.startswith(prefix + " "):
                raise fail(f"expected '{prefix} ...', got {line!r}")
            return line[len(prefix) + 1:]

        if take("version") != "1":
            raise fail("unsupported version")
        try:
            n_layers = int(take("layers"))
        except ValueError as exc:
            raise fail("bad layer count") from exc
        layers = []
        for idx in range(n_layers):
            if take("layer") != str(idx):
                raise fail(f"expected layer {idx}")
            try:
                k = int(take("components"))
                pi = np.array([float(t) for t in take("pi").split()])
                mu = np.array([float(t) for t in take("mu").split()])
                sg = np.array([float(t) for t in take("sigma").split()])
            except ValueError as exc:
                raise fail(f"bad numeric field in layer {idx}") from exc
            if not (len(pi) == len(mu) == len(sg) == k):
                raise fail(f"layer {idx} parameter lengths disagree with K={k}")
            layers.append(Mixture1D(weights=pi, means=mu, sigmas=sg))
        return cls(layers=tuple(layers))


@dataclass(frozen=True)
class ConditionalMatrix:
    """hdp_model.py:302-317."""

    matrix: np.ndarray
    direction: str

    def __post_init__(self) -> None:
        if self.direction not in ("parent_given_child", "child_given_parent"):
            raise ConfigError(f"unknown direction {self.direction!r}")


def conditional_parent_given_child(mixture: Mixture1D, d_child: int, d_parent: int,
                                   block_size: int) -> ConditionalMatrix:
    """hdp_model.py:320-331."""
    return ConditionalMatrix(E.conditional_matrix(mixture, d_child, d_parent, block_size),
                             "parent_given_child")


def bayes_child_given_parent(conditional: ConditionalMatrix, prior: np.ndarray) -> ConditionalMatrix:
    """hdp_model.py:334-363."""
    if conditional.direction != "parent_given_child":
        raise ConfigError("bayes inversion expects a parent_given_child matrix")
    prior = np.asarray(prior, dtype=np.float64)
    n_parent, n_child = conditional.matrix.shape
    if prior.shape != (n_child,):
        raise ConfigError(f"prior length {prior.shape} does not match child range {n_child}")
    if np.any(prior < 0):
        raise ConfigError("prior has negative entries")
    bm, n_dead = E.bayes_batched(conditional.matrix, prior[None, :])
    if n_dead[0]:
        logger.warning("%d of %d posterior rows had zero mass; using uniform fallback",
                       int(n_dead[0]), n_parent)
    return ConditionalMatrix(bm[0], "child_given_parent")


@dataclass(frozen=True)
class DisparityIntervalTable:
    """hdp_model.py:473-495."""

    intervals: tuple[np.ndarray, ...]
    delta: float

    @property
    def n_rows(self) -> int:
        return len(self.intervals)

    def sizes(self) -> np.ndarray:
        return np.array([iv.size for iv in self.intervals], dtype=np.int64)

    def masks(self) -> list[int]:
        out = []
        for iv in self.intervals:
            m = 0
            for j in iv.tolist():
                m |= 1 << j
            out.append(m)
        return out


def predict_intervals(bayes: ConditionalMatrix, delta: float) -> DisparityIntervalTable:
    """hdp_model.py:498-525."""
    if bayes.direction != "child_given_parent":
        raise ConfigError("interval prediction expects a child_given_parent matrix")
    if delta <= 0:
        raise ConfigError(f"delta must be positive, got {delta}")
    chosen = E.predict_masks(np.asarray(bayes.matrix, np.float64)[None], delta)[0]
    return DisparityIntervalTable(
        intervals=tuple(np.flatnonzero(row).astype(np.int64) for row in chosen), delta=delta)


def estimate_prior(left_layer: PyramidLayer, right_layer: PyramidLayer,
                   params: CostParams | None = None, sample_stride: int = 5, window: int = 7,
                   max_offset: int = 1) -> np.ndarray:
    """hdp_model.py:425-470 -- the matching runs on the GPU (float64 exact)."""
    params = params or CostParams()
    if sample_stride < 1 or window < 1 or window % 2 == 0:
        raise ConfigError("sample_stride must be >= 1 and window odd and positive")
    torch = E._t()
    dev = E.L.device()
    il = torch.from_numpy(np.ascontiguousarray(left_layer.intensities, np.float64)[None]).to(dev)
    ir = torch.from_numpy(np.ascontiguousarray(right_layer.intensities, np.float64)[None]).to(dev)
    ul, _, gl, _ = E.prepare(il, True, False)
    ur, _, gr, _ = E.prepare(ir, True, False)
    lev = E.Level(0, left_layer.height, left_layer.width, left_layer.channels, left_layer.d_max,
                  il, ir, None, None, ul, gl, ur, gr)
    counts, kept = E.prior_counts(lev, sample_stride, window, max_offset,
                                  E.CostConsts(params.alpha, params.tau_color, params.tau_grad))
    counts, kept = counts.cpu().numpy(), kept.cpu().numpy()
    if kept[0] == 0:
        logger.warning("no cross-checked samples survived; prior falls back to uniform")
    return E.priors_from_counts(counts, kept)[0]
