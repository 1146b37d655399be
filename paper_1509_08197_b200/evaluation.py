"""Method dispatch into the hot path (drop-in for the caller the reference
uses, treestereo/evaluation.py:125-167).  Dataset scoring, benchmarking
tables and CSV/JSONL reporting are host-side tooling, out of scope
(SURVEY.md §2); error_rate is kept as the small metric the tests use."""

from __future__ import annotations

import numpy as np

from .aggregation import AggregationParams, PipelineResult, run_baseline_pipeline, run_hdp_pipeline
from .cost_volume import CostParams
from .errors import ConfigError, DataError
from .hdp_model import GmmModel
from .raster_io import DisparityMap, StereoPair

KNOWN_METHODS = ("mst", "rt", "hdp+mst", "hdp+rt", "m+mst", "m+rt", "m+hdp+mst", "m+hdp+rt")


def parse_method(name: str) -> tuple[bool, bool, str]:
    """evaluation.py:135-151: label -> (median_prefilter, hdp, tree_kind)."""
    parts = name.strip().lower().split("+")
    median = hdp = False
    if parts and parts[0] == "m":
        median = True
        parts = parts[1:]
    if parts and parts[0] == "hdp":
        hdp = True
        parts = parts[1:]
    if len(parts) != 1 or parts[0] not in ("mst", "rt"):
        raise ConfigError(f"unknown method {name!r}; expected a combination like "
                          f"{', '.join(KNOWN_METHODS)}")
    return median, hdp, parts[0]


def run_method(pair: StereoPair, method: str, params: AggregationParams,
               cost_params: CostParams | None = None,
               model: GmmModel | None = None) -> PipelineResult:
    """evaluation.py:154-167."""
    median, hdp, tree = parse_method(method)
    if hdp:
        if model is None:
            raise ConfigError(f"method {method!r} needs an offset model")
        return run_hdp_pipeline(pair, model, params, cost_params, tree, median)
    return run_baseline_pipeline(pair, params, cost_params, tree, median)


def error_rate(predicted: DisparityMap, ground_truth: DisparityMap,
               occlusion: np.ndarray | None = None, threshold: int = 1) -> float:
    """evaluation.py:27-54: percent of evaluated pixels with |pred - gt| >= threshold."""
    if predicted.values.shape != ground_truth.values.shape:
        raise DataError(f"prediction {predicted.values.shape} vs ground truth "
                        f"{ground_truth.values.shape}")
    if threshold < 1:
        raise ConfigError(f"threshold must be >= 1, got {threshold}")
    evaluated = predicted.valid & ground_truth.valid
    if occlusion is not None:
        if occlusion.shape != predicted.values.shape:
            raise DataError("occlusion mask shape mismatch")
        evaluated &= ~occlusion
    n = int(evaluated.sum())
    if n == 0:
        raise DataError("no pixels left to evaluate")
    diff = np.abs(predicted.values.astype(np.int64) - ground_truth.values.astype(np.int64))
    return 100.0 * float((diff[evaluated] >= threshold).sum()) / n
