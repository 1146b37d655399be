"""Method dispatch into the hot path and on-device evaluation (drop-in for
treestereo/evaluation.py).

run_method / parse_method are the caller of the hot path the reference uses
(evaluation.py:135-167).  error_rate, occlusion_from_gt and evaluate_pair
(evaluation.py:27-124) run on the GPU (hdp_error_counts,
hdp_occlusion_from_gt): integer counts on the device, the percentage formed on
the host with the reference's expression, so the numbers are identical.
error_rates_device scores a whole batch of device-resident maps without a host
round trip of the maps.  Dataset walking, bench tables and CSV/JSONL writers
are host tooling, out of scope."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .aggregation import AggregationParams, PipelineResult, run_baseline_pipeline, run_hdp_pipeline
from .cost_volume import CostParams
from .errors import ConfigError, DataError
from .hdp_model import GmmModel
from .raster_io import DisparityMap, StereoPair

KNOWN_METHODS = ("mst", "rt", "hdp+mst", "hdp+rt", "m+mst", "m+rt", "m+hdp+mst", "m+hdp+rt")
# the segment tree the reference names but does not implement (ST, "st")
EXTENSION_METHODS = ("st", "hdp+st", "m+st", "m+hdp+st")


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
    if len(parts) != 1 or parts[0] not in ("mst", "rt", "st"):
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


def _dev_i32(a):
    torch = L.torch_mod()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(L.device())


def _dev_u8(a):
    if a is None:
        return None
    torch = L.torch_mod()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint8)).to(L.device())


def error_counts_device(pred, gt, thresholds=(1, 2), pred_valid=None, gt_valid=None, occlusion=None):
    """(B, len(thresholds) + 1) int64 host counts for device tensors pred / gt
    (B, ...) int32 and optional uint8 masks of the same shape: column 0 = the
    evaluated pixels, column 1 + i = evaluated pixels with |pred - gt| >=
    thresholds[i]."""
    torch = L.torch_mod()
    b = pred.shape[0] if pred.dim() > 2 else 1
    npix = pred.numel() // b
    thr = torch.tensor(list(thresholds), dtype=torch.int32, device=pred.device)
    counts = torch.empty((b, len(thresholds) + 1), dtype=torch.int64, device=pred.device)
    pred, gt = pred.contiguous(), gt.contiguous()  # referenced until the launch
    L.call("hdp_error_counts", L.ptr(pred), L.ptr(gt),
           L.ptr(pred_valid), L.ptr(gt_valid), L.ptr(occlusion), b, npix, L.ptr(thr), len(thresholds),
           L.ptr(counts), L.stream())
    return counts.cpu().numpy()


def error_rates_device(pred, gt, occlusion=None, thresholds=(1, 2)) -> np.ndarray:
    """Batched error_rate on device-resident maps: (B, len(thresholds)) percents."""
    c = error_counts_device(pred, gt, thresholds, occlusion=occlusion)
    if np.any(c[:, 0] == 0):
        raise DataError("no pixels left to evaluate")
    return np.array([[100.0 * float(c[b, 1 + i]) / int(c[b, 0]) for i in range(len(thresholds))]
                     for b in range(c.shape[0])])


def error_rate(predicted: DisparityMap, ground_truth: DisparityMap,
               occlusion: np.ndarray | None = None, threshold: int = 1) -> float:
    """evaluation.py:27-54: percent of evaluated pixels with |pred - gt| >= threshold."""
    if predicted.values.shape != ground_truth.values.shape:
        raise DataError(f"prediction {predicted.values.shape} vs ground truth "
                        f"{ground_truth.values.shape}")
    if threshold < 1:
        raise ConfigError(f"threshold must be >= 1, got {threshold}")
    if occlusion is not None and occlusion.shape != predicted.values.shape:
        raise DataError("occlusion mask shape mismatch")
    c = error_counts_device(_dev_i32(predicted.values)[None], _dev_i32(ground_truth.values)[None],
                            (threshold,), _dev_u8(predicted.valid)[None], _dev_u8(ground_truth.valid)[None],
                            None if occlusion is None else _dev_u8(occlusion)[None])
    n = int(c[0, 0])
    if n == 0:
        raise DataError("no pixels left to evaluate")
    return 100.0 * float(c[0, 1]) / n


def occlusion_from_gt(gt_left: DisparityMap, gt_right: DisparityMap) -> np.ndarray:
    """evaluation.py:57-76 on the GPU: left pixels whose match is off-image,
    invalid in the right map, or fails the +-1 cross-check.  (A match past the
    right border -- negative ground truth, which the reference does not guard
    -- counts as off-image here.)"""
    if gt_left.values.shape != gt_right.values.shape:
        raise DataError("left/right ground truth shapes differ")
    torch = L.torch_mod()
    h, w = gt_left.values.shape
    out = torch.empty((h, w), dtype=torch.uint8, device=L.device())
    # the device copies must stay referenced until the kernel has run
    gl, gr = _dev_i32(gt_left.values), _dev_i32(gt_right.values)
    vl, vr = _dev_u8(gt_left.valid), _dev_u8(gt_right.valid)
    L.call("hdp_occlusion_from_gt", L.ptr(gl), L.ptr(gr), L.ptr(vl), L.ptr(vr), 1, h, w, L.ptr(out), L.stream())
    return out.cpu().numpy().astype(bool)


@dataclass
class ErrorReport:
    """evaluation.py:79-101."""

    name: str
    method: str
    err_ge_1: float
    err_ge_2: float
    n_evaluated: int
    seconds: float | None = None
    extra: dict = field(default_factory=dict)

    def row(self) -> dict:
        out = {"name": self.name, "method": self.method, "err_ge_1": round(self.err_ge_1, 4),
               "err_ge_2": round(self.err_ge_2, 4), "n_evaluated": self.n_evaluated}
        if self.seconds is not None:
            out["seconds"] = round(self.seconds, 4)
        out.update(self.extra)
        return out


def evaluate_pair(name: str, method: str, predicted: DisparityMap, ground_truth: DisparityMap,
                  occlusion: np.ndarray | None = None, seconds: float | None = None) -> ErrorReport:
    """evaluation.py:104-124: err>=1, err>=2 and the evaluated count from one
    device pass."""
    if predicted.values.shape != ground_truth.values.shape:
        raise DataError(f"prediction {predicted.values.shape} vs ground truth "
                        f"{ground_truth.values.shape}")
    if occlusion is not None and occlusion.shape != predicted.values.shape:
        raise DataError("occlusion mask shape mismatch")
    c = error_counts_device(_dev_i32(predicted.values)[None], _dev_i32(ground_truth.values)[None], (1, 2),
                            _dev_u8(predicted.valid)[None], _dev_u8(ground_truth.valid)[None],
                            None if occlusion is None else _dev_u8(occlusion)[None])
    n = int(c[0, 0])
    if n == 0:
        raise DataError("no pixels left to evaluate")
    return ErrorReport(name=name, method=method, err_ge_1=100.0 * float(c[0, 1]) / n,
                       err_ge_2=100.0 * float(c[0, 2]) / n, n_evaluated=n, seconds=seconds)


def search_ratios_percent(result: PipelineResult) -> list[float]:
    """evaluation.py:127-129."""
    return [100.0 * r for r in result.metrics["search_ratios"]]
