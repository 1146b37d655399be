"""Boundary value types: the same dataclasses the reference's hot path
consumes and returns (treestereo/raster_io.py:27-97).  File I/O is out of
scope; only the validated containers live here."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, DataError


@dataclass(frozen=True)
class RasterImage:
    """8-bit raster (H, W, C), C in {1, 3} (raster_io.py:27-49)."""

    data: np.ndarray

    def __post_init__(self) -> None:
        if self.data.ndim != 3 or self.data.shape[2] not in (1, 3):
            raise DataError(f"expected (H, W, 1|3) array, got shape {self.data.shape}")
        if self.data.dtype != np.uint8:
            raise DataError(f"expected uint8 samples, got {self.data.dtype}")

    @property
    def height(self) -> int:
        return self.data.shape[0]

    @property
    def width(self) -> int:
        return self.data.shape[1]

    @property
    def channels(self) -> int:
        return self.data.shape[2]


@dataclass
class DisparityMap:
    """int32 disparities + validity mask (raster_io.py:52-78)."""

    values: np.ndarray
    valid: np.ndarray
    scale: int = 1

    def __post_init__(self) -> None:
        self.values = np.asarray(self.values, dtype=np.int32)
        self.valid = np.asarray(self.valid, dtype=bool)
        if self.values.shape != self.valid.shape or self.values.ndim != 2:
            raise DataError("disparity values and validity mask must share a 2-D shape")
        if self.scale < 1:
            raise ConfigError(f"disparity scale must be >= 1, got {self.scale}")

    @property
    def height(self) -> int:
        return self.values.shape[0]

    @property
    def width(self) -> int:
        return self.values.shape[1]


@dataclass(frozen=True)
class StereoPair:
    """Rectified pair with a disparity bound (raster_io.py:81-97)."""

    left: RasterImage
    right: RasterImage
    d_max: int
    name: str = "pair"

    def __post_init__(self) -> None:
        if self.left.data.shape != self.right.data.shape:
            raise DataError(
                f"stereo views disagree in shape: {self.left.data.shape} vs {self.right.data.shape}"
            )
        if self.d_max < 1:
            raise ConfigError(f"d_max must be >= 1, got {self.d_max}")
