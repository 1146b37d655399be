"""B200-native HDP tree stereo: the reference `treestereo` hot path (cost
volume, MST / disparity-forest build, two-pass tree aggregation + WTA, HDP
pyramid prediction) as hand-written sm_100a CUDA behind the reference's
Python API.  See DESIGN.md."""

__version__ = "0.1.0"

from .errors import ConfigError, DataError, InternalError, TreeStereoError

__all__ = ["__version__", "ConfigError", "DataError", "InternalError", "TreeStereoError"]
