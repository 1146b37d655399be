"""Error types of the drop-in API.

Same classes, meaning and exit codes as the reference (treestereo/errors.py:
8-29): ConfigError -> 2 (bad parameters), DataError -> 3 (bad or inconsistent
data), InternalError -> 4 (violated invariant).  The C-ABI returns the same
codes (include/hdp_stereo.h) and ``_lib.check`` maps them back onto these.
"""


class TreeStereoError(Exception):
    exit_code = 1


class ConfigError(TreeStereoError):
    exit_code = 2


class DataError(TreeStereoError):
    exit_code = 3


class InternalError(TreeStereoError):
    exit_code = 4
