"""The C-ABI library loads on a CPU-only host and exports exactly what
include/hdp_stereo.h declares; status codes map onto the reference errors."""

from __future__ import annotations

import os
import re
import subprocess

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "hdp_stereo.h")
LIB = os.path.join(REPO, "paper_1509_08197_b200", "libhdpstereo.so")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hdp_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-j8", "-C",
                        os.path.join(REPO, "paper_1509_08197_b200", "csrc")], check=True)
    from paper_1509_08197_b200 import _lib

    return _lib.load()


def test_header_declares_the_entry_points():
    names = declared_functions()
    for must in ("hdp_mst", "hdp_hdpf", "hdp_forest_create", "hdp_aggregate_wta",
                 "hdp_prior_counts", "hdp_cost_volume", "hdp_block_mean", "hdp_prepare"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (hdp_[a-z0-9_]+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, f"declared but not exported: {missing}"
    extra = sorted(exported - set(declared_functions()))
    assert not extra, f"exported but not declared: {extra}"


def test_binding_covers_every_symbol(lib):
    from paper_1509_08197_b200 import _lib

    assert set(_lib.SIGNATURES) == set(declared_functions())


def test_abi_version_and_error_mapping(lib):
    from paper_1509_08197_b200 import _lib
    from paper_1509_08197_b200.errors import ConfigError, DataError, InternalError

    assert lib.hdp_abi_version() == _lib.ABI_VERSION
    _lib.check(0)
    for code, exc in ((2, ConfigError), (3, DataError), (4, InternalError), (5, InternalError)):
        with pytest.raises(exc):
            _lib.check(code)


def test_config_errors_without_a_gpu(lib):
    """Argument validation happens before any device work."""
    from paper_1509_08197_b200 import _lib
    from paper_1509_08197_b200.errors import ConfigError

    with pytest.raises(ConfigError):
        _lib.call("hdp_block_mean", None, None, 1, 4, 4, 3, 1, None)  # block_size < 2
    with pytest.raises(ConfigError):
        _lib.call("hdp_hdpf", 1, 4, 4, None, None, None, None, None, 1, 1, 1.5, None, -1.0, None, None,
                  None, None, None)  # beta > 1
    with pytest.raises(ConfigError):
        _lib.call("hdp_segment_tree", 1, 4, 4, None, None, None, None, -1.0, None, None, None,
                  None)  # segment-tree k < 0
    with pytest.raises(ConfigError):
        _lib.call("hdp_error_counts", None, None, None, None, None, 1, 4, None, 0, None, None)  # no threshold
    assert lib.hdp_launch_count() == 0


def test_kernels_target_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_product_path_never_imports_the_oracle():
    pkg = os.path.join(REPO, "paper_1509_08197_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(root, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), f
