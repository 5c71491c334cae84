"""Every non-default leaf variant kept behind a switch
passes the same parity checks as the default path.

The switches are read once per process, so each variant runs the random-
instance and hub-row parity tests of test_gpu_parity.py in a subprocess
with its environment variable set.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

VARIANTS = [
    {"SPD_HOT": "1"},  # per-access evict_last / evict_first C-row loads
    {"SPD_HOT": "2"},  # hot-row copy under a persisting window
    {"SPD_HOT": "3"},  # plain int32 crd
    {"SPD_SPMV_STAGE": "1"},  # staged-product SpMV / SpTTV
    {"SPD_SPMV_ROWS": "0"},  # window-scan SpMV instead of lane per row
    {"SPD_SPMV_ROWS": "1"},
    {"SPD_NZ": "0"},  # direct row-pointer walks
    {"SPD_DYN": "0"},  # static grid stride for the N=32 SpMM leaf
    {"SPD_SPMMV": "0"},  # lane-per-column SpMM / SpMTTKRP walks for N != 32
    {"SPD_ZCONC": "0"},  # zero-fill before the leaf
    {"SPD_XC": "2"},  # compacted-column SpMV on every matrix
    {"SPD_XC": "0"},  # never (the wide-x test then reads x directly)
]


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_switch_variant_parity(env):
    full = dict(os.environ, **env)
    r = subprocess.run(
        [sys.executable, "-m", "pytest", os.path.join(HERE, "test_gpu_parity.py"), "-m", "gpu", "-x", "-q",
         "-p", "no:cacheprovider", "-k", "restatement_random or long_hub or widths or long_empty or wide_x or restage or degenerate or golden"],
        env=full, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
