"""Every leaf choice that an automatic rule or a tuning knob can flip
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
    {"SPD_CH_SPMV": "100"},  # SpMV chunks shorter than a window, not a multiple of 32
    {"SPD_CH_SPMV": "700"},  # several SpMV windows per chunk, a partial last one
    {"SPD_SPMV_MINB": "6"},  # the 6-CTA SpMV instantiation on the small matrices too
    {"SPD_ZCONC": "0"},  # zero-fill before the leaf instead of concurrent with it
    {"SPD_CH": "64"},  # tiny SpMM / SpMTTKRP chunks: every row crosses chunk records
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
