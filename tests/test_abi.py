"""The C-ABI boundary (CPU): the in-tree library loads, exports exactly what
include/spdistal_b200.h declares, maps errors onto the reference's classes,
and fails loudly without a GPU (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

from paper_2207_13901_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spdistal_b200.h")
PKG = os.path.join(ROOT, "paper_2207_13901_b200")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spd_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ["spd_tensor_upload", "spd_partition_universe", "spd_partition_nonzero",
                 "spd_spmv", "spd_spmm", "spd_sddmm", "spd_spttv", "spd_spmttkrp", "spd_spadd3",
                 "spd_context_init_comm", "spd_last_error"]:
        assert must in syms


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(declared_symbols()) == set(N.SIGNATURES), "bindings out of sync with the header"


def test_abi_version():
    assert N.lib().spd_abi_version() == 100


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = C.c_void_p()
    st = N.lib().spd_context_create(0, None, C.byref(h))
    assert st == N.SPD_ERR_RUNTIME
    assert b"no CUDA device" in N.lib().spd_last_error()
    with pytest.raises(N.SpdError):
        N.check(st)


def test_null_arguments_are_validation_errors():
    assert N.lib().spd_context_synchronize(None) == N.SPD_ERR_VALIDATION
    assert N.lib().spd_tensor_destroy(None) == N.SPD_OK


def test_product_never_touches_the_oracle():
    """Only tests/, smoke() and bench's baseline legs may use oracle/."""
    for dirpath, _, files in os.walk(PKG):
        if "build" in dirpath:
            continue
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".c", ".h")):
                src = open(os.path.join(dirpath, f), errors="replace").read()
                assert "oracle_bind" not in src and "liboracle" not in src and "libdspar_ref" not in src, f


def test_synth_library_loads():
    s = N.synth()
    assert s.syn_max_threads() >= 1


def test_gpu_dependent_partitioning_fails_loudly_without_a_gpu():
    """The reference's planner linked with the GPU deppart has no CPU
    fallback: without a device every partitioning call raises."""
    import subprocess

    import torch

    exe = os.path.join(ROOT, "oracle", "_ref", "dspar_ref_tests_gpudeppart")
    if torch.cuda.is_available() or not os.path.exists(exe):
        pytest.skip("needs the GPU-deppart suite on a machine without a GPU")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert "deppart on gpu: no CUDA device available" in r.stderr


def test_production_leaves_do_not_spill():
    """The SpMV / SpTTV leaf and the C2 SpMM leaf keep their working set in
    registers at their launch bounds (ptxas log of the in-tree build; a
    spill on these kernels costs a local-memory round trip per chunk)."""
    log = os.path.join(PKG, "build", "leaf_rows.ptxas.log")
    if not os.path.exists(log):
        pytest.skip("library not built from source here")
    cur, spills = None, {}
    for line in open(log):
        m = re.search(r"Compiling entry function '([^']*)'", line)
        if m:
            cur = m.group(1)
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            spills[cur] = int(m.group(1)) + int(m.group(2))
    prod = {k: v for k, v in spills.items() if "k_spmv_win" in k or "k_spmm32_nz" in k}
    assert len(prod) >= 5, sorted(spills)
    assert all(v == 0 for v in prod.values()), prod
