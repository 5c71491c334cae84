"""ctypes bindings of the C-ABI in include/spdistal_b200.h.

The shared library is built in-tree (``make -C paper_2207_13901_b200``); there
is no CPU fallback: importing a compute entry point without the library, or
calling one without a CUDA device, raises.
"""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libspdistal_b200.so")
SYNTH_PATH = os.path.join(HERE, "libspd_synth.so")

SPD_OK, SPD_ERR_RUNTIME, SPD_ERR_VALIDATION = 0, 1, 2
SPD_DENSE, SPD_COMPRESSED = 0, 1

i64 = C.c_int64
i64p = C.POINTER(C.c_int64)
dblp = C.POINTER(C.c_double)
vp = C.c_void_p


class spd_range(C.Structure):
    _fields_ = [("lo", i64), ("hi", i64)]


class spd_color(C.Structure):
    _fields_ = [("color", spd_range), ("q", spd_range), ("par", spd_range), ("top", spd_range)]


class spd_stats(C.Structure):
    _fields_ = [
        ("workers", i64),
        ("combines", i64),
        ("imbalance", C.c_double),
        ("kernel_ms", C.c_double),
        ("launches", i64),
    ]


# Every symbol the header declares, with (restype, argtypes).
SIGNATURES = {
    "spd_last_error": (C.c_char_p, []),
    "spd_abi_version": (C.c_int, []),
    "spd_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "spd_context_create": (C.c_int, [C.c_int, vp, C.POINTER(vp)]),
    "spd_context_destroy": (C.c_int, [vp]),
    "spd_context_synchronize": (C.c_int, [vp]),
    "spd_nccl_unique_id": (C.c_int, [vp]),
    "spd_context_init_comm": (C.c_int, [vp, vp, C.c_int, C.c_int]),
    "spd_context_rank": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "spd_context_abort": (C.c_int, [vp]),
    "spd_allgather": (C.c_int, [vp, vp, i64]),
    "spd_tensor_upload": (
        C.c_int,
        [vp, C.c_int, i64p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(i64p),
         C.POINTER(i64p), dblp, C.POINTER(vp)],
    ),
    "spd_deppart_image": (C.c_int, [vp, vp, i64, i64, i64, vp, vp, vp, vp, i64, i64p, C.POINTER(C.c_int)]),
    "spd_deppart_preimage": (C.c_int, [vp, vp, i64, i64, i64, vp, vp, vp, vp, i64, i64p, C.POINTER(C.c_int)]),
    "spd_deppart_image_host": (C.c_int, [vp, vp, i64, i64, i64, vp, vp, vp, vp, i64, i64p, C.POINTER(C.c_int)]),
    "spd_deppart_preimage_host": (C.c_int, [vp, vp, i64, i64, i64, vp, vp, vp, vp, i64, i64p, C.POINTER(C.c_int)]),
    "spd_deppart_by_bounds_host": (C.c_int, [vp, C.c_int, i64p, i64, i64p, i64p, i64p, i64, i64p,
                                              C.POINTER(C.c_int)]),
    "spd_deppart_by_bounds": (C.c_int, [vp, C.c_int, i64p, i64, i64p, vp, vp, i64, i64p, C.POINTER(C.c_int)]),
    "spd_tensor_restage": (C.c_int, [vp, vp, C.POINTER(i64p), C.POINTER(i64p), dblp]),
    "spd_ledger_bytes": (C.c_int, [vp, vp, C.c_int, C.c_int, i64, i64p]),
    "spd_ledger_missing": (C.c_int, [vp, i64, C.POINTER(i64p), i64p, C.POINTER(i64p), i64p, i64p]),
    "spd_tensor_repartition": (C.c_int, [vp, vp, C.c_int, C.POINTER(vp), i64p]),
    "spd_tensor_upload_piece": (
        C.c_int,
        [vp, C.c_int, i64p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(i64p), C.POINTER(i64p), dblp,
         C.c_int, C.POINTER(vp)],
    ),
    "spd_tensor_upload_rowptr": (
        C.c_int,
        [vp, C.c_int, i64p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(i64p),
         C.POINTER(i64p), dblp, C.c_int, C.POINTER(vp)],
    ),
    "spd_tensor_wrap_device": (
        C.c_int,
        [vp, C.c_int, i64p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(vp),
         C.POINTER(vp), vp, C.POINTER(vp)],
    ),
    "spd_tensor_destroy": (C.c_int, [vp]),
    "spd_tensor_num_levels": (C.c_int, [vp, C.POINTER(C.c_int)]),
    "spd_tensor_level": (C.c_int, [vp, C.c_int, C.POINTER(C.c_int), i64p, i64p]),
    "spd_tensor_nvals": (C.c_int, [vp, i64p]),
    "spd_tensor_device_ptrs": (C.c_int, [vp, C.c_int, C.POINTER(vp), C.POINTER(vp)]),
    "spd_tensor_vals_ptr": (C.c_int, [vp, C.POINTER(vp)]),
    "spd_tensor_download_level": (C.c_int, [vp, C.c_int, i64p, i64p]),
    "spd_tensor_download_rowptr": (C.c_int, [vp, C.c_int, i64p]),
    "spd_tensor_download_vals": (C.c_int, [vp, dblp]),
    "spd_tensor_download_vals_range": (C.c_int, [vp, i64, i64, dblp]),
    "spd_partition_universe": (C.c_int, [vp, vp, i64, C.POINTER(spd_color)]),
    "spd_partition_nonzero": (C.c_int, [vp, vp, C.c_int, i64, C.POINTER(spd_color)]),
    "spd_partition_materialize": (C.c_int, [vp, vp, C.c_int, C.c_int, i64, i64p, i64, i64p]),
    "spd_partition_bucket": (C.c_int, [vp, vp, C.c_int, i64, i64p]),
    "spd_bucket_positions": (C.c_int, [vp, i64, i64p, i64, i64p]),
    "spd_bucket_grid_work": (C.c_int, [vp, i64p, i64, i64p]),
    "spd_spmv": (C.c_int, [vp, vp, vp, vp, i64, i64, C.POINTER(spd_stats)]),
    "spd_spmm": (C.c_int, [vp, vp, vp, i64, vp, i64, i64, C.POINTER(spd_stats)]),
    "spd_sddmm": (C.c_int, [vp, vp, vp, vp, i64, i64, i64, vp, i64, i64, C.POINTER(spd_stats)]),
    "spd_spttv": (C.c_int, [vp, vp, vp, vp, i64, i64, C.POINTER(spd_stats)]),
    "spd_spmttkrp": (C.c_int, [vp, vp, vp, vp, i64, vp, i64, i64, C.POINTER(spd_stats)]),
    "spd_spadd3": (C.c_int, [vp, vp, vp, vp, C.POINTER(vp), i64, i64, C.POINTER(spd_stats)]),
    "spd_tensor_global_span": (C.c_int, [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]),
    "spd_gather_rows": (C.c_int, [vp, vp, C.c_int, C.POINTER(vp)]),
    "spd_tensor_load": (C.c_int, [vp, C.c_char_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), i64p,
                                  C.POINTER(vp), i64p]),
    "spd_tensor_store": (C.c_int, [vp, C.c_char_p]),
    "spd_tensor_place": (C.c_int, [vp, C.c_int, vp, C.c_int, C.POINTER(vp), i64p]),
    "spd_tensor_piece_span": (C.c_int, [vp, i64p, i64p]),
    "spd_capture_begin": (C.c_int, [vp]),
    "spd_capture_end": (C.c_int, [vp, C.POINTER(vp)]),
    "spd_graph_launch": (C.c_int, [vp, vp]),
    "spd_graph_destroy": (C.c_int, [vp]),
    "spd_tensor_pack": (C.c_int, [vp, C.c_int, i64p, C.POINTER(C.c_int), C.POINTER(C.c_int), i64,
                                  C.POINTER(i64p), dblp, C.c_int, C.POINTER(vp)]),
    "spd_last_work": (C.c_int, [vp, i64p, i64]),
    "spd_context_set_colour_blocks": (C.c_int, [vp, i64, i64p]),
    "spd_context_colour_blocks": (C.c_int, [vp, i64, i64p]),
    "spd_split_colour_blocks": (C.c_int, [dblp, i64, C.c_int, i64p]),
    "spd_colour_costs": (C.c_int, [vp, vp, i64p, i64p, i64p]),
    "spd_last_owned": (C.c_int, [vp, i64, i64, i64p, i64p]),
    "spd_context_timing": (C.c_int, [vp, C.c_int]),
    "spd_context_read_timing": (C.c_int, [vp, dblp, i64, i64p]),
    "spd_context_launches": (C.c_int, [vp, i64p]),
}

SYNTH_SIGNATURES = {
    "syn_dense": (None, [i64, C.c_uint64, C.c_int, dblp]),
    "syn_uniform_csr": (i64, [i64, i64, i64, C.c_uint64, C.c_int, i64p, i64p, dblp]),
    "syn_rmat_csr": (
        i64,
        [C.c_int, i64, C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_int, C.c_int, i64,
         i64p, i64p, dblp],
    ),
    "syn_powerlaw_csf": (
        i64,
        [i64, i64, i64, i64, C.c_uint64, C.c_int, i64p, i64p, i64p, i64p, dblp, i64p],
    ),
    "syn_max_threads": (C.c_int, []),
    "syn_set_threads": (None, [C.c_int]),
}


class SpdError(RuntimeError):
    """Runtime-class failure (std::runtime_error / logic_error / ClosureViolation)."""


class SpdValidationError(ValueError):
    """ValidationError / ParseError class failure (exit code 2 in the reference CLI)."""


_lib = None
_synth = None


def _bind(lib, sigs):
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib():
    """The product library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C paper_2207_13901_b200` "
                "(there is no CPU fallback)")
        _lib = _bind(C.CDLL(LIB_PATH), SIGNATURES)
    return _lib


def synth():
    global _synth
    if _synth is None:
        if not os.path.exists(SYNTH_PATH):
            raise ImportError(f"{SYNTH_PATH} is missing: run `make -C paper_2207_13901_b200`")
        _synth = _bind(C.CDLL(SYNTH_PATH), SYNTH_SIGNATURES)
    return _synth


def check(status):
    if status == SPD_OK:
        return
    msg = lib().spd_last_error().decode(errors="replace")
    if status == SPD_ERR_VALIDATION:
        raise SpdValidationError(msg)
    raise SpdError(msg)
