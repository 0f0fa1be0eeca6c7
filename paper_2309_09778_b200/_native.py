"""ctypes binding of the C ABI in include/permez_b200.h (libpermez_b200.so).

The shared library is built in-tree (``paper_2309_09778_b200/_lib``) by
``__graft_entry__.build()``.  There is no CPU fallback: if the library or a
CUDA device is missing, every entry point raises ``DeviceError``.
"""
from __future__ import annotations

import ctypes
import os

from .errors import DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
# PMZ_LIB_PATH: load a variant build instead (A/B experiments under tools/)
LIB_PATH = os.environ.get("PMZ_LIB_PATH") or os.path.join(_HERE, "_lib", "libpermez_b200.so")

c_double, c_int32, c_uint32, c_uint64, c_int64 = (ctypes.c_double, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint64,
                                                   ctypes.c_int64)
VP = ctypes.c_void_p


class Params(ctypes.Structure):
    _fields_ = [
        ("b_r", c_double), ("b_a", c_double), ("onepbr2", c_double), ("eps0", c_double), ("repair_t", c_double),
        ("coverage_target", c_double), ("slope", c_double), ("w1", c_double * 8), ("w2", c_double * 2),
        ("block_rows", c_int32), ("block_cols", c_int32), ("partition_rows", c_int32), ("S", c_int32),
        ("H", c_int32), ("m", c_int32), ("precision", c_int32), ("reserved", c_int32), ("d_code_dump", c_uint64),
    ]


class Geom(ctypes.Structure):
    _fields_ = [("rows", c_uint64), ("cols", c_uint64), ("block_row0", c_uint64), ("global_rows", c_uint64)]


class Result(ctypes.Structure):
    _fields_ = [
        ("header_bytes", c_uint64), ("record_bytes", c_uint64), ("nblocks", c_uint64), ("ntrivial", c_uint64),
        ("nbal", c_uint64), ("nrepair", c_uint64), ("ncodes", c_uint64), ("coverage", c_uint64 * 18),
        ("m", c_int32), ("max_code_len", c_int32), ("unresolved", c_uint32), ("launches", c_uint32),
    ]


class Header(ctypes.Structure):
    _fields_ = [
        ("rows", c_uint64), ("cols", c_uint64), ("block_rows", c_uint32), ("block_cols", c_uint32),
        ("partition_rows", c_uint32), ("version", c_uint32), ("elem", c_uint32), ("m", c_uint32), ("S", c_uint32),
        ("H", c_uint32), ("b_r", c_double), ("coverage_target", c_double), ("slope", c_double),
        ("w1", c_double * 8), ("w2", c_double * 2), ("nblocks", c_uint64), ("header_bytes", c_uint64),
        ("lens_offset", c_uint64),
    ]


class NpFix(ctypes.Structure):
    """pmz_np_fix: a block whose general-double log2 numpy must decide (D22)."""
    _fields_ = [("block", c_int64), ("arg", c_double * 2), ("lg", c_double * 2), ("mask", c_int32),
                ("pad", c_int32)]


_SIGS = {
    "pmz_abi_version": (c_int32, []),
    "pmz_code_dump_elems": (c_int32, [ctypes.POINTER(Params), ctypes.POINTER(Geom), ctypes.POINTER(c_uint64)]),
    "pmz_status_string": (ctypes.c_char_p, [c_int32]),
    "pmz_workspace_size": (c_int32, [ctypes.POINTER(Params), ctypes.POINTER(Geom), ctypes.POINTER(c_uint64)]),
    "pmz_max_container_size": (c_int32, [ctypes.POINTER(Params), ctypes.POINTER(Geom), ctypes.POINTER(c_uint64)]),
    "pmz_compress_analyze": (c_int32, [VP, ctypes.POINTER(Geom), ctypes.POINTER(Params), VP, c_int64, VP, c_uint64,
                                       VP]),
    "pmz_ws_coverage": (VP, [VP, ctypes.POINTER(Params), ctypes.POINTER(Geom)]),
    "pmz_compress_codes": (c_int32, [VP, ctypes.POINTER(Geom), ctypes.POINTER(Params), VP, c_int64, VP, c_uint64,
                                     VP]),
    "pmz_ws_histogram": (VP, [VP, ctypes.POINTER(Params), ctypes.POINTER(Geom)]),
    "pmz_compress_finish": (c_int32, [VP, ctypes.POINTER(Geom), ctypes.POINTER(Params), c_int32, VP, c_uint64, VP,
                                      VP, c_uint64, VP, ctypes.POINTER(Result)]),
    "pmz_compress_finish_async": (c_int32, [VP, ctypes.POINTER(Geom), ctypes.POINTER(Params), c_int32, VP, c_uint64,
                                            VP, VP, c_uint64, VP]),
    "pmz_compress_encode": (c_int32, [VP, ctypes.POINTER(Geom), ctypes.POINTER(Params), VP, c_uint64, VP]),
    "pmz_compress_write_async": (c_int32, [ctypes.POINTER(Geom), ctypes.POINTER(Params), c_int32, VP, c_uint64, VP,
                                           VP, c_uint64, VP]),
    "pmz_compress_result": (c_int32, [ctypes.POINTER(Geom), ctypes.POINTER(Params), c_int32, VP, c_uint64, VP,
                                      ctypes.POINTER(Result)]),
    "pmz_compress_enqueue": (c_int32, [VP, ctypes.POINTER(Geom), ctypes.POINTER(Params), VP, c_int64, c_int32, VP,
                                       c_uint64, VP, VP, c_uint64, VP]),
    "pmz_compress": (c_int32, [VP, ctypes.POINTER(Geom), ctypes.POINTER(Params), VP, c_int64, VP, c_uint64, VP, VP,
                               c_uint64, VP, ctypes.POINTER(Result)]),
    "pmz_parse_header": (c_int32, [VP, c_uint64, ctypes.POINTER(Header)]),
    "pmz_index_blocks": (c_int32, [VP, c_uint64, ctypes.POINTER(Header), VP]),
    "pmz_index_blocks_range": (c_int32, [VP, c_uint64, ctypes.POINTER(Header), c_uint64, c_uint64, c_uint64, VP]),
    "pmz_decompress_workspace_size": (c_int32, [ctypes.POINTER(Header), ctypes.POINTER(c_uint64)]),
    "pmz_decompress": (c_int32, [VP, c_uint64, ctypes.POINTER(Header), c_double, VP, VP, VP, c_uint64, VP]),
    "pmz_decompress_enqueue": (c_int32, [VP, c_uint64, ctypes.POINTER(Header), c_double, VP, VP, VP, c_uint64, VP]),
    "pmz_decompress_result": (c_int32, [ctypes.POINTER(Header), VP, c_uint64, VP]),
    "pmz_train_gradient": (c_int32, [VP, ctypes.POINTER(Geom), ctypes.POINTER(Params), VP, c_int64, VP, VP, c_uint64,
                                     VP]),
    "pmz_train_gradient_batch": (c_int32, [VP, VP, c_uint64, ctypes.POINTER(Params), VP, VP, c_uint64, VP]),
    "pmz_segy_samples": (c_int32, [VP, c_uint64, c_uint32, c_int32, VP, VP]),
    "pmz_transform_params": (c_int32, [VP, ctypes.POINTER(Geom), ctypes.POINTER(Params), VP, VP, VP, c_uint64, VP]),
    "pmz_forward_map": (c_int32, [VP, c_uint64, VP, VP, VP]),
    "pmz_inverse_map": (c_int32, [VP, c_uint64, VP, VP, VP, VP]),
    "pmz_log2_f32_batch": (c_int32, [VP, c_uint64, VP, VP, c_int32, VP]),
    "pmz_block_stats": (c_int32, [VP, c_uint64, VP, VP, VP]),
    "pmz_derive_params": (c_int32, [VP, c_double, VP, VP, VP]),
    "pmz_zero_sub_floor": (c_int32, [VP, c_uint64, c_double, VP, VP]),
    "pmz_compress_stats": (c_int32, [VP, ctypes.POINTER(Geom), ctypes.POINTER(Params), VP, c_uint64, VP]),
    "pmz_compress_transform": (c_int32, [VP, ctypes.POINTER(Geom), ctypes.POINTER(Params), VP, c_int64, VP, c_uint64,
                                         VP]),
    "pmz_compress_np_fixups": (c_int64, [ctypes.POINTER(Geom), ctypes.POINTER(Params), VP, c_uint64, VP, VP, c_int64]),
    "pmz_compress_np_apply": (c_int32, [ctypes.POINTER(Geom), ctypes.POINTER(Params), VP, c_uint64, VP, VP, c_int64]),
    "pmz_decompress_prepare": (c_int32, [VP, c_uint64, ctypes.POINTER(Header), c_double, VP, VP, c_uint64, VP]),
    "pmz_decompress_status": (c_int32, [ctypes.POINTER(Header), VP, c_uint64, VP, ctypes.POINTER(Result)]),
    "pmz_decompress_run": (c_int32, [VP, c_uint64, ctypes.POINTER(Header), c_double, VP, VP, VP, c_uint64, VP]),
    "pmz_decompress_np_fixups": (c_int64, [ctypes.POINTER(Header), VP, c_uint64, VP, VP, c_int64]),
    "pmz_decompress_np_apply": (c_int32, [ctypes.POINTER(Header), c_double, VP, c_uint64, VP, VP, c_int64]),
    "pmz_pack_blocks_host": (c_int32, [VP, c_int64, c_int32, c_int32, VP, VP, c_int64, VP, c_int32]),
}

EXPORTS = tuple(_SIGS)
_lib = None


def resolve_np_log2(read, apply, cap: int = 4096) -> int:
    """Host half of the numpy-exact per-block logarithms (DESIGN D22): ``read``
    = pmz_*_np_fixups bound to a workspace (synchronises the stream),
    ``apply`` = pmz_*_np_apply.  Fills lg[i] = np.log2(arg[i]) -- the
    reference's own arithmetic (transform.py:120, :123) -- and hands the
    entries back.  Returns the number of listed blocks."""
    import numpy as np
    buf = (NpFix * cap)()
    n = int(read(buf, cap))
    if n < 0:
        return n
    if n > cap:
        buf = (NpFix * n)()
        n = int(read(buf, n))
        if n < 0:
            return n
    if n == 0:
        return 0
    a = np.frombuffer(buf, dtype=np.dtype([("block", "<i8"), ("arg", "<f8", 2), ("lg", "<f8", 2), ("mask", "<i4"),
                                           ("pad", "<i4")]), count=n)
    a["lg"] = np.log2(a["arg"])  # both args: the unflagged one is ignored by the device
    s = int(apply(buf, n))
    return s if s < 0 else n


def load():
    """Load the native library (raises DeviceError when it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"native library missing: {LIB_PATH} (run __graft_entry__.build())")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.pmz_abi_version() != 2:
            raise DeviceError("ABI version mismatch")
        _lib = lib
    return _lib
