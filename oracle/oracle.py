"""ctypes front-end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Loaded only by ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg, always as the checker or the CPU
baseline -- never by the product package ``paper_2309_09778_b200``.

The oracle restates the reference path (``transform.py`` + the SPEC-only
predictor/quantizer/entropy/pipeline modules) in C: ``permez_oracle.c``.
Host-side scalars that the reference evaluates in Python/numpy
(``b_a = float(np.log2(1.0 + b_r))``, transform.py:118; ``(1.0 + b_r) ** 2``,
transform.py:160-162) are evaluated here exactly as the reference writes them
and handed to the C code, so both sides start from the same bits.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libpermez_oracle.so")
_lib = None

EPS0_F32 = float(np.finfo(np.float32).tiny)  # transform.py:37-39 float_floor(float32)


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


class OrcCfg(ctypes.Structure):
    _fields_ = [
        ("b_r", ctypes.c_double),
        ("b_a", ctypes.c_double),
        ("onepbr2", ctypes.c_double),
        ("eps0", ctypes.c_double),
        ("repair_t", ctypes.c_double),
        ("coverage_target", ctypes.c_double),
        ("slope", ctypes.c_double),
        ("w1", ctypes.c_double * 8),
        ("w2", ctypes.c_double * 2),
        ("block_rows", ctypes.c_int32),
        ("block_cols", ctypes.c_int32),
        ("partition_rows", ctypes.c_int32),
        ("S", ctypes.c_int32),
        ("H", ctypes.c_int32),
        ("m", ctypes.c_int32),
        ("pad", ctypes.c_int32),
    ]


class OrcParams(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in (
        "factor_pos", "factor_neg", "eps0", "b_r", "b_a", "boundary", "zero_code", "zero_threshold", "lg_pos",
        "lg_neg")]


class OrcResult(ctypes.Structure):
    _fields_ = [
        ("nblocks", ctypes.c_int64),
        ("ntrivial", ctypes.c_int64),
        ("nbal", ctypes.c_int64),
        ("nrepair", ctypes.c_int64),
        ("ncodes", ctypes.c_int64),
        ("m", ctypes.c_int32),
        ("pad", ctypes.c_int32),
        ("header_bytes", ctypes.c_uint64),
        ("total_bytes", ctypes.c_uint64),
        ("mreq", ctypes.c_uint64 * 18),
    ]


class OrcHeader(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
        ("block_rows", ctypes.c_int32), ("block_cols", ctypes.c_int32), ("partition_rows", ctypes.c_int32),
        ("m", ctypes.c_int32), ("S", ctypes.c_int32), ("H", ctypes.c_int32), ("version", ctypes.c_int32),
        ("elem", ctypes.c_int32),
        ("b_r", ctypes.c_double), ("coverage_target", ctypes.c_double), ("slope", ctypes.c_double),
        ("w1", ctypes.c_double * 8), ("w2", ctypes.c_double * 2),
        ("nblocks", ctypes.c_int64), ("header_bytes", ctypes.c_int64),
    ]


_NP_LOG2_FN = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.c_double)
# np.log2 of the per-block doubles that are not float32 values (transform.py:120,
# :123): the reference's own arithmetic, installed into the C oracle
_np_log2_hook = _NP_LOG2_FN(lambda x: float(np.log2(np.float64(x))))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.isdir("/root/reference") or os.environ.get("PMZ_ORACLE_MAKE"):
            build()  # incremental (make); the GPU box only uses the prebuilt library
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_set_np_log2.argtypes = [_NP_LOG2_FN]
        L.orc_set_np_log2(_np_log2_hook)
        P = ctypes.c_void_p
        L.orc_log2.restype = ctypes.c_double
        L.orc_log2.argtypes = [ctypes.c_double]
        L.orc_exp2.restype = ctypes.c_double
        L.orc_exp2.argtypes = [ctypes.c_double]
        L.orc_derive_params.argtypes = [ctypes.c_double] * 5 + [ctypes.POINTER(OrcParams)]
        L.orc_forward_map.argtypes = [P, ctypes.c_int64, ctypes.POINTER(OrcParams), P]
        L.orc_inverse_map.argtypes = [P, ctypes.c_int64, ctypes.POINTER(OrcParams), P]
        L.orc_predict.restype = ctypes.c_double
        L.orc_predict.argtypes = [ctypes.POINTER(OrcCfg), P]
        L.orc_quantize.restype = ctypes.c_int32
        L.orc_quantize.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int32]
        L.orc_dequantize.restype = ctypes.c_double
        L.orc_dequantize.argtypes = [ctypes.c_int32, ctypes.c_double, ctypes.c_int32]
        L.orc_build_codebook.restype = ctypes.c_int
        L.orc_build_codebook.argtypes = [P, ctypes.c_int32, P]
        L.orc_canonical_codes.restype = ctypes.c_int
        L.orc_canonical_codes.argtypes = [P, ctypes.c_int32, P]
        L.orc_num_blocks.restype = ctypes.c_int64
        L.orc_num_blocks.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32]
        L.orc_compress.restype = ctypes.c_int64
        L.orc_compress.argtypes = [P, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(OrcCfg), P, ctypes.c_int64, P,
                                   ctypes.c_int64, ctypes.POINTER(OrcResult), P, ctypes.c_int32]
        L.orc_read_header.restype = ctypes.c_int
        L.orc_read_header.argtypes = [P, ctypes.c_int64, ctypes.POINTER(OrcHeader)]
        L.orc_decompress.restype = ctypes.c_int
        L.orc_decompress.argtypes = [P, ctypes.c_int64, ctypes.c_double, P, ctypes.c_int64,
                                     ctypes.POINTER(ctypes.c_int64)]
        L.orc_slow_counts.argtypes = [P]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------
# host-side scalars, evaluated exactly as the reference writes them
# --------------------------------------------------------------------------

def host_b_a(b_r: float) -> float:
    return float(np.log2(1.0 + b_r))  # transform.py:118


def host_onepbr2(b_r: float) -> float:
    return (1.0 + b_r) ** 2  # transform.py:160-162


def init_weights(S: int):
    """init_model: hidden columns = Lorenzo coefficients, bias 0, w2 = (0.5, 0.5)."""
    if S == 3:
        w1 = [[1.0, 1.0], [1.0, 1.0], [-1.0, -1.0], [0.0, 0.0]]
    else:
        w1 = [[1.0, 1.0], [0.0, 0.0]]
    return np.array(w1, dtype=np.float64), np.array([0.5, 0.5], dtype=np.float64)


@dataclass
class OracleConfig:
    b_r: float = 1e-2
    block_rows: int = 256
    block_cols: int = 256
    partition_rows: int = 32
    repair_factor: float = 1.5
    coverage_target: float = 0.99
    sample_rate: float = 0.10
    seed: int = 0
    m: int = 0
    S: int = 3
    w1: np.ndarray | None = None
    w2: np.ndarray | None = None
    slope: float = 0.01

    def to_c(self) -> OrcCfg:
        c = OrcCfg()
        c.b_r = self.b_r
        c.b_a = host_b_a(self.b_r)
        c.onepbr2 = host_onepbr2(self.b_r)
        c.eps0 = EPS0_F32
        c.repair_t = self.repair_factor * self.b_r
        c.coverage_target = self.coverage_target
        c.slope = self.slope
        w1, w2 = (self.w1, self.w2) if self.w1 is not None else init_weights(self.S)
        flat = np.asarray(w1, dtype=np.float64).reshape(-1)
        for i, v in enumerate(flat):
            c.w1[i] = float(v)
        for i, v in enumerate(np.asarray(w2, dtype=np.float64).reshape(-1)):
            c.w2[i] = float(v)
        c.block_rows, c.block_cols, c.partition_rows = self.block_rows, self.block_cols, self.partition_rows
        c.S, c.H, c.m = self.S, 2, self.m
        return c


def ceil_frac(rate: float, n: int) -> int:
    """ceil(rate * n) robust to binary representation of the rate (D16)."""
    return int(math.ceil(rate * n - 1e-9))


def split_blocks(nblocks: int, sample_rate: float, seed: int):
    """sample_training_blocks + split_train_validation (D16, D21)."""
    if nblocks == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    k = max(ceil_frac(sample_rate, nblocks), min(nblocks, 5))
    if sample_rate == 1.0:
        ids = np.arange(nblocks, dtype=np.int64)  # all blocks, original order
    else:
        ids = np.random.default_rng(seed).permutation(nblocks)[:k].astype(np.int64)
    ntr = ceil_frac(0.8, k)
    train, val = ids[:ntr], ids[ntr:]
    if val.size == 0:
        val = ids
    return train, val


def grid_view(data: np.ndarray):
    """1-D -> 1xN (S=1); 2-D as is; n-D -> (prod(shape[:-1]), shape[-1]) (D18)."""
    a = np.ascontiguousarray(data, dtype=np.float32)
    if a.ndim == 1:
        return a.reshape(1, -1), 1
    if a.ndim == 2:
        return a, 3
    return a.reshape(-1, a.shape[-1]), 3


def compress(data: np.ndarray, cfg: OracleConfig, nthreads: int = 0, return_codes: bool = False):
    L = lib()
    x, S = grid_view(data)
    cfg = OracleConfig(**{**cfg.__dict__, "S": S}) if cfg.S != S else cfg
    rows, cols = x.shape
    nb = L.orc_num_blocks(rows, cols, cfg.block_rows, cfg.block_cols)
    _, val = split_blocks(nb, cfg.sample_rate, cfg.seed)
    c = cfg.to_c()
    res = OrcResult()
    nthreads = nthreads or os.cpu_count() or 1
    codes = np.zeros((rows, cols), np.uint16) if return_codes else None
    need = L.orc_compress(_ptr(x), rows, cols, ctypes.byref(c), _ptr(val), val.size, None, 0, ctypes.byref(res),
                          None, nthreads)
    if need not in (-16,) and need < 0:
        raise RuntimeError(f"oracle compress failed: status {need}")
    out = np.zeros(int(res.total_bytes), np.uint8)
    n = L.orc_compress(_ptr(x), rows, cols, ctypes.byref(c), _ptr(val), val.size, _ptr(out), out.size,
                       ctypes.byref(res), _ptr(codes) if codes is not None else None, nthreads)
    if n < 0:
        raise RuntimeError(f"oracle compress failed: status {n}")
    info = {f: getattr(res, f) for f in ("nblocks", "ntrivial", "nbal", "nrepair", "ncodes", "m", "header_bytes",
                                         "total_bytes")}
    info["mreq"] = list(res.mreq)
    info["val_ids"] = val
    if return_codes:
        return out.tobytes(), info, codes
    return out.tobytes(), info


def read_header(buf: bytes) -> dict:
    h = OrcHeader()
    b = np.frombuffer(buf, np.uint8)
    st = lib().orc_read_header(_ptr(b), b.size, ctypes.byref(h))
    if st != 0:
        raise RuntimeError(f"oracle header parse failed: status {st}")
    return {f: getattr(h, f) for f, _ in OrcHeader._fields_ if f not in ("w1", "w2")}


def decompress(buf: bytes) -> np.ndarray:
    h = read_header(buf)
    out = np.zeros((h["rows"], h["cols"]), np.float32)
    b = np.frombuffer(buf, np.uint8)
    used = ctypes.c_int64(0)
    st = lib().orc_decompress(_ptr(b), b.size, host_b_a(h["b_r"]), _ptr(out), out.size, ctypes.byref(used))
    if st != 0:
        raise RuntimeError(f"oracle decompress failed: status {st}")
    return out


def params(factor_pos: float, factor_neg: float, b_r: float, eps0: float = EPS0_F32) -> dict:
    p = OrcParams()
    lib().orc_derive_params(factor_pos, factor_neg, b_r, host_b_a(b_r), eps0, ctypes.byref(p))
    return {f: getattr(p, f) for f, _ in OrcParams._fields_}


def log2(x: float) -> float:
    return lib().orc_log2(x)


def exp2(y: float) -> float:
    return lib().orc_exp2(y)


def build_codebook(freq: np.ndarray) -> np.ndarray:
    f = np.ascontiguousarray(freq, dtype=np.uint64)
    lens = np.zeros(f.size, np.uint8)
    st = lib().orc_build_codebook(_ptr(f), f.size, _ptr(lens))
    if st != 0:
        raise RuntimeError(f"build_codebook status {st}")
    return lens


def canonical_codes(lens: np.ndarray) -> np.ndarray:
    l = np.ascontiguousarray(lens, dtype=np.uint8)
    c = np.zeros(l.size, np.uint32)
    st = lib().orc_canonical_codes(_ptr(l), l.size, _ptr(c))
    if st != 0:
        raise RuntimeError(f"canonical_codes status {st}")
    return c


def slow_counts():
    a = np.zeros(3, np.int64)
    lib().orc_slow_counts(_ptr(a))
    return a.tolist()


def ibm_to_ieee(words: np.ndarray) -> np.ndarray:
    """Oracle of the IBM hex-float conversion (read_segy):
    (-1)^s * 0.fraction * 16^(exponent - 64), evaluated exactly in double and
    rounded once to float32."""
    w = np.asarray(words, dtype=np.uint32)
    frac = (w & 0xFFFFFF).astype(np.float64)
    e = ((w >> 24) & 0x7F).astype(np.int64)
    v = np.ldexp(frac, (4 * (e - 64) - 24).astype(np.int32))
    with np.errstate(over="ignore"):
        f = v.astype(np.float32)
    return np.where((w >> 31) == 1, -f, f).astype(np.float32)
