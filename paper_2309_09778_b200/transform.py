"""Drop-in of the reference's domain-transform module (transform.py:1-210),
executed by this package's sm_100a kernels through the C ABI.

Same names (``__all__``, transform.py:24-34), the same frozen dataclasses
(``BlockStats`` :42-58, ``TransformParams`` :61-81), the same argument
meaning, return types (floats for scalar inputs, float64 arrays otherwise)
and the same exceptions (errors.py).  Where the reference computes with
numpy, this module runs:

* ``compute_block_stats``       -> ``pmz_block_stats`` (device reduction)
* ``derive_transform_params``   -> ``pmz_derive_params`` (device; the log2 of
  a general double that lies within 2^-56 of a rounding midpoint is handed to
  np.log2, DESIGN D22)
* ``forward_map``               -> ``pmz_forward_map``
* ``inverse_map``               -> ``pmz_inverse_map``
* ``zero_sub_floor_magnitudes`` -> ``pmz_zero_sub_floor``

Exactness against the reference: per-block parameters and the forward map
of every float32-valued input are bit-identical to numpy (the exhaustive
np.log2 exception table; every value the compress path maps is a float32);
the forward map of other doubles is correctly rounded (numpy's SIMD log2
differs by one ulp on ~4e-5 of random doubles); the inverse map's float32
cast is bit-identical, its float64 value correctly rounded (numpy's exp2 is
one ulp off on ~5 % of doubles).  Inputs may be numpy arrays, scalars or
torch tensors; they are moved to the CUDA device.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError, DegenerateBlock, DeviceError, NonFiniteInput, NonRepresentableFactor, \
    SubnormalMinimum, check

__all__ = [
    "BlockStats",
    "TransformParams",
    "compute_block_stats",
    "make_transform_params",
    "derive_transform_params",
    "forward_map",
    "inverse_map",
    "zero_sub_floor_magnitudes",
    "float_floor",
]


def float_floor(dtype) -> float:
    """Smallest positive normal value of the element type (transform.py:37-39)."""
    return float(np.finfo(np.dtype(dtype)).tiny)


@dataclass(frozen=True)
class BlockStats:
    """Per-block magnitude statistics (transform.py:42-58); ``abs_min`` /
    ``abs_max`` are None for an all-zero (degenerate) block."""

    abs_min: float | None
    abs_max: float | None
    has_zero: bool
    has_negative: bool
    count: int

    @property
    def is_degenerate(self) -> bool:
        return self.abs_min is None


@dataclass(frozen=True)
class TransformParams:
    """Factors, bounds and thresholds of the mapping (transform.py:61-81)."""

    factor_pos: float
    factor_neg: float
    epsilon0: float
    b_r: float
    b_a: float
    boundary: float
    zero_code_value: float
    zero_threshold: float
    lg_pos: float
    lg_neg: float

    def as_array(self) -> np.ndarray:
        """The ten fields in declaration order (the ABI's params10)."""
        return np.array([self.factor_pos, self.factor_neg, self.epsilon0, self.b_r, self.b_a, self.boundary,
                         self.zero_code_value, self.zero_threshold, self.lg_pos, self.lg_neg], np.float64)


def _device():
    if not torch.cuda.is_available():
        raise DeviceError("CUDA device required (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _to_device_f64(x) -> torch.Tensor:
    dev = _device()
    if isinstance(x, torch.Tensor):
        return x.detach().to(device=dev, dtype=torch.float64).contiguous().reshape(-1)
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64)).reshape(-1)
    return torch.from_numpy(a).to(dev)


def _shape_of(x):
    return tuple(x.shape) if isinstance(x, torch.Tensor) else np.shape(x)


def _ptr(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())


def compute_block_stats(block) -> BlockStats:
    """compute_block_stats (transform.py:84-107): DegenerateBlock on an empty
    block, NonFiniteInput on NaN/Inf; ``abs_min`` ignores exact zeros."""
    d = _to_device_f64(block)
    if d.numel() == 0:
        raise DegenerateBlock("empty block")
    lib = N.load()
    out = torch.empty(6, dtype=torch.float64, device=d.device)
    scratch = torch.empty(8, dtype=torch.int64, device=d.device)
    check(lib.pmz_block_stats(_ptr(d), d.numel(), _ptr(out), _ptr(scratch), _stream()), "block_stats")
    amin, amax, has_zero, has_neg, nonfinite, count = out.cpu().tolist()
    if nonfinite:
        raise NonFiniteInput("block contains NaN or Inf")
    if amax == 0.0:
        return BlockStats(None, None, bool(has_zero), bool(has_neg), int(count))
    return BlockStats(abs_min=float(amin), abs_max=float(amax), has_zero=bool(has_zero), has_negative=bool(has_neg),
                      count=int(count))


def derive_transform_params(factor_pos: float, factor_neg: float, b_r: float, epsilon0: float) -> TransformParams:
    """derive_transform_params (transform.py:110-135) on the device."""
    dev = _device()
    lib = N.load()
    b_a = float(np.log2(1.0 + b_r))  # transform.py:118, the host scalar the ABI takes
    d_in = torch.tensor([factor_pos, factor_neg, b_r, epsilon0], dtype=torch.float64, device=dev)
    d_out = torch.empty(10, dtype=torch.float64, device=dev)
    d_mask = torch.zeros(1, dtype=torch.int32, device=dev)
    check(lib.pmz_derive_params(_ptr(d_in), b_a, _ptr(d_out), _ptr(d_mask), _stream()), "derive_params")
    o = d_out.cpu().numpy()
    mask = int(d_mask.item())
    if mask:
        # a general-double logarithm within 2^-56 of a rounding midpoint: the
        # reference's own numpy expressions (transform.py:119-123) decide
        lg_pos, lg_neg = float(np.log2(factor_pos)), float(np.log2(factor_neg))
        zc = float(np.log2(epsilon0) + lg_pos)
        o[5:10] = [float(lg_neg + np.log2(factor_pos - epsilon0) - b_a), zc, zc + b_a, lg_pos, lg_neg]
    return TransformParams(*[float(v) for v in o])


def make_transform_params(stats: BlockStats, b_r: float, epsilon0: float | None = None) -> TransformParams:
    """make_transform_params (transform.py:138-167): ConfigError for b_r
    outside (0, 1), DegenerateBlock, SubnormalMinimum, NonRepresentableFactor."""
    if not (0.0 < b_r < 1.0):
        raise ConfigError(f"relative error bound must be in (0, 1), got {b_r}")
    if stats.is_degenerate:
        raise DegenerateBlock("all-zero block has no transform parameters")
    if epsilon0 is None:
        epsilon0 = float_floor(np.float32)
    abs_min, abs_max = stats.abs_min, stats.abs_max
    if abs_min <= epsilon0:
        raise SubnormalMinimum(f"abs_min={abs_min!r} <= epsilon0={epsilon0!r}; reclassify "
                               "sub-floor magnitudes as zeros and recompute stats")
    factor_pos = abs_min
    factor_neg = ((abs_max + epsilon0) * factor_pos * (1.0 + b_r) ** 2) / (abs_min - epsilon0)  # :160-162
    if not np.isfinite(factor_neg):
        raise NonRepresentableFactor(f"factor_neg overflows for abs_min={abs_min!r}, abs_max={abs_max!r}")
    return derive_transform_params(factor_pos, factor_neg, b_r, epsilon0)


def _p10(p: TransformParams):
    return (ctypes.c_double * 10)(*p.as_array().tolist())


def _ret(out: torch.Tensor, x):
    if np.ndim(x) == 0 and not isinstance(x, torch.Tensor):
        return float(out.item())
    return out.cpu().numpy().reshape(_shape_of(x))


def forward_map(x, p: TransformParams):
    """forward_map (transform.py:170-185): scalars or arrays, float64 out."""
    d = _to_device_f64(x)
    out = torch.empty_like(d)
    check(N.load().pmz_forward_map(_ptr(d), d.numel(), _p10(p), _ptr(out), _stream()), "forward_map")
    return _ret(out, x)


def inverse_map(v, p: TransformParams, dtype=np.float64):
    """inverse_map (transform.py:188-202): float64 out (``dtype=np.float32``
    returns the emitted element type, the round-to-nearest cast D20)."""
    d = _to_device_f64(v)
    if np.dtype(dtype) == np.float32:
        out32 = torch.empty(d.numel(), dtype=torch.float32, device=d.device)
        check(N.load().pmz_inverse_map(_ptr(d), d.numel(), _p10(p), None, _ptr(out32), _stream()), "inverse_map")
        return _ret(out32, v)
    out = torch.empty_like(d)
    check(N.load().pmz_inverse_map(_ptr(d), d.numel(), _p10(p), _ptr(out), None, _stream()), "inverse_map")
    return _ret(out, v)


def zero_sub_floor_magnitudes(data, epsilon0: float) -> np.ndarray:
    """zero_sub_floor_magnitudes (transform.py:205-210): a float64 copy with
    |x| <= epsilon0 set to 0."""
    d = _to_device_f64(data)
    out = torch.empty_like(d)
    check(N.load().pmz_zero_sub_floor(_ptr(d), d.numel(), float(epsilon0), _ptr(out), _stream()),
          "zero_sub_floor")
    return out.cpu().numpy().reshape(_shape_of(data))
