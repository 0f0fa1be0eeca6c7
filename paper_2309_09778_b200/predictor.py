"""Predictor module surface: Lorenzo coefficients, the
three-layer perceptron model and its serialization.

The perceptron is *evaluated* only on the GPU, inside the compress/decompress
wavefront kernels (csrc/common.cuh ``predict``); this module holds the weights
that travel by value into those kernels and the container's model blob
(D12).  Training (``train_step``) is outside this path (SURVEY.md
§8(f) row f1).
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field
from math import comb

import numpy as np

from .errors import Corrupt, ConfigError

LEAKY_SLOPE = 0.01


def lorenzo_coefficients(n: int = 1, dims: int = 2) -> dict:
    """(-1)^(k1+k2+1) C(n,k1) C(n,k2) over stencil offsets."""
    if n < 1:
        raise ConfigError("Lorenzo order must be >= 1")
    if dims == 1:
        return {(k,): (-1) ** (k + 1) * comb(n, k) for k in range(1, n + 1)}
    out = {}
    for k1 in range(n + 1):
        for k2 in range(n + 1):
            if (k1, k2) != (0, 0):
                out[(k1, k2)] = (-1) ** (k1 + k2 + 1) * comb(n, k1) * comb(n, k2)
    return out


@dataclass
class PerceptronModel:
    """w1: (S+1) x H (input + bias -> hidden), w2: H; leaky ReLU hidden layer."""
    w1: np.ndarray
    w2: np.ndarray
    leaky_slope: float = LEAKY_SLOPE
    S: int = 3
    H: int = 2
    dims: int = field(default=2)

    def __post_init__(self):
        self.w1 = np.asarray(self.w1, dtype=np.float64).reshape(self.S + 1, self.H)
        self.w2 = np.asarray(self.w2, dtype=np.float64).reshape(self.H)
        if self.H != 2 or self.S not in (1, 3):
            raise ConfigError("only S in {1,3}, H = 2 are supported (SPEC.md:127, 491)")
        if not (np.all(np.isfinite(self.w1)) and np.all(np.isfinite(self.w2))):
            raise ConfigError("non-finite perceptron weights")

    def to_bytes(self) -> bytes:
        """Model blob: S u32, H u32, slope f64, w1 row-major f64, w2 f64 (D12)."""
        return (struct.pack("<IId", self.S, self.H, float(self.leaky_slope)) + self.w1.astype("<f8").tobytes() +
                self.w2.astype("<f8").tobytes())

    @classmethod
    def from_bytes(cls, b: bytes) -> "PerceptronModel":
        if len(b) < 16:
            raise Corrupt("model blob too short")
        S, H, slope = struct.unpack_from("<IId", b, 0)
        if H != 2 or S not in (1, 3) or len(b) != 16 + 8 * (S + 1) * H + 8 * H:
            raise Corrupt("bad model blob")
        w = np.frombuffer(b, "<f8", offset=16)
        return cls(w[: (S + 1) * H].copy(), w[(S + 1) * H:].copy(), slope, S, H, 2 if S == 3 else 1)


def init_model(surface_size: int = 3, leaky_slope: float = LEAKY_SLOPE) -> PerceptronModel:
    """init_model: every hidden column = Lorenzo coefficients, bias 0; w2 = (0.5, 0.5)."""
    if surface_size == 3:
        col = [1.0, 1.0, -1.0, 0.0]  # W, N, NW (offsets (0,1), (1,0), (1,1)) + bias
    elif surface_size == 1:
        col = [1.0, 0.0]
    else:
        raise ConfigError("surface size must be 3 (2-D) or 1 (1-D)")
    w1 = np.array([[c, c] for c in col], dtype=np.float64)
    return PerceptronModel(w1, np.array([0.5, 0.5]), leaky_slope, surface_size, 2, 2 if surface_size == 3 else 1)
