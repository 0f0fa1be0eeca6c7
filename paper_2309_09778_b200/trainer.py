"""Trainer pieces on the hot path (§8 rows a17, a18, a23).

Only the seeded block sampling + 8:2 split that name the validation blocks
live here (host-side integer work); ``select_m``'s residual
histogram and ``estimate_codebook``'s validation histogram + Huffman build run
on the GPU inside the compress stages (csrc/compress.cuh, csrc/encode.cuh).
The training sweep itself is training.py.
"""
from __future__ import annotations

import math

import numpy as np

from .errors import ConfigError, EmptyDataset

SAMPLE_RATE = 0.10
COVERAGE_TARGET = 0.99
MIN_SAMPLED = 5


def _ceil(x: float) -> int:
    # ceil of a product of a decimal fraction; robust to its binary representation (D16)
    return int(math.ceil(x - 1e-9))


def sample_training_blocks(n_blocks: int, rate: float = SAMPLE_RATE, seed: int = 0) -> np.ndarray:
    """Seeded uniform shuffle selection of ceil(rate*N) blocks (D16).

    D21: inputs too small for a 5-block sample take min(N, 5) blocks."""
    if not (0.0 < rate <= 1.0):
        raise ConfigError("sample rate must be in (0, 1]")
    if n_blocks <= 0:
        raise EmptyDataset("no blocks to sample")
    k = max(_ceil(rate * n_blocks), min(n_blocks, MIN_SAMPLED))
    if rate == 1.0:
        return np.arange(n_blocks, dtype=np.int64)
    return np.random.default_rng(seed).permutation(n_blocks)[:k].astype(np.int64)


def split_train_validation(samples: np.ndarray):
    """First ceil(0.8 k) train, the rest validate.  D21: when
    fewer than 5 blocks exist the whole sample also serves as validation."""
    k = len(samples)
    ntr = _ceil(0.8 * k)
    train, val = samples[:ntr], samples[ntr:]
    if val.size == 0:
        val = samples
    return train, val


def validation_blocks(n_blocks: int, rate: float = SAMPLE_RATE, seed: int = 0) -> np.ndarray:
    if n_blocks == 0:
        return np.zeros(0, np.int64)
    return split_train_validation(sample_training_blocks(n_blocks, rate, seed))[1]
