"""Seeded synthetic stand-ins for the BASELINE.json configs.

The paper's SEG-Y corpus is proprietary and absent; these fields reproduce the
shapes, sizes and value distributions BASELINE.json names.  Generation uses
torch (CPU or CUDA) so the 8 GiB C5 field can be built directly in HBM; each
test generates its input once and hands the same array to both the CUDA path
and the oracle, so generator numerics never enter a parity comparison.
"""
from __future__ import annotations

import math

import numpy as np
import torch

# name -> (shape, rel error bounds, seed, description)
CONFIGS = {
    "C1": ((1 << 20,), (1e-2,), 0, "1-D sines + noise x100, 1% exact zeros, mixed sign"),
    "C2": ((1800, 3600), (1e-2, 1e-3), 1, "exp(GRF k^-3), 30% sign-flipped on a smooth mask"),
    "C3": ((512, 512, 512), (1e-2,), 2, "lognormal exp(2 GRF k^-2.5), all positive"),
    "C4": ((100, 500, 500), (1e-2, 1e-4), 3, "GRF k^-3 + N(0,1e-3), 2 zero planes"),
    "C5": ((1024, 1024, 2048), (1e-2,), 4, "GRF k^-3 mixed sign (8 GiB)"),
}


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def grf(shape, beta: float, gen: torch.Generator, device) -> torch.Tensor:
    """Gaussian random field with power spectrum |k|^-beta (k=0 zeroed), standardized."""
    noise = torch.randn(shape, generator=gen, device=device, dtype=torch.float32)
    # CPU: numpy's pocketfft (float32 in, complex64 out).  torch's CPU FFT corrupts the heap
    # now and then on this image ("free(): corrupted unsorted chunks" inside irfftn of a
    # 20x500x500 field, with no other native code loaded), which would abort a test run.
    cpu = torch.device(device).type == "cpu"
    f = torch.from_numpy(np.fft.rfftn(noise.numpy())) if cpu else torch.fft.rfftn(noise)
    del noise
    k2 = None
    for ax, n in enumerate(shape):
        if ax == len(shape) - 1:
            k = torch.fft.rfftfreq(n, device=device)
        else:
            k = torch.fft.fftfreq(n, device=device)
        view = [1] * len(shape)
        view[ax] = k.numel()
        kk = (k * k).reshape(view)
        k2 = kk if k2 is None else k2 + kk
    amp = torch.where(k2 > 0, k2.clamp_min(1e-30) ** (-beta / 4.0), torch.zeros_like(k2))
    f.mul_(amp)
    del amp, k2
    out = torch.from_numpy(np.ascontiguousarray(np.fft.irfftn(f.numpy(), s=shape, axes=tuple(range(len(shape)))))) if cpu \
        else torch.fft.irfftn(f, s=shape)
    del f
    out -= out.mean()
    out /= out.std()
    return out


def generate(name: str, device="cpu", shape=None) -> torch.Tensor:
    """Build config ``name`` (C1..C5) as a float32 tensor; ``shape`` overrides the size."""
    shp, _, seed, _ = CONFIGS[name]
    shp = tuple(shape) if shape is not None else shp
    g = _gen(seed, device)
    if name == "C1":
        n = shp[0]
        i = torch.arange(n, device=device, dtype=torch.float64)
        x = torch.sin(2 * math.pi * i / 4096) + 0.3 * torch.sin(2 * math.pi * i / 97)
        x = x + 0.01 * torch.randn(n, generator=g, device=device, dtype=torch.float64)
        x = (100.0 * x).to(torch.float32)
        nz = max(1, n // 100)
        idx = torch.randperm(n, generator=g, device=device)[:nz]
        x[idx] = 0.0
        return x
    if name == "C2":
        base = torch.exp(grf(shp, 3.0, g, device))
        mask = grf(shp, 4.0, g, device)
        thr = torch.quantile(mask.reshape(-1)[:: max(1, mask.numel() // 1_000_000)].double(), 0.7).float()
        return torch.where(mask > thr, -base, base).to(torch.float32)
    if name == "C3":
        return torch.exp(2.0 * grf(shp, 2.5, g, device)).to(torch.float32)
    if name == "C4":
        x = grf(shp, 3.0, g, device)
        x += 1e-3 * torch.randn(shp, generator=g, device=device, dtype=torch.float32)
        n0 = shp[0]
        planes = [n0 // 3, n0 // 3 + 1] if n0 >= 2 else [0]
        for p in planes:
            x[p] = 0.0
        return x.to(torch.float32)
    if name == "C5":
        return grf(shp, 3.0, g, device).to(torch.float32)
    raise KeyError(name)
