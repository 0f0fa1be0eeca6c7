"""The perceptron trainer:
``train_step``, ``sweep``, ``simulate_roundtrip`` and ``select_best`` of the
reference's inline training flow, on the device.

* The objective -- mean over the samples of (predict(surface) - target)^2
  plus l2 * ||weights||^2 -- and its gradient (backpropagation through the
  leaky-ReLU hidden layer) are summed by CUDA kernels (csrc/train.cuh) in a
  fixed order, so a sweep is bit-reproducible.
* Training samples are every element (partition anchors excepted, D1) of
  the seeded training blocks, surfaces from the TRUE
  forward-mapped values, exactly what compress_block predicts from.
* ``sweep`` trains every HyperConfig with ONE full-batch gradient-descent
  pass from ``init_model`` ("one training round"), validates each
  candidate with ``simulate_roundtrip`` -- the real device compress +
  decompress of the validation blocks -- and
  ``select_best`` keeps the bound-respecting candidate with the smallest
  compression ratio, ties to the smaller l2 then the smaller lr.

The default grid is {lr: 1e-3, 1e-4} x {l2: 0, 1e-4, 1e-2}.
No oracle exists for this module (the reference ships no trainer code): its
tests pin the SPEC's properties (finite-difference gradients, lr = 0
identity, zero-loss fixed point, L2 shrinkage, determinism, selection rules).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError, DivergedTraining, SweepExhausted, check
from .predictor import PerceptronModel, init_model
from .trainer import sample_training_blocks, split_train_validation

DEFAULT_LR = (1e-3, 1e-4)
DEFAULT_L2 = (0.0, 1e-4, 1e-2)


@dataclass(frozen=True)
class HyperConfig:
    lr: float
    l2: float

    def __post_init__(self):
        if not (self.lr > 0) or not (self.l2 >= 0):
            raise ConfigError("HyperConfig needs lr > 0 and l2 >= 0 (SPEC.md:323)")


@dataclass
class TrainBatch:
    """surfaces: (n, S) float64 CUDA tensor, targets: (n,) float64 CUDA tensor."""
    surfaces: torch.Tensor
    targets: torch.Tensor

    def __post_init__(self):
        if self.surfaces.ndim != 2 or self.targets.ndim != 1 or self.surfaces.shape[0] != self.targets.shape[0]:
            raise ConfigError("TrainBatch: surfaces (n, S) and targets (n,) of equal length")
        if self.targets.numel() == 0:
            raise ConfigError("TrainBatch must be non-empty")


@dataclass
class ValidationReport:
    compression_ratio: float
    max_rel_error: float
    coverage: float
    chosen_m: int


@dataclass
class TrainingOutcome:
    model: PerceptronModel
    report: ValidationReport
    config: HyperConfig | None


def default_grid():
    return [HyperConfig(lr, l2) for lr in DEFAULT_LR for l2 in DEFAULT_L2]


def parse_grid(spec: str):
    """CLI --grid "lr:1e-3,1e-4;l2:0,1e-4,1e-2"."""
    vals = {}
    for part in spec.split(";"):
        if not part.strip():
            continue
        key, _, rest = part.partition(":")
        try:
            vals[key.strip()] = [float(v) for v in rest.split(",") if v.strip()]
        except ValueError:
            raise ConfigError(f"bad --grid part {part!r}")
    lrs, l2s = vals.get("lr", list(DEFAULT_LR)), vals.get("l2", list(DEFAULT_L2))
    return [HyperConfig(lr, l2) for lr in lrs for l2 in l2s]


def _params(model: PerceptronModel) -> N.Params:
    p = N.Params()
    p.b_r, p.b_a, p.slope = 1e-2, float(np.log2(1.01)), float(model.leaky_slope)
    for i, v in enumerate(model.w1.reshape(-1)):
        p.w1[i] = float(v)
    for i, v in enumerate(model.w2.reshape(-1)):
        p.w2[i] = float(v)
    p.S, p.H = model.S, model.H
    p.block_rows, p.block_cols, p.partition_rows = 256, 256, 32
    return p


def _weights(model: PerceptronModel) -> np.ndarray:
    return np.concatenate([model.w1.reshape(-1), model.w2.reshape(-1)])


def _step(model: PerceptronModel, sums: np.ndarray, lr: float, l2: float):
    """Gradient-descent update from the device sums (12 doubles: d/dw1 (S+1)xH,
    d/dw2, sum r^2, count): w -= lr * (grad mean + 2 l2 w).  Loss is pre-update."""
    nw1 = (model.S + 1) * model.H
    n = sums[11]
    if n <= 0:
        raise ConfigError("no training samples")
    g = np.concatenate([sums[:nw1], sums[8:10]]) / n
    w = _weights(model)
    g = g + 2.0 * l2 * w
    w_new = w - lr * g
    loss = float(sums[10] / n)
    if not np.all(np.isfinite(w_new)):
        raise DivergedTraining(f"non-finite weights after a step with lr={lr}, l2={l2}")
    out = PerceptronModel(w_new[:nw1].copy(), w_new[nw1:].copy(), model.leaky_slope, model.S, model.H, model.dims)
    return out, loss


def batch_sums(model: PerceptronModel, batch: TrainBatch) -> np.ndarray:
    """Device sums of the objective's terms over a TrainBatch (csrc/train.cuh)."""
    if batch.surfaces.shape[1] != model.S:
        raise ConfigError("surface size does not match the model")
    lib = N.load()
    dev = batch.targets.device
    surf = batch.surfaces.to(torch.float64).contiguous()
    tgt = batch.targets.to(torch.float64).contiguous()
    out = torch.zeros(12, dtype=torch.float64, device=dev)
    ws = torch.empty(296 * 12 * 8, dtype=torch.uint8, device=dev)
    p = _params(model)
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    check(lib.pmz_train_gradient_batch(ctypes.c_void_p(surf.data_ptr()), ctypes.c_void_p(tgt.data_ptr()),
                                       tgt.numel(), ctypes.byref(p), ctypes.c_void_p(out.data_ptr()),
                                       ctypes.c_void_p(ws.data_ptr()), ws.numel(), stream), "train_gradient_batch")
    return out.cpu().numpy()


def train_step(model: PerceptronModel, batch: TrainBatch, lr: float, l2: float):
    """One full gradient-descent pass over the batch:
    returns (updated model, mean squared loss before the update)."""
    if not (lr >= 0) or not (l2 >= 0):
        raise ConfigError("train_step needs lr >= 0 and l2 >= 0")
    return _step(model, batch_sums(model, batch), lr, l2)


def field_sums(codec, x: torch.Tensor, cfg, blocks: np.ndarray, model: PerceptronModel) -> np.ndarray:
    """Device sums over every element (anchors excepted) of the listed blocks
    of the field x, surfaces from the forward-mapped TRUE values."""
    from .pipeline import grid_view_shape, make_params
    (rows, cols), S = grid_view_shape(tuple(x.shape))
    p = make_params(_with_model(cfg, model), S)
    g = N.Geom(rows, cols, 0, rows)
    lib = codec.lib
    wsz = ctypes.c_uint64(0)
    check(lib.pmz_workspace_size(ctypes.byref(p), ctypes.byref(g), ctypes.byref(wsz)), "workspace_size")
    ws = codec._buf("_ws", wsz.value)
    d_blocks = torch.as_tensor(np.asarray(blocks, np.int64), device=codec.device)
    out = torch.zeros(12, dtype=torch.float64, device=codec.device)
    check(lib.pmz_train_gradient(ctypes.c_void_p(x.data_ptr()), ctypes.byref(g), ctypes.byref(p),
                                 ctypes.c_void_p(d_blocks.data_ptr()), int(d_blocks.numel()),
                                 ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                 ctypes.c_void_p(torch.cuda.current_stream(codec.device).cuda_stream)),
          "train_gradient")
    return out.cpu().numpy()


def _with_model(cfg, model):
    from dataclasses import replace
    return replace(cfg, model=model)


def _block_slices(shape2d, br: int, bc: int, ids):
    rows, cols = shape2d
    nbc = (cols + bc - 1) // bc
    for b in ids:
        bi, bj = divmod(int(b), nbc)
        yield slice(bi * br, min(rows, (bi + 1) * br)), slice(bj * bc, min(cols, (bj + 1) * bc))


def simulate_roundtrip(codec, x: torch.Tensor, cfg, model: PerceptronModel, val_blocks) -> ValidationReport:
    """The real device compress + decompress of the validation blocks
    (SPEC.md:371-377): blocks of one shape are stacked into one field (block
    boundaries preserved) whose every block validates (select_m and the
    codebook from all of them); CR counts the block records (headers of the
    simulation containers excluded), the error is measured on the decoded
    f32 values (zeros exact)."""
    from .pipeline import decompress, grid_view_shape
    (rows, cols), _ = grid_view_shape(tuple(x.shape))
    x2 = x.reshape(rows, cols)
    groups = {}
    for rs, cs in _block_slices((rows, cols), cfg.block_rows, cfg.block_cols, val_blocks):
        blk = x2[rs, cs]
        groups.setdefault(tuple(blk.shape), []).append(blk)
    c_bytes = o_bytes = 0
    max_rel, cov_num, cov_den, m = 0.0, 0, 0, 0
    mcfg = _with_model(cfg, model)
    for (h, w), blks in groups.items():
        # full-height blocks stack without moving a block boundary; shorter
        # (bottom-edge) blocks go one by one
        fields = [torch.cat(blks, 0)] if h == cfg.block_rows else blks
        for f in fields:
            f = f.contiguous()
            nb = (f.shape[0] + cfg.block_rows - 1) // cfg.block_rows * ((f.shape[1] + cfg.block_cols - 1) // cfg.block_cols)
            d_val = torch.arange(nb, dtype=torch.int64, device=codec.device)
            buf, info = codec.compress_device(f, mcfg, d_val=d_val)
            c_bytes += info.nbytes - info.header_bytes
            o_bytes += f.numel() * 4
            m = max(m, info.m)
            cov = np.asarray(info.coverage, dtype=np.float64)
            cov_den += cov.sum()
            cov_num += cov[: info.m + 1].sum()
            y = torch.from_numpy(decompress(buf.cpu().numpy().tobytes(), device=codec.device,
                                            shape=tuple(f.shape))).to(codec.device)
            xz = torch.where(f.abs() <= 1.1754943508222875e-38, torch.zeros_like(f), f).double()
            nz = xz != 0
            if bool((y[~nz] != 0).any()):
                max_rel = float("inf")
            elif bool(nz.any()):
                max_rel = max(max_rel, float(((y.double()[nz] - xz[nz]).abs() / xz[nz].abs()).max()))
    return ValidationReport(c_bytes / max(o_bytes, 1), max_rel, cov_num / cov_den if cov_den else 1.0, m)


def sweep(codec, x: torch.Tensor, cfg, configs=None, train_blocks=None, val_blocks=None):
    """Every HyperConfig trained by one gradient-descent pass from init_model
    over the training blocks, then validated by simulate_roundtrip; returns
    [(config, model or None, report or None, error or None)] in config order
    (a diverging config is recorded, the sweep goes on)."""
    from .pipeline import grid_view_shape
    configs = list(configs) if configs is not None else default_grid()
    if not configs:
        raise ConfigError("sweep needs at least one HyperConfig")
    (rows, cols), S = grid_view_shape(tuple(x.shape))
    if train_blocks is None or val_blocks is None:
        nb = ((rows + cfg.block_rows - 1) // cfg.block_rows) * ((cols + cfg.block_cols - 1) // cfg.block_cols)
        tr, va = split_train_validation(sample_training_blocks(nb, cfg.sample_rate, cfg.seed))
        train_blocks = tr if train_blocks is None else train_blocks
        val_blocks = va if val_blocks is None else val_blocks
    m0 = cfg.model if cfg.model is not None else init_model(S)
    x2 = x.reshape(rows, cols).contiguous()
    sums = field_sums(codec, x2, cfg, train_blocks, m0)  # every config starts from m0: one gradient
    out = []
    for hc in configs:
        try:
            model, _ = _step(m0, sums, hc.lr, hc.l2)
            out.append((hc, model, simulate_roundtrip(codec, x2, cfg, model, val_blocks), None))
        except DivergedTraining as ex:
            out.append((hc, None, None, ex))
    return out


def select_best(results, b_r: float, bound_factor: float = 1.5) -> TrainingOutcome:
    """Among the reports within bound_factor * b_r (1.5 in
    the SPEC, the compress repair factor otherwise): the smallest
    compression ratio, ties to the smaller l2, then the smaller lr."""
    ok = [(r.compression_ratio, hc.l2, hc.lr, i) for i, (hc, mdl, r, e) in enumerate(results)
          if r is not None and r.max_rel_error <= bound_factor * b_r]
    if not ok:
        raise SweepExhausted("no candidate satisfies the error bound")
    i = min(ok)[3]
    hc, mdl, r, _ = results[i]
    return TrainingOutcome(mdl, r, hc)


def train(codec, x: torch.Tensor, cfg, configs=None) -> TrainingOutcome:
    """The inline training of a compress run: sweep, select;
    SweepExhausted falls back to init_model."""
    from .pipeline import grid_view_shape
    res = sweep(codec, x, cfg, configs)
    try:
        return select_best(res, cfg.rel_error, cfg.repair_factor)
    except SweepExhausted:
        _, S = grid_view_shape(tuple(x.shape))
        return TrainingOutcome(init_model(S), ValidationReport(float("nan"), float("nan"), float("nan"), 0), None)
