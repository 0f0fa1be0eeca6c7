"""Command line front end:
``compress`` / ``decompress`` / ``bench`` over container files, with the
reference's flags and one exit code per error family (errors.EXIT_CODES).

    python -m paper_2309_09778_b200 compress --input x.f32 --format raw32 --dims 1800x3600 \\
        --rel-error 1e-2 --output x.pmz
    python -m paper_2309_09778_b200 decompress --input x.pmz --output y.f32 --original x.f32
    python -m paper_2309_09778_b200 bench --input gen:C2 --bench-bounds 1e-2,1e-3

Every subcommand prints one metrics CSV line per compression (evaluate,
SPEC.md:540-549): dataset, b_r, CR, max relative error, compress and
decompress MB/s (device time of the call, file I/O excluded).  The compute
runs on the GPU through the library; there is no CPU path.  ``--threads`` is
accepted for flag compatibility (the device decides its own parallelism;
output is deterministic for any value).  ``--train`` / ``--grid``
run the inline training sweep (training.py); ``--save-model`` /
``--load-model`` write / read the model blob; ``--format segy`` reads rev-0
SEG-Y (format codes 1 and 5, ingest.py).
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

from . import errors as E
from .predictor import PerceptronModel

CSV_HEADER = "dataset,rel_error,rows,cols,bytes_in,bytes_out,compression_ratio,max_rel_error,compress_MBps,decompress_MBps"


def _dims(s: str):
    try:
        r, c = (int(v) for v in s.lower().split("x"))
    except ValueError:
        raise E.ConfigError(f"bad dims {s!r}: expected RxC")
    if r <= 0 or c <= 0:
        raise E.ConfigError(f"bad dims {s!r}")
    return r, c


def _generate(kind: str, dims, seed: int) -> np.ndarray:
    """gen:<kind>: the BASELINE configs C1..C4 (synthetic.py) or the SPEC's
    acceptance datasets sine2d / gaussian-field / white-noise."""
    from . import synthetic
    if kind in ("C1", "C2", "C3", "C4"):
        return synthetic.generate(kind, shape=dims).numpy()
    r, c = dims or (512, 512)
    rng = np.random.default_rng(seed)
    if kind == "sine2d":  # sin(2 pi r / rows) sin(2 pi c / cols) + 2.0, strictly positive
        i, j = np.meshgrid(np.arange(r), np.arange(c), indexing="ij")
        return (np.sin(2 * np.pi * i / r) * np.sin(2 * np.pi * j / c) + 2.0).astype(np.float32)
    if kind == "constant":
        return np.full((r, c), 1.0, np.float32)
    if kind == "gaussian-field":
        import torch
        g = torch.Generator().manual_seed(seed)
        return synthetic.grf((r, c), 3.0, g, "cpu").numpy().astype(np.float32)
    if kind == "white-noise":
        return rng.normal(0, 1, (r, c)).astype(np.float32)
    raise E.ConfigError(f"unknown generator {kind!r}")


def _read_input(a) -> tuple[np.ndarray, str]:
    src = a.input
    if src.startswith("gen:"):
        return _generate(src[4:], _dims(a.dims) if a.dims else None, a.seed), src
    fmt = a.format or ("raw32" if src.endswith((".f32", ".raw")) else "npy" if src.endswith(".npy") else
                       "segy" if src.endswith((".sgy", ".segy")) else None)
    if not os.path.exists(src):
        raise E.IngestError(f"cannot read {src!r}")
    if fmt == "segy":  # traces as rows, sample conversion on the device (ingest.py)
        from . import ingest
        return ingest.read_segy(src, a.device).cpu().numpy(), os.path.basename(src)
    try:
        if fmt == "npy":
            x = np.load(src)
        elif fmt == "raw64":
            raise E.ConfigError("--format raw64: 64-bit elements are not supported by the device path (raw32 only)")
        elif fmt == "raw32":
            x = np.fromfile(src, dtype=np.float32)
            if a.dims:
                r, c = _dims(a.dims)
                if x.size != r * c:
                    raise E.IngestError(f"{src!r} holds {x.size} values, --dims asks for {r * c}")
                x = x.reshape(r, c)
        else:
            raise E.ConfigError(f"unknown --format {fmt!r} (raw32 | npy | segy | gen:<kind>)")
    except OSError as ex:
        raise E.IngestError(f"cannot read {src!r}: {ex}")
    if x.dtype != np.float32:
        raise E.ConfigError("only 32-bit element type is supported on the device path")
    return x, os.path.basename(src)


def _model(a, x=None, rel=None):
    """--load-model (a model blob), else the inline training sweep when
    --train / --grid is given (training.py), else init_model;
    --save-model writes the model used."""
    model = None
    if a.load_model:
        try:
            with open(a.load_model, "rb") as f:
                model = PerceptronModel.from_bytes(f.read())
        except OSError as ex:
            raise E.IngestError(f"cannot read model {a.load_model!r}: {ex}")
    elif (a.train or a.grid) and x is not None:
        import torch
        from . import pipeline as P, training
        br, bc = _dims(a.block_size)
        cfg = P.CompressConfig(rel_error=rel, block_rows=br, block_cols=bc, partition_rows=a.partition_rows,
                               repair_factor=a.repair_factor, coverage_target=a.coverage_target,
                               sample_rate=a.sample_rate, seed=a.seed)
        codec = P._codec(a.device)
        grid = training.parse_grid(a.grid) if a.grid else None
        model = training.train(codec, torch.from_numpy(np.ascontiguousarray(x)).to(codec.device), cfg, grid).model
    if a.save_model:
        from .predictor import init_model
        m = model if model is not None else init_model(1 if (x is not None and (x.ndim == 1 or x.shape[0] == 1)) else 3)
        with open(a.save_model, "wb") as f:
            f.write(m.to_bytes())
    return model


def _max_rel(x: np.ndarray, y: np.ndarray) -> float:
    tiny = float(np.finfo(np.float32).tiny)
    xz = np.where(np.abs(x) <= tiny, 0, x).astype(np.float64).reshape(-1)
    yy = y.astype(np.float64).reshape(-1)
    nz = xz != 0
    if np.any(yy[~nz] != 0):
        return float("inf")
    return float((np.abs(yy[nz] - xz[nz]) / np.abs(xz[nz])).max(initial=0.0))


def _compress_one(x: np.ndarray, rel: float, a, model):
    import torch
    from . import pipeline as P
    br, bc = _dims(a.block_size)
    cfg = P.CompressConfig(rel_error=rel, block_rows=br, block_cols=bc, partition_rows=a.partition_rows,
                           repair_factor=a.repair_factor, coverage_target=a.coverage_target,
                           sample_rate=a.sample_rate, seed=a.seed, model=model)
    codec = P._codec(a.device)
    d = torch.from_numpy(np.ascontiguousarray(x)).to(codec.device)
    codec.compress_device(d, cfg)  # warm (tables, workspace)
    torch.cuda.synchronize(codec.device)
    t0 = time.perf_counter()
    buf, info = codec.compress_device(d, cfg)
    torch.cuda.synchronize(codec.device)
    tc = time.perf_counter() - t0
    return buf.cpu().numpy().tobytes(), info, tc


def _decompress_one(container: bytes, a, shape=None):
    import torch
    from . import pipeline as P
    codec = P._codec(a.device)
    buf = np.frombuffer(container, dtype=np.uint8)
    h = codec.parse_header(buf)
    offs = codec.index_blocks(buf, h)
    d_buf = torch.from_numpy(buf.copy()).to(codec.device)
    d_off = torch.from_numpy(offs.view(np.int64)).to(codec.device)
    codec.decompress_device(d_buf, h, d_off)
    torch.cuda.synchronize(codec.device)
    t0 = time.perf_counter()
    y = codec.decompress_device(d_buf, h, d_off)
    torch.cuda.synchronize(codec.device)
    td = time.perf_counter() - t0
    y = y.cpu().numpy()
    return (y.reshape(shape) if shape is not None else y), td


def _csv(name, rel, x, nout, max_rel, tc, td):
    r, c = (x.shape + (1,))[:2] if x.ndim > 1 else (1, x.size)
    return (f"{name},{rel:g},{r},{c},{x.nbytes},{nout},{nout / x.nbytes:.6f},{max_rel:.6g},"
            f"{x.nbytes / tc / 1e6 if tc else float('nan'):.1f},{x.nbytes / td / 1e6 if td else float('nan'):.1f}")


def cmd_compress(a) -> int:
    x, name = _read_input(a)
    if not a.output:
        raise E.ConfigError("--output is required")
    cont, info, tc = _compress_one(x, a.rel_error, a, _model(a, x, a.rel_error))
    with open(a.output, "wb") as f:
        f.write(cont)
    y, td = _decompress_one(cont, a, x.shape)
    print(CSV_HEADER)
    print(_csv(name, a.rel_error, x, len(cont), _max_rel(x, y), tc, td))
    return 0


def cmd_decompress(a) -> int:
    if not os.path.exists(a.input):
        raise E.IngestError(f"cannot read {a.input!r}")
    with open(a.input, "rb") as f:
        cont = f.read()
    y, td = _decompress_one(cont, a)
    if a.output:
        (np.save if a.output.endswith(".npy") else lambda p, v: v.tofile(p))(a.output, y)
    if a.original:
        x, _ = _read_input(argparse.Namespace(**{**vars(a), "input": a.original}))
        print(f"max_rel_error,{_max_rel(x.reshape(y.shape), y):.6g}")
    print(f"decompress_MBps,{y.nbytes / td / 1e6:.1f}")
    return 0


def cmd_bench(a) -> int:
    x, name = _read_input(a)
    print(CSV_HEADER)
    for tok in a.bench_bounds.split(","):
        rel = float(tok)
        cont, info, tc = _compress_one(x, rel, a, _model(a, x, rel))
        y, td = _decompress_one(cont, a, x.shape)
        print(_csv(name, rel, x, len(cont), _max_rel(x, y), tc, td), flush=True)
    return 0


def parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2309_09778_b200", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("compress", "decompress", "bench"):
        s = sub.add_parser(name)
        s.add_argument("--input", required=True, help="file, or gen:<C1..C4|sine2d|gaussian-field|white-noise>")
        s.add_argument("--output")
        s.add_argument("--format", choices=["raw32", "raw64", "npy", "segy"])
        s.add_argument("--dims", help="RxC of a raw input / generator size")
        s.add_argument("--rel-error", type=float, default=1e-2)
        s.add_argument("--block-size", default="256x256")
        s.add_argument("--partition-rows", type=int, default=32)
        s.add_argument("--sample-rate", type=float, default=0.1)
        s.add_argument("--coverage-target", type=float, default=0.99)
        s.add_argument("--repair-factor", type=float, default=1.5)
        s.add_argument("--grid", help='trainer sweep grid, e.g. "lr:1e-3,1e-4;l2:0,1e-4,1e-2" (implies --train)')
        s.add_argument("--train", action="store_true", help="inline training sweep (default grid) before compressing")
        s.add_argument("--threads", type=int, default=int(os.environ.get("PERMEZ_THREADS", "1")))
        s.add_argument("--seed", type=int, default=0)
        s.add_argument("--save-model")
        s.add_argument("--load-model")
        s.add_argument("--original")
        s.add_argument("--bench-bounds", default="1e-2,1e-3,1e-4")
        s.add_argument("--device", default=None)
    return ap


def main(argv=None) -> int:
    a = parser().parse_args(argv)
    try:
        if a.threads < 1:
            raise E.ConfigError("--threads must be >= 1")
        if a.grid:
            from . import training
            training.parse_grid(a.grid)  # validate before any device work
        if not (0.0 < a.rel_error < 1.0):
            raise E.ConfigError("--rel-error must lie in (0, 1)")
        return {"compress": cmd_compress, "decompress": cmd_decompress, "bench": cmd_bench}[a.cmd](a)
    except E.PermezError as ex:
        print(f"error: {type(ex).__name__}: {ex}", file=sys.stderr)
        return E.exit_code(ex)


if __name__ == "__main__":
    sys.exit(main())
