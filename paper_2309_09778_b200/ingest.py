"""Dataset ingest: SEG-Y rev-0
files with fixed-length traces, sample format 1 (IBM hex float) or 5 (IEEE),
traces stacked as rows.  The host parses the 3600-byte file header and checks
the trace framing; the trace records go to the device in one copy and the
sample conversion runs there (csrc/segy.cuh, ``pmz_segy_samples``)."""
from __future__ import annotations

import ctypes
import os
import struct

import numpy as np
import torch

from . import _native as N
from .errors import InconsistentTraceLength, SizeMismatch, TruncatedFile, UnsupportedFormatCode, check, EmptyDataset

TEXT_HEADER = 3200
BIN_HEADER = 400
TRACE_HEADER = 240


def segy_layout(head: bytes, file_size: int):
    """(format code, samples per trace, traces) from the binary header
    (big-endian int16: samples per trace at 3220, format code at 3224)."""
    if file_size < TEXT_HEADER + BIN_HEADER:
        raise TruncatedFile("shorter than the 3600-byte SEG-Y file header")
    ns, = struct.unpack_from(">H", head, TEXT_HEADER + 20)
    fmt, = struct.unpack_from(">h", head, TEXT_HEADER + 24)
    if fmt not in (1, 5):
        raise UnsupportedFormatCode(f"sample format code {fmt} (supported: 1 IBM float, 5 IEEE float)")
    if ns == 0:
        raise EmptyDataset("zero samples per trace")
    rec = TRACE_HEADER + 4 * ns
    body = file_size - TEXT_HEADER - BIN_HEADER
    if body <= 0 or body % rec:
        raise TruncatedFile(f"{body} bytes of trace records is not a whole number of {rec}-byte traces")
    return fmt, ns, body // rec


def read_segy(path: str, device=None) -> torch.Tensor:
    """read_segy -> (traces, samples) float32 CUDA tensor."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        data = f.read()
    fmt, ns, ntr = segy_layout(data, size)
    rec = TRACE_HEADER + 4 * ns
    tr = np.frombuffer(data, np.uint8, count=ntr * rec, offset=TEXT_HEADER + BIN_HEADER)
    per_trace = np.frombuffer(tr.reshape(ntr, rec)[:, 114:116].tobytes(), ">u2")
    if np.any((per_trace != 0) & (per_trace != ns)):
        raise InconsistentTraceLength("a trace header declares a different sample count (fixed-length traces only)")
    d_tr = torch.from_numpy(tr.copy()).pin_memory().to(dev, non_blocking=True)
    out = torch.empty((ntr, ns), dtype=torch.float32, device=dev)
    lib = N.load()
    check(lib.pmz_segy_samples(ctypes.c_void_p(d_tr.data_ptr()), ntr, ns, fmt, ctypes.c_void_p(out.data_ptr()),
                               ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)), "segy")
    return out


def read_raw(path: str, rows: int, cols: int, dtype=np.float32, big_endian: bool = False) -> np.ndarray:
    """read_raw: row-major array of rows x cols."""
    if rows <= 0 or cols <= 0:
        raise EmptyDataset("zero-sized raw request")
    dt = np.dtype(dtype).newbyteorder(">" if big_endian else "<")
    if os.path.getsize(path) != rows * cols * dt.itemsize:
        raise SizeMismatch(f"{path!r}: {os.path.getsize(path)} bytes, expected {rows * cols * dt.itemsize}")
    return np.fromfile(path, dtype=dt).astype(np.dtype(dtype).newbyteorder("=")).reshape(rows, cols)
