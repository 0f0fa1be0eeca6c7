"""Pipeline module: the compress / decompress entry points
of the reference package, executed by the sm_100a kernels behind the C ABI.

Host side (this file): argument checking, the seeded validation split, buffer
ownership (torch CUDA tensors), stream plumbing and the container framing
helpers.  Device side (csrc/): every per-element and per-block operation of
compress_block, verify_and_repair, estimate_codebook, build_codebook, encode,
decode_next, decompress_block and the domain transform.

There is deliberately no CPU fallback; without the native library or a CUDA
device every call raises ``DeviceError``.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError, DeviceError, check
from .predictor import PerceptronModel, init_model
from .trainer import COVERAGE_TARGET, SAMPLE_RATE, validation_blocks

EPS0_F32 = float(np.finfo(np.float32).tiny)  # transform.py:37-39 float_floor(float32)
REPAIR_FACTOR_SPEC = 1.5


@dataclass
class CompressConfig:
    """Reference parameters (SPEC.md:607 flags): --rel-error, --block-size RxC,
    --partition-rows, --coverage-target, --sample-rate, --seed; the model is
    the PerceptronModel (weights) and ``repair_factor`` the verify_and_repair
    tolerance multiple (D8: SPEC 1.5, BASELINE runs 1.0)."""
    rel_error: float = 1e-2
    block_rows: int = 256
    block_cols: int = 256
    partition_rows: int = 32
    repair_factor: float = REPAIR_FACTOR_SPEC
    coverage_target: float = COVERAGE_TARGET
    sample_rate: float = SAMPLE_RATE
    seed: int = 0
    m: int = 0
    model: PerceptronModel | None = None
    # "fp64": the reference's arithmetic, container version 1 (bit-exact parity);
    # "fp32": the north star's FP32 perceptron perf mode, container version 2
    # (2-D fields; codes may differ from fp64 where float32 rounding moves them)
    precision: str = "fp64"
    # optional uint16 CUDA tensor of Codec.code_dump_numel() elements: receives
    # every final code (raster per partition, 0xFFFF at anchors) -- for counting
    # code mismatches between the two precisions
    code_dump: object = None


@dataclass
class CompressInfo:
    nbytes: int
    header_bytes: int
    nblocks: int
    ntrivial: int
    nbal: int
    nrepair: int
    ncodes: int
    m: int
    max_code_len: int
    coverage: list = field(default_factory=list)
    shape: tuple = ()
    val_blocks: np.ndarray | None = None
    launches: int = 0


def host_b_a(b_r: float) -> float:
    return float(np.log2(1.0 + b_r))  # transform.py:118


def grid_view_shape(shape):
    """1-D -> (1, N), S=1; 2-D as is; n-D -> (prod(lead), last) (D18)."""
    if len(shape) == 1:
        return (1, int(shape[0])), 1
    if len(shape) == 2:
        return (int(shape[0]), int(shape[1])), 3
    return (int(np.prod(shape[:-1])), int(shape[-1])), 3


def make_params(cfg: CompressConfig, S: int) -> N.Params:
    if not (0.0 < cfg.rel_error < 1.0):
        raise ConfigError(f"relative error bound must be in (0, 1), got {cfg.rel_error}")
    if cfg.repair_factor <= 0:
        raise ConfigError("repair_factor must be > 0")
    model = cfg.model if cfg.model is not None else init_model(S)
    if model.S != S:
        raise ConfigError(f"model surface size {model.S} does not match the data ({S})")
    p = N.Params()
    p.b_r = cfg.rel_error
    p.b_a = host_b_a(cfg.rel_error)
    p.onepbr2 = (1.0 + cfg.rel_error) ** 2  # transform.py:160-162, Python float pow
    p.eps0 = EPS0_F32
    p.repair_t = cfg.repair_factor * cfg.rel_error
    p.coverage_target = cfg.coverage_target
    p.slope = float(model.leaky_slope)
    for i, v in enumerate(model.w1.reshape(-1)):
        p.w1[i] = float(v)
    for i, v in enumerate(model.w2.reshape(-1)):
        p.w2[i] = float(v)
    p.block_rows, p.block_cols, p.partition_rows = cfg.block_rows, cfg.block_cols, cfg.partition_rows
    p.S, p.H, p.m = S, 2, cfg.m
    if cfg.precision not in ("fp64", "fp32"):
        raise ConfigError(f"precision must be 'fp64' or 'fp32', got {cfg.precision!r}")
    p.precision = 1 if cfg.precision == "fp32" else 0
    if p.precision and S != 3:
        raise ConfigError("the FP32 perf mode is defined for 2-D fields (S = 3)")
    p.d_code_dump = int(cfg.code_dump.data_ptr()) if cfg.code_dump is not None else 0
    return p


def _ptr(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream_ptr(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _require_cuda(device):
    if not torch.cuda.is_available():
        raise DeviceError("CUDA device required (no CPU fallback)")
    return torch.device(device if device is not None else "cuda")


class Codec:
    """Reusable device codec: owns the workspace and output buffers so
    repeated calls (benchmarks, streaming) allocate nothing."""

    def __init__(self, device=None):
        self.device = _require_cuda(device)
        self.lib = N.load()
        self._ws = None
        self._dws = None
        self._out = None

    # ---- buffers ------------------------------------------------------
    def _buf(self, name: str, nbytes: int) -> torch.Tensor:
        cur = getattr(self, name)
        if cur is None or cur.numel() < nbytes:
            cur = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=self.device)
            setattr(self, name, cur)
        return cur

    # ---- numpy-exact per-block logarithms (DESIGN D22) ---------------------
    def np_fix_compress(self, p, g, ws: torch.Tensor, stream) -> int:
        """Resolve the blocks whose general-double log2 (np.log2(factor_neg),
        transform.py:120) the device left to numpy.  Synchronises ``stream``."""
        lib = self.lib
        return N.resolve_np_log2(
            lambda b, cap: lib.pmz_compress_np_fixups(ctypes.byref(g), ctypes.byref(p), _ptr(ws), ws.numel(), stream,
                                                      b, cap),
            lambda b, n: lib.pmz_compress_np_apply(ctypes.byref(g), ctypes.byref(p), _ptr(ws), ws.numel(), stream, b,
                                                   n))

    def np_fix_decompress(self, h, ws: torch.Tensor, stream) -> int:
        lib = self.lib
        return N.resolve_np_log2(
            lambda b, cap: lib.pmz_decompress_np_fixups(ctypes.byref(h), _ptr(ws), ws.numel(), stream, b, cap),
            lambda b, n: lib.pmz_decompress_np_apply(ctypes.byref(h), host_b_a(h.b_r), _ptr(ws), ws.numel(), stream,
                                                     b, n))

    def _write(self, p, g, write_header, out, block_offsets, ws, stream, res) -> int:
        s = self.lib.pmz_compress_write_async(ctypes.byref(g), ctypes.byref(p), int(write_header), _ptr(out),
                                              out.numel(), _ptr(block_offsets), _ptr(ws), ws.numel(), stream)
        if s:
            return s
        return self.lib.pmz_compress_result(ctypes.byref(g), ctypes.byref(p), 1, _ptr(ws), ws.numel(), stream,
                                            ctypes.byref(res))

    def analyze(self, x, p, g, d_val, ws, stream):
        """Stage 1: block stats + parameters, the host's np.log2 for the
        listed blocks, then forward map + coverage (pmz_compress_stats /
        _np_fixups / _np_apply / pmz_compress_transform)."""
        lib = self.lib
        check(lib.pmz_compress_stats(_ptr(x), ctypes.byref(g), ctypes.byref(p), _ptr(ws), ws.numel(), stream),
              "compress_stats")
        check(min(self.np_fix_compress(p, g, ws, stream), 0), "np_fixups")
        check(lib.pmz_compress_transform(_ptr(x), ctypes.byref(g), ctypes.byref(p), _ptr(d_val), int(d_val.numel()),
                                         _ptr(ws), ws.numel(), stream), "compress_transform")

    # ---- compression --------------------------------------------------
    def plan(self, shape, cfg: CompressConfig):
        (rows, cols), S = grid_view_shape(tuple(shape))
        p = make_params(cfg, S)
        g = N.Geom(rows, cols, 0, rows)
        nb = ((rows + cfg.block_rows - 1) // cfg.block_rows) * ((cols + cfg.block_cols - 1) // cfg.block_cols) \
            if rows and cols else 0
        val = validation_blocks(nb, cfg.sample_rate, cfg.seed)
        return p, g, nb, val

    def code_dump_numel(self, shape, cfg: CompressConfig) -> int:
        """Elements of a CompressConfig.code_dump buffer for a field of ``shape``."""
        p, g, _, _ = self.plan(shape, cfg)
        n = ctypes.c_uint64(0)
        check(self.lib.pmz_code_dump_elems(ctypes.byref(p), ctypes.byref(g), ctypes.byref(n)), "code_dump_elems")
        return int(n.value)

    def compress_device(self, x: torch.Tensor, cfg: CompressConfig | None = None, out_capacity: int | None = None,
                        plan=None, d_val: torch.Tensor | None = None, block_offsets: torch.Tensor | None = None):
        """Compress a float32 CUDA tensor; returns (container uint8 CUDA tensor
        view, CompressInfo).  The container bytes are the full reference layout."""
        cfg = cfg or CompressConfig()
        if x.dtype != torch.float32:
            raise ConfigError("only float32 element type is supported on the device path")
        if not x.is_cuda:
            raise DeviceError("compress_device expects a CUDA tensor")
        x = x.contiguous()
        p, g, nb, val = plan if plan is not None else self.plan(x.shape, cfg)
        if d_val is None:
            d_val = torch.as_tensor(val, dtype=torch.int64, device=self.device)
        lib = self.lib
        wsz = ctypes.c_uint64(0)
        check(lib.pmz_workspace_size(ctypes.byref(p), ctypes.byref(g), ctypes.byref(wsz)), "workspace_size")
        ws = self._buf("_ws", wsz.value)
        if out_capacity is None:
            out_capacity = int(x.numel() * 4 * 1.25) + 65536 + 64 * max(nb, 1) * 12
        out = self._buf("_out", out_capacity)
        res = N.Result()
        stream = _stream_ptr(self.device)
        self.analyze(x, p, g, d_val, ws, stream)
        check(lib.pmz_compress_codes(_ptr(x), ctypes.byref(g), ctypes.byref(p), _ptr(d_val), int(d_val.numel()),
                                     _ptr(ws), ws.numel(), stream), "compress_codes")
        check(lib.pmz_compress_encode(_ptr(x), ctypes.byref(g), ctypes.byref(p), _ptr(ws), ws.numel(), stream),
              "compress_encode")
        s = self._write(p, g, 1, out, block_offsets, ws, stream, res)
        if s == -16:  # capacity: write again into a buffer of the exact size (the encoded state is kept)
            out = self._buf("_out", int(res.header_bytes + res.record_bytes))
            s = self._write(p, g, 1, out, block_offsets, ws, stream, res)
        check(s, "compress")
        n = int(res.header_bytes + res.record_bytes)
        info = CompressInfo(n, int(res.header_bytes), int(res.nblocks), int(res.ntrivial), int(res.nbal),
                            int(res.nrepair), int(res.ncodes), int(res.m), int(res.max_code_len),
                            list(res.coverage), tuple(x.shape), val, int(res.launches))
        return out[:n], info

    def compress_staged(self, x: torch.Tensor, cfg: CompressConfig, *, block_row0: int = 0,
                        global_rows: int | None = None, global_shape=None, allreduce=None,
                        write_header: bool = True, out_capacity: int | None = None,
                        block_offsets: torch.Tensor | None = None, events=None, d_val: torch.Tensor | None = None):
        """Stage-by-stage compress of one shard (whole block-rows starting at
        global block-row ``block_row0``).  ``allreduce(tensor)`` sums a device
        int64 tensor across shards (NCCL) between stages: the select_m coverage
        histogram and the validation-code histogram, so every shard derives the
        same m and codebook.  ``events`` (5 CUDA events) time
        the stages (stage_names_compress) on the launching stream."""
        if x.dtype != torch.float32 or not x.is_cuda:
            raise ConfigError("compress_staged expects a float32 CUDA tensor")
        x = x.contiguous()
        (rows, cols), S = grid_view_shape(tuple(x.shape))
        if global_shape is not None:
            (grows, _), S = grid_view_shape(tuple(global_shape))
        else:
            grows = global_rows if global_rows is not None else rows
        p = make_params(cfg, S)
        g = N.Geom(rows, cols, block_row0, grows)
        nbc = (cols + cfg.block_cols - 1) // cfg.block_cols
        nb_local = ((rows + cfg.block_rows - 1) // cfg.block_rows) * nbc
        if d_val is None:
            gnb = ((grows + cfg.block_rows - 1) // cfg.block_rows) * nbc
            val = validation_blocks(gnb, cfg.sample_rate, cfg.seed)
            lo = block_row0 * nbc
            val = val[(val >= lo) & (val < lo + nb_local)] - lo
            d_val = torch.as_tensor(val, dtype=torch.int64, device=self.device)
        lib = self.lib
        wsz = ctypes.c_uint64(0)
        check(lib.pmz_workspace_size(ctypes.byref(p), ctypes.byref(g), ctypes.byref(wsz)), "workspace_size")
        ws = self._buf("_ws", wsz.value)
        if out_capacity is None:
            cap = ctypes.c_uint64(0)
            check(lib.pmz_max_container_size(ctypes.byref(p), ctypes.byref(g), ctypes.byref(cap)), "max_size")
            out_capacity = int(cap.value)
        out = self._buf("_out", out_capacity)
        stream = _stream_ptr(self.device)
        nv = int(d_val.numel())
        if events is not None:
            events[0].record()
        self.analyze(x, p, g, d_val, ws, stream)
        if allreduce is not None:
            off = lib.pmz_ws_coverage(_ptr(ws), ctypes.byref(p), ctypes.byref(g)) - ws.data_ptr()
            allreduce(ws[off: off + 18 * 8].view(torch.int64))
        if events is not None:
            events[1].record()
        check(lib.pmz_compress_codes(_ptr(x), ctypes.byref(g), ctypes.byref(p), _ptr(d_val), nv, _ptr(ws),
                                     ws.numel(), stream), "compress_codes")
        if allreduce is not None:
            off = lib.pmz_ws_histogram(_ptr(ws), ctypes.byref(p), ctypes.byref(g)) - ws.data_ptr()
            allreduce(ws[off: off + (65536 + 1) * 8].view(torch.int64))
        if events is not None:
            events[2].record()
        check(lib.pmz_compress_encode(_ptr(x), ctypes.byref(g), ctypes.byref(p), _ptr(ws), ws.numel(), stream),
              "compress_encode")
        if events is not None:
            events[3].record()
        res = N.Result()
        s = self._write(p, g, write_header, out, block_offsets, ws, stream, res)
        check(s, "compress_finish")
        if events is not None:
            events[4].record()
        n = int(res.header_bytes + res.record_bytes)
        info = CompressInfo(n, int(res.header_bytes), int(res.nblocks), int(res.ntrivial), int(res.nbal),
                            int(res.nrepair), int(res.ncodes), int(res.m), int(res.max_code_len),
                            list(res.coverage), tuple(x.shape), None, int(res.launches))
        return out[:n], info

    def compress_staged_async(self, x: torch.Tensor, cfg: CompressConfig, *, block_row0: int, global_rows: int,
                              d_val: torch.Tensor, allreduce=None, ws: torch.Tensor | None = None,
                              out: torch.Tensor | None = None, block_offsets: torch.Tensor | None = None):
        """compress_staged without a host synchronisation: the stages and the
        two histogram all-reduces are only enqueued on the current stream
        (NCCL collectives are stream-ordered), so several shards' fields can
        be in flight; ``ws``/``out`` are the caller's per-slot buffers.  Read
        the outcome with ``staged_result``."""
        (rows, cols), S = grid_view_shape(tuple(x.shape))
        p = make_params(cfg, S)
        g = N.Geom(rows, cols, block_row0, global_rows)
        lib = self.lib
        stream = _stream_ptr(self.device)
        nv = int(d_val.numel())
        self.analyze(x, p, g, d_val, ws, stream)  # (one host synchronisation: the numpy log2 fixups)
        if allreduce is not None:
            off = lib.pmz_ws_coverage(_ptr(ws), ctypes.byref(p), ctypes.byref(g)) - ws.data_ptr()
            allreduce(ws[off: off + 18 * 8].view(torch.int64))
        check(lib.pmz_compress_codes(_ptr(x), ctypes.byref(g), ctypes.byref(p), _ptr(d_val), nv, _ptr(ws),
                                     ws.numel(), stream), "compress_codes")
        if allreduce is not None:
            off = lib.pmz_ws_histogram(_ptr(ws), ctypes.byref(p), ctypes.byref(g)) - ws.data_ptr()
            allreduce(ws[off: off + (65536 + 1) * 8].view(torch.int64))
        check(lib.pmz_compress_finish_async(_ptr(x), ctypes.byref(g), ctypes.byref(p), 1, _ptr(out), out.numel(),
                                            _ptr(block_offsets), _ptr(ws), ws.numel(), stream), "compress_finish")
        return p, g

    def staged_result(self, p, g, ws: torch.Tensor, out: torch.Tensor) -> CompressInfo:
        """Synchronise the current stream and decode the status of a field
        enqueued by ``compress_staged_async``."""
        res = N.Result()
        check(self.lib.pmz_compress_result(ctypes.byref(g), ctypes.byref(p), 1, _ptr(ws), ws.numel(),
                                           _stream_ptr(self.device), ctypes.byref(res)), "compress")
        return CompressInfo(int(res.header_bytes + res.record_bytes), int(res.header_bytes), int(res.nblocks),
                            int(res.ntrivial), int(res.nbal), int(res.nrepair), int(res.ncodes), int(res.m),
                            int(res.max_code_len), list(res.coverage), (int(g.rows), int(g.cols)), None,
                            int(res.launches))

    # ---- decompression ------------------------------------------------
    @staticmethod
    def parse_header(buf: np.ndarray) -> N.Header:
        lib = N.load()
        h = N.Header()
        check(lib.pmz_parse_header(buf.ctypes.data_as(ctypes.c_void_p), buf.size, ctypes.byref(h)), "read_container")
        return h

    @staticmethod
    def index_blocks(buf: np.ndarray, h: N.Header) -> np.ndarray:
        lib = N.load()
        offs = np.zeros(int(h.nblocks) + 1, np.uint64)
        check(lib.pmz_index_blocks(buf.ctypes.data_as(ctypes.c_void_p), buf.size, ctypes.byref(h),
                                   offs.ctypes.data_as(ctypes.c_void_p)), "read_container")
        return offs

    # stage names of the ``events`` of compress_staged / decompress_device
    stage_names_compress = ("analyze (block stats, numpy fixups, select_m coverage)",
                            "codes (select_m, validation codes / latency path: verify_and_repair)",
                            "encode (codebook; throughput path: k_c_main = forward map + compress_block + "
                            "verify_and_repair of every block)",
                            "write (record sizes/offsets, header, block records)")
    stage_names_decompress = ("prepare (block records, parameters, decode tables)",
                              "run (decode, decompress_block, inverse map)")
    last_decompress_launches = 0

    def decompress_device(self, d_buf: torch.Tensor, h: N.Header, d_offsets: torch.Tensor,
                          out: torch.Tensor | None = None, events=None) -> torch.Tensor:
        """decompress_block of every block + inverse map into a float32 CUDA
        grid.  ``events`` (3 CUDA events) time the prepare and run stages on
        the launching stream."""
        lib = self.lib
        wsz = ctypes.c_uint64(0)
        check(lib.pmz_decompress_workspace_size(ctypes.byref(h), ctypes.byref(wsz)), "workspace")
        ws = self._buf("_dws", wsz.value)
        if out is None:
            out = torch.empty((int(h.rows), int(h.cols)), dtype=torch.float32, device=self.device)
        stream = _stream_ptr(self.device)
        b_a = host_b_a(h.b_r)
        if events is not None:
            events[0].record()
        check(lib.pmz_decompress_prepare(_ptr(d_buf), d_buf.numel(), ctypes.byref(h), b_a, _ptr(d_offsets), _ptr(ws),
                                         ws.numel(), stream), "decompress")
        check(min(self.np_fix_decompress(h, ws, stream), 0), "np_fixups")
        if events is not None:
            events[1].record()
        check(lib.pmz_decompress_run(_ptr(d_buf), d_buf.numel(), ctypes.byref(h), b_a, _ptr(d_offsets), _ptr(out),
                                     _ptr(ws), ws.numel(), stream), "decompress")
        if events is not None:
            events[2].record()
        res = N.Result()
        check(lib.pmz_decompress_status(ctypes.byref(h), _ptr(ws), ws.numel(), stream, ctypes.byref(res)),
              "decompress")
        self.last_decompress_launches = int(res.launches)
        return out


_codecs: dict = {}


class GraphedCompressor:
    """The whole single-GPU compress pipeline of one geometry captured into two
    CUDA graphs (block stats; then transform + codes + finish, ~16 kernels)
    around the host's numpy log2 fixups, replayed per call; the outcome is read with pmz_compress_result (one small
    device->host copy).  Buffers are fixed at construction: the input is
    ``x`` (a float32 CUDA tensor the caller keeps alive and refills), or, with
    ``host_input`` (a pinned float32 CPU tensor), a device copy that the graph
    itself refills from it (host->device copy inside the graph).  ``run``
    returns (container bytes as a CUDA uint8 view, CompressInfo)."""

    def __init__(self, codec: Codec, cfg: CompressConfig, x: torch.Tensor | None = None,
                 host_input: torch.Tensor | None = None, block_offsets: torch.Tensor | None = None):
        if (x is None) == (host_input is None):
            raise ConfigError("GraphedCompressor needs exactly one of x (device) or host_input (pinned host)")
        self.codec, self.cfg = codec, cfg
        if host_input is not None:
            if host_input.dtype != torch.float32 or host_input.is_cuda:
                raise ConfigError("host_input must be a float32 CPU tensor (pinned for asynchronous copies)")
            self.host = host_input
            self.x = torch.empty(host_input.shape, dtype=torch.float32, device=codec.device)
        else:
            if x.dtype != torch.float32 or not x.is_cuda or not x.is_contiguous():
                raise ConfigError("x must be a contiguous float32 CUDA tensor")
            self.host, self.x = None, x
        self.p, self.g, self.nb, self.val = codec.plan(self.x.shape, cfg)
        self.d_val = torch.as_tensor(self.val, dtype=torch.int64, device=codec.device)
        lib = codec.lib
        wsz, cap = ctypes.c_uint64(0), ctypes.c_uint64(0)
        check(lib.pmz_workspace_size(ctypes.byref(self.p), ctypes.byref(self.g), ctypes.byref(wsz)), "workspace_size")
        check(lib.pmz_max_container_size(ctypes.byref(self.p), ctypes.byref(self.g), ctypes.byref(cap)), "max_size")
        self.ws = torch.empty(max(int(wsz.value), 1), dtype=torch.uint8, device=codec.device)
        self.out = torch.empty(max(int(cap.value), 1), dtype=torch.uint8, device=codec.device)
        self.block_offsets = block_offsets
        # eager run: sets kernel attributes, validates the configuration
        self._enqueue_stats()
        self._fix()
        self._enqueue_rest()
        self._result()
        torch.cuda.synchronize(codec.device)
        self.graph_stats = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph_stats):
            self._enqueue_stats()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._enqueue_rest()

    def _enqueue_stats(self):
        if self.host is not None:
            self.x.copy_(self.host, non_blocking=True)
        check(self.codec.lib.pmz_compress_stats(_ptr(self.x), ctypes.byref(self.g), ctypes.byref(self.p),
                                                _ptr(self.ws), self.ws.numel(), _stream_ptr(self.codec.device)),
              "compress_stats")

    def _fix(self):
        # the only host step: np.log2 of the listed blocks' general doubles (D22)
        check(min(self.codec.np_fix_compress(self.p, self.g, self.ws, _stream_ptr(self.codec.device)), 0), "np_fixups")

    def _enqueue_rest(self):
        lib = self.codec.lib
        stream = _stream_ptr(self.codec.device)
        nv = int(self.d_val.numel())
        check(lib.pmz_compress_transform(_ptr(self.x), ctypes.byref(self.g), ctypes.byref(self.p), _ptr(self.d_val),
                                         nv, _ptr(self.ws), self.ws.numel(), stream), "compress_transform")
        check(lib.pmz_compress_codes(_ptr(self.x), ctypes.byref(self.g), ctypes.byref(self.p), _ptr(self.d_val), nv,
                                     _ptr(self.ws), self.ws.numel(), stream), "compress_codes")
        check(lib.pmz_compress_finish_async(_ptr(self.x), ctypes.byref(self.g), ctypes.byref(self.p), 1,
                                            _ptr(self.out),
                                            self.out.numel(), _ptr(self.block_offsets), _ptr(self.ws),
                                            self.ws.numel(), stream), "compress_finish")

    def _result(self):
        res = N.Result()
        check(self.codec.lib.pmz_compress_result(ctypes.byref(self.g), ctypes.byref(self.p), 1, _ptr(self.ws),
                                                 self.ws.numel(), _stream_ptr(self.codec.device), ctypes.byref(res)),
              "compress")
        n = int(res.header_bytes + res.record_bytes)
        info = CompressInfo(n, int(res.header_bytes), int(res.nblocks), int(res.ntrivial), int(res.nbal),
                            int(res.nrepair), int(res.ncodes), int(res.m), int(res.max_code_len),
                            list(res.coverage), tuple(self.x.shape), self.val, int(res.launches))
        return self.out[:n], info

    def launch(self):
        """Replay the captured pipeline on the current stream: the stats graph,
        the host's numpy log2 fixups (one synchronisation), then the rest
        (asynchronous)."""
        self.graph_stats.replay()
        self._fix()
        self.graph.replay()

    def result(self):
        """Synchronise and return (container CUDA view, CompressInfo) of the last launch."""
        return self._result()

    def run(self):
        self.launch()
        return self.result()


class PipelinedCompressor:
    """Streaming compression of a sequence of same-shaped fields with several
    in flight: ``depth`` slots, each with its own CUDA stream, device input,
    workspace, output and captured pipeline (GraphedCompressor).  ``submit``
    enqueues the host->device copy of the field (from pinned host memory) and
    the graph replay on the next slot's stream; ``collect`` returns the oldest
    result: the status read-back, then a device->host copy of exactly the
    container bytes into pinned memory.  While one slot's result is read, the
    other slots' copies and kernels proceed, so the PCIe transfers (full
    duplex) overlap the compute of neighbouring fields."""

    def __init__(self, codec: Codec, cfg: CompressConfig, shape, depth: int = 3):
        if depth < 1:
            raise ConfigError("depth must be >= 1")
        self.codec, self.cfg, self.depth = codec, cfg, depth
        self.slots = []
        for _ in range(depth):
            stream = torch.cuda.Stream(codec.device)
            with torch.cuda.stream(stream):
                x = torch.empty(tuple(shape), dtype=torch.float32, device=codec.device)
                x.zero_()
                gc = GraphedCompressor(codec, cfg, x=x)
                host_out = torch.empty(max(int(gc.out.numel()), 1), dtype=torch.uint8, pin_memory=True)
            self.slots.append({"stream": stream, "gc": gc, "x": x, "host_out": host_out, "busy": False,
                               "done": torch.cuda.Event()})
        self._next = 0
        self._queue = []  # slot indices in submission order

    def submit(self, host_field: torch.Tensor):
        """Enqueue one field (a float32 CPU tensor, pinned for an asynchronous
        copy).  Blocks only when every slot is in flight (collect first)."""
        if len(self._queue) == self.depth:
            raise ConfigError("all slots in flight: collect() before submitting more")
        i = self._next
        self._next = (i + 1) % self.depth
        sl = self.slots[i]
        with torch.cuda.stream(sl["stream"]):
            # the slot's previous container copy-out must have landed before
            # its graph runs again (collect(block=False) leaves it in flight)
            sl["stream"].wait_event(sl["done"])
            sl["x"].copy_(host_field, non_blocking=True)
            sl["gc"].launch()
        self._queue.append(i)
        return i

    def collect(self, block: bool = True):
        """(container bytes as a pinned uint8 CPU view, CompressInfo) of the
        oldest submitted field.  With ``block=False`` the device->host copy of
        the container is only enqueued: submit the next field right away (its
        host->device copy then overlaps this copy-out on the full-duplex link)
        and call ``wait()`` before reading the bytes."""
        if not self._queue:
            raise ConfigError("nothing submitted")
        i = self._queue.pop(0)
        sl = self.slots[i]
        with torch.cuda.stream(sl["stream"]):
            buf, info = sl["gc"].result()      # synchronises this slot's stream (status read-back)
            sl["host_out"][: info.nbytes].copy_(buf, non_blocking=True)
            sl["done"].record(sl["stream"])
        self._last = sl["done"]
        if block:
            sl["done"].synchronize()
        return sl["host_out"][: info.nbytes], info

    def wait(self):
        """Wait for the copy-out of the last collected field."""
        if getattr(self, "_last", None) is not None:
            self._last.synchronize()


class PipelinedDecompressor:
    """Streaming decompression of a sequence of containers of one geometry
    with several in flight (the mirror of PipelinedCompressor): ``depth``
    slots, each with its own CUDA stream, device container buffer, block
    index, workspace and output.  ``submit`` enqueues the host->device copy
    of the container (pinned host bytes), the decode kernels
    (pmz_decompress_prepare, the numpy log2 fixups, pmz_decompress_run) and the device->host copy of the float32 grid
    into pinned memory; ``collect`` synchronises the oldest slot, maps its
    device status (pmz_decompress_result) and returns the grid."""

    def __init__(self, codec: Codec, container: bytes | np.ndarray, depth: int = 3):
        if depth < 1:
            raise ConfigError("depth must be >= 1")
        buf = np.frombuffer(container, dtype=np.uint8) if isinstance(container, (bytes, bytearray)) else container
        self.codec, self.depth = codec, depth
        self.h = Codec.parse_header(buf)
        lib = codec.lib
        wsz = ctypes.c_uint64(0)
        check(lib.pmz_decompress_workspace_size(ctypes.byref(self.h), ctypes.byref(wsz)), "workspace")
        self.shape = (int(self.h.rows), int(self.h.cols))
        self.cap = int(buf.size) + 64
        self.slots = []
        for _ in range(depth):
            stream = torch.cuda.Stream(codec.device)
            self.slots.append({
                "stream": stream,
                "buf": torch.empty(self.cap, dtype=torch.uint8, device=codec.device),
                "offs": torch.empty(int(self.h.nblocks) + 1, dtype=torch.int64, device=codec.device),
                "ws": torch.empty(max(int(wsz.value), 1), dtype=torch.uint8, device=codec.device),
                "h_offs": torch.empty(int(self.h.nblocks) + 1, dtype=torch.int64, pin_memory=True),
                "done": torch.cuda.Event(),
                "out": torch.empty(self.shape, dtype=torch.float32, device=codec.device),
                "host_out": torch.empty(self.shape, dtype=torch.float32, pin_memory=True),
                "n": 0})
        self._next = 0
        self._queue = []

    def submit(self, host_container: torch.Tensor, block_offsets: np.ndarray | None = None):
        """Enqueue one container: a pinned uint8 CPU tensor of the same
        geometry; ``block_offsets`` (pmz_index_blocks) is computed when absent."""
        if len(self._queue) == self.depth:
            raise ConfigError("all slots in flight: collect() before submitting more")
        n = int(host_container.numel())
        h = Codec.parse_header(host_container.numpy())  # m / codebook / header size vary per container
        if (h.rows, h.cols, h.block_rows, h.block_cols, h.partition_rows) != \
                (self.h.rows, self.h.cols, self.h.block_rows, self.h.block_cols, self.h.partition_rows):
            raise ConfigError("PipelinedDecompressor: container of another geometry")
        if block_offsets is None:
            block_offsets = Codec.index_blocks(host_container.numpy(), h)
        i = self._next
        self._next = (i + 1) % self.depth
        sl = self.slots[i]
        lib = self.codec.lib
        if n > sl["buf"].numel():  # the slot is idle (collected): grow its container buffer
            sl["buf"] = torch.empty(n + (n >> 3), dtype=torch.uint8, device=self.codec.device)
        with torch.cuda.stream(sl["stream"]):
            sl["buf"][:n].copy_(host_container, non_blocking=True)
            sl["h_offs"].copy_(torch.from_numpy(np.asarray(block_offsets).view(np.int64)))  # slot is idle: safe
            sl["offs"].copy_(sl["h_offs"], non_blocking=True)
            sl["h"] = h
            stream = ctypes.c_void_p(sl["stream"].cuda_stream)
            check(lib.pmz_decompress_prepare(_ptr(sl["buf"]), n, ctypes.byref(h), host_b_a(h.b_r), _ptr(sl["offs"]),
                                             _ptr(sl["ws"]), sl["ws"].numel(), stream), "decompress")
            check(min(self.codec.np_fix_decompress(h, sl["ws"], stream), 0), "np_fixups")
            check(lib.pmz_decompress_run(_ptr(sl["buf"]), n, ctypes.byref(h), host_b_a(h.b_r), _ptr(sl["offs"]),
                                         _ptr(sl["out"]), _ptr(sl["ws"]), sl["ws"].numel(), stream), "decompress")
        sl["n"] = n
        self._queue.append(i)
        return i

    def collect(self, block: bool = True) -> torch.Tensor:
        """The oldest submitted container's float32 grid (a pinned CPU tensor
        view, valid until its slot is reused).  The status is read first
        (synchronising the slot's kernels), then the grid is copied out; with
        ``block=False`` that copy is left in flight -- submit the next
        container right away (its host->device copy overlaps this copy-out)
        and call ``wait()`` before reading the grid."""
        if not self._queue:
            raise ConfigError("nothing submitted")
        i = self._queue.pop(0)
        sl = self.slots[i]
        check(self.codec.lib.pmz_decompress_result(ctypes.byref(sl["h"]), _ptr(sl["ws"]), sl["ws"].numel(),
                                                   ctypes.c_void_p(sl["stream"].cuda_stream)), "decompress")
        with torch.cuda.stream(sl["stream"]):
            sl["host_out"].copy_(sl["out"], non_blocking=True)
            sl["done"].record(sl["stream"])
        self._last = sl["done"]
        if block:
            sl["done"].synchronize()
        return sl["host_out"]

    def wait(self):
        """Wait for the copy-out of the last collected container."""
        if getattr(self, "_last", None) is not None:
            self._last.synchronize()


def _codec(device=None) -> Codec:
    dev = _require_cuda(device)
    key = str(dev)
    if key not in _codecs:
        _codecs[key] = Codec(dev)
    return _codecs[key]


def compress(data, rel_error: float = 1e-2, block_size=(256, 256), partition_rows: int = 32,
             model: PerceptronModel | None = None, repair_factor: float = REPAIR_FACTOR_SPEC,
             coverage_target: float = COVERAGE_TARGET, sample_rate: float = SAMPLE_RATE, seed: int = 0,
             m: int = 0, device=None, return_info: bool = False, train: bool = False, grid=None):
    """cmd_compress minus ingest: array in, container bytes
    out.  ``train=True`` (or a ``grid`` of HyperConfigs) runs the inline
    training sweep first (training.py) and compresses with the
    selected model; the default is ``model`` or init_model (BASELINE runs)."""
    cfg = CompressConfig(rel_error, int(block_size[0]), int(block_size[1]), partition_rows, repair_factor,
                         coverage_target, sample_rate, seed, m, model)
    codec = _codec(device)
    if isinstance(data, torch.Tensor):
        x = data.to(device=codec.device, dtype=torch.float32)
    else:
        a = np.ascontiguousarray(np.asarray(data), dtype=np.float32)
        x = torch.from_numpy(a).to(codec.device)
    if train or grid is not None:
        from dataclasses import replace
        from . import training
        cfg = replace(cfg, model=training.train(codec, x, cfg, grid).model)
    buf, info = codec.compress_device(x, cfg)
    host = buf.cpu().numpy().tobytes()
    return (host, info) if return_info else host


def decompress(container: bytes, device=None, shape=None) -> np.ndarray:
    """cmd_decompress: container bytes in, float32 array out."""
    codec = _codec(device)
    buf = np.frombuffer(container, dtype=np.uint8)
    h = codec.parse_header(buf)
    offs = codec.index_blocks(buf, h)
    d_buf = torch.from_numpy(buf.copy()).to(codec.device)
    d_off = torch.from_numpy(offs.view(np.int64)).to(codec.device)
    out = codec.decompress_device(d_buf, h, d_off)
    res = out.cpu().numpy()
    if shape is not None:
        return res.reshape(shape)
    if h.rows == 1 and h.S == 1:
        return res.reshape(-1)
    return res


def code_mismatches(a: torch.Tensor, b: torch.Tensor) -> dict:
    """Compare two code dumps of the same field (CompressConfig.code_dump,
    both pre-filled with the same value so the padding agrees): positions whose
    final code differs, and positions that are a balance point (code 0) in
    exactly one of them -- the north star's perceptron-rounding mismatch
    counters for the FP32 perf mode against the FP64 path."""
    valid = (a != 0xFFFF) & (a != 0xFFFE)
    diff = (a != b) & valid
    bal = ((a == 0) != (b == 0)) & valid
    return {"codes": int(valid.sum()), "code_mismatches": int(diff.sum()), "balance_mismatches": int(bal.sum())}
