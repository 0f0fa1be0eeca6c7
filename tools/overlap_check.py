"""Can the validation passes (coverage, histogram) run beside k_stats?  Times
stats(field B) on one stream while transform + codes(field A) run on another,
against the two run back to back."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2309_09778_b200 as P  # noqa: E402
from paper_2309_09778_b200 import _native as N  # noqa: E402
from paper_2309_09778_b200.pipeline import _ptr, make_params  # noqa: E402

dev = torch.device("cuda", 0)
x = bench.field_2d("C5", dev)
cfg = P.CompressConfig(rel_error=1e-2, repair_factor=1.0)
codec = P.Codec(dev)
lib = codec.lib
p, g, nb, val = codec.plan(x.shape, cfg)
d_val = torch.as_tensor(val, dtype=torch.int64, device=dev)
wsz = ctypes.c_uint64(0)
lib.pmz_workspace_size(ctypes.byref(p), ctypes.byref(g), ctypes.byref(wsz))
wsA = torch.empty(wsz.value, dtype=torch.uint8, device=dev)
wsB = torch.empty(wsz.value, dtype=torch.uint8, device=dev)
sA, sB = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
pa, pb = ctypes.c_void_p(sA.cuda_stream), ctypes.c_void_p(sB.cuda_stream)


def stats(ws, st):
    assert lib.pmz_compress_stats(_ptr(x), ctypes.byref(g), ctypes.byref(p), _ptr(ws), ws.numel(), st) == 0


def valpass(ws, st):
    assert lib.pmz_compress_transform(_ptr(x), ctypes.byref(g), ctypes.byref(p), _ptr(d_val), d_val.numel(), _ptr(ws),
                                      ws.numel(), st) == 0
    assert lib.pmz_compress_codes(_ptr(x), ctypes.byref(g), ctypes.byref(p), _ptr(d_val), d_val.numel(), _ptr(ws),
                                  ws.numel(), st) == 0


stats(wsA, pa)
codec.np_fix_compress(p, g, wsA, pa)
torch.cuda.synchronize()
for mode in ("serial", "overlap", "serial", "overlap"):
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sA)
        sB.wait_stream(sA)
        if mode == "serial":
            stats(wsB, pa)
            valpass(wsA, pa)
        else:
            stats(wsB, pb)
            valpass(wsA, pa)
            sA.wait_stream(sB)
        e1.record(sA)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(mode, " ".join(f"{t:.3f}" for t in ts), flush=True)
