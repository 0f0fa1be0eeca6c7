"""Per-kernel decompress (and compress) timing on the bench workload for A/B
experiments: CUPTI kernel durations via torch.profiler, total by CUDA events.

usage: PMZ_LIB_PATH=variant.so python tools/dec_bench.py [--field C2|C4s] [--compress]
Prints one summary block; writes the decompressed output hash so variants can
be compared for bit-identity."""
import argparse
import collections
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2309_09778_b200 import synthetic  # noqa: E402
from paper_2309_09778_b200.pipeline import Codec, CompressConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--field", default="C2")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--compress", action="store_true")
a = ap.parse_args()

shape = {"C1": None, "C2": None, "C3q": (128, 512, 512), "C4": None}[a.field]
name = "C3" if a.field == "C3q" else a.field
x = synthetic.generate(name, shape=shape).cuda()
codec = Codec()
cfg = CompressConfig(rel_error=1e-2, repair_factor=1.0)
buf, info = codec.compress_device(x, cfg)
hb = buf.cpu().numpy()
h = Codec.parse_header(hb)
offs = torch.as_tensor(Codec.index_blocks(hb, h).astype(np.int64)).cuda()
dbuf = buf.clone()
out = torch.empty(tuple(int(v) for v in (h.rows, h.cols)), dtype=torch.float32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def run_dec():
    try:
        codec.decompress_device(dbuf, h, offs, out)
    except Exception:  # ablation builds (tools only) produce wrong parses
        if not os.environ.get("DB_IGNORE_ERR"):
            raise


def run_cmp():
    codec.compress_device(x, cfg)


fn = run_cmp if a.compress else run_dec
for _ in range(3):
    fn()
torch.cuda.synchronize()
tot = 0.0
for i in range(a.iters):
    flush.fill_(i & 0xff)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    tot += e0.elapsed_time(e1)
tot /= a.iters
acc = collections.defaultdict(float)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for i in range(a.iters):
        flush.fill_(i & 0xff)
        fn()
    torch.cuda.synchronize()
seq = collections.defaultdict(list)
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA and "pmz" in ev.name:
        seq[ev.name.split("(")[0][:48]].append(ev.device_time)
for nm, v in seq.items():  # several launches per call: one line per launch index
    k = max(1, len(v) // a.iters)
    for j in range(k):
        acc[nm + (f" #{j}" if k > 1 else "")] = sum(v[j::k]) / a.iters
torch.cuda.synchronize()
dig = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:12] if not a.compress else \
    hashlib.sha1(codec.compress_device(x, cfg)[0].cpu().numpy().tobytes()).hexdigest()[:12]
lib = os.path.basename(os.environ.get("PMZ_LIB_PATH", "default"))
if hasattr(codec.lib, "pmz_d3prof_read") and not a.compress:
    import ctypes
    torch.cuda.synchronize()
    run_dec()
    torch.cuda.synchronize()
    np_ = int(out.numel() // 8192 + 64)
    arr = np.zeros(np_ * 8, np.uint64)
    big = np.zeros(1 << 20, np.uint64)
    codec.lib.pmz_d3prof_read(big.ctypes.data_as(ctypes.c_void_p), ctypes.c_uint64(big.nbytes))
    arr[:] = big[:arr.size]
    A = arr.reshape(-1, 8)
    A = A[A[:, 0] != 0].astype(np.int64)
    t0 = A[:, 0].min()
    ph = np.diff(A[:, :5], axis=1)
    print("d3prof parts", len(A), "start spread (cyc) p50/max", np.percentile(A[:, 0] - t0, 50), (A[:, 0] - t0).max(),
          "end max", (A[:, 4] - t0).max())
    print("   partitions on the word-map path:", int((A[:, 6] == 1).sum()), "of", len(A))
    T = np.stack([A[:, 0], A[:, 1], A[:, 2], A[:, 3], A[:, 5], A[:, 4]], 1)
    ph = np.diff(T, axis=1)
    for i, nm in enumerate(["maps", "chain", "write", "lookback", "gather"]):
        print(f"   {nm:8s} cycles p50 {np.percentile(ph[:, i], 50):9.0f} p90 {np.percentile(ph[:, i], 90):9.0f} max {ph[:, i].max():9.0f}")
if hasattr(codec.lib, "pmz_cbprof_read") and a.compress:
    import ctypes
    cb = np.zeros(8, np.int64)
    codec.lib.pmz_cbprof_read(cb.ctypes.data_as(ctypes.c_void_p))
    print("codebook phase cycles (leaves, sort, merge, depths, codes):", np.diff(cb[:6]).tolist())
mode = "compress" if a.compress else "decompress"
print(f"== {lib} {a.field} {mode}: {tot * 1e3:.1f} us/call  {x.numel() * 4 / tot / 1e6:.1f} GB/s  "
      f"CR={info.nbytes / (x.numel() * 4):.4f}  hash={dig}")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"   {v:9.1f} us  {k}")
