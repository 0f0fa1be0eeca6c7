"""Host-to-host (pinned) compress / decompress of a BASELINE config through
hostpipe.HostPipeline: wall-clock ms per call, GB/s, and the bytes moved."""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2309_09778_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--slab-mb", type=int, default=128)
ap.add_argument("--check", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda", 0)
x = bench.field_2d(a.config, dev)
cfg = P.CompressConfig(rel_error=1e-2, repair_factor=1.0)
codec = P.Codec(dev)
h_in = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
h_in.copy_(x)
ref = None
if a.check:
    buf, info = codec.compress_device(x, cfg)
    ref = buf.cpu()
del x
torch.cuda.empty_cache()
pipe = P.HostPipeline(codec, slab_bytes=a.slab_mb << 20)
h_out = torch.empty(int(h_in.numel() * 4 * 0.6) + (1 << 20), dtype=torch.uint8, pin_memory=True)
h_y = torch.empty(h_in.shape, dtype=torch.float32, pin_memory=True)
nbytes = h_in.numel() * 4
for it in range(a.steps + 1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n, info = pipe.compress(h_in, cfg, h_out)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    pipe.decompress(h_out[:n], h_y)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"slab {a.slab_mb} MiB: compress {1e3 * (t1 - t0):.1f} ms {nbytes / (t1 - t0) / 1e9:.1f} GB/s | "
          f"decompress {1e3 * (t2 - t1):.1f} ms {nbytes / (t2 - t1) / 1e9:.1f} GB/s | n={n} m={info.m}", flush=True)
if ref is not None:
    print("container identical:", bool(torch.equal(h_out[:n], ref)), "launches", info.launches)
