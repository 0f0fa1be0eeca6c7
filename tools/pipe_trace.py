"""Timeline of one HostPipeline.decompress (or compress) call: copies and
kernels per stream from torch.profiler (CUPTI), to see what overlaps."""
import argparse
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2309_09778_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--slab-mb", type=int, default=128)
ap.add_argument("--compress", action="store_true")
ap.add_argument("--from-ms", type=float, default=60.0)
ap.add_argument("--to-ms", type=float, default=85.0)
a = ap.parse_args()
dev = torch.device("cuda", 0)
x = bench.field_2d("C5", dev)
cfg = P.CompressConfig(rel_error=1e-2, repair_factor=1.0)
codec = P.Codec(dev)
h_in = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
h_in.copy_(x)
del x
torch.cuda.empty_cache()
pipe = P.HostPipeline(codec, slab_bytes=a.slab_mb << 20)
h_out = torch.empty(int(h_in.numel() * 4 * 0.6), dtype=torch.uint8, pin_memory=True)
h_y = torch.empty(h_in.shape, dtype=torch.float32, pin_memory=True)
n, info = pipe.compress(h_in, cfg, h_out)
pipe.decompress(h_out[:n], h_y)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    if a.compress:
        pipe.compress(h_in, cfg, h_out)
    else:
        pipe.decompress(h_out[:n], h_y)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in ev)
rows = []
for e in ev:
    s, d = (e.time_range.start - t0) / 1e3, (e.time_range.end - e.time_range.start) / 1e3
    if d >= float(os.environ.get("MIN_MS", "0.05")) and a.from_ms <= s <= a.to_ms:
        rows.append((s, d, e.name[:40]))
for s, d, nm in sorted(rows):
    print(f"{s:9.3f} ms  +{d:7.3f}  {nm}")
print("total", (max(e.time_range.end for e in ev) - t0) / 1e3, "ms")
