"""Compress/decompress throughput of the GraphedCompressor on a BASELINE
config at full size (device-resident input, CUDA events).
usage: python tools/scale_check.py C3 [eps] [n_compress] [n_decompress]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2309_09778_b200 as P  # noqa: E402
from paper_2309_09778_b200 import synthetic  # noqa: E402

name = sys.argv[1]
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-2
NC = int(sys.argv[3]) if len(sys.argv) > 3 else 6
ND = int(sys.argv[4]) if len(sys.argv) > 4 else 4
t0 = time.time()
x = synthetic.generate(name, device="cuda").contiguous()
torch.cuda.synchronize()
print(f"{name}: shape {tuple(x.shape)} ({x.numel() * 4 / 2**20:.0f} MiB) generated in {time.time() - t0:.1f}s")
codec = P.Codec("cuda:0")
cfg = P.CompressConfig(rel_error=eps, repair_factor=1.0)
gc = P.GraphedCompressor(codec, cfg, x=x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ms = []
for i in range(NC):
    flush.fill_(i)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    gc.launch()
    b.record()
    buf, info = gc.result()
    ms.append(a.elapsed_time(b))
c = sorted(ms[1:] or ms)[len(ms[1:] or ms) // 2]
print(f"compress: {c:.3f} ms  {x.numel() * 4 / c / 1e6:.1f} GB/s  CR {info.nbytes / (x.numel() * 4):.4f}  m {info.m}")
h = P.Codec.parse_header(buf.cpu().numpy())
offs = torch.from_numpy(P.Codec.index_blocks(buf.cpu().numpy(), h).view("int64")).cuda()
dms = []
for i in range(ND):
    flush.fill_(i)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    y = codec.decompress_device(buf, h, offs)
    b.record()
    torch.cuda.synchronize()
    dms.append(a.elapsed_time(b))
d = sorted(dms[1:] or dms)[len(dms[1:] or dms) // 2]
print(f"decompress: {d:.3f} ms  {x.numel() * 4 / d / 1e6:.1f} GB/s")
