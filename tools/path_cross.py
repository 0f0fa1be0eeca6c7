"""Latency-path vs throughput-path crossover: compress / decompress ms of
C2-like fields with a growing partition count, both paths (PMZ_PATH)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2309_09778_b200 as P  # noqa: E402
from paper_2309_09778_b200 import synthetic  # noqa: E402

codec = P.Codec("cuda:0")
cfg = P.CompressConfig(rel_error=1e-2, repair_factor=1.0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
shapes = [(8192, 1024), (16384, 1024), (32768, 1024), (65536, 1024), (131072, 1024), (262144, 1024)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]


def med(f, n=5):
    ms = []
    for i in range(n):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return sorted(ms[1:])[len(ms[1:]) // 2]


for shp in shapes:
    x = synthetic.generate("C4" if os.environ.get("GEN") == "C4" else "C2", shape=shp).cuda().contiguous()
    nparts = ((shp[0] + 255) // 256) * ((shp[1] + 255) // 256) * 8
    row = [f"{shp[0]}x{shp[1]} (~{nparts} partitions)"]
    for path in ("latency", "throughput"):
        os.environ["PMZ_PATH"] = path
        buf, info = codec.compress_device(x, cfg)
        buf = buf.clone()
        hb = buf.cpu().numpy()
        h = P.Codec.parse_header(hb)
        offs = torch.from_numpy(P.Codec.index_blocks(hb, h).view("int64")).cuda()
        c = med(lambda: codec.compress_device(x, cfg))
        d = med(lambda: codec.decompress_device(buf, h, offs))
        row.append(f"{path[:3]}: c {c:.3f} d {d:.3f} ms")
    print(" | ".join(row), flush=True)
