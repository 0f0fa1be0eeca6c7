"""Serial vs pipelined end-to-end compress throughput on C2 (pinned host in,
pinned host out, every step)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2309_09778_b200 as P  # noqa: E402
from paper_2309_09778_b200 import synthetic  # noqa: E402

x = synthetic.generate("C2")
h_in = x.pin_memory()
codec = P.Codec("cuda:0")
cfg = P.CompressConfig(rel_error=1e-2, repair_factor=1.0)
K = 40
# serial (graph with H2D inside, one at a time)
gce = P.GraphedCompressor(codec, cfg, host_input=h_in)
h_out = torch.empty(gce.out.numel(), dtype=torch.uint8, pin_memory=True)
for _ in range(3):
    b, i = gce.run()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(K):
    gce.launch()
    b, i = gce.result()
    h_out[: i.nbytes].copy_(b, non_blocking=True)
    torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / K
print(f"serial   : {dt * 1e3:.3f} ms/field  {x.numel() * 4 / dt / 1e9:.1f} GB/s")
for depth in (2, 3):
    pc = P.PipelinedCompressor(codec, cfg, x.shape, depth=depth)
    for _ in range(depth):
        pc.submit(h_in)
    for _ in range(depth):
        pc.collect()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n_sub = 0
    for _ in range(depth):
        pc.submit(h_in)
        n_sub += 1
    ref = None
    for k in range(K):
        buf, info = pc.collect()
        if ref is None:
            ref = bytes(buf.numpy())
        if n_sub < K:
            pc.submit(h_in)
            n_sub += 1
    dt = (time.perf_counter() - t0) / K
    assert bytes(buf.numpy()) == ref
    print(f"depth {depth}  : {dt * 1e3:.3f} ms/field  {x.numel() * 4 / dt / 1e9:.1f} GB/s")
