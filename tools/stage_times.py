"""Warm per-stage compress timing (CUDA events on the launching stream) on the
bench workload: analyze (stats + forward/quantize), codes (select_m + verify +
validation histogram), finish (codebook .. record writer)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_09778_b200 import synthetic  # noqa: E402
from paper_2309_09778_b200.pipeline import Codec, CompressConfig  # noqa: E402

x = synthetic.generate("C2", shape=(1800, 3600)).cuda()
codec = Codec()
cfg = CompressConfig(rel_error=1e-2, repair_factor=1.0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
acc = [0.0, 0.0, 0.0]
n = 20
for it in range(n + 3):
    flush.fill_(it & 0xff)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    codec.compress_staged(x, cfg, events=ev)
    torch.cuda.synchronize()
    if it >= 3:
        for i in range(3):
            acc[i] += ev[i].elapsed_time(ev[i + 1]) * 1e3 / n
print("analyze %.1f us  codes %.1f us  finish %.1f us  total %.1f us" % (acc[0], acc[1], acc[2], sum(acc)))
