"""Compress-only stage timing on a BASELINE config (A/B experiments through
env knobs such as PMZ_FUSED); prints ms per stage, mean of --steps runs."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2309_09778_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--fp32", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda", 0)
x = bench.field_2d(a.config, dev)
cfg = P.CompressConfig(rel_error=1e-2, repair_factor=1.0, precision="fp32" if a.fp32 else "fp64")
codec = P.Codec(dev)
for _ in range(3):
    codec.compress_staged(x, cfg, block_row0=0, global_rows=x.shape[0])
st = []
for _ in range(a.steps):
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(codec.stage_names_compress) + 1)]
    codec.compress_staged(x, cfg, block_row0=0, global_rows=x.shape[0], events=ev)
    torch.cuda.synchronize()
    st.append([ev[i].elapsed_time(ev[i + 1]) for i in range(len(ev) - 1)])
s = np.mean(np.array(st), axis=0)
print(os.environ.get("PMZ_FUSED", "-"), "total %.3f" % s.sum(), " ".join("%.3f" % v for v in s), flush=True)
