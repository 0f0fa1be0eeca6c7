"""Decompress-only stage timing on a BASELINE config (A/B experiments through
PMZ_LIB_PATH variants): ms per stage, mean of --steps runs, output hash."""
import argparse
import hashlib
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
a = ap.parse_args()
dev = torch.device("cuda", 0)
x = bench.field_2d(a.config, dev)
cfg = P.CompressConfig(rel_error=1e-2, repair_factor=1.0)
codec = P.Codec(dev)
buf, info = codec.compress_device(x, cfg)
hb = buf.cpu().numpy()
h = P.Codec.parse_header(hb)
offs = torch.from_numpy(P.Codec.index_blocks(hb, h).view(np.int64)).to(dev)
dbuf = buf.clone()
y = torch.empty_like(x)
for _ in range(2):
    codec.decompress_device(dbuf, h, offs, out=y)
st = []
for _ in range(a.steps):
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    codec.decompress_device(dbuf, h, offs, out=y, events=ev)
    torch.cuda.synchronize()
    st.append([ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])])
s = np.mean(np.array(st), axis=0)
hsh = hashlib.sha1(y[:: max(1, y.shape[0] // 4096)].cpu().numpy().tobytes()).hexdigest()[:12]
print(os.path.basename(os.environ.get("PMZ_LIB_PATH", "default")), "total %.3f" % s.sum(), " ".join("%.3f" % v for v in s), hsh, flush=True)
