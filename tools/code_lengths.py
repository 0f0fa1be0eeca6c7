"""Distribution of codeword lengths actually emitted for a config (validation
histogram x the container's code lengths): how often the decoder leaves its
first-level table.  usage: python tools/code_lengths.py C5"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2309_09778_b200 as P  # noqa: E402
from paper_2309_09778_b200 import synthetic  # noqa: E402
from paper_2309_09778_b200.pipeline import grid_view_shape  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
x = synthetic.generate(name, device="cuda")
(r, c), _ = grid_view_shape(tuple(x.shape))
x = x.reshape(r, c)
codec = P.Codec("cuda:0")
cfg = P.CompressConfig(rel_error=1e-2, repair_factor=1.0)
buf, info = codec.compress_staged(x, cfg)
p = P.pipeline.make_params(cfg, 3)
g = P._native.Geom(r, c, 0, r)
off = codec.lib.pmz_ws_histogram(ctypes.c_void_p(codec._ws.data_ptr()), ctypes.byref(p), ctypes.byref(g)) - \
    codec._ws.data_ptr()
hist = codec._ws[off: off + 65537 * 8].view(torch.int64).cpu().numpy()[: 1 << info.m].astype(np.float64)
hb = buf[: info.header_bytes].cpu().numpy()
h = P.Codec.parse_header(hb)
lens = hb[h.lens_offset: h.lens_offset + (1 << info.m)].astype(np.int64)
tot = hist.sum()
print(f"{name}: m={info.m} maxlen={lens.max()} mean bits/code={(hist * lens).sum() / tot:.3f}")
for L in (8, 10, 12, 13, 14, 15, 16, 18, 20):
    print(f"  P(len > {L:2d}) = {hist[lens > L].sum() / tot:.5f}")
