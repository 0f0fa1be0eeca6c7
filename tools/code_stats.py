"""Codeword-length statistics of a config's container (decoder table sizing):
the code lengths from the header, weighted by the final codes of the field
(CompressConfig.code_dump)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2309_09778_b200 as P  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C5"
dev = torch.device("cuda", 0)
x = bench.field_2d(cfgname, dev)
codec = P.Codec(dev)
cfg = P.CompressConfig(rel_error=1e-2, repair_factor=1.0)
dump = torch.empty(codec.code_dump_numel(tuple(x.shape), cfg), dtype=torch.int16, device=dev)
cfg.code_dump = dump
buf, info = codec.compress_device(x, cfg)
hb = buf.cpu().numpy()
h = P.Codec.parse_header(hb)
m = int(h.m)
lens = hb[int(h.lens_offset): int(h.lens_offset) + (1 << m)].astype(np.int64)
c = dump.view(torch.int32 if False else torch.int16).to(torch.int32) & 0xFFFF
hist = torch.bincount(c.reshape(-1), minlength=1 << 16).cpu().numpy()[: 1 << m].astype(np.float64)
w = np.bincount(lens, weights=hist, minlength=33)
w /= w.sum()
print("m", m, "maxlen", lens.max(), "symbols", int((lens > 0).sum()))
print("count by len", np.bincount(lens, minlength=33)[1:].tolist())
print("weighted", " ".join(f"{l}:{w[l]:.5f}" for l in range(1, 33) if w[l] > 0))
for lb in (12, 13, 14, 15, 16):
    print(f"P(len>{lb}) = {w[lb + 1:].sum():.6f}")
for lb in (13, 14):
    u = sum(float(np.sum(lens == l)) * 2.0 ** (lb - l) for l in range(lb + 1, 33))
    print(f"prefix units beyond {lb} bits: {u:.1f}")
