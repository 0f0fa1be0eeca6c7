"""Regenerate tools/micro/data/{c2.f32,c2.pmz} from the bench workload (GPU)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_2309_09778_b200 import synthetic  # noqa: E402
from paper_2309_09778_b200.pipeline import Codec, CompressConfig  # noqa: E402

d = os.path.join(os.path.dirname(__file__), "data")
os.makedirs(d, exist_ok=True)
x = synthetic.generate("C2", shape=(1800, 3600)).cuda()  # host generator, as bench.py
x.cpu().numpy().astype(np.float32).tofile(os.path.join(d, "c2.f32"))
buf, info = Codec().compress_device(x, CompressConfig(rel_error=1e-2, repair_factor=1.0))
buf.cpu().numpy().tofile(os.path.join(d, "c2.pmz"))
print("wrote", info.nbytes, "bytes")
