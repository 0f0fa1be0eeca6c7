"""One FP32-perf-mode compress + decompress of a BASELINE config (ncu target)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2309_09778_b200 as P  # noqa: E402
from paper_2309_09778_b200 import synthetic  # noqa: E402

x = synthetic.generate(sys.argv[1], device="cuda").contiguous()
codec = P.Codec("cuda:0")
buf, info = codec.compress_device(x, P.CompressConfig(rel_error=1e-2, repair_factor=1.0, precision="fp32"))
h = P.Codec.parse_header(buf.cpu().numpy())
offs = torch.from_numpy(P.Codec.index_blocks(buf.cpu().numpy(), h).view("int64")).cuda()
y = codec.decompress_device(buf, h, offs)
torch.cuda.synchronize()
print("ok", info.m, info.nbytes)
