"""Check: the sharded compress stages with their NCCL all-reduces captured in
one CUDA graph (one rank here; torchrun --nproc-per-node 1).  Prints the
replay time per field and whether replays reproduce the eager container."""
import ctypes
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2309_09778_b200 as P  # noqa: E402
from paper_2309_09778_b200 import _native as N, synthetic  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
x = synthetic.generate("C2").to(dev)
cfg = P.CompressConfig(rel_error=1e-2, repair_factor=1.0)
codec = P.Codec(dev)
val = torch.as_tensor(P.pipeline.validation_blocks(8 * 15, cfg.sample_rate, cfg.seed), dtype=torch.int64, device=dev)
lib = codec.lib
p0 = P.pipeline.make_params(cfg, 3)
g0 = N.Geom(x.shape[0], x.shape[1], 0, x.shape[0])
wsz, cap = ctypes.c_uint64(0), ctypes.c_uint64(0)
lib.pmz_workspace_size(ctypes.byref(p0), ctypes.byref(g0), ctypes.byref(wsz))
lib.pmz_max_container_size(ctypes.byref(p0), ctypes.byref(g0), ctypes.byref(cap))
ws = torch.empty(int(wsz.value), dtype=torch.uint8, device=dev)
out = torch.empty(int(cap.value), dtype=torch.uint8, device=dev)


def ar(t):
    dist.all_reduce(t)


s = torch.cuda.Stream(dev)
with torch.cuda.stream(s):
    pg = codec.compress_staged_async(x, cfg, block_row0=0, global_rows=x.shape[0], d_val=val, allreduce=ar, ws=ws,
                                     out=out)
    info = codec.staged_result(*pg, ws, out)
ref = out[: info.nbytes].clone()
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=s):
    codec.compress_staged_async(x, cfg, block_row0=0, global_rows=x.shape[0], d_val=val, allreduce=ar, ws=ws, out=out)
torch.cuda.synchronize()
for _ in range(3):
    graph.replay()
torch.cuda.synchronize()
with torch.cuda.stream(s):
    info2 = codec.staged_result(*pg, ws, out)
print("graph replay container identical:", info2.nbytes == info.nbytes and torch.equal(out[: info.nbytes], ref))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    graph.replay()
e1.record()
torch.cuda.synchronize()
print(f"replay {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per field")
dist.destroy_process_group()
