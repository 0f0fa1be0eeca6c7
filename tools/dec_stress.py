"""Repeated compress -> decompress of one BASELINE config; counts decode
failures and mismatches between runs (races show up as intermittent ones).
usage: python tools/dec_stress.py C2 [iters]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2309_09778_b200 as P  # noqa: E402
from paper_2309_09778_b200 import synthetic  # noqa: E402

name = sys.argv[1]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
x = synthetic.generate(name).cuda().contiguous()
codec = P.Codec("cuda:0")
cfg = P.CompressConfig(rel_error=1e-2, repair_factor=1.0)
gc = P.GraphedCompressor(codec, cfg, x=x)
gc.launch()
buf, info = gc.result()
h = P.Codec.parse_header(buf.cpu().numpy())
offs = torch.from_numpy(P.Codec.index_blocks(buf.cpu().numpy(), h).view("int64")).cuda()
ref = None
fail = mism = 0
msgs = {}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
mode = sys.argv[3] if len(sys.argv) > 3 else "plain"  # plain | flush | graph (flush + compress replay)
for i in range(iters):
    if mode in ("flush", "graph"):
        flush.fill_(i & 255)
    if mode == "graph":
        gc.launch()
        gc.result()
        flush.fill_((i + 1) & 255)
    try:
        y = codec.decompress_device(buf, h, offs)
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        fail += 1
        msgs[str(e)[:80]] = msgs.get(str(e)[:80], 0) + 1
        continue
    if ref is None:
        ref = y.clone()
    elif not torch.equal(y.view(torch.int32), ref.view(torch.int32)):
        mism += 1
print(f"{name} {mode}: {iters} decodes, {fail} failures, {mism} mismatches {msgs}")
