"""Two ranks driving the GPU compress path of their shards (AC6, SPEC.md:621:
identical bitstream for any worker count).  Both processes run on the one
B200 of the test box -- their kernels never wait on each other; the only
exchanges are the two histogram all-reduces and the record-size all-gather,
here over gloo (host memory) instead of NCCL.  The re-assembled container
must equal the single-GPU container and the oracle's, byte for byte, through
both compress paths."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROWS, COLS = 2048, 1536  # 8 x 6 blocks: 5 validation blocks (sample rate 0.1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _field():
    from paper_2309_09778_b200 import synthetic
    return synthetic.generate("C2", shape=(ROWS, COLS)).numpy()


def _worker(rank, world, port, path, out_path):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["PMZ_PATH"] = path
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2309_09778_b200 as P
    from paper_2309_09778_b200.sharding import compress_shard, plan_shard
    x = _field()
    cfg = P.CompressConfig(rel_error=1e-2, repair_factor=1.0)
    plan = plan_shard(ROWS, COLS, cfg.block_rows, cfg.block_cols, world, rank)
    codec = P.Codec("cuda:0")
    xs = torch.from_numpy(np.ascontiguousarray(x[plan.row0:plan.row1])).cuda()
    buf, hdr, start, total, info = compress_shard(codec, xs, cfg, plan)
    mine = buf[:info.nbytes].cpu().numpy().tobytes()
    with open(f"{out_path}.{rank}", "wb") as f:
        f.write(int(start).to_bytes(8, "little") + int(total).to_bytes(8, "little") + mine)
    dist.destroy_process_group()


@pytest.mark.parametrize("path", ["latency", "throughput"])
def test_two_ranks_gpu_container_identical(tmp_path, oracle, path):
    import torch
    import paper_2309_09778_b200 as P
    x = _field()
    ref, _ = oracle.compress(x, oracle.OracleConfig(b_r=1e-2, repair_factor=1.0))
    os.environ["PMZ_PATH"] = path
    try:
        single, _ = P.Codec("cuda:0").compress_device(torch.from_numpy(x).cuda(),
                                                       P.CompressConfig(rel_error=1e-2, repair_factor=1.0))
    finally:
        os.environ.pop("PMZ_PATH", None)
    assert single.cpu().numpy().tobytes() == ref
    world, port = 2, _free_port()
    out = str(tmp_path / "shard")
    mp.spawn(_worker, args=(world, port, path, out), nprocs=world, join=True)
    assembled = bytearray()
    for r in range(world):
        d = open(f"{out}.{r}", "rb").read()
        start, total = int.from_bytes(d[:8], "little"), int.from_bytes(d[8:16], "little")
        assert start == len(assembled) and total == len(ref)
        assembled += d[16:]
    assert bytes(assembled) == ref
