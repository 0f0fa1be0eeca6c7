"""Multi-process (gloo, world_size 2, CPU) tests of the sharding host logic:
block-row partitioning, the shard-local validation sets, the record-size
all-gather and the container assembly.  The per-shard records are cut from an
oracle container (the checker) by block index, so the test proves that
offsets exchanged between ranks re-assemble the single-process container
byte for byte."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_plan_covers_every_block_once():
    from paper_2309_09778_b200.sharding import plan_shard
    for rows in (1, 255, 256, 257, 1800, 5000):
        for world in (1, 2, 3, 4, 8):
            plans = [plan_shard(rows, 700, 256, 256, world, r) for r in range(world)]
            assert plans[0].row0 == 0 and plans[-1].row1 == rows
            for a, b in zip(plans, plans[1:]):
                assert a.row1 == b.row0 and b.row0 % 256 == 0
            assert sum(p.nblocks for p in plans) == ((rows + 255) // 256) * 3


def test_local_validation_sets_partition_the_global_set():
    from paper_2309_09778_b200.sharding import local_validation_blocks, plan_shard
    from paper_2309_09778_b200.trainer import validation_blocks
    rows, cols = 4000, 900
    glob = np.sort(validation_blocks(((rows + 255) // 256) * 4, 0.1, 7))
    for world in (1, 2, 4):
        got = []
        for r in range(world):
            p = plan_shard(rows, cols, 256, 256, world, r)
            got.extend((local_validation_blocks(p, 0.1, 7) + p.block0).tolist())
        assert sorted(got) == glob.tolist()


def _worker(rank, world, port, path, out_path):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2309_09778_b200.sharding import exchange_record_sizes, make_allreduce, plan_shard, record_offsets
    data = np.load(path)
    buf, boffs, hdr = data["buf"].tobytes(), data["boffs"], int(data["hdr"])
    rows, cols = int(data["rows"]), int(data["cols"])
    plan = plan_shard(rows, cols, 256, 256, world, rank)
    lo, hi = plan.block0, plan.block0 + plan.nblocks
    mine = buf[boffs[lo]:boffs[hi]]
    # histograms are summed across shards (stand-in tensors: each rank its own part)
    h = torch.tensor([rank + 1, 10 * (rank + 1)], dtype=torch.int64)
    make_allreduce()(h)
    sizes = exchange_record_sizes(len(mine))
    offs = record_offsets(sizes, hdr)
    with open(f"{out_path}.{rank}", "wb") as f:
        f.write(int(offs[rank]).to_bytes(8, "little") + mine + bytes(h.numpy().astype("<i8").tobytes()))
    dist.destroy_process_group()


def test_gloo_two_ranks_reassemble_container(tmp_path, oracle):
    from paper_2309_09778_b200 import synthetic
    x = synthetic.generate("C2", shape=(700, 600)).numpy()
    buf, info = oracle.compress(x, oracle.OracleConfig(b_r=1e-2))
    from paper_2309_09778_b200.pipeline import Codec
    a = np.frombuffer(buf, np.uint8)
    h = Codec.parse_header(a)
    boffs = Codec.index_blocks(a, h)
    path = str(tmp_path / "c.npz")
    np.savez(path, buf=a, boffs=boffs.astype(np.int64), hdr=h.header_bytes, rows=700, cols=600)
    world, port = 2, _free_port()
    out = str(tmp_path / "out")
    mp.spawn(_worker, args=(world, port, path, out), nprocs=world, join=True)
    assembled = bytearray(buf[:h.header_bytes])
    for r in range(world):
        d = open(f"{out}.{r}", "rb").read()
        off = int.from_bytes(d[:8], "little")
        assert off == len(assembled)
        recs = d[8:-16]
        assembled += recs
        hist = np.frombuffer(d[-16:], "<i8")
        assert hist.tolist() == [3, 30]  # (1 + 2), (10 + 20): every rank sees the sum
    assert bytes(assembled) == buf
