"""Host-to-host slab pipeline (hostpipe.HostPipeline): the container written
slab by slab -- validation blocks uploaded first, their coverage / code
histograms handed to every slab, header from the first slab -- must be the
single-call container byte for byte (so it is the oracle's, which the parity
tests pin), and the slab-wise decode must give the single-call grid bit for
bit.  AC6: the bitstream does not depend on how the field is
cut across workers."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _pin(t):
    p = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    p.copy_(t)
    return p


@pytest.mark.parametrize("shape,slab_rows,eps", [
    ((2048, 1024), 512, 1e-2),     # 4 slabs of 2 block-rows
    ((1800, 3600), 256, 1e-3),     # C2 geometry: ragged last block-row / block-column, 8 slabs
    ((4096, 512), 256, 1e-2),      # 16 slabs of one block-row
])
def test_slab_pipeline_matches_single_call(oracle, shape, slab_rows, eps):
    import paper_2309_09778_b200 as P
    from paper_2309_09778_b200 import synthetic
    x = synthetic.generate("C2", shape=shape).contiguous()
    cfg = P.CompressConfig(rel_error=eps, repair_factor=1.0)
    codec = P.Codec("cuda:0")
    ref, rinfo = codec.compress_device(x.cuda(), cfg)
    ref = ref.cpu().numpy().tobytes()
    pipe = P.HostPipeline(codec, slab_bytes=slab_rows * shape[1] * 4)
    h_out = torch.empty(len(ref) + (1 << 16), dtype=torch.uint8, pin_memory=True)
    n, info = pipe.compress(_pin(x), cfg, h_out)
    got = h_out[:n].numpy().tobytes()
    assert n == len(ref) and got == ref
    assert (info.m, info.nbal, info.nrepair, info.nblocks) == (rinfo.m, rinfo.nbal, rinfo.nrepair, rinfo.nblocks)
    assert pipe.last_h2d_bytes >= x.numel() * 4 and pipe.last_d2h_bytes == n
    # the oracle's container (small enough to run here)
    if x.numel() <= (1 << 22):
        oc, _ = oracle.compress(x.numpy(), oracle.OracleConfig(b_r=eps, repair_factor=1.0))
        assert got == oc
    # slab-wise decode == single-call decode, bit for bit
    y_ref = P.decompress(ref, device="cuda:0")
    y = pipe.decompress(_pin(torch.from_numpy(np.frombuffer(got, np.uint8).copy())))
    assert np.array_equal(y.numpy().view(np.uint32).reshape(y_ref.shape), y_ref.view(np.uint32))


def test_slab_pipeline_fp32_mode_and_small_field():
    import paper_2309_09778_b200 as P
    from paper_2309_09778_b200 import synthetic
    codec = P.Codec("cuda:0")
    # FP32 perceptron mode through the slabs
    x = synthetic.generate("C2", shape=(2048, 768)).contiguous()
    cfg = P.CompressConfig(rel_error=1e-2, repair_factor=1.0, precision="fp32")
    ref, _ = codec.compress_device(x.cuda(), cfg)
    ref = ref.cpu().numpy().tobytes()
    pipe = P.HostPipeline(codec, slab_bytes=512 * 768 * 4)
    h_out = torch.empty(len(ref) + 4096, dtype=torch.uint8, pin_memory=True)
    n, _ = pipe.compress(_pin(x), cfg, h_out)
    assert h_out[:n].numpy().tobytes() == ref
    y = pipe.decompress(_pin(h_out[:n].clone()))
    assert np.array_equal(y.numpy().view(np.uint32), P.decompress(ref, device="cuda:0").view(np.uint32))
    # a field of one slab takes the single-call path
    xs = synthetic.generate("C2", shape=(300, 520)).contiguous()
    cfg = P.CompressConfig(rel_error=1e-2, repair_factor=1.0)
    r2, _ = codec.compress_device(xs.cuda(), cfg)
    h2 = torch.empty(r2.numel() + 4096, dtype=torch.uint8, pin_memory=True)
    n2, _ = P.HostPipeline(codec).compress(_pin(xs), cfg, h2)
    assert h2[:n2].numpy().tobytes() == r2.cpu().numpy().tobytes()
    # too small an output buffer is an error, not a truncated container
    with pytest.raises(P.errors.ConfigError):
        pipe.compress(_pin(x), P.CompressConfig(rel_error=1e-2, repair_factor=1.0),
                      torch.empty(1024, dtype=torch.uint8, pin_memory=True))


# ---- two ranks, each streaming its shard through the slab pipeline (AC6) -----
ROWS, COLS = 2048, 1536


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2309_09778_b200 as P
    from paper_2309_09778_b200 import synthetic
    from paper_2309_09778_b200.sharding import make_allreduce, plan_shard
    x = synthetic.generate("C2", shape=(ROWS, COLS))
    cfg = P.CompressConfig(rel_error=1e-2, repair_factor=1.0)
    plan = plan_shard(ROWS, COLS, cfg.block_rows, cfg.block_cols, world, rank)
    pipe = P.HostPipeline(P.Codec("cuda:0"), slab_bytes=256 * COLS * 4)  # 4 slabs of one block-row per rank
    h_out = torch.empty(ROWS * COLS * 4, dtype=torch.uint8, pin_memory=True)
    n, info = pipe.compress(_pin(x[plan.row0:plan.row1].contiguous()), cfg, h_out, block_row0=plan.block_row0,
                            global_rows=ROWS, allreduce=make_allreduce(None), write_header=(rank == 0))
    with open(f"{out_path}.{rank}", "wb") as f:
        f.write(h_out[:n].numpy().tobytes())
    dist.destroy_process_group()


def test_two_ranks_slab_pipeline_container_identical(tmp_path, oracle):
    import torch.multiprocessing as mp
    from paper_2309_09778_b200 import synthetic
    x = synthetic.generate("C2", shape=(ROWS, COLS)).numpy()
    ref, _ = oracle.compress(x, oracle.OracleConfig(b_r=1e-2, repair_factor=1.0))
    out = str(tmp_path / "shard")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert open(f"{out}.0", "rb").read() + open(f"{out}.1", "rb").read() == ref


@pytest.mark.slow
def test_slab_pipeline_c3_full_size():
    """C3 at full size (512 MiB, 16384 partitions) in 8 slabs of 64 MiB: the
    slab container equals the single-call one (which tests/test_gpu_fullsize.py
    pins to the oracle byte for byte); slab decode equals the device decode."""
    import paper_2309_09778_b200 as P
    from paper_2309_09778_b200 import synthetic
    from paper_2309_09778_b200.pipeline import grid_view_shape
    x = synthetic.generate("C3", device="cuda")
    (r, c), _ = grid_view_shape(tuple(x.shape))
    x = x.reshape(r, c).contiguous()
    cfg = P.CompressConfig(rel_error=1e-2, repair_factor=1.0)
    codec = P.Codec("cuda:0")
    ref, rinfo = codec.compress_device(x, cfg)
    ref = ref.cpu()
    h = P.Codec.parse_header(ref.numpy())
    offs = torch.from_numpy(P.Codec.index_blocks(ref.numpy(), h).view(np.int64)).cuda()
    y_ref = codec.decompress_device(ref.cuda(), h, offs).cpu()
    pipe = P.HostPipeline(codec, slab_bytes=64 << 20)
    h_out = torch.empty(ref.numel() + (1 << 16), dtype=torch.uint8, pin_memory=True)
    n, info = pipe.compress(_pin(x.cpu()), cfg, h_out)
    assert n == ref.numel() and torch.equal(h_out[:n], ref)
    assert (info.m, info.nbal, info.nrepair, info.ncodes) == (rinfo.m, rinfo.nbal, rinfo.nrepair, rinfo.ncodes)
    y = pipe.decompress(h_out[:n])
    assert torch.equal(y.view(torch.int32), y_ref.view(torch.int32))


def test_decompress_shard_of_a_container():
    """HostPipeline.decompress(shard_rows=...): header + the records of one
    shard of whole block-rows (what a rank of a sharded run holds) decode to
    that shard's rows of the full decode."""
    import paper_2309_09778_b200 as P
    from paper_2309_09778_b200 import synthetic
    x = synthetic.generate("C2", shape=(2048, 1024)).contiguous()
    codec = P.Codec("cuda:0")
    buf, _ = codec.compress_device(x.cuda(), P.CompressConfig(rel_error=1e-2, repair_factor=1.0))
    full = buf.cpu().numpy()
    h = P.Codec.parse_header(full)
    offs = P.Codec.index_blocks(full, h)
    y_full = P.decompress(full.tobytes(), device="cuda:0")
    nbc, hb = 4, int(h.header_bytes)
    pipe = P.HostPipeline(codec, slab_bytes=256 * 1024 * 4)  # slabs of one block-row
    for br0, br1 in ((0, 3), (3, 8)):  # two shards: block-rows [0, 3) and [3, 8)
        part = np.concatenate([full[:hb], full[int(offs[br0 * nbc]): int(offs[br1 * nbc])]])
        y = pipe.decompress(_pin(torch.from_numpy(part)), shard_rows=(br1 - br0) * 256)
        assert np.array_equal(y.numpy().view(np.uint32), y_full[br0 * 256: br1 * 256].view(np.uint32))
