"""FP32 perceptron perf mode (BASELINE.json north_star):
float32 surfaces, predictor, quantizer and recurrence on the throughput path,
container version 2.  Every point still satisfies the bound (the encoder
simulates the float32 decoder exactly); codes differ from the FP64 path only
where float32 rounding moves them -- counted, never silently."""
import numpy as np
import pytest
import torch

import paper_2309_09778_b200 as P
from paper_2309_09778_b200 import errors as E
from paper_2309_09778_b200.pipeline import CompressConfig, make_params


def test_precision_parameter_checks():
    with pytest.raises(E.ConfigError):
        make_params(CompressConfig(precision="fp16"), 3)
    with pytest.raises(E.ConfigError):  # 1-D fields have no FP32 mode
        make_params(CompressConfig(precision="fp32"), 1)
    p = make_params(CompressConfig(precision="fp32"), 3)
    assert p.precision == 1 and p.d_code_dump == 0
    assert make_params(CompressConfig(), 3).precision == 0


def _bound(x, y, b_r):
    tiny = float(np.finfo(np.float32).tiny)
    xz = np.where(np.abs(x) <= tiny, 0, x).astype(np.float64)
    y = y.astype(np.float64)
    assert np.all(y[xz == 0] == 0)
    nz = np.abs(xz) > tiny * (1 + 2 * b_r)
    return float((np.abs(y[nz] - xz[nz]) / np.abs(xz[nz])).max())


@pytest.mark.gpu
@pytest.mark.parametrize("name,shape,b_r", [("C2", (2048, 1536), 1e-2), ("C2", (1800, 3600), 1e-3),
                                            ("C4", (20, 500, 500), 1e-2)])
def test_fp32_roundtrip_bound_and_mismatch_counts(name, shape, b_r):
    from paper_2309_09778_b200 import synthetic
    from paper_2309_09778_b200.pipeline import code_mismatches
    codec = P.Codec("cuda:0")
    x = synthetic.generate(name, shape=shape).numpy()
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    n = codec.code_dump_numel(xd.shape, CompressConfig(rel_error=b_r))
    dumps, bufs, infos = {}, {}, {}
    for prec in ("fp64", "fp32"):
        d = torch.full((n,), 0xFFFE, dtype=torch.int32, device="cuda").to(torch.uint16)
        cfg = CompressConfig(rel_error=b_r, repair_factor=1.0, precision=prec, code_dump=d)
        buf, info = codec.compress_device(xd, cfg)
        bufs[prec], infos[prec], dumps[prec] = buf.cpu().numpy().tobytes(), info, d
    h = P.Codec.parse_header(np.frombuffer(bufs["fp32"], np.uint8))
    assert int(h.version) == 2 and int(P.Codec.parse_header(np.frombuffer(bufs["fp64"], np.uint8)).version) == 1
    y32 = P.decompress(bufs["fp32"], device="cuda:0").reshape(x.shape)
    assert _bound(x.reshape(-1), y32.reshape(-1), b_r) <= b_r
    cm = code_mismatches(dumps["fp64"], dumps["fp32"])
    assert cm["codes"] == infos["fp64"].ncodes == infos["fp32"].ncodes
    assert cm["code_mismatches"] / cm["codes"] < 0.05, cm
    assert abs(len(bufs["fp32"]) - len(bufs["fp64"])) / len(bufs["fp64"]) < 0.05


@pytest.mark.gpu
@pytest.mark.parametrize("shape,br,bc,pr", [((2048, 1536), 256, 256, 32), ((1100, 900), 256, 256, 32),
                                           ((700, 330), 64, 128, 16)])
def test_fp32_container_independent_of_chain_length(shape, br, bc, pr):
    """The FP32 sweep gives the same container whether a warp takes one
    partition or a chain of consecutive partitions of a block (PMZ_CHAIN; the
    size rule gives small fields 1, C5 8), and the code dump agrees too."""
    import os
    from paper_2309_09778_b200 import synthetic
    codec = P.Codec("cuda:0")
    xd = synthetic.generate("C2", shape=shape).cuda()
    got = {}
    for chain in ("1", "3", "8"):
        os.environ["PMZ_CHAIN"] = chain
        try:
            n = codec.code_dump_numel(xd.shape, CompressConfig(block_rows=br, block_cols=bc, partition_rows=pr))
            d = torch.full((n,), 0xFFFE, dtype=torch.int32, device="cuda").to(torch.uint16)
            cfg = CompressConfig(rel_error=1e-2, repair_factor=1.0, block_rows=br, block_cols=bc, partition_rows=pr,
                                 precision="fp32", code_dump=d)
            buf, info = codec.compress_device(xd, cfg)
            got[chain] = (buf.cpu().numpy().tobytes(), d.cpu(), info.nbal, info.nrepair)
        finally:
            os.environ.pop("PMZ_CHAIN", None)
    for chain in ("3", "8"):
        assert got[chain][0] == got["1"][0], chain
        assert torch.equal(got[chain][1].view(torch.int16), got["1"][1].view(torch.int16)), chain
        assert got[chain][2:] == got["1"][2:], chain
