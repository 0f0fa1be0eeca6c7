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
