"""CPU tests of the product's host side: the C-ABI library loads and exports
every symbol include/permez_b200.h declares; container header parsing and
block indexing (host C++ code, no GPU) agree with the oracle's container;
exception mapping; trainer split; model blob.  No compute kernel is called."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "permez_b200.h")).read()
    return sorted(set(re.findall(r"PMZ_API\s+[\w\s\*]*?\b(pmz_\w+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    from paper_2309_09778_b200 import _native as N
    lib = N.load()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(N.EXPORTS)
    assert lib.pmz_abi_version() == 2
    assert lib.pmz_status_string(-14) == b"Corrupt"


def test_status_mapping():
    from paper_2309_09778_b200 import errors as E
    assert isinstance(E.status_error(-2), E.NonFiniteInput)
    assert isinstance(E.status_error(-12), E.BadMagic)
    assert isinstance(E.status_error(-15), E.BalanceUnderflow)
    assert issubclass(E.Corrupt, E.ContainerError) and issubclass(E.ContainerError, E.PermezError)
    assert E.exit_code(E.Corrupt("x")) == 6 and E.exit_code(E.ConfigError("x")) == 2


def _container(oracle, shape=(300, 520), **kw):
    from paper_2309_09778_b200 import synthetic
    x = synthetic.generate("C2", shape=shape).numpy()
    buf, info = oracle.compress(x, oracle.OracleConfig(**kw))
    return x, buf, info


def test_parse_header_and_index_match_oracle(oracle):
    from paper_2309_09778_b200.pipeline import Codec
    x, buf, info = _container(oracle, b_r=1e-3)
    a = np.frombuffer(buf, np.uint8)
    h = Codec.parse_header(a)
    oh = oracle.read_header(buf)
    assert (h.rows, h.cols, h.m, h.nblocks, h.header_bytes) == (oh["rows"], oh["cols"], oh["m"], oh["nblocks"],
                                                               oh["header_bytes"])
    assert h.b_r == 1e-3 and h.S == 3 and h.H == 2
    offs = Codec.index_blocks(a, h)
    assert offs[0] == h.header_bytes and offs[-1] == len(buf)
    assert np.all(np.diff(offs.astype(np.int64)) > 0)


@pytest.mark.parametrize("mutate,exc", [
    (lambda b: b"QMEZ" + b[4:], "BadMagic"),
    (lambda b: b[:4] + b"\x03\x00" + b[6:], "UnsupportedVersion"),  # 1: FP64 parity, 2: FP32 perf mode
    (lambda b: b[:51] + bytes([3]) + b[52:], "Corrupt"),        # m out of range
    (lambda b: b[:20], "Corrupt"),
])
def test_header_corruption(oracle, mutate, exc):
    from paper_2309_09778_b200 import errors as E
    from paper_2309_09778_b200.pipeline import Codec
    _, buf, _ = _container(oracle, shape=(64, 64))
    with pytest.raises(getattr(E, exc)):
        Codec.parse_header(np.frombuffer(mutate(buf), np.uint8).copy())


def test_index_detects_truncation_and_trailing_bytes(oracle):
    from paper_2309_09778_b200 import errors as E
    from paper_2309_09778_b200.pipeline import Codec
    _, buf, _ = _container(oracle)
    a = np.frombuffer(buf, np.uint8)
    h = Codec.parse_header(a)
    with pytest.raises((E.TruncatedStream, E.Corrupt)):
        Codec.index_blocks(a[:-5].copy(), h)
    with pytest.raises(E.Corrupt):
        Codec.index_blocks(np.concatenate([a, np.zeros(3, np.uint8)]), h)


@pytest.mark.parametrize("n", [1, 4, 5, 10, 100, 120, 4096])
def test_trainer_split_matches_oracle(oracle, n):
    from paper_2309_09778_b200.trainer import validation_blocks
    assert np.array_equal(np.sort(validation_blocks(n, 0.1, 0)), np.sort(oracle.split_blocks(n, 0.1, 0)[1]))


def test_sampling_kats():
    from paper_2309_09778_b200 import trainer as T
    assert len(T.sample_training_blocks(100, 0.1, 1)) == 10
    assert list(T.sample_training_blocks(7, 1.0, 1)) == list(range(7))
    assert np.array_equal(T.sample_training_blocks(50, 0.2, 3), T.sample_training_blocks(50, 0.2, 3))
    tr, va = T.split_train_validation(np.arange(10))
    assert (len(tr), len(va)) == (8, 2)
    tr, va = T.split_train_validation(np.arange(5))
    assert (len(tr), len(va)) == (4, 1)


def test_model_blob_roundtrip():
    from paper_2309_09778_b200.predictor import PerceptronModel, init_model
    m = init_model(3)
    b = m.to_bytes()
    assert len(b) == 16 + 8 * 8 + 16
    m2 = PerceptronModel.from_bytes(b)
    assert np.array_equal(m2.w1, m.w1) and np.array_equal(m2.w2, m.w2) and m2.leaky_slope == 0.01


def test_header_model_blob_is_reference_layout(oracle):
    """The container's model blob equals PerceptronModel.to_bytes()."""
    from paper_2309_09778_b200.predictor import init_model
    _, buf, _ = _container(oracle, shape=(64, 64))
    ml = int.from_bytes(buf[52:60], "little")
    assert buf[60:60 + ml] == init_model(3).to_bytes()


def test_no_cpu_fallback_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    import paper_2309_09778_b200 as P
    from paper_2309_09778_b200 import errors as E
    with pytest.raises(E.DeviceError):
        P.compress(np.ones((4, 4), np.float32))


def test_hostpipe_slab_plan():
    """hostpipe.plan_slabs: contiguous slabs of whole block-rows covering the field."""
    from paper_2309_09778_b200.hostpipe import plan_slabs
    for nbr, br, cols, sb in [(4096, 256, 2048, 128 << 20), (8, 256, 3600, 1 << 20), (1, 256, 500, 1 << 30),
                              (196, 256, 500, 10 << 20), (0, 256, 512, 1 << 20)]:
        sl = plan_slabs(nbr, br, cols, sb)
        assert [a for a, _ in sl] == ([0] + [b for _, b in sl[:-1]] if sl else [])
        assert (sl[-1][1] if sl else 0) == nbr and all(b > a for a, b in sl)
        per = max(1, sb // (br * cols * 4))
        assert all(b - a == per for a, b in sl[:-1]) and (not sl or sl[-1][1] - sl[-1][0] <= per)
    assert len(plan_slabs(4096, 256, 2048, 128 << 20)) == 64  # C5: 64 slabs of 64 block-rows


def test_index_blocks_range_matches_full_walk(oracle):
    """pmz_index_blocks_range over consecutive block ranges reproduces the
    whole-container walk (the host pipeline indexes one slab at a time), keeps
    its framing checks and only the range that ends the container checks the
    container's end."""
    import ctypes
    from paper_2309_09778_b200 import _native as N
    from paper_2309_09778_b200 import errors as E
    from paper_2309_09778_b200.pipeline import Codec
    _, buf, _ = _container(oracle, shape=(1100, 900), b_r=1e-2)  # 5 x 4 blocks, ragged edges
    a = np.frombuffer(buf, np.uint8).copy()
    h = Codec.parse_header(a)
    full = Codec.index_blocks(a, h)
    lib = N.load()

    def rng(arr, b0, b1, pos0):
        out = np.zeros(b1 - b0 + 1, np.uint64)
        s = lib.pmz_index_blocks_range(arr.ctypes.data_as(ctypes.c_void_p), arr.size, ctypes.byref(h), b0, b1, pos0,
                                       out.ctypes.data_as(ctypes.c_void_p))
        return s, out

    nb = int(h.nblocks)
    pos, got = int(h.header_bytes), []
    for b0 in range(0, nb, 4):  # one block-row at a time
        s, out = rng(a, b0, min(nb, b0 + 4), pos)
        assert s == 0
        got.extend(out[:-1].tolist())
        pos = int(out[-1])
    got.append(pos)
    assert got == full.tolist()
    assert rng(a, 3, 2, 0)[0] == -1 and rng(a, 0, nb + 1, int(h.header_bytes))[0] == -1  # ConfigError
    # an inner range does not see trailing bytes, the final one does; truncation is seen where it bites
    longer = np.concatenate([a, np.zeros(3, np.uint8)])
    assert rng(longer, 0, 4, int(h.header_bytes))[0] == 0
    assert isinstance(E.status_error(rng(longer, nb - 4, nb, int(full[nb - 4]))[0]), E.Corrupt)
    assert rng(a[: int(full[2])].copy(), 0, 4, int(h.header_bytes))[0] in (-10, -14)
