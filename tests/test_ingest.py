"""SEG-Y ingest (AC10): header
framing and errors on CPU, the device IBM->IEEE conversion bit-exact against
the oracle on a 64-case corpus, and an IEEE (format 5) fixture round trip
through compress/decompress within the bound."""
import struct

import numpy as np
import pytest

from paper_2309_09778_b200 import ingest
from paper_2309_09778_b200.errors import InconsistentTraceLength, TruncatedFile, UnsupportedFormatCode


def segy_bytes(samples_be_words: np.ndarray, fmt: int, ns_override=None) -> bytes:
    """A rev-0 SEG-Y file: EBCDIC-blank textual header, binary header with the
    sample count (3220) and format code (3224), one 240-byte header per trace."""
    ntr, ns = samples_be_words.shape
    head = bytearray(b"\x40" * 3200) + bytearray(400)
    struct.pack_into(">H", head, 3200 + 20, ns)
    struct.pack_into(">h", head, 3200 + 24, fmt)
    out = bytearray(head)
    for t in range(ntr):
        th = bytearray(240)
        struct.pack_into(">H", th, 114, ns if ns_override is None or t == 0 else ns_override)
        out += th + samples_be_words[t].astype(">u4").tobytes()
    return bytes(out)


def ibm_corpus() -> np.ndarray:
    """64 words spanning signs, exponents (incl. the extremes) and fractions
    (normalized, unnormalized, zero)."""
    fr = [0x100000, 0x800000, 0xFFFFFF, 0x000001, 0x0F0000, 0x123456, 0x000000, 0x7FFFFF]
    ex = [0, 1, 32, 63, 64, 65, 96, 127]
    w = [(s << 31) | (e << 24) | f for i, (e, f) in enumerate((e, f) for e in ex for f in fr)
         for s in [i & 1]]
    return np.array(w, dtype=np.uint32)


def test_ibm_oracle_kats(oracle):
    assert oracle.ibm_to_ieee(np.array([0x41100000]))[0] == np.float32(1.0)
    assert oracle.ibm_to_ieee(np.array([0xC1100000]))[0] == np.float32(-1.0)
    assert oracle.ibm_to_ieee(np.array([0x42640000]))[0] == np.float32(100.0)
    assert len(ibm_corpus()) == 64


def test_segy_header_errors(tmp_path):
    w = np.zeros((3, 8), np.uint32)
    p = tmp_path / "a.sgy"
    p.write_bytes(segy_bytes(w, 3))
    with pytest.raises(UnsupportedFormatCode):
        ingest.segy_layout(p.read_bytes(), p.stat().st_size)
    good = segy_bytes(w, 1)
    assert ingest.segy_layout(good, len(good)) == (1, 8, 3)
    with pytest.raises(TruncatedFile):
        ingest.segy_layout(good[:-5], len(good) - 5)
    with pytest.raises(TruncatedFile):
        ingest.segy_layout(good[:1000], 1000)


@pytest.mark.gpu
def test_segy_ibm_corpus_bit_exact(tmp_path, oracle):
    words = ibm_corpus().reshape(4, 16)
    p = tmp_path / "ibm.sgy"
    p.write_bytes(segy_bytes(words, 1))
    y = ingest.read_segy(str(p), "cuda:0").cpu().numpy()
    ref = oracle.ibm_to_ieee(words)
    assert np.array_equal(y.view(np.uint32), ref.view(np.uint32))
    q = tmp_path / "bad.sgy"
    q.write_bytes(segy_bytes(words, 1, ns_override=15))
    with pytest.raises(InconsistentTraceLength):
        ingest.read_segy(str(q), "cuda:0")


@pytest.mark.gpu
def test_segy_ieee_fixture_roundtrip(tmp_path):
    import paper_2309_09778_b200 as P
    from paper_2309_09778_b200 import synthetic
    x = synthetic.generate("C2", shape=(96, 700)).numpy()  # 96 traces x 700 samples
    p = tmp_path / "ieee.sgy"
    p.write_bytes(segy_bytes(x.view(np.uint32), 5))
    y = ingest.read_segy(str(p), "cuda:0").cpu().numpy()
    assert np.array_equal(y, x)
    buf = P.compress(y, rel_error=1e-3, device="cuda:0")
    z = P.decompress(buf, device="cuda:0")
    nz = x != 0
    assert np.all(z[~nz] == 0) and np.max(np.abs(z[nz] - x[nz]) / np.abs(x[nz])) <= 1.5e-3
