"""CLI: flag handling and the
per-family exit codes on CPU; file round trips and the bench sweep on the GPU."""
import numpy as np
import pytest

from paper_2309_09778_b200 import cli


def test_exit_codes_per_family(tmp_path, capsys):
    out = str(tmp_path / "x.pmz")
    assert cli.main(["compress", "--input", str(tmp_path / "missing.f32"), "--output", out]) == 7  # IngestError
    assert cli.main(["compress", "--input", "gen:C2", "--rel-error", "0", "--output", out]) == 2  # ConfigError
    assert cli.main(["compress", "--input", str(tmp_path / "x.sgy"), "--format", "segy", "--output", out]) == 7
    assert cli.main(["compress", "--input", "gen:C2", "--grid", "lr:0", "--output", out]) == 2  # lr > 0
    assert cli.main(["compress", "--input", "gen:C2", "--threads", "0", "--output", out]) == 2
    assert cli.main(["decompress", "--input", str(tmp_path / "missing.pmz")]) == 7
    raw = tmp_path / "a.f32"
    np.zeros(10, np.float32).tofile(raw)
    assert cli.main(["compress", "--input", str(raw), "--dims", "3x4", "--output", out]) == 7  # size mismatch
    capsys.readouterr()


def test_generators_follow_spec(tmp_path):
    """sine2d = sin(2 pi r/rows) sin(2 pi c/cols) + 2.0 (strictly
    positive, no zeros); constant -> all equal; same seed -> identical; raw64
    is reported unsupported (ConfigError, exit 2)."""
    x = cli._generate("sine2d", (64, 48), 0)
    r, c = np.meshgrid(np.arange(64), np.arange(48), indexing="ij")
    ref = (np.sin(2 * np.pi * r / 64) * np.sin(2 * np.pi * c / 48) + 2.0).astype(np.float32)
    assert x.dtype == np.float32 and np.array_equal(x, ref) and x.min() >= 1.0
    k = cli._generate("constant", (5, 7), 0)
    assert np.all(k == k.flat[0])
    assert np.array_equal(cli._generate("white-noise", (9, 9), 4), cli._generate("white-noise", (9, 9), 4))
    raw = tmp_path / "a.f64"
    np.zeros(12, np.float64).tofile(raw)
    assert cli.main(["compress", "--input", str(raw), "--format", "raw64", "--dims", "3x4",
                     "--output", str(tmp_path / "o.pmz")]) == 2


@pytest.mark.gpu
def test_cli_roundtrip_and_original(tmp_path, capsys):
    x = np.ascontiguousarray(np.random.default_rng(3).normal(0, 1, (200, 300)).astype(np.float32) * 10)
    src, cont, dst = tmp_path / "x.f32", tmp_path / "x.pmz", tmp_path / "y.f32"
    x.tofile(src)
    assert cli.main(["compress", "--input", str(src), "--dims", "200x300", "--rel-error", "1e-3",
                     "--output", str(cont)]) == 0
    line = capsys.readouterr().out.strip().splitlines()[-1].split(",")
    assert float(line[7]) <= 1.5e-3  # max_rel_error column, SPEC default repair factor 1.5
    assert cli.main(["decompress", "--input", str(cont), "--output", str(dst), "--original", str(src),
                     "--dims", "200x300"]) == 0
    out = capsys.readouterr().out
    y = np.fromfile(dst, np.float32).reshape(200, 300)
    assert float(out.split("max_rel_error,")[1].split()[0]) <= 1.5e-3
    import paper_2309_09778_b200 as P
    assert np.array_equal(y, P.decompress(cont.read_bytes(), device="cuda:0"))
    b = bytearray(cont.read_bytes())
    b[:4] = b"XXXX"
    (tmp_path / "bad.pmz").write_bytes(bytes(b))
    assert cli.main(["decompress", "--input", str(tmp_path / "bad.pmz")]) == 6  # ContainerError (BadMagic)


@pytest.mark.gpu
def test_cli_bench_rows_and_cr_monotone(capsys):
    assert cli.main(["bench", "--input", "gen:sine2d", "--dims", "256x256", "--bench-bounds", "1e-4,1e-3,1e-2"]) == 0
    rows = [r.split(",") for r in capsys.readouterr().out.strip().splitlines()]
    assert rows[0][0] == "dataset" and len(rows) == 4
    cr = [float(r[6]) for r in rows[1:]]
    assert cr[0] >= cr[1] >= cr[2]  # AC8: CR non-increasing as b_r grows


@pytest.mark.gpu
def test_cli_train_save_load_model(tmp_path, capsys):
    """--train runs the sweep; the saved model blob reloads and gives the
    identical container (SPEC.md:607 --save-model / --load-model)."""
    c1, c2, mb = tmp_path / "a.pmz", tmp_path / "b.pmz", tmp_path / "m.bin"
    base = ["compress", "--input", "gen:C2", "--dims", "400x600", "--rel-error", "1e-2"]
    assert cli.main(base + ["--train", "--save-model", str(mb), "--output", str(c1)]) == 0
    assert cli.main(base + ["--load-model", str(mb), "--output", str(c2)]) == 0
    capsys.readouterr()
    assert c1.read_bytes() == c2.read_bytes()
    from paper_2309_09778_b200.predictor import PerceptronModel, init_model
    m = PerceptronModel.from_bytes(mb.read_bytes())
    assert not np.array_equal(m.w1, init_model(3).w1)
