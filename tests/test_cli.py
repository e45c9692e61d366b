"""CLI and signal files (mirror of reference tests/test_cli.py, test_sigio.py)."""

import json

import numpy as np
import pytest

from paper_2203_09384_b200.cli import main, parse_lengths
from paper_2203_09384_b200.sigio import read_signal, write_signal
from paper_2203_09384_b200 import DomainError, ShapeError


def test_parse_lengths():
    assert parse_lengths("8:64:pow2") == [8, 16, 32, 64]
    assert parse_lengths("8,16") == [8, 16]
    assert parse_lengths("32") == [32]
    for bad in ("8:64", "8:64:lin", "64:8:pow2", ","):
        with pytest.raises(ValueError):
            parse_lengths(bad)


@pytest.mark.parametrize("ext", ["csv", "json"])
@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_text_round_trip(tmp_path, ext, dtype):
    rng = np.random.default_rng(1)
    x = (rng.standard_normal(33) + 1j * rng.standard_normal(33)).astype(dtype)
    path = tmp_path / f"s.{ext}"
    write_signal(path, x)
    prec = "single" if dtype == np.complex64 else "double"
    assert np.array_equal(read_signal(path, precision=prec), x)


def test_npy_batch_round_trip_and_errors(tmp_path):
    x = np.arange(12, dtype=np.complex64).reshape(3, 4)
    write_signal(tmp_path / "b.npy", x)
    assert np.array_equal(read_signal(tmp_path / "b.npy"), x)
    with pytest.raises(ShapeError):
        write_signal(tmp_path / "b.csv", x)
    (tmp_path / "bad.csv").write_text("re,im\n1,2\n3\n")
    with pytest.raises(DomainError):
        read_signal(tmp_path / "bad.csv")
    (tmp_path / "bad.json").write_text("[[1, 2], [3]]")
    with pytest.raises(DomainError):
        read_signal(tmp_path / "bad.json")
    (tmp_path / "h.csv").write_text("re,im\n1,2\n")
    assert read_signal(tmp_path / "h.csv")[0] == 1 + 2j


def test_plan_command(capsys):
    assert main(["plan", "--length", "2048", "--precision", "double"]) == 0
    out = capsys.readouterr().out
    assert "stages: 8,8,8,4" in out and "precision: double" in out and "gpu_passes: 16,16,8" in out


def test_exit_codes(capsys):
    assert main(["plan", "--length", "4096"]) == 3
    assert main(["plan", "--length", "12"]) == 2
    assert main(["plan"]) == 2
    assert main(["transform", "--length", "8", "--input", "/nonexistent/x.csv"]) == 4


@pytest.mark.gpu
def test_transform_and_verify_on_gpu(tmp_path, capsys, cuda):
    out = tmp_path / "y.npy"
    assert main(["transform", "--length", "1024", "--signal", "random", "--batch", "64", "--output", str(out)]) == 0
    import oracle

    y = np.load(out)
    x = oracle.generate_batch(64, 1024, 0)
    assert np.max(np.linalg.norm(y - oracle.direct_dft(x), axis=1) / np.linalg.norm(oracle.direct_dft(x), axis=1)) < 1e-4
    assert main(["verify", "--length", "2048", "--fail-under-p", "0.999"]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep["chi2_reduced"] <= 0.01 and rep["p_value"] >= 0.999
    assert main(["verify", "--length", "512", "--batch", "256", "--signal", "random", "--precision", "double",
                 "--report", str(tmp_path / "r.json")]) == 0
    assert json.loads((tmp_path / "r.json").read_text())["max_rel_l2"] < 1e-12
    rec = tmp_path / "rec.csv"
    assert main(["bench", "--lengths", "8,64", "--iterations", "5", "--records", str(rec),
                 "--summary", str(tmp_path / "s.json")]) == 0
    assert len(rec.read_text().splitlines()) == 1 + 2 * 6
