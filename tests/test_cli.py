"""CLI parity with the reference's command line (convkit cli.py).

tests/golden/cli/ holds transcripts of the REFERENCE's own CLI
(tests/golden/make_cli_golden.py): gzipped IDX files, architecture files and
the metrics.log / stdout it produced.  The B200 CLI must reproduce them
byte for byte (--no-timing), load the reference's weights.npz and write one
the reference can load, and keep the exit-code contract (cli.py:1-12).
"""

from __future__ import annotations

import contextlib
import io
import os

import numpy as np
import pytest

from paper_1102_0183_b200 import cli
from paper_1102_0183_b200.datasets import load_cifar10, load_idx, load_norb, write_idx
from paper_1102_0183_b200.errors import DataFormatError
from tests.conftest import GOLDEN, has_cuda

G = os.path.join(GOLDEN, "cli")


def run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        code = cli.main(argv)
    return code, buf.getvalue()


def golden_text(name):
    with open(os.path.join(G, name)) as f:
        return f.read()


def test_inspect_matches_reference():
    code, text = run(["inspect", "--arch", os.path.join(G, "deform.net")])
    assert code == 0
    assert text == golden_text("deform.inspect.txt")


def test_idx_loader_reads_gzipped_golden_files():
    d = load_idx(os.path.join(G, "train-images-idx3-ubyte.gz"),
                 os.path.join(G, "train-labels-idx1-ubyte.gz"))
    assert (len(d), d.channels, d.height, d.width) == (240, 1, 29, 29)
    assert d.raw.dtype == np.uint8 and d.labels.max() <= 9


def test_idx_roundtrip_and_errors(tmp_path):
    imgs = np.random.default_rng(0).integers(0, 256, (5, 7, 9), dtype=np.uint8)
    write_idx(imgs, [0, 1, 2, 3, 4], tmp_path / "i", tmp_path / "l")
    d = load_idx(tmp_path / "i", tmp_path / "l")
    assert np.array_equal(d.raw[:, 0], imgs)
    blob = (tmp_path / "i").read_bytes()
    (tmp_path / "t").write_bytes(blob[:-1])
    with pytest.raises(DataFormatError):
        load_idx(tmp_path / "t", tmp_path / "l")
    (tmp_path / "m").write_bytes(b"\0\0\x08\x04" + blob[4:])
    with pytest.raises(DataFormatError):
        load_idx(tmp_path / "m", tmp_path / "l")


def test_cifar_and_norb_loaders(tmp_path):
    rng = np.random.default_rng(1)
    rec = rng.integers(0, 256, (4, 3073), dtype=np.uint8)
    rec[:, 0] = [0, 9, 3, 1]
    (tmp_path / "b").write_bytes(rec.tobytes())
    d = load_cifar10([tmp_path / "b"])
    assert d.raw.shape == (4, 3, 32, 32) and list(d.labels) == [0, 9, 3, 1]
    assert np.array_equal(d.raw[2].reshape(-1), rec[2, 1:])
    rec[1, 0] = 10
    (tmp_path / "bad").write_bytes(rec.tobytes())
    with pytest.raises(DataFormatError):
        load_cifar10([tmp_path / "bad"])
    import struct
    px = rng.integers(0, 256, (3, 2, 6, 5), dtype=np.uint8)
    (tmp_path / "dat").write_bytes(struct.pack("<iiiiii", 0x1E3D4C55, 4, 3, 2, 6, 5) +
                                   px.tobytes())
    (tmp_path / "cat").write_bytes(struct.pack("<iiiii", 0x1E3D4C54, 1, 3, 1, 1) +
                                   np.array([0, 4, 2], "<i4").tobytes())
    d = load_norb(tmp_path / "dat", tmp_path / "cat")
    assert np.array_equal(d.raw, px) and list(d.labels) == [0, 4, 2] and d.n_classes == 5


@pytest.mark.parametrize("argv,code", [
    (["inspect", "--arch", "/nonexistent.net"], cli.EXIT_CONFIG),
    (["gradcheck", "--arch", os.path.join(G, "plain.net")], cli.EXIT_CONFIG),
    (["train", "--arch", os.path.join(G, "plain.net"), "--precision", "double",
      "--data", G], cli.EXIT_CONFIG),
    (["train", "--arch", os.path.join(G, "plain.net"), "--data", "/nonexistent"],
     cli.EXIT_CONFIG),
])
def test_exit_codes(argv, code):
    assert run(argv)[0] == code


def test_bad_data_exit_code(tmp_path):
    (tmp_path / "train-images-idx3-ubyte").write_bytes(b"junk")
    (tmp_path / "train-labels-idx1-ubyte").write_bytes(b"junk")
    (tmp_path / "t10k-images-idx3-ubyte").write_bytes(b"junk")
    (tmp_path / "t10k-labels-idx1-ubyte").write_bytes(b"junk")
    code, _ = run(["train", "--arch", os.path.join(G, "plain.net"), "--data", str(tmp_path)])
    assert code == cli.EXIT_DATA_FORMAT


def test_unknown_config_key(tmp_path):
    arch = tmp_path / "x.net"
    arch.write_text(golden_text("plain.net") + "bogus = 1\n")
    code, _ = run(["train", "--arch", str(arch), "--data", G])
    assert code == cli.EXIT_CONFIG


@pytest.mark.parametrize("tag,arch,extra", [
    ("plain", "plain.net", []),
    ("deform", "deform.net", []),
    ("runs2", "plain.net", ["--runs", "2", "--epochs", "2"]),
])
@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_train_log_byte_identical(tmp_path, tag, arch, extra):
    out = tmp_path / tag
    code, _ = run(["train", "--arch", os.path.join(G, arch), "--data", G, "--seed", "3",
                   "--no-timing", "--out", str(out), *extra])
    assert code == 0
    assert (out / "metrics.log").read_text() == golden_text(f"{tag}.metrics.log")
    if tag == "plain":
        ref = np.load(os.path.join(G, "plain.weights.npz"))
        mine = np.load(out / "weights.npz")
        assert sorted(ref.files) == sorted(mine.files)
        for k in ref.files:
            np.testing.assert_allclose(mine[k], ref[k], rtol=0, atol=1e-5, err_msg=k)
        code, text = run(["eval", "--arch", os.path.join(G, arch), "--data", G,
                          "--weights", os.path.join(G, "plain.weights.npz")])
        assert code == 0 and text == golden_text("plain.eval.txt")



@pytest.mark.parametrize("tag,arch,extra", [
    ("plain", "plain.net", []),
    ("runs2", "plain.net", ["--runs", "2", "--epochs", "2"]),
    ("deform", "deform.net", []),
])
@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_reference_frontend_over_b200_engine(tmp_path, tag, arch, extra):
    """SURVEY §8(f)2 backend switch: the reference's unchanged convkit.cli
    (from baseline/_ref) with its engine symbols rebound to this package
    reproduces its own transcripts byte for byte."""
    from tests.conftest import reference_convkit
    if reference_convkit() is None:
        pytest.skip("reference package not available")
    out = tmp_path / tag
    code, _ = run(["--reference-frontend", "train", "--arch", os.path.join(G, arch),
                   "--data", G, "--seed", "3", "--no-timing", "--out", str(out), *extra])
    assert code == 0
    assert (out / "metrics.log").read_text() == golden_text(f"{tag}.metrics.log")
    if tag == "plain":
        code, text = run(["--reference-frontend", "eval", "--arch", os.path.join(G, arch),
                          "--data", G, "--weights", os.path.join(G, "plain.weights.npz")])
        assert code == 0 and text == golden_text("plain.eval.txt")


def test_reference_frontend_exit_codes():
    from tests.conftest import reference_convkit
    if reference_convkit() is None:
        pytest.skip("reference package not available")
    assert run(["--reference-frontend", "inspect", "--arch", "/nonexistent.net"])[0] == \
        cli.EXIT_CONFIG
    code, text = run(["--reference-frontend", "inspect", "--arch", os.path.join(G, "deform.net")])
    assert code == 0 and text == golden_text("deform.inspect.txt")
