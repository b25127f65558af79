"""Golden CLI transcripts from the REFERENCE's own command line (convkit cli.py).

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nbcache \\
        python tests/golden/make_cli_golden.py

Writes tests/golden/cli/: gzipped MNIST-format IDX files of synthetic glyphs
(convkit.synth), two architecture files (one with the paper's deformation
keys), and the reference's metrics.log / stdout for `train` (1 run and a
2-run experiment, --no-timing), `eval` of the saved weights and `inspect`.
"""

from __future__ import annotations

import contextlib
import gzip
import io
import os
import shutil
import tempfile

import numpy as np

from convkit import cli
from convkit.datasets import write_idx
from convkit.synth import make_glyph_images

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli")

ARCH_PLAIN = """input 1x29x29
conv 8M k4x4 s0x0
maxpool 2x2
conv 12M k5x5 s0x0
maxpool 3x3
fc 30N
output 10

eta0 = 2e-3
eta_decay = 0.9
epochs = 3
"""
ARCH_DEFORM = ARCH_PLAIN + """deform_rotate = 10
deform_scale = 0.1
deform_elastic_sigma = 6
deform_elastic_alpha = 6
"""


def gz(src, dst):
    with open(src, "rb") as f, open(dst, "wb") as raw:
        with gzip.GzipFile(fileobj=raw, mode="wb", mtime=0) as g:
            g.write(f.read())


def run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        code = cli.main(argv)
    return code, buf.getvalue()


def main():
    os.makedirs(OUT, exist_ok=True)
    tmp = tempfile.mkdtemp()
    tr, trl = make_glyph_images(240, 10, 29, 1, "train")
    te, tel = make_glyph_images(120, 10, 29, 1, "test")
    write_idx(tr, trl, f"{tmp}/train-images-idx3-ubyte", f"{tmp}/train-labels-idx1-ubyte")
    write_idx(te, tel, f"{tmp}/t10k-images-idx3-ubyte", f"{tmp}/t10k-labels-idx1-ubyte")
    for n in os.listdir(tmp):
        gz(f"{tmp}/{n}", f"{OUT}/{n}.gz")
    for name, text in (("plain.net", ARCH_PLAIN), ("deform.net", ARCH_DEFORM)):
        with open(f"{OUT}/{name}", "w") as f:
            f.write(text)
    data = OUT
    for tag, arch, extra in (("plain", "plain.net", []), ("deform", "deform.net", []),
                             ("runs2", "plain.net", ["--runs", "2", "--epochs", "2"])):
        out_dir = f"{tmp}/{tag}"
        code, _ = run(["train", "--arch", f"{OUT}/{arch}", "--data", data, "--seed", "3",
                       "--no-timing", "--out", out_dir, *extra])
        assert code == 0, (tag, code)
        shutil.copy(f"{out_dir}/metrics.log", f"{OUT}/{tag}.metrics.log")
        if tag == "plain":
            w = dict(np.load(f"{out_dir}/weights.npz"))
            np.savez_compressed(f"{OUT}/plain.weights.npz", **w)
            code, text = run(["eval", "--arch", f"{OUT}/{arch}", "--data", data,
                              "--weights", f"{out_dir}/weights.npz"])
            assert code == 0
            with open(f"{OUT}/plain.eval.txt", "w") as f:
                f.write(text)
    code, text = run(["inspect", "--arch", f"{OUT}/deform.net"])
    with open(f"{OUT}/deform.inspect.txt", "w") as f:
        f.write(text)
    shutil.rmtree(tmp)
    print("written", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
