"""bench.py keeps the driver's contract: one JSON line on stdout with the
required keys, a roofline / cpu_baseline / e2e / clocks / gpu_launches block,
the per-config blocks, and the reference arm's line (rank 0: the reference
itself from baseline/_ref when importable, else the oracle port) with the same
config object."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from tests.conftest import ROOT, has_cuda

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]

REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
            "e2e", "gpu_launches", "roofline", "cpu_baseline", "clocks"]


def run_bench(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


FOUR = ("value", "roofline", "cpu_baseline", "e2e")


def test_bench_line_contract():
    d = run_bench("--config", "C1", "--blocks", "C2", "--steps", "3", "--warmup", "3",
                  "--imgs-per-step", "64", "--cpu-seconds", "0.3", "--cpu-windows", "1")
    for k in REQUIRED:
        assert k in d, k
    assert d["value"] > 0 and d["gpu_launches"] == 3     # C1: one launch per step
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert 0 < d["roofline"]["frac"] < 1
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["eval_tc"]["label_agreement_with_exact"] >= 0.995
    assert d["deform"]["value"] > 0
    assert d["latency"]["phases_per_image"] >= 2
    for blk in (d, d["eval"], d["configs"]["C2"], d["configs"]["C2"]["eval"], d["committee"]):
        for k in FOUR:
            assert blk.get(k) is not None, k
    assert 0 < d["eval"]["roofline"]["frac"] < 1


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "1",
                  "--imgs-per-step", "16")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    ours = run_bench("--config", "C1", "--blocks", "", "--steps", "3", "--warmup", "3",
                     "--imgs-per-step", "16", "--no-cpu-baseline", "--no-committee",
                     "--no-deform", "--no-tc", "--no-e2e")
    assert d["config"] == ours["config"]          # same step definition in both arms
