"""The multi-GPU driver on the real engine (one B200 here: world size 1 over
NCCL; the N>1 host logic is covered by tests/test_multigpu_host.py on gloo).
Sharded evaluation and the distributed committee must reproduce the
single-process evaluate / run_experiment integers exactly."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from tests.conftest import has_cuda

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]

import paper_1102_0183_b200 as ck  # noqa: E402
from paper_1102_0183_b200 import multigpu  # noqa: E402
from paper_1102_0183_b200.configs import spec_for  # noqa: E402


@pytest.fixture(scope="module")
def nccl_world():
    import torch
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_sharded_evaluate_equals_evaluate(nccl_world):
    spec = spec_for("C1")
    train = ck.make_glyph_dataset(300, 10, 29, seed=1)
    test = ck.make_glyph_dataset(1001, 10, 29, seed=1, split="test")
    net = ck.NetworkState(spec, 0)
    ck.train_epoch(net, train, ck.TrainConfig(epochs=1, eta0=1e-3), 0)
    err, labels = multigpu.sharded_evaluate(net, test)
    np.testing.assert_array_equal(labels, ck.predict_batch(net, test))
    assert err == ck.evaluate(net, test)
    err_tc, labels_tc = multigpu.sharded_evaluate(net, test, engine="tc")
    np.testing.assert_array_equal(labels_tc, ck.predict_batch(net, test, engine="tc"))
    assert np.mean(labels_tc == labels) >= 0.995
    flat = net.flat_parameters()
    multigpu.broadcast_parameters(net, 0)
    np.testing.assert_array_equal(net.flat_parameters(), flat)
    net.close()


def test_committee_equals_run_experiment(nccl_world):
    spec = spec_for("C1")
    train = ck.make_glyph_dataset(120, 10, 29, seed=3)
    test = ck.make_glyph_dataset(200, 10, 29, seed=3, split="test")
    cfg = ck.TrainConfig(epochs=2, eta0=1e-3, seed=5, test_every=1)
    summary, labels = multigpu.run_committee(spec, train, test, cfg, runs=3)
    solo = ck.run_experiment(spec, train, test, cfg, runs=3)
    assert summary.seeds == solo.seeds
    for got, want in zip(summary.runs, solo.runs):
        assert [(e.train_err, e.test_err) for e in got.epochs] == \
            [(e.train_err, e.test_err) for e in want.epochs]
        assert (got.tfbv, got.bt, got.best_epoch) == (want.tfbv, want.bt, want.best_epoch)
    for m in range(3):
        net = ck.NetworkState(spec, cfg.seed + m)
        for e in range(cfg.epochs):
            ck.train_epoch(net, train, cfg, e)
        np.testing.assert_array_equal(labels[m], ck.predict_batch(net, test))
        assert summary.runs[m].epochs[-1].test_err == ck.evaluate(net, test)
        net.close()
