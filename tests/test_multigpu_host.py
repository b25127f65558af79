"""Host logic of the multi-GPU driver (paper_1102_0183_b200.multigpu) on CPU:
world_size 2 over gloo, with a stand-in shard predictor in place of the CUDA
engine.  Checks that sharded evaluation returns exactly the single-process
error count and label vector, on every rank, for even, ragged and tiny test
sets, and that weights broadcast bit-exactly."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_1102_0183_b200 as ck
from paper_1102_0183_b200.multigpu import nets_for_rank, shard_range


def test_shard_range_partitions_every_size():
    for n in (0, 1, 2, 7, 10, 10_000, 10_001):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                first, count = shard_range(n, r, world)
                assert count >= 0
                seen.extend(range(first, first + count))
            assert seen == list(range(n)), (n, world)


def test_committee_members_cover_all_nets_once():
    for runs in (1, 3, 8, 9):
        for world in (1, 2, 4, 8):
            got = sorted(m for r in range(world) for m in nets_for_rank(runs, r, world))
            assert got == list(range(runs))


def test_bad_rank_rejected():
    with pytest.raises(ck.ConfigError):
        shard_range(10, 2, 2)


def _fake_labels(idx):
    # deterministic "predictions": right for most images, wrong for some
    return np.where(idx % 7 == 3, (idx + 1) % 10, idx % 10).astype(np.int32)


class _FakeNet:
    def __init__(self, flat):
        self.flat = np.array(flat, dtype=np.float32)

    def flat_parameters(self):
        return self.flat.copy()

    def set_flat_parameters(self, flat):
        self.flat = np.asarray(flat, dtype=np.float32).copy()


def _worker(rank, world, port, n_images, out_dir):
    import torch.distributed as dist

    from paper_1102_0183_b200 import multigpu
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        labels = (np.arange(n_images) % 10).astype(np.int32)
        data = ck.Dataset(np.zeros((n_images, 1, 2, 2), np.float32), labels, 10, "test")

        def predictor(first, count):
            return _fake_labels(np.arange(first, first + count))

        err, pred = multigpu.sharded_evaluate(None, data, predictor=predictor)
        net = _FakeNet(np.full(5, rank, np.float32) + np.arange(5, dtype=np.float32) / 3)
        multigpu.broadcast_parameters(net, src=0)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), err=err, pred=pred, flat=net.flat)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n_images", [10_000, 10_001, 3, 1])
def test_sharded_evaluation_matches_single_process(tmp_path, n_images):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), n_images, str(tmp_path)), nprocs=world)
    want_pred = _fake_labels(np.arange(n_images))
    want_err = 100.0 * np.count_nonzero(want_pred != np.arange(n_images) % 10) / n_images
    want_flat = np.arange(5, dtype=np.float32) / 3          # rank 0's weights
    for r in range(world):
        got = np.load(tmp_path / f"r{r}.npz")
        assert float(got["err"]) == want_err
        assert np.array_equal(got["pred"], want_pred)
        assert np.array_equal(got["flat"], want_flat)


# -- the committee driver over gloo with a stand-in backend ----------------------

class _FakeBackend:
    """Deterministic stand-in for the CUDA engine: a 'net' is its seed plus
    the epochs it has seen; its predictions depend on both."""

    def create(self, spec, seed):
        return {"seed": seed, "epochs": 0}

    def train_epoch(self, nets, data, config, epoch):
        for n in nets:
            assert n["epochs"] == epoch
            n["epochs"] += 1

    def predict(self, net, data):
        idx = np.arange(len(data))
        wrong = (idx * (net["seed"] + 3) + net["epochs"] * 5) % 11 == 0
        return np.where(wrong, (data.labels + 1) % 10, data.labels).astype(np.int32)

    def close(self, net):
        net["closed"] = True


def _committee_data():
    train = ck.Dataset(np.zeros((37, 1, 2, 2), np.float32), np.arange(37) % 10, 10, "train")
    test = ck.Dataset(np.zeros((23, 1, 2, 2), np.float32), (np.arange(23) * 3) % 10, 10, "test")
    return train, test


def _committee_worker(rank, world, port, runs, out_dir):
    import torch.distributed as dist

    from paper_1102_0183_b200 import multigpu
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        train, test = _committee_data()
        cfg = ck.TrainConfig(epochs=3, eta0=1e-3, seed=4, test_every=2)
        summary, labels = multigpu.run_committee(None, train, test, cfg, runs,
                                                 backend=_FakeBackend())
        errs = np.array([[(e.train_err, e.test_err) for e in r.epochs] for r in summary.runs])
        np.savez(os.path.join(out_dir, f"c{rank}.npz"), errs=errs, labels=labels,
                 tfbv=[r.tfbv for r in summary.runs], bt=[r.bt for r in summary.runs],
                 best=[r.best_epoch for r in summary.runs], seeds=summary.seeds,
                 mean=summary.tfbv_mean)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("runs", [3, 1, 4])
def test_run_committee_matches_single_process(tmp_path, runs):
    """training.run_experiment's protocol split over 2 ranks (gloo) gives the
    single-process per-epoch errors, TfbV / bT and final labels on every rank."""
    from paper_1102_0183_b200.training import committee_records, summarize
    world = 2
    mp.spawn(_committee_worker, args=(world, _free_port(), runs, str(tmp_path)), nprocs=world)
    train, test = _committee_data()
    cfg = ck.TrainConfig(epochs=3, eta0=1e-3, seed=4, test_every=2)
    seeds = [cfg.seed + r for r in range(runs)]
    records, labels = committee_records(None, train, test, cfg, seeds, _FakeBackend())
    want = summarize(records, seeds)
    errs = np.array([[(e.train_err, e.test_err) for e in r.epochs] for r in want.runs])
    for r in range(world):
        got = np.load(tmp_path / f"c{r}.npz")
        np.testing.assert_array_equal(got["errs"], errs)      # NaN where untested
        np.testing.assert_array_equal(got["labels"], labels)
        np.testing.assert_array_equal(got["tfbv"], [x.tfbv for x in want.runs])
        np.testing.assert_array_equal(got["bt"], [x.bt for x in want.runs])
        np.testing.assert_array_equal(got["best"], [x.best_epoch for x in want.runs])
        np.testing.assert_array_equal(got["seeds"], seeds)
        assert float(got["mean"]) == want.tfbv_mean


# -- bench.py's N>1 control flow, rehearsed on CPU over gloo ---------------------

def test_bench_dry_run_two_ranks():
    """torchrun --nproc-per-node 2 bench.py --gpus 2 --dry-run: one JSON line
    (rank 0 only), value from the MAX over ranks, sharded labels gathered in
    order, errors reduced, rank 0's weights broadcast, committee split."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
         "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
         os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "4", "--warmup", "3",
         "--dry-run"], capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"]
    # rank 1 sleeps twice as long: the reported time is its (the max), not rank 0's
    assert d["ms_per_step"] >= 1.8 * d["my_ms_per_step"]
    assert d["eval"]["labels_ok"]
    idx = np.arange(10_000)
    assert d["eval"]["wrong"] == int(np.count_nonzero(idx % 7 == 3))
    assert d["broadcast_weights"] == [0.0] * 5
    assert d["committee_members"] == 8
