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
