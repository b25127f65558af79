"""Multi-GPU driver: sharded test-set evaluation and committees.

Online training is sequential -- every update depends on the previous image
-- so a single net never spans GPUs ("replicas only").  What
partitions is (a) the images of a test-set evaluation and (b) the independent
nets of a committee (training.run_experiment, training.py:181-199).  One
process per GPU (torch.distributed, NCCL over NVLink); the only collectives
are an all-gather of int32 predicted labels, an all-reduce of int64 error
counts and, to evaluate one trained net everywhere, a broadcast of its
weights.  Every result equals the single-GPU (and CPU reference) result
exactly: labels and error counts are integers.

The collective plumbing is backend-agnostic (tensors live on the backend's
device: CUDA for NCCL, CPU for gloo), so the host logic is tested on CPU with
gloo and a stand-in predictor; the product predictor is ck_net_eval.
"""

from __future__ import annotations

import numpy as np

from .data import Dataset
from .errors import ConfigError


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [first, first+count) of n items for rank (ceil split)."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError(f"bad rank {rank} of {world}")
    per = (n + world - 1) // world
    first = min(rank * per, n)
    return first, max(0, min(per, n - first))


def nets_for_rank(n_nets: int, rank: int, world: int) -> list[int]:
    """Committee members trained on this rank (contiguous blocks, so a GPU
    trains its members together in one launch)."""
    first, count = shard_range(n_nets, rank, world)
    return list(range(first, first + count))


def _backend_device(group=None):
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def gather_shards(local: np.ndarray, n_total: int, group=None) -> np.ndarray:
    """All-gather equally padded per-rank int32 shards into the full vector
    (identical on every rank)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    per = (n_total + world - 1) // world
    dev = _backend_device(group)
    buf = torch.zeros(per, dtype=torch.int32, device=dev)
    if len(local):
        buf[:len(local)] = torch.as_tensor(np.asarray(local, dtype=np.int32), device=dev)
    out = torch.zeros(per * world, dtype=torch.int32, device=dev)
    dist.all_gather_into_tensor(out, buf, group=group)
    return out[:n_total].cpu().numpy()


def all_reduce_count(count: int, group=None) -> int:
    import torch
    import torch.distributed as dist
    t = torch.tensor([int(count)], dtype=torch.int64, device=_backend_device(group))
    dist.all_reduce(t, group=group)
    return int(t.item())


def _device_predictor(net, data: Dataset, engine: str = "exact"):
    """Shard predictor backed by the CUDA engine (ck_net_eval, or the
    tensor-core path with engine="tc")."""
    from .device import device_dataset, torch_cuda
    from .training import eval_range_async

    torch = torch_cuda()
    dd = device_dataset(data, net.device)

    def predict(first: int, count: int) -> np.ndarray:
        if count == 0:
            return np.zeros(0, np.int32)
        pred = torch.empty(count, dtype=torch.int32, device=torch.device("cuda", net.device))
        eval_range_async(net, dd, first, count, pred, engine=engine)
        return pred.cpu().numpy()

    return predict


def sharded_evaluate(net, data: Dataset, group=None, predictor=None, engine: str = "exact"):
    """training.evaluate over a test set split across the ranks of ``group``.

    Returns (error percent, predicted labels of ALL images) on every rank.
    ``predictor(first, count) -> labels`` defaults to the CUDA engine
    (``engine`` = "exact" bit-exact SIMT path, "tc" tensor-core path).
    """
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    first, count = shard_range(len(data), rank, world)
    predict = predictor or _device_predictor(net, data, engine)
    local = np.asarray(predict(first, count), dtype=np.int32)
    wrong = int(np.count_nonzero(local != data.labels[first:first + count]))
    labels = gather_shards(local, len(data), group)
    wrong = all_reduce_count(wrong, group)
    return 100.0 * wrong / len(data), labels


def broadcast_parameters(net, src: int = 0, group=None) -> None:
    """Copy rank ``src``'s weights into ``net`` on every rank."""
    import torch
    import torch.distributed as dist
    flat = torch.as_tensor(net.flat_parameters(), device=_backend_device(group))
    dist.broadcast(flat, src, group=group)
    net.set_flat_parameters(flat.cpu().numpy())


def run_committee(spec, train_data: Dataset, test_data: Dataset, config, runs: int,
                  group=None, backend=None, **net_kwargs):
    """run_experiment (training.py:181-199) with the committee split over the
    ranks of ``group``: rank r trains members nets_for_rank(runs, r, world)
    (seeds config.seed + member) together, one launch per epoch, with
    run_training's protocol per member (validation on the training set every
    epoch, the test set on the test_every cadence, TfbV / bT).  Each rank's
    per-epoch errors and final test labels are all-gathered, so every rank
    returns (ExperimentSummary, final test labels (runs, n_test)) -- the same
    values a single-process run_experiment produces for the same seeds."""
    import torch
    import torch.distributed as dist

    from .training import CudaBackend, EpochStats, RunRecord, committee_records, summarize

    if runs < 1:
        raise ConfigError(f"need at least one run, got {runs}")
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    mine = nets_for_rank(runs, rank, world)
    backend = backend or CudaBackend(**net_kwargs)
    records, labels = committee_records(spec, train_data, test_data, config,
                                        [config.seed + m for m in mine], backend)
    per = (runs + world - 1) // world           # member slots per rank (padded)
    ep = config.epochs
    dev = _backend_device(group)
    stats = torch.zeros((per, ep, 4), dtype=torch.float64, device=dev)
    lab = torch.zeros((per, len(test_data)), dtype=torch.int32, device=dev)
    for j, rec in enumerate(records):
        stats[j] = torch.as_tensor([[st.lr, st.train_err, st.test_err, st.seconds]
                                    for st in rec.epochs], dtype=torch.float64, device=dev)
        lab[j] = torch.as_tensor(labels[j], device=dev)
    all_stats = torch.zeros((world * per, ep, 4), dtype=torch.float64, device=dev)
    all_lab = torch.zeros((world * per, len(test_data)), dtype=torch.int32, device=dev)
    dist.all_gather_into_tensor(all_stats, stats, group=group)
    dist.all_gather_into_tensor(all_lab, lab, group=group)
    all_stats = all_stats.cpu().numpy()
    all_lab = all_lab.cpu().numpy()
    out_records, out_labels = [], np.zeros((runs, len(test_data)), dtype=np.int32)
    for r in range(world):
        for j, m in enumerate(nets_for_rank(runs, r, world)):
            rec = RunRecord()
            for e in range(ep):
                lr, tr, te, sec = all_stats[r * per + j, e]
                rec.epochs.append(EpochStats(e, float(lr), float(tr), float(te), float(sec)))
            rec.finalize()
            out_records.append(rec)
            out_labels[m] = all_lab[r * per + j]
    return summarize(out_records, [config.seed + m for m in range(runs)]), out_labels
