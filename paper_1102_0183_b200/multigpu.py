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
                  group=None, **net_kwargs):
    """run_experiment with the committee split over the ranks: rank r trains
    members nets_for_rank(runs, r, world) (seeds config.seed + member) in one
    launch per epoch, evaluates them, and the per-member test errors and
    predicted labels are all-gathered.  Returns (test error % per member,
    labels (runs, n_test)) on every rank -- the values a single-GPU
    run_experiment produces."""
    import torch.distributed as dist

    from .network import NetworkState
    from .training import predict_batch, train_committee_epoch

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    mine = nets_for_rank(runs, rank, world)
    nets = [NetworkState(spec, config.seed + m, **net_kwargs) for m in mine]
    for epoch in range(config.epochs):
        if nets:
            train_committee_epoch(nets, train_data, config, epoch)
    errs = np.zeros(runs, dtype=np.int64)
    labels = np.zeros((runs, len(test_data)), dtype=np.int32)
    for m, net in zip(mine, nets):
        labels[m] = predict_batch(net, test_data)
        errs[m] = int(np.count_nonzero(labels[m] != test_data.labels))
        net.close()
    # members are disjoint across ranks: a sum-reduce assembles them
    import torch
    dev = _backend_device(group)
    t_err = torch.as_tensor(errs, device=dev)
    t_lab = torch.as_tensor(labels, device=dev)
    dist.all_reduce(t_err, group=group)
    dist.all_reduce(t_lab, group=group)
    return 100.0 * t_err.cpu().numpy() / len(test_data), t_lab.cpu().numpy()
