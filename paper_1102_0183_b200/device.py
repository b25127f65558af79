"""Device plumbing (PyTorch is used only for memory and streams).

Datasets are uploaded once per (dataset, device) as uint8 (n, C, H, W) plus
the 256-entry normalisation LUT and int32 labels; the CUDA engine reads them
in place for every epoch and every evaluation.
"""

from __future__ import annotations

import numpy as np

from .data import Dataset, byte_lut
from .errors import StateError


def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        raise StateError("no CUDA device is visible (the engine has no CPU fallback)")
    return torch


def current_stream_handle(device: int = 0) -> int:
    torch = torch_cuda()
    return torch.cuda.current_stream(device).cuda_stream


class DeviceDataset:
    """Resident copy of a Dataset on one GPU."""

    def __init__(self, data: Dataset, device: int = 0):
        torch = torch_cuda()
        dev = torch.device("cuda", device)
        self.n = len(data)
        self.device = device
        self.in_shape = (data.channels, data.height, data.width)
        pinned = getattr(data, "_pinned", None)
        if pinned is not None:      # page-locked host copies: async uploads
            self.images = pinned["images"].to(dev, non_blocking=True)
            self.lut = pinned["lut"].to(dev, non_blocking=True)
            self.labels = pinned["labels"].to(dev, non_blocking=True)
            return
        if data.raw is not None:
            self.images = torch.from_numpy(np.require(data.raw, requirements=["C", "W"])).to(dev)
            self.lut = torch.from_numpy(byte_lut()).to(dev)
        else:   # arbitrary float32 inputs: the engine reads them directly
            self.images = torch.from_numpy(
                np.ascontiguousarray(data.images, dtype=np.float32)).to(dev)
            self.lut = None
        self.labels = torch.from_numpy(np.ascontiguousarray(data.labels, np.int32)).to(dev)

    @property
    def images_ptr(self) -> int:
        return self.images.data_ptr()

    @property
    def lut_ptr(self) -> int | None:
        return None if self.lut is None else self.lut.data_ptr()


def pin_dataset(data: Dataset) -> Dataset:
    """Keep page-locked host copies of ``data``'s bytes, LUT and labels so
    that every upload (DeviceDataset) is an async copy from pinned memory."""
    if data.raw is None:
        raise StateError("only byte datasets (from_bytes) can be pinned")
    torch = torch_cuda()
    data._pinned = {
        "images": torch.from_numpy(np.ascontiguousarray(data.raw)).pin_memory(),
        "lut": torch.from_numpy(byte_lut()).pin_memory(),
        "labels": torch.from_numpy(np.ascontiguousarray(data.labels, np.int32)).pin_memory(),
    }
    return data


def upload_bytes(data: Dataset) -> int:
    """Host->device bytes one DeviceDataset upload of ``data`` moves."""
    n = data.raw.nbytes if data.raw is not None else len(data) * data.channels * \
        data.height * data.width * 4
    return int(n + 4 * len(data) + (1024 if data.raw is not None else 0))


def device_dataset(data: Dataset, device: int = 0) -> DeviceDataset:
    cache = getattr(data, "_device_cache", None)
    if cache is None:
        return DeviceDataset(data, device)
    if device not in cache:
        cache[device] = DeviceDataset(data, device)
    return cache[device]
