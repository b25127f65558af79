"""Datasets as the engine consumes them: uint8 images plus a 256-entry LUT.

``normalize`` / ``from_bytes`` / ``Dataset`` follow convkit datasets.py:28-98:
a pixel byte b maps to f32(b / 127.5 - 1) computed in f64.  The device never
recomputes that expression; it indexes ``byte_lut()`` (the same 256 f32
values), so device inputs are bit-identical to the reference's.

``make_glyph_images`` is a light, numpy-only stand-in for the reference's
glyph generator (synth.py:30-54, which needs the affine/elastic deformation
pipeline): seeded class prototypes, per-sample shifts and N(0, 8) pixel
noise clipped to [0, 255].  Like the reference's glyphs it has large
constant backgrounds, so pooling sees exact ties.  Parity fixtures that must
match the reference bit for bit use the reference's own glyphs
(tests/golden/).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DataFormatError


def normalize(raw) -> np.ndarray:
    return np.asarray(raw, dtype=np.float64) / 127.5 - 1.0


def byte_lut() -> np.ndarray:
    """f32 value of every byte under ``normalize``."""
    return normalize(np.arange(256)).astype(np.float32)


@dataclass
class Dataset:
    """Labelled images; ``raw`` keeps the source bytes when known."""

    images: np.ndarray          # (n, c, h, w) float32, normalised
    labels: np.ndarray          # (n,) int32
    n_classes: int
    split: str
    raw: np.ndarray | None = None   # (n, c, h, w) uint8

    def __post_init__(self):
        if self.images.ndim != 4 or len(self.labels) != len(self.images):
            raise DataFormatError("images must be (n, c, h, w) with one label each")
        if len(self.images) == 0:
            raise DataFormatError("dataset is empty")
        bad = (self.labels < 0) | (self.labels >= self.n_classes)
        if bad.any():
            raise DataFormatError(
                f"label {int(self.labels[bad.argmax()])} outside [0, {self.n_classes})")
        self._device_cache = {}

    def __len__(self):
        return len(self.images)

    @property
    def channels(self) -> int:
        return self.images.shape[1]

    @property
    def height(self) -> int:
        return self.images.shape[2]

    @property
    def width(self) -> int:
        return self.images.shape[3]

    def limit(self, n: int | None) -> "Dataset":
        if n is None or n >= len(self):
            return self
        if n < 1:
            raise DataFormatError(f"limit must be >= 1, got {n}")
        raw = None if self.raw is None else self.raw[:n]
        return Dataset(self.images[:n], self.labels[:n], self.n_classes, self.split, raw)


def from_bytes(images_u8, labels, n_classes: int, split: str, dtype=None) -> Dataset:
    images_u8 = np.asarray(images_u8, dtype=np.uint8)
    if images_u8.ndim == 3:
        images_u8 = images_u8[:, np.newaxis]
    images = byte_lut()[images_u8] if dtype in (None, np.float32) else \
        normalize(images_u8).astype(dtype)
    return Dataset(images, np.asarray(labels, dtype=np.int32), n_classes, split,
                   np.ascontiguousarray(images_u8))


def _prototype(cls: int, size: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng([seed, cls, 0x917])
    yy, xx = np.mgrid[0:size, 0:size].astype(np.float64)
    img = np.zeros((size, size))
    centre = (size - 1) / 2.0
    for _ in range(4):
        # a stroke: a short segment between two random points, blurred
        p0 = centre + rng.uniform(-0.3, 0.3, 2) * size
        p1 = centre + rng.uniform(-0.3, 0.3, 2) * size
        for t in np.linspace(0.0, 1.0, 12):
            py, px = p0 + t * (p1 - p0)
            img += np.exp(-((yy - py) ** 2 + (xx - px) ** 2) / (2 * (size / 14.0) ** 2))
    img /= img.max()
    return 255.0 * np.clip((img - 0.25) / 0.5, 0.0, 1.0)


def make_glyph_images(n: int, n_classes: int = 10, size: int = 28, seed: int = 0,
                      split: str = "train"):
    """(n, size, size) uint8 glyphs and labels i % n_classes."""
    protos = np.stack([_prototype(c, size, seed) for c in range(n_classes)])
    tag = 0 if split == "train" else 1
    rng = np.random.default_rng([seed, tag, 0xA2])
    shifts = rng.integers(-2, 3, size=(n, 2))
    noise = rng.normal(0.0, 8.0, size=(n, size, size))
    labels = (np.arange(n) % n_classes).astype(np.int32)
    images = np.empty((n, size, size), dtype=np.uint8)
    for i in range(n):
        g = np.roll(protos[labels[i]], tuple(shifts[i]), axis=(0, 1))
        images[i] = np.clip(g + noise[i], 0, 255).astype(np.uint8)
    return images, labels


def make_glyph_dataset(n: int, n_classes: int = 10, size: int = 28, seed: int = 0,
                       split: str = "train", channels: int = 1) -> Dataset:
    """Multi-channel glyph set: channel c drawn with seed + c."""
    chans = []
    labels = None
    for c in range(channels):
        img, labels = make_glyph_images(n, n_classes, size, seed + c, split)
        chans.append(img)
    return from_bytes(np.stack(chans, axis=1), labels, n_classes, split)
