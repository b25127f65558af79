"""On-line training image deformation on the device (convkit.augment).

Same API as the reference module (augment.py:23-170): ``DeformationConfig``
(per-parameter maxima), ``DeformationParams`` (one sample's concrete warp),
``sample_params`` and ``deform_channels``.  The hot path is
``deform_epoch``: every image of an epoch is deformed in ONE kernel launch
(csrc/ck_deform.cu) — parameters drawn on the device from numpy's
``default_rng([seed, epoch, i])`` stream (SeedSequence + PCG64 restated
bit-exactly), affine + Gaussian-smoothed elastic displacement, one bilinear
``grid-constant`` resampling pass with the border median as background —
into a float32 (n, C, H, W) buffer the training kernel reads directly.
"""

from __future__ import annotations

import dataclasses

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import current_stream_handle, torch_cuda
from .errors import ConfigError


class DeformCfg(C.Structure):
    """Mirror of ``ck_deform_cfg``."""
    _fields_ = [("translate_max", C.c_double), ("rotate_max", C.c_double),
                ("scale_max", C.c_double), ("shear_max", C.c_double),
                ("elastic_sigma", C.c_double), ("elastic_alpha_max", C.c_double)]


class DeformParamsC(C.Structure):
    """Mirror of ``ck_deform_params`` (64 bytes)."""
    _fields_ = [("translate_x", C.c_double), ("translate_y", C.c_double),
                ("rotate", C.c_double), ("scale_x", C.c_double), ("scale_y", C.c_double),
                ("shear_h", C.c_double), ("elastic_alpha", C.c_double),
                ("seed", C.c_uint32), ("pad", C.c_uint32)]


PARAMS_DTYPE = np.dtype([("translate_x", "<f8"), ("translate_y", "<f8"), ("rotate", "<f8"),
                         ("scale_x", "<f8"), ("scale_y", "<f8"), ("shear_h", "<f8"),
                         ("elastic_alpha", "<f8"), ("seed", "<u4"), ("pad", "<u4")])
assert PARAMS_DTYPE.itemsize == C.sizeof(DeformParamsC)


@dataclass
class DeformationParams:
    """One sample's concrete deformation (augment.py:23-40)."""

    translate: tuple[float, float] = (0.0, 0.0)
    rotate: float = 0.0
    scale: tuple[float, float] = (1.0, 1.0)
    shear_h: float = 0.0
    elastic_sigma: float = 6.0
    elastic_alpha: float = 0.0
    seed: int = 0

    def is_identity(self) -> bool:
        return (self.translate == (0.0, 0.0) and self.rotate == 0.0
                and self.scale == (1.0, 1.0) and self.shear_h == 0.0
                and self.elastic_alpha == 0.0)


@dataclass
class DeformationConfig:
    """Per-parameter maxima each training sample draws from (augment.py:43-60)."""

    translate_max: float = 0.0
    rotate_max: float = 0.0
    scale_max: float = 0.0
    shear_max: float = 0.0
    elastic_sigma: float = 6.0
    elastic_alpha_max: float = 0.0

    def __post_init__(self):
        for name in ("translate_max", "rotate_max", "scale_max", "shear_max",
                     "elastic_alpha_max"):
            if getattr(self, name) < 0:
                raise ConfigError(f"{name} must be >= 0")
        if self.elastic_alpha_max > 0 and self.elastic_sigma <= 0:
            raise ConfigError("elastic_sigma must be > 0 when elastic is on")

    def enabled(self) -> bool:
        return any(getattr(self, n) > 0 for n in
                   ("translate_max", "rotate_max", "scale_max", "shear_max",
                    "elastic_alpha_max"))

    def c_struct(self) -> DeformCfg:
        return DeformCfg(self.translate_max, self.rotate_max, self.scale_max,
                         self.shear_max, self.elastic_sigma, self.elastic_alpha_max)


def sample_params(config: DeformationConfig, rng_seed) -> DeformationParams:
    """One sample's deformation, deterministically from the seed
    (augment.py:63-80; the device kernel draws the identical stream)."""
    rng = np.random.default_rng(rng_seed)
    tx, ty, rot, sx, sy, shear = rng.uniform(-1.0, 1.0, 6)
    alpha = rng.uniform(0.0, 1.0)
    seed = int(rng.integers(0, 2**31 - 1))
    return DeformationParams(
        translate=(tx * config.translate_max, ty * config.translate_max),
        rotate=rot * config.rotate_max,
        scale=(1.0 + sx * config.scale_max, 1.0 + sy * config.scale_max),
        shear_h=shear * config.shear_max, elastic_sigma=config.elastic_sigma,
        elastic_alpha=alpha * config.elastic_alpha_max, seed=seed)


def gaussian_taps(sigma: float, truncate: float = 3.0) -> np.ndarray:
    """scipy.ndimage._gaussian_kernel1d(sigma, 0, int(truncate*sigma + 0.5)):
    the normalised f64 taps the elastic smoothing uses (augment.py:111-113)."""
    if sigma <= 0:
        raise ConfigError(f"elastic sigma must be > 0, got {sigma}")
    radius = int(truncate * float(sigma) + 0.5)
    x = np.arange(-radius, radius + 1)
    phi = np.exp(-0.5 / (sigma * sigma) * x ** 2)
    return phi / phi.sum()


def _check_scale(scale_x: float, scale_y: float) -> None:
    if scale_x == 0 or scale_y == 0:
        raise ConfigError("scale factor 0 would collapse the image")


class _Taps:
    """Device copies of the Gaussian taps, one per (sigma, device)."""
    cache: dict = {}

    @classmethod
    def get(cls, sigma: float, device: int):
        key = (float(sigma), device)
        if key not in cls.cache:
            torch = torch_cuda()
            w = gaussian_taps(sigma)
            cls.cache[key] = (torch.from_numpy(w).to(torch.device("cuda", device)),
                              len(w) // 2)
        return cls.cache[key]


def deform_epoch(dd, config: DeformationConfig, seed: int, epoch: int, out=None,
                 params_out=None, stream=None):
    """Deform every image i of device dataset ``dd`` with
    ``sample_params(config, [seed, epoch, i])`` (training.py:140-144) into a
    float32 (n, C, H, W) device tensor (``out`` or a new one); one launch."""
    torch = torch_cuda()
    n = dd.n
    c, h, w = dd.in_shape
    dev = torch.device("cuda", dd.device)
    if out is None:
        out = torch.empty((n, c, h, w), dtype=torch.float32, device=dev)
    if not isinstance(config, DeformationConfig):   # e.g. convkit's (same fields)
        config = DeformationConfig(**{f.name: getattr(config, f.name)
                                      for f in dataclasses.fields(DeformationConfig)})
    taps, radius = _Taps.get(config.elastic_sigma if config.elastic_sigma > 0 else 1.0,
                             dd.device)
    cfg = config.c_struct()
    _lib.call("ck_deform_epoch", dd.images_ptr, dd.lut_ptr, c, h, w, n, C.byref(cfg),
              taps.data_ptr(), radius, int(seed), int(epoch),
              None if params_out is None else params_out.data_ptr(), out.data_ptr(),
              current_stream_handle(dd.device) if stream is None else stream)
    return out


def params_array(params: list[DeformationParams]) -> np.ndarray:
    a = np.zeros(len(params), dtype=PARAMS_DTYPE)
    for i, p in enumerate(params):
        _check_scale(*p.scale)
        a[i] = (p.translate[0], p.translate[1], p.rotate, p.scale[0], p.scale[1], p.shear_h,
                p.elastic_alpha, p.seed, 0)
    return a


def deform_batch(images: np.ndarray, params: list[DeformationParams],
                 device: int = 0) -> np.ndarray:
    """deform_channels for a batch of float32 (n, C, H, W) host images with
    explicit per-image parameters (all sharing one elastic sigma)."""
    torch = torch_cuda()
    images = np.ascontiguousarray(images, dtype=np.float32)
    n, c, h, w = images.shape
    if len(params) != n:
        raise ConfigError(f"{len(params)} parameter sets for {n} images")
    sigmas = {p.elastic_sigma for p in params if p.elastic_alpha > 0}
    if len(sigmas) > 1:
        raise ConfigError("one elastic sigma per batch")
    sigma = sigmas.pop() if sigmas else 1.0
    dev = torch.device("cuda", device)
    src = torch.from_numpy(images).to(dev)
    prm = torch.from_numpy(params_array(params).view(np.uint8)).to(dev)
    out = torch.empty_like(src)
    taps, radius = _Taps.get(sigma, device)
    _lib.call("ck_deform_apply", src.data_ptr(), None, c, h, w, n, prm.data_ptr(),
              taps.data_ptr(), radius, out.data_ptr(), current_stream_handle(device))
    return out.cpu().numpy()


def deform_channels(channels: np.ndarray, params: DeformationParams,
                    device: int = 0) -> np.ndarray:
    """Apply one sample's deformation to every channel of a (c, h, w) image
    (augment.py:150-170); identity parameters return ``channels`` itself."""
    if params.is_identity():
        return channels
    return deform_batch(np.asarray(channels)[None], [params], device)[0]


def border_intensity(channel: np.ndarray) -> float:
    """Median intensity of the outer one-pixel frame (augment.py:143-147)."""
    frame = np.concatenate([channel[0], channel[-1], channel[1:-1, 0], channel[1:-1, -1]])
    return float(np.median(frame))


__all__ = ["DeformationConfig", "DeformationParams", "sample_params", "deform_channels",
           "deform_batch", "deform_epoch", "gaussian_taps", "border_intensity"]
