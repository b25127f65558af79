"""Coefficients of the fixed image-processing (contrast / edge) layer.

Only the coefficient construction lives on the host; the correlation itself
is the CUDA ``ck_contrast`` kernel (f64 accumulate, replicated border, one
rounding to f32 — the arithmetic of ``scipy.ndimage.correlate(mode="nearest")``
used by the reference, filters.py:153-175).

Coefficients follow the reference:
  * Sobel / Scharr x-kernels and their transposes        (filters.py:20-25)
  * hat<N>: zero-sum unit-norm difference of Gaussians, sigma N/8 and N/4,
    off-center = -on-center                              (filters.py:88-123)
  * selection expansion and output order: original channels, then per
    expanded filter, per channel                         (filters.py:129-175)
"""

from __future__ import annotations

import re

import numpy as np

from .errors import ConfigError

SOBEL_X = np.array([[-1.0, 0.0, 1.0], [-2.0, 0.0, 2.0], [-1.0, 0.0, 1.0]])
SCHARR_X = np.array([[-3.0, 0.0, 3.0], [-10.0, 0.0, 10.0], [-3.0, 0.0, 3.0]])

_HAT = re.compile(r"hat(\d+)")


def make_contrast_filters(size: int, sigma_center: float, sigma_surround: float):
    """(on_center, off_center) DoG pair: zero mean, unit L2 norm, off = -on."""
    if size < 1 or size % 2 == 0:
        raise ConfigError(f"contrast filter size must be odd, got {size}")
    if not 0 < sigma_center < sigma_surround:
        raise ConfigError(f"need 0 < sigma_center < sigma_surround, got "
                          f"{sigma_center} and {sigma_surround}")
    half = size // 2
    axis = np.arange(-half, half + 1, dtype=np.float64)
    gx, gy = np.meshgrid(axis, axis)
    radius2 = gx * gx + gy * gy

    def normalised_gaussian(sigma):
        g = np.exp(-radius2 / (2.0 * sigma * sigma))
        return g / g.sum()

    on = normalised_gaussian(sigma_center) - normalised_gaussian(sigma_surround)
    on -= on.mean()
    on /= np.sqrt((on * on).sum())
    return on, -on


def expand_selection(selection) -> list[str]:
    """sobel -> sobel_x, sobel_y; hatN -> hatN_on, hatN_off."""
    names: list[str] = []
    for item in selection:
        if item in ("sobel", "scharr"):
            names.extend((f"{item}_x", f"{item}_y"))
            continue
        m = _HAT.fullmatch(item)
        if m is None:
            raise ConfigError(f"unknown filter selection {item!r}")
        size = int(m.group(1))
        if size % 2 == 0:
            raise ConfigError(f"hat size {size} must be odd")
        names.extend((f"hat{size}_on", f"hat{size}_off"))
    return names


def filter_coefficients(name: str) -> np.ndarray:
    """(fh, fw) float64 coefficients of one expanded filter name."""
    if name == "sobel_x":
        return SOBEL_X.copy()
    if name == "sobel_y":
        return SOBEL_X.T.copy()
    if name == "scharr_x":
        return SCHARR_X.copy()
    if name == "scharr_y":
        return SCHARR_X.T.copy()
    if name.startswith("hat") and name.endswith(("_on", "_off")):
        size = int(name[3:].split("_")[0])
        on, off = make_contrast_filters(size, size / 8.0, size / 4.0)
        return np.ascontiguousarray(on if name.endswith("_on") else off)
    raise ConfigError(f"unknown filter {name!r}")


def selection_bank(selection) -> list[np.ndarray]:
    """Coefficient arrays in output order for an imgproc selection."""
    return [filter_coefficients(n) for n in expand_selection(selection)]
