"""CPU restatement of the reference's on-line deformation (TEST INFRASTRUCTURE ONLY).

Follows ``convkit.augment`` (/root/reference/pkg/src/convkit/augment.py) and
restates the third-party arithmetic it relies on, so the device kernel
(csrc/ck_deform.cu) can be checked step by step:

* numpy 2.3 ``default_rng(seed)``: ``SeedSequence`` entropy pool + PCG64
  (XSL-RR 128/64), ``next_double = (u64 >> 11) * 2**-53``, ``uniform(lo, hi)
  = lo + (hi - lo) * next_double``, ``integers(0, 2**31 - 1)`` through the
  buffered 32-bit Lemire bound (numpy/random/src/distributions).
  Pure-Python integers here; pinned against numpy in tests/test_deform_host.py.
* scipy 1.18 ``ndimage.gaussian_filter(..., mode="constant", truncate=3.0)``:
  ``_gaussian_kernel1d`` weights, one ``correlate1d`` per axis (axis 0 then 1),
  symmetric-kernel order ``out = x[0]*w[0]; out += (x[-j] + x[+j]) * w[-j]``
  for j = radius..1 (ni_filters.c NI_Correlate1D), zero padding.
* scipy ``ndimage.map_coordinates(order=1, mode="grid-constant", cval=bg)``:
  start = floor(c), w0 = 1 - (c - floor c), w1 = 1 - w0, taps outside the
  image read ``bg``; value = sum over corners (row-major) of
  coeff * w_row * w_col, accumulated from 0.0 in f64, rounded to f32.
* ``augment.sample_params`` (augment.py:63-80), ``_affine_source_grid``
  (:83-105), ``_elastic_field`` (:108-114), ``border_intensity`` (:143-147),
  ``deform_channels`` (:150-170).

Only tests/ may import this module.
"""

from __future__ import annotations

import math

import numpy as np

MASK32 = 0xFFFFFFFF
MASK64 = (1 << 64) - 1
MASK128 = (1 << 128) - 1

# numpy/random/bit_generator.pyx SeedSequence constants
INIT_A = 0x43B0D7E5
MULT_A = 0x931E8875
INIT_B = 0x8B51F9DD
MULT_B = 0x58F38DED
MIX_MULT_L = 0xCA01F9DD
MIX_MULT_R = 0x4973F715
XSHIFT = 16
POOL_SIZE = 4

# pcg64.h PCG_DEFAULT_MULTIPLIER_128
PCG_MULT = (2549297995355413924 << 64) + 4865540595714422341


def _entropy_words(seed) -> list[int]:
    """``_coerce_to_uint32_array`` for a non-negative int or a sequence of them."""
    vals = seed if isinstance(seed, (list, tuple, np.ndarray)) else [seed]
    words = []
    for v in vals:
        v = int(v)
        if v < 0:
            raise ValueError("negative entropy")
        if v == 0:
            words.append(0)
        while v > 0:
            words.append(v & MASK32)
            v >>= 32
    return words


def seed_sequence_state(seed, n_words64: int = 4) -> list[int]:
    """SeedSequence(seed).generate_state(n_words64, np.uint64)."""
    entropy = _entropy_words(seed)
    hc = INIT_A

    def hashmix(value):
        nonlocal hc
        value = (value ^ hc) & MASK32
        hc = (hc * MULT_A) & MASK32
        value = (value * hc) & MASK32
        return value ^ (value >> XSHIFT)

    def mix(x, y):
        r = (MIX_MULT_L * x - MIX_MULT_R * y) & MASK32
        return r ^ (r >> XSHIFT)

    pool = [hashmix(entropy[i] if i < len(entropy) else 0) for i in range(POOL_SIZE)]
    for s in range(POOL_SIZE):
        for d in range(POOL_SIZE):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(POOL_SIZE, len(entropy)):
        for d in range(POOL_SIZE):
            pool[d] = mix(pool[d], hashmix(entropy[s]))
    hb = INIT_B
    out32 = []
    for i in range(2 * n_words64):
        v = pool[i % POOL_SIZE]
        v = (v ^ hb) & MASK32
        hb = (hb * MULT_B) & MASK32
        v = (v * hb) & MASK32
        out32.append(v ^ (v >> XSHIFT))
    return [out32[2 * i] | (out32[2 * i + 1] << 32) for i in range(n_words64)]


class PCG64:
    """numpy.random.PCG64 seeded from a SeedSequence (pcg64_srandom_r)."""

    def __init__(self, seed):
        s = seed_sequence_state(seed, 4)
        initstate = (s[0] << 64) | s[1]
        initseq = (s[2] << 64) | s[3]
        self.inc = ((initseq << 1) | 1) & MASK128
        self.state = 0
        self._step()
        self.state = (self.state + initstate) & MASK128
        self._step()
        self.has32 = False
        self.buf32 = 0

    def _step(self):
        self.state = (self.state * PCG_MULT + self.inc) & MASK128

    def next64(self) -> int:
        self._step()
        s = self.state
        x = ((s >> 64) ^ s) & MASK64
        rot = s >> 122
        return ((x >> rot) | (x << ((64 - rot) & 63))) & MASK64

    def next32(self) -> int:
        if self.has32:
            self.has32 = False
            return self.buf32
        v = self.next64()
        self.has32 = True
        self.buf32 = v >> 32
        return v & MASK32

    def next_double(self) -> float:
        return float(self.next64() >> 11) * (1.0 / 9007199254740992.0)

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.next_double()

    def bounded32(self, rng: int) -> int:
        """integers(0, rng + 1) for rng < 2**32 - 1 (buffered Lemire, unmasked)."""
        excl = rng + 1
        m = self.next32() * excl
        left = m & MASK32
        if left < excl:
            thresh = (MASK32 - rng) % excl
            while left < thresh:
                m = self.next32() * excl
                left = m & MASK32
        return m >> 32


def sample_params(cfg, seed):
    """augment.sample_params (augment.py:63-80) on the restated generator.
    ``cfg`` has the DeformationConfig fields; returns a dict."""
    g = PCG64(seed)
    tx, ty, rot, sx, sy, shear = [g.uniform(-1.0, 1.0) for _ in range(6)]
    alpha = g.uniform(0.0, 1.0)
    eseed = g.bounded32(2**31 - 2)
    return dict(translate=(tx * cfg.translate_max, ty * cfg.translate_max),
                rotate=rot * cfg.rotate_max,
                scale=(1.0 + sx * cfg.scale_max, 1.0 + sy * cfg.scale_max),
                shear_h=shear * cfg.shear_max, elastic_sigma=cfg.elastic_sigma,
                elastic_alpha=alpha * cfg.elastic_alpha_max, seed=eseed)


def is_identity(p) -> bool:
    return (p["translate"] == (0.0, 0.0) and p["rotate"] == 0.0 and p["scale"] == (1.0, 1.0)
            and p["shear_h"] == 0.0 and p["elastic_alpha"] == 0.0)


def gaussian_weights(sigma: float, truncate: float = 3.0) -> np.ndarray:
    """scipy _gaussian_kernel1d(sigma, 0, int(truncate*sigma + 0.5))."""
    radius = int(truncate * float(sigma) + 0.5)
    x = np.arange(-radius, radius + 1)
    phi = np.exp(-0.5 / (sigma * sigma) * x ** 2)
    return phi / phi.sum()


def correlate1d_sym(line: np.ndarray, w: np.ndarray) -> np.ndarray:
    """NI_Correlate1D, symmetric odd kernel, constant-0 border, f64."""
    r = len(w) // 2
    n = len(line)
    pad = np.zeros(n + 2 * r)
    pad[r:r + n] = line
    out = pad[r:r + n] * w[r]
    for j in range(r, 0, -1):
        out = out + (pad[r - j:r - j + n] + pad[r + j:r + j + n]) * w[r - j]
    return out


def gaussian_filter2d(a: np.ndarray, w: np.ndarray) -> np.ndarray:
    t = np.stack([correlate1d_sym(a[:, c], w) for c in range(a.shape[1])], axis=1)
    return np.stack([correlate1d_sym(t[r], w) for r in range(a.shape[0])], axis=0)


def elastic_field(width, height, sigma, alpha, seed):
    """augment._elastic_field (augment.py:108-114) on the restated generator."""
    g = PCG64(seed)
    f = np.array([g.uniform(-1.0, 1.0) for _ in range(2 * height * width)]).reshape(
        2, height, width)
    w = gaussian_weights(sigma)
    return alpha * np.stack([gaussian_filter2d(f[0], w), gaussian_filter2d(f[1], w)])


def affine_grid(width, height, p):
    """augment._affine_source_grid (augment.py:83-105); the 2x2 inverse is
    taken in closed form (numpy uses LAPACK: last-ulp differences)."""
    sx, sy = p["scale"]
    rot = math.radians(p["rotate"])
    sh = math.radians(p["shear_h"])
    c, s, t = math.cos(rot), math.sin(rot), math.tan(sh)
    # m = R @ Shear @ Scale
    m00, m01 = c * sx, (c * t - s) * sy
    m10, m11 = s * sx, (s * t + c) * sy
    det = m00 * m11 - m01 * m10
    i00, i01, i10, i11 = m11 / det, -m01 / det, -m10 / det, m00 / det
    cx, cy = (width - 1) / 2.0, (height - 1) / 2.0
    dx, dy = p["translate"][0] * width, p["translate"][1] * height
    cols, rows = np.meshgrid(np.arange(width, dtype=np.float64),
                             np.arange(height, dtype=np.float64))
    rx, ry = cols - cx - dx, rows - cy - dy
    return i10 * rx + i11 * ry + cy, i00 * rx + i01 * ry + cx


def interp_bilinear(img: np.ndarray, rows: np.ndarray, cols: np.ndarray, bg: float):
    """map_coordinates(order=1, mode='grid-constant', cval=bg) -> img.dtype."""
    h, w = img.shape
    out = np.empty(rows.shape, dtype=img.dtype)
    for idx in np.ndindex(rows.shape):
        r, c = float(rows[idx]), float(cols[idx])
        r0, c0 = math.floor(r), math.floor(c)
        wr0 = 1.0 - (r - r0)
        wc0 = 1.0 - (c - c0)
        wr = (wr0, 1.0 - wr0)
        wc = (wc0, 1.0 - wc0)
        t = 0.0
        for i in range(2):
            for j in range(2):
                rr, cc = r0 + i, c0 + j
                v = float(img[rr, cc]) if (0 <= rr < h and 0 <= cc < w) else bg
                t += v * wr[i] * wc[j]
        out[idx] = t
    return out


def border_intensity(ch: np.ndarray) -> float:
    frame = np.concatenate([ch[0], ch[-1], ch[1:-1, 0], ch[1:-1, -1]])
    return float(np.median(frame))


def deform_channels(channels: np.ndarray, p) -> np.ndarray:
    """augment.deform_channels (augment.py:150-170)."""
    if is_identity(p):
        return channels
    _, h, w = channels.shape
    rows, cols = affine_grid(w, h, p)
    if p["elastic_alpha"] > 0:
        d = elastic_field(w, h, p["elastic_sigma"], p["elastic_alpha"], p["seed"])
        rows = rows + d[0]
        cols = cols + d[1]
    out = np.empty_like(channels)
    for c in range(channels.shape[0]):
        out[c] = interp_bilinear(channels[c], rows, cols, border_intensity(channels[c]))
    return out
