"""CPU pins of the deformation restatement (oracle/deform.py).

* the restated numpy generator (SeedSequence + PCG64, uniform, the bounded
  integer draw) equals numpy's default_rng bit for bit;
* the restated Gaussian smoothing and bilinear grid-constant resampling equal
  scipy.ndimage bit for bit;
* the restated deform_channels reproduces the REFERENCE's outputs
  (tests/golden/deform.npz, made by running convkit.augment) and a deformed
  online epoch of the reference's train_epoch (training.py:140-144);
* the package's host-side API (augment.sample_params, DeformationConfig
  validation) matches the reference's.
"""

from __future__ import annotations

import numpy as np
import pytest
from scipy import ndimage

from oracle import deform as D
from oracle.oracle import OracleNet
from paper_1102_0183_b200 import augment, parse_architecture, targets_for
from paper_1102_0183_b200.data import byte_lut
from paper_1102_0183_b200.errors import ConfigError

from tests.golden.cases import DEFORM_CFGS, DEFORM_SHAPES

TINY = "input 1x13x13; conv 3M k3x3 s1x1; maxpool 2x2; conv 4M k3x3 s0x0; fc 8N; output 3"

SEEDS = [0, 1, 12345, [0, 0, 5], [7, 3, 59999], [2**40 + 3, 1], 2**31 - 5, [5, 2, 0]]


@pytest.mark.parametrize("seed", SEEDS, ids=str)
def test_restated_generator_matches_numpy(seed):
    g = D.PCG64(seed)
    raw = np.random.default_rng(seed).bit_generator.random_raw(8)
    assert [g.next64() for _ in range(8)] == [int(v) for v in raw]
    g = D.PCG64(seed)
    r = np.random.default_rng(seed)
    assert [g.uniform(-1.0, 1.0) for _ in range(6)] == list(r.uniform(-1.0, 1.0, 6))
    assert g.uniform(0.0, 1.0) == r.uniform(0.0, 1.0)
    assert g.bounded32(2**31 - 2) == int(r.integers(0, 2**31 - 1))


def test_bounded_draw_over_many_streams():
    for s in range(500):
        cfg = augment.DeformationConfig(rotate_max=1.0)
        p = D.sample_params(cfg, [1, 2, s])
        q = augment.sample_params(cfg, [1, 2, s])
        assert p["seed"] == q.seed and p["rotate"] == q.rotate


@pytest.mark.parametrize("sigma", [6.0, 4.0, 1.5, 0.7])
def test_gaussian_matches_scipy(sigma):
    a = np.random.default_rng(int(sigma * 10)).uniform(-1, 1, (29, 31))
    got = D.gaussian_filter2d(a, D.gaussian_weights(sigma))
    ref = ndimage.gaussian_filter(a, sigma, mode="constant", truncate=3.0)
    assert np.array_equal(got, ref)
    assert np.array_equal(augment.gaussian_taps(sigma), D.gaussian_weights(sigma))


def test_bilinear_matches_scipy():
    rng = np.random.default_rng(3)
    img = rng.uniform(-1, 1, (17, 19)).astype(np.float32)
    rows = rng.uniform(-3, 20, (17, 19))
    cols = rng.uniform(-3, 22, (17, 19))
    rows[0, :6] = [-1.0, -0.5, 0.0, 16.0, 16.5, 7.0]
    cols[0, :6] = [0.0, 18.0, -1e-17, 18.0000001, 3.0, 7.0]
    got = D.interp_bilinear(img, rows, cols, 0.3)
    ref = ndimage.map_coordinates(img, [rows, cols], order=1, mode="grid-constant", cval=0.3)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("shape", list(DEFORM_SHAPES))
@pytest.mark.parametrize("cfg_name", list(DEFORM_CFGS))
def test_oracle_deform_matches_reference(golden, shape, cfg_name):
    g = golden("deform")
    cfg = augment.DeformationConfig(**DEFORM_CFGS[cfg_name])
    x = byte_lut()[g[f"{shape}_u8"]]
    want_p = g[f"{shape}_{cfg_name}_params"]
    want = g[f"{shape}_{cfg_name}_out"]
    for i in range(len(x)):
        p = D.sample_params(cfg, [5, 2, i])
        got_p = [*p["translate"], p["rotate"], *p["scale"], p["shear_h"],
                 p["elastic_alpha"], float(p["seed"])]
        assert got_p == list(want_p[i])
        hp = augment.sample_params(cfg, [5, 2, i])       # package host API
        assert [*hp.translate, hp.rotate, *hp.scale, hp.shear_h, hp.elastic_alpha,
                float(hp.seed)] == list(want_p[i])
        out = D.deform_channels(x[i], p)
        # numpy's LAPACK 2x2 inverse vs the closed form: last-ulp coordinates
        np.testing.assert_allclose(out, want[i], rtol=0, atol=1e-6)
        assert np.count_nonzero(out != want[i]) <= out.size // 100


def test_oracle_deformed_epoch_matches_reference(golden):
    g = golden("deform")
    spec = parse_architecture(TINY)
    net = OracleNet(spec, 4)
    x = byte_lut()[g["epoch_u8"]]
    labels = g["epoch_labels"]
    cfg = augment.DeformationConfig(**DEFORM_CFGS["all"])
    order = np.random.default_rng([5, 1, 0x5FFE]).permutation(len(x))
    total = 0.0
    for i in order:
        xi = D.deform_channels(x[i], D.sample_params(cfg, [5, 1, int(i)]))
        total += net.train_step(xi, targets_for(int(labels[i]), 3), 1e-2)
    assert abs(total / len(x) - float(g["epoch_loss"])) <= 1e-6
    np.testing.assert_allclose(net.flat_parameters(), g["epoch_params"], rtol=0, atol=1e-6)


def test_config_validation_mirrors_reference():
    with pytest.raises(ConfigError):
        augment.DeformationConfig(rotate_max=-1.0)
    with pytest.raises(ConfigError):
        augment.DeformationConfig(elastic_alpha_max=1.0, elastic_sigma=0.0)
    assert not augment.DeformationConfig().enabled()
    assert augment.DeformationConfig(shear_max=1.0).enabled()
    assert augment.sample_params(augment.DeformationConfig(), 3).is_identity()


def test_border_intensity():
    img = np.zeros((5, 5))
    img[0, :] = 2.0
    assert augment.border_intensity(np.full((5, 5), -1.0)) == -1.0
    assert augment.border_intensity(img) == 0.0
