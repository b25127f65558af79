"""Host-side logic of the package (no GPU): architecture grammar, geometry,
connection tables, filters, data LUT, the C-ABI library and its exports, and
the CPU oracle's C2 trajectory against the reference."""

from __future__ import annotations

import ctypes as C
import hashlib
import os
import re
import warnings

import numpy as np
import pytest

import paper_1102_0183_b200 as ck
from paper_1102_0183_b200 import configs
from paper_1102_0183_b200 import _lib
from paper_1102_0183_b200.errors import (ConfigError, GeometryError, GeometryWarning,
                                         PrecisionError)
from tests.conftest import ROOT


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# -- grammar and geometry (reference tests/test_arch.py) --------------------

def test_mnist_chain_sizes():
    spec = ck.parse_architecture(
        "input 1x29x29; conv 20M k4x4 s0x0; maxpool 2x2; conv 40M k5x5 s0x0; "
        "maxpool 3x3; fc 150N; output 10")
    assert [l.out_width for l in spec.layers] == [29, 26, 13, 9, 3, 1, 1]
    assert [l.out_maps for l in spec.layers] == [1, 20, 20, 40, 40, 150, 10]


def test_cifar_chain_widths():
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        spec = ck.parse_architecture(
            "input 3x32x32; conv 300M k3x3 s0x0; maxpool 2x2; conv 300M k2x2 s0x0 rand30; "
            "maxpool 2x2; conv 300M k3x3 s0x0 rand30; maxpool 2x2; fc 300N; output 10")
    assert [l.out_width for l in spec.layers] == [32, 30, 15, 14, 7, 5, 2, 1, 1]
    assert any(issubclass(x.category, GeometryWarning) for x in w)   # 5 -> 2 truncation


def test_imgproc_map_count_and_position():
    spec = ck.parse_architecture("input 2x48x48; imgproc hat21; conv 5M k5x5 s0x0; output 6")
    assert spec.layers[1].out_maps == 6
    with pytest.raises(ConfigError):
        ck.parse_architecture("input 1x20x20; conv 2M k3x3 s0x0; imgproc sobel; output 2")
    with pytest.raises(ConfigError):
        ck.parse_architecture("input 1x20x20; imgproc hat4; output 2")


def test_skip_placement_eq1():
    assert ck.output_map_size(29, 5, 1) == 13
    for prev in range(1, 20):
        for k in range(1, prev + 1):
            for s in range(3):
                n = ck.output_map_size(prev, k, s)
                assert (n - 1) * (s + 1) + k <= prev < n * (s + 1) + k


@pytest.mark.parametrize("text,err", [
    ("conv 2M k3x3 s0x0; output 2", ConfigError),
    ("input 1x8x8; fc 3N", ConfigError),
    ("input 1x8x8; conv 2M k9x9 s0x0; output 2", GeometryError),
    ("input 1x8x8; maxpool 9x1; output 2", GeometryError),
    ("input 1x8x8; fc 3N; conv 2M k2x2 s0x0; output 2", ConfigError),
    ("input 1x8x8; conv 2M k3x3 s0x0 rand3; output 2", ConfigError),
    ("input 1x8x8; bogus 3; output 2", ConfigError),
])
def test_bad_architectures(text, err):
    with pytest.raises(err):
        ck.parse_architecture(text)


def test_experiment_settings_split():
    spec, cfg = ck.parse_experiment("input 1x8x8\neta0 = 0.001 # comment\noutput 3")
    assert cfg == {"eta0": "0.001"} and spec.n_classes == 3
    with pytest.raises(ConfigError):
        ck.parse_architecture("input 1x8x8; eta0=1; output 3")


# -- connection tables (reference tests/test_topology.py) -------------------

def test_arena_tiling_and_transpose():
    t = ck.build_random_table(6, 5, 3, [1, 2], (3, 2))
    blocks = []
    for d, row in enumerate(t.forward):
        for s in row:
            blocks.append((t.weight_index[d, s], 6))
        blocks.append((t.bias_offset[d], 1))
    covered = np.zeros(t.arena_size, int)
    for off, n in blocks:
        covered[off:off + n] += 1
    assert (covered == 1).all()
    for s, row in enumerate(t.backward):
        for d in row:
            assert s in t.forward[d]
    assert sorted(t._bwd_dests.tolist()) == sorted(t._pair_dest.tolist())


def test_random_table_degree_coverage_and_seed():
    t = ck.build_random_table(300, 300, 30, [0x7AB1E, 3], (2, 2))
    assert all(len(r) == 30 and r == sorted(r) for r in t.forward)
    assert len({s for r in t.forward for s in r}) == 300
    t2 = ck.build_random_table(300, 300, 30, [0x7AB1E, 3], (2, 2))
    assert t.forward == t2.forward


def test_tables_match_reference_digests(golden):
    g = golden("configs")
    for cfg in ("C1", "C2", "C3", "C4", "C4F"):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            spec = ck.parse_architecture(str(g[f"{cfg}_arch"]))
        prev = None
        for idx, ls in enumerate(spec.layers):
            if ls.kind == "convolutional":
                if ls.connectivity == "random":
                    t = ck.build_random_table(prev.out_maps, ls.maps, ls.in_degree,
                                              [0x7AB1E, idx], ls.kernel)
                else:
                    t = ck.build_full_table(prev.out_maps, ls.maps, ls.kernel)
                assert sha(t._fwd_offsets) + sha(t._fwd_srcs) + sha(t._fwd_widx) == \
                    str(g[f"{cfg}_L{idx}_fwd_digest"])
                assert sha(t._bwd_offsets) + sha(t._bwd_dests) + sha(t._bwd_widx) == \
                    str(g[f"{cfg}_L{idx}_bwd_digest"])
            prev = ls


# -- filters and data -------------------------------------------------------

def test_contrast_pair_properties():
    on, off = ck.make_contrast_filters(21, 21 / 8, 21 / 4)
    np.testing.assert_array_equal(off, -on)
    assert abs(on.sum()) < 1e-12 and abs((on * on).sum() - 1) < 1e-12
    np.testing.assert_allclose(on, on.T, atol=1e-15)
    assert ck.expand_selection(["hat21", "sobel"]) == ["hat21_on", "hat21_off",
                                                       "sobel_x", "sobel_y"]


def test_sobel_ramp_response_is_8():
    from oracle import oracle
    ramp = np.tile(np.arange(12, dtype=np.float32), (10, 1))[None]
    resp = oracle.contrast(ramp, ck.filter_coefficients("sobel_x")[None])
    assert (resp[0, :, 1:-1] == 8.0).all()


def test_byte_lut_is_reference_normalisation():
    lut = ck.byte_lut()
    ref = (np.arange(256, dtype=np.float64) / 127.5 - 1.0).astype(np.float32)
    np.testing.assert_array_equal(lut, ref)
    d = ck.from_bytes(np.arange(256, dtype=np.uint8).reshape(4, 8, 8), [0, 1, 2, 3], 4, "x")
    np.testing.assert_array_equal(d.images.ravel(), ref)


def test_glyph_generator_has_constant_background():
    imgs, labels = ck.make_glyph_images(50, 10, 29, seed=1)
    assert imgs.shape == (50, 29, 29) and labels.tolist() == [i % 10 for i in range(50)]
    assert (imgs == 0).mean() > 0.2          # saturated background -> pooling ties


def test_network_rejects_double_precision():
    spec = ck.parse_architecture("input 1x8x8; fc 3N; output 2")
    with pytest.raises(PrecisionError):
        ck.NetworkState(spec, 0, dtype=np.float64)


def test_init_matches_reference_digest(golden):
    from oracle import oracle
    g = golden("configs")
    for cfg in ("C1", "C4", "C4F"):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            spec = ck.parse_architecture(str(g[f"{cfg}_arch"]))
        assert sha(oracle.OracleNet(spec, 0).flat_parameters()) == str(g[f"{cfg}_params0_digest"])


# -- the C ABI library --------------------------------------------------------

def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "ckb200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ck_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_lib.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 25
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) == set(_lib.EXPORTED_SYMBOLS)


def test_library_abi_and_error_path_without_gpu():
    lib = _lib.load()
    assert lib.ck_abi_version() == 1
    # argument validation runs before any CUDA call and maps to the reference types
    with pytest.raises(ConfigError):
        _lib.call("ck_net_create", None, 0, 0, None)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True)
    assert "sm_100a" in out.stdout


# -- oracle trajectory against the reference (BASELINE configs[1]) -----------

def test_oracle_c2_trajectory_matches_reference(golden):
    from oracle import oracle
    g = golden("c2_traj")
    spec = ck.parse_architecture(
        "input 1x29x29; conv 40M k4x4 s0x0; maxpool 2x2; conv 60M k5x5 s0x0; "
        "maxpool 3x3; fc 150N; output 10")
    net = oracle.OracleNet(spec, 7)
    x = ck.byte_lut()[g["images_u8"]]
    labels = g["labels"]
    losses = []
    for step in range(1, 1001):
        i = (step - 1) % len(labels)
        losses.append(net.train_step(x[i], oracle.targets_for(int(labels[i]), 10), 1e-3))
        if step in (1, 10, 100, 1000):
            got = net.flat_parameters()[g["psel"]]
            np.testing.assert_allclose(got, g[f"params_sub_{step}"], rtol=0, atol=1e-6)
    np.testing.assert_allclose(losses, g["losses"], rtol=1e-5)
    xt = ck.byte_lut()[g["test_u8"]]
    pred = [net.predict(xt[i]) for i in range(len(xt))]
    np.testing.assert_array_equal(pred, g["test_pred"])


# -- oracle trajectories of the larger nets (tests/golden/traj_<C>.npz) -------

@pytest.mark.parametrize("cfg", ["C3", "C4", "C4F"])
def test_oracle_trajectory_matches_reference(golden, cfg):
    """C3 / C4 (200 online steps) and C4' (100): the oracle's weights follow
    the reference's to 1e-6 at every checkpoint, test labels identical."""
    from oracle import oracle
    g = golden(f"traj_{cfg}")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        spec = ck.parse_architecture(str(g["arch"]))
    assert str(g["arch"]) == configs.ARCH[cfg]
    net = oracle.OracleNet(spec, int(g["seed"]))
    x = ck.byte_lut()[g["images_u8"]]
    labels = g["labels"]
    n_cls = spec.n_classes
    steps = int(g["steps"])
    checkpoints = set(g["checkpoints"].tolist())
    losses = []
    for step in range(1, steps + 1):
        i = (step - 1) % len(labels)
        losses.append(net.train_step(x[i], oracle.targets_for(int(labels[i]), n_cls), 1e-3))
        if step in checkpoints:
            got = net.flat_parameters()[g["psel"]]
            np.testing.assert_allclose(got, g[f"params_sub_{step}"], rtol=0, atol=1e-6,
                                       err_msg=f"step {step}")
    np.testing.assert_allclose(losses, g["losses"], rtol=1e-5)
    xt = ck.byte_lut()[g["test_u8"]]
    out = np.stack([net.forward(xt[i]).copy() for i in range(len(xt))])
    np.testing.assert_allclose(out, g["test_out"], rtol=0, atol=1e-5)
    np.testing.assert_array_equal(out.argmax(axis=1), g["test_pred"])
