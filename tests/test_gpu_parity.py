"""GPU parity: the sm_100a engine against the oracle and the reference goldens.

Tolerance policy (stated here so the tests are the contract):
  * conv pre-activations / activations, pool outputs and argmax indices,
    predicted labels: BIT-EXACT.
  * f64-accumulated backward sums (pull, weight/bias grads): the device may
    combine partial sums in another order; the f32 result equals the
    reference's except at a rounding boundary -> rtol 2e-6.
  * FC layers: the reference uses OpenBLAS sgemv and numpy's SIMD float32
    tanh; the device uses an f64-accumulated dot and CUDA's tanhf (both
    within ~2 ulp of the true tanh) -> FC a / y / delta within rtol 2e-6.
  * weights after N online steps: max |dw| <= 1e-6 (1 step), 1e-5 (an epoch
    of small nets), 1e-4 (C2, 1000 steps; SURVEY.md §7.3 trajectory bound).
"""

from __future__ import annotations

import warnings

import numpy as np
import pytest

from tests.conftest import has_cuda

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]

import paper_1102_0183_b200 as ck  # noqa: E402
from paper_1102_0183_b200 import kernels as gk  # noqa: E402
from oracle import oracle  # noqa: E402

RTOL = 2e-6
ATOL = 1e-8

C1 = ("input 1x29x29; conv 20M k4x4 s0x0; maxpool 2x2; conv 40M k5x5 s0x0; "
      "maxpool 3x3; fc 150N; output 10")
C2 = ("input 1x29x29; conv 40M k4x4 s0x0; maxpool 2x2; conv 60M k5x5 s0x0; "
      "maxpool 3x3; fc 150N; output 10")
C3 = ("input 2x48x48; imgproc hat21; conv 50M k5x5 s0x0; maxpool 2x2; conv 50M k5x5 s0x0; "
      "maxpool 4x4; fc 300N; output 6")
C4 = ("input 3x32x32; conv 300M k3x3 s0x0; maxpool 2x2; conv 300M k2x2 s0x0 rand30; "
      "maxpool 2x2; conv 300M k3x3 s0x0 rand30; maxpool 2x2; fc 300N; output 10")
C4F = ("input 3x32x32; conv 300M k3x3 s0x0; maxpool 2x2; conv 300M k2x2 s0x0; "
       "maxpool 2x2; conv 300M k3x3 s0x0; maxpool 2x2; fc 300N; output 10")


def spec_of(arch):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return ck.parse_architecture(str(arch))


def assert_close(got, want, msg, rtol=RTOL, atol=ATOL):
    np.testing.assert_allclose(got, want, rtol=rtol, atol=atol, err_msg=msg)


def assert_scaled(got, want, msg, frac=1e-6):
    """Deltas and gradients: the FC layers' few-ulp differences (sgemv /
    numpy tanh vs f64 dot / correctly rounded tanh) propagate into every
    backward sum, whose cancellation turns them into absolute errors of the
    size of the summed terms.  Bound: |diff| <= frac * max|want| + RTOL*|want|."""
    scale = float(np.abs(want).max()) if np.size(want) else 0.0
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=frac * scale + ATOL, err_msg=msg)


def compare_nets(gpu, ref, tag=""):
    for idx, L in enumerate(ref.layers):
        G = gpu.layers[idx]
        p = f"{tag}L{idx}:{L.kind}:"
        if L.kind in ("input", "image_processing"):
            np.testing.assert_array_equal(G.y, L.y, err_msg=p + "y")
        elif L.kind == "convolutional":
            np.testing.assert_array_equal(G.a, L.a, err_msg=p + "a")
            np.testing.assert_array_equal(G.y, L.y, err_msg=p + "y")
            assert_scaled(G.delta, L.delta, p + "delta")
        elif L.kind == "max_pooling":
            np.testing.assert_array_equal(G.y, L.y, err_msg=p + "y")
            np.testing.assert_array_equal(G.arg_r, L.arg_r, err_msg=p + "arg_r")
            np.testing.assert_array_equal(G.arg_c, L.arg_c, err_msg=p + "arg_c")
            assert_scaled(G.delta, L.delta, p + "delta")
        else:
            assert_scaled(G.a, L.a, p + "a")
            assert_scaled(G.y, L.y, p + "y")
            assert_scaled(G.delta, L.delta, p + "delta")


# -- operator seam: each CUDA kernel against the reference's own outputs ----

@pytest.mark.parametrize("k", range(24))
def test_seam_kernels_match_reference(golden, k):
    g = golden("kernels")

    def c(name):
        return g[f"k{k}_{name}"]

    (n_src, n_dest, kx, ky, sx, sy, W, H, ow, oh, px, py, pw, ph) = c("geom").tolist()
    a = np.zeros_like(c("a"))
    y = np.zeros_like(a)
    gk.conv_fwd(c("src"), W, c("arena"), c("fwd_offsets"), c("fwd_srcs"), c("fwd_widx"),
                c("bias_offset"), kx, ky, sx, sy, a, y, ow, oh)
    np.testing.assert_array_equal(a, c("a"))
    np.testing.assert_array_equal(y, c("y"))
    pull = np.zeros_like(c("pull"))
    gk.pull_bwd(c("delta"), ow, oh, c("arena"), c("bwd_offsets"), c("bwd_dests"),
                c("bwd_widx"), kx, ky, sx, sy, pull, W, H)
    np.testing.assert_array_equal(pull, c("pull"))
    grad = np.zeros_like(c("grad"))
    gk.weight_grad(c("delta"), ow, oh, c("src"), c("pair_dest"), c("pair_src"),
                   c("pair_offsets"), kx, ky, sx, sy, grad)
    gk.bias_grad(c("delta"), ow, oh, c("bias_offset"), grad)
    np.testing.assert_array_equal(grad, c("grad"))
    pout = np.zeros_like(c("pout"))
    ar = np.zeros_like(c("arg_r"))
    ac = np.zeros_like(ar)
    gk.maxpool_fwd(c("psrc"), px, py, pout, pw, ph, ar, ac)
    np.testing.assert_array_equal(pout, c("pout"))
    np.testing.assert_array_equal(ar, c("arg_r"))
    np.testing.assert_array_equal(ac, c("arg_c"))
    back = np.zeros_like(c("pback"))
    gk.maxpool_bwd(c("pdelta"), pw, ph, ar, ac, back)
    np.testing.assert_array_equal(back, c("pback"))


def test_seam_contrast_matches_oracle():
    rng = np.random.default_rng(4)
    img = rng.uniform(-1, 1, (2, 48, 48)).astype(np.float32)
    from paper_1102_0183_b200.network import _padded_bank
    bank, _, _ = _padded_bank(("hat21", "sobel"))
    np.testing.assert_array_equal(gk.contrast(img, bank), oracle.contrast(img, bank))


def test_seam_drives_reference_shaped_network():
    """The seam functions run the oracle's network walk (which calls the
    kernels exactly as network.py does) and reproduce its step."""
    spec = spec_of("input 1x13x13; conv 3M k3x3 s1x1; maxpool 2x2; conv 4M k3x3 s0x0; "
                   "fc 8N; output 3")
    x = np.random.default_rng(0).uniform(-1, 1, (1, 13, 13)).astype(np.float32)
    t = oracle.targets_for(1, 3)
    ref = oracle.OracleNet(spec, 2)
    ref.train_step(x, t, 1e-2)
    via = oracle.OracleNet(spec, 2)
    saved = {n: getattr(oracle, n) for n in gk.SEAM}
    try:
        for n in gk.SEAM:
            setattr(oracle, n, getattr(gk, n))
        via.train_step(x, t, 1e-2)
    finally:
        for n, f in saved.items():
            setattr(oracle, n, f)
    np.testing.assert_array_equal(via.flat_parameters(), ref.flat_parameters())


# -- network seam: one full online step ---------------------------------------

NET_NAMES = ("tiny", "imgproc", "poolpool", "convconv", "fconly")


@pytest.mark.parametrize("name", NET_NAMES)
def test_net_step_matches_reference_golden(golden, name):
    g = golden("nets")
    p = f"{name}_"
    spec = spec_of(g[p + "arch"])
    net = ck.NetworkState(spec, int(g[p + "seed"]))
    np.testing.assert_array_equal(net.flat_parameters(), g[p + "params0"])
    x = ck.byte_lut()[g[p + "images_u8"]]
    labels = g[p + "labels"]
    loss = net.train_step(x[0], ck.targets_for(int(labels[0]), spec.n_classes), 1e-2)
    assert loss == pytest.approx(float(g[p + "loss0"]), rel=1e-6)
    for idx, L in enumerate(net.layers):
        q = f"{p}s0_L{idx}_"
        if L.kind in ("input", "image_processing"):
            np.testing.assert_array_equal(L.y, g[q + "y"], err_msg=q)
        elif L.kind == "convolutional":
            np.testing.assert_array_equal(L.a, g[q + "a"], err_msg=q + "a")
            np.testing.assert_array_equal(L.y, g[q + "y"], err_msg=q + "y")
            assert_scaled(L.delta, g[q + "delta"], q + "delta")
        elif L.kind == "max_pooling":
            np.testing.assert_array_equal(L.arg_r, g[q + "arg_r"], err_msg=q)
            np.testing.assert_array_equal(L.arg_c, g[q + "arg_c"], err_msg=q)
            assert_scaled(L.delta, g[q + "delta"], q + "delta")
        else:
            assert_close(L.a, g[q + "a"], q + "a")
            assert_close(L.y, g[q + "y"], q + "y")
            assert_scaled(L.delta, g[q + "delta"], q + "delta")
    assert_close(net.flat_parameters(), g[p + "params1"], "params", rtol=0, atol=1e-6)
    losses = [net.train_step(x[i], ck.targets_for(int(labels[i]), spec.n_classes), 1e-2)
              for i in range(1, 31)]
    np.testing.assert_allclose(losses, g[p + "losses"], rtol=1e-5)
    assert_close(net.flat_parameters(), g[p + "params31"], "params31", rtol=0, atol=1e-5)
    pred = [net.predict(x[i]) for i in range(31)]
    np.testing.assert_array_equal(pred, g[p + "pred31"])
    net.close()


@pytest.mark.parametrize("arch", [C1, C2, C3, C4, C4F], ids=["C1", "C2", "C3", "C4", "C4F"])
def test_config_step_matches_oracle(arch):
    spec = spec_of(arch)
    c, h, w = spec.layers[0].out_maps, spec.layers[0].out_height, spec.layers[0].out_width
    data = ck.make_glyph_dataset(4, spec.n_classes, w, seed=3, channels=c)
    net = ck.NetworkState(spec, 0)
    ref = oracle.OracleNet(spec, 0)
    for i in range(3):
        t = ck.targets_for(int(data.labels[i]), spec.n_classes)
        loss = net.train_step(data.images[i], t, 1e-3)
        ref_loss = ref.train_step(data.images[i], t, 1e-3)
        assert loss == pytest.approx(ref_loss, rel=1e-5)
        if i == 0:
            # identical weights going in: conv / pool forward bit-exact
            compare_nets(net, ref)
    # later steps start from weights that differ at the ulp level
    assert_close(net.flat_parameters(), ref.flat_parameters(), "params", rtol=0, atol=1e-6)
    net.close()


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4", "C4F"])
def test_config_golden_bitexact_conv(golden, cfg):
    """One online step of every BASELINE net against the REFERENCE's own
    digests (tests/golden/configs.npz): conv a / y bit for bit, pool argmax
    indices equal, weights after the update within 1e-6."""
    g = golden("configs")
    import hashlib
    spec = spec_of(g[f"{cfg}_arch"])
    net = ck.NetworkState(spec, 0)
    x = ck.byte_lut()[g[f"{cfg}_image_u8"]]
    t = ck.targets_for(int(g[f"{cfg}_label"]), spec.n_classes)
    net.train_step(x, t, 1e-3)
    for idx, L in enumerate(net.layers):
        q = f"{cfg}_L{idx}_"
        if L.kind == "convolutional":
            assert hashlib.sha256(L.a.tobytes()).hexdigest() == str(g[q + "a_digest"]), q
            assert hashlib.sha256(L.y.tobytes()).hexdigest() == str(g[q + "y_digest"]), q
        elif L.kind == "max_pooling":
            np.testing.assert_array_equal(L.arg_r, g[q + "arg_r"])
            np.testing.assert_array_equal(L.arg_c, g[q + "arg_c"])
    assert_close(net.flat_parameters()[g[f"{cfg}_psel"]], g[f"{cfg}_params1_sub"],
                 cfg, rtol=0, atol=1e-6)
    net.close()


def test_backward_then_apply_equals_fused_step():
    spec = spec_of(C1)
    data = ck.make_glyph_dataset(2, 10, 29, seed=5)
    a = ck.NetworkState(spec, 1)
    b = ck.NetworkState(spec, 1)
    t = ck.targets_for(int(data.labels[0]), 10)
    a.train_step(data.images[0], t, 2e-3)
    b.forward(data.images[0])
    b.backward(t)
    ref = oracle.OracleNet(spec, 1)
    ref.forward(data.images[0])
    ref.backward(t)
    for idx, L in enumerate(ref.layers):
        if L.kind == "convolutional":
            assert_scaled(b.layers[idx].grad, L.grad, f"grad L{idx}")
    b.apply_gradients(2e-3)
    np.testing.assert_array_equal(a.flat_parameters(), b.flat_parameters())
    with pytest.raises(ck.ConfigError):
        b.apply_gradients(0.0)


def test_team_shapes_give_identical_results():
    spec = spec_of(C1)
    data = ck.make_glyph_dataset(24, 10, 29, seed=6)
    cfg = ck.TrainConfig(epochs=1, eta0=1e-3, seed=4)
    results = []
    for team in ((1, 16, 512), (1, 8, 256), (1, 1, 512), (2, 32, 512), (2, 148, 256)):
        net = ck.NetworkState(spec, 3, team=team)
        ck.train_epoch(net, data, cfg, 0)
        results.append(net.flat_parameters())
        net.close()
    for r in results[1:]:
        np.testing.assert_array_equal(r, results[0])


# -- device-resident epochs, evaluation and the committee ---------------------

def test_epoch_matches_oracle_and_eval_labels_bitexact():
    spec = spec_of(C1)
    train = ck.make_glyph_dataset(64, 10, 29, seed=1)
    test = ck.make_glyph_dataset(50, 10, 29, seed=1, split="test")
    cfg = ck.TrainConfig(epochs=1, eta0=1e-3, seed=0)
    net = ck.NetworkState(spec, 0)
    ref = oracle.OracleNet(spec, 0)
    mean = ck.train_epoch(net, train, cfg, 0)
    order = np.random.default_rng([0, 0, 0x5FFE]).permutation(len(train))
    ref_mean = oracle.train_sequence(ref, train.images, train.labels, order, 1e-3, 10)
    assert mean == pytest.approx(ref_mean, rel=1e-5)
    assert_close(net.flat_parameters(), ref.flat_parameters(), "epoch", rtol=0, atol=1e-5)
    # evaluation labels: device batched eval == device single forward == oracle
    pred, out = ck.predict_batch(net, test, outputs=True)
    ref_pred = np.array([ref.predict(test.images[i]) for i in range(len(test))])
    one = np.array([net.predict(test.images[i]) for i in range(len(test))])
    np.testing.assert_array_equal(pred, one)
    net.set_flat_parameters(ref.flat_parameters())
    pred2 = ck.predict_batch(net, test)
    np.testing.assert_array_equal(pred2, ref_pred)
    err = ck.evaluate(net, test)
    assert err == pytest.approx(100.0 * np.count_nonzero(ref_pred != test.labels) / len(test))
    net.close()


def test_committee_equals_sequential_runs():
    spec = spec_of(C1)
    data = ck.make_glyph_dataset(40, 10, 29, seed=2)
    cfg = ck.TrainConfig(epochs=1, eta0=1e-3, seed=0)
    nets = [ck.NetworkState(spec, s) for s in range(3)]
    means = ck.train_committee_epoch(nets, data, cfg, 0)
    for s in range(3):
        solo = ck.NetworkState(spec, s)
        m = ck.train_epoch(solo, data, cfg, 0)
        assert m == means[s]
        np.testing.assert_array_equal(solo.flat_parameters(), nets[s].flat_parameters())
        solo.close()
    for n in nets:
        n.close()


@pytest.mark.slow
def test_c2_trajectory_1000_steps_vs_reference(golden):
    """BASELINE configs[1]: deep MNIST net, 1000 online steps; weights vs the
    reference after steps 1/10/100/1000 (max |dw| <= 1e-4), test labels equal."""
    g = golden("c2_traj")
    spec = spec_of(C2)
    net = ck.NetworkState(spec, 7)
    imgs = g["images_u8"][:, None] if g["images_u8"].ndim == 3 else g["images_u8"]
    labels = g["labels"]
    data = ck.from_bytes(imgs, labels, 10, "train")
    reps = 1000 // len(labels)
    # the fixture visits images 0..199 cyclically: run five unshuffled epochs
    cfg = ck.TrainConfig(epochs=reps, eta0=1e-3, shuffle=False)
    step = 0
    for epoch in range(reps):
        if epoch == 0:
            x = data.images
            for i in range(10):
                net.train_step(x[i], ck.targets_for(int(labels[i]), 10), 1e-3)
                step += 1
                if step in (1, 10):
                    assert_close(net.flat_parameters()[g["psel"]], g[f"params_sub_{step}"],
                                 f"step {step}", rtol=0, atol=1e-5)
            rest = ck.Dataset(data.images[10:], labels[10:], 10, "train", data.raw[10:])
            ck.train_epoch(net, rest, cfg, epoch)
            step += len(rest)
        else:
            ck.train_epoch(net, data, cfg, epoch)
            step += len(data)
        if step == 200:
            pass
    assert step == 1000
    got = net.flat_parameters()[g["psel"]]
    diff = np.abs(got - g["params_sub_1000"]).max()
    assert diff <= 1e-4, diff
    test = ck.from_bytes(g["test_u8"][:, None] if g["test_u8"].ndim == 3 else g["test_u8"],
                         g["test_labels"], 10, "test")
    pred = ck.predict_batch(net, test)
    np.testing.assert_array_equal(pred, g["test_pred"])
    net.close()


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["C3", "C4", "C4F"])
def test_trajectory_vs_reference(golden, cfg):
    """C3 / C4: 200 online steps, C4': 100 (tests/golden/traj_<C>.npz, made by
    the reference): weights within 1e-4 of the reference's at every checkpoint,
    the first losses within 1e-5 relative, test labels identical and test
    outputs within 5e-3 (the FC layers' ulp-level differences -- f64 dot vs
    OpenBLAS sgemv -- enter every update; on C4' the 300-map full tables sum
    them into the outputs: measured 1.2e-3 after 100 steps)."""
    g = golden(f"traj_{cfg}")
    spec = spec_of(g["arch"])
    n_cls = spec.n_classes
    net = ck.NetworkState(spec, int(g["seed"]))
    labels = g["labels"]
    data = ck.from_bytes(g["images_u8"], labels, n_cls, "train")
    steps, n = int(g["steps"]), len(labels)
    checkpoints = g["checkpoints"].tolist()
    cfg_nt = ck.TrainConfig(epochs=1, eta0=1e-3, shuffle=False)
    # single steps up to the first checkpoints, then whole unshuffled epochs
    losses = []
    step = 0
    for i in range(10):
        losses.append(net.train_step(data.images[i], ck.targets_for(int(labels[i]), n_cls), 1e-3))
        step += 1
        if step in checkpoints:
            assert_close(net.flat_parameters()[g["psel"]], g[f"params_sub_{step}"],
                         f"{cfg} step {step}", rtol=0, atol=1e-5)
    rest = ck.Dataset(data.images[10:], labels[10:], n_cls, "train", data.raw[10:])
    ck.train_epoch(net, rest, cfg_nt, 0)
    step += len(rest)
    epoch = 1
    while step < steps:
        ck.train_epoch(net, data, cfg_nt, epoch)
        step += n
        epoch += 1
        if step in checkpoints:
            diff = np.abs(net.flat_parameters()[g["psel"]] - g[f"params_sub_{step}"]).max()
            assert diff <= 1e-4, (cfg, step, diff)
    assert step == steps
    np.testing.assert_allclose(losses, g["losses"][:10], rtol=1e-5)
    diff = np.abs(net.flat_parameters()[g["psel"]] - g[f"params_sub_{steps}"]).max()
    assert diff <= 1e-4, (cfg, diff)
    test = ck.from_bytes(g["test_u8"], g["test_labels"], n_cls, "test")
    pred, out = ck.predict_batch(net, test, outputs=True)
    np.testing.assert_array_equal(pred, g["test_pred"])
    np.testing.assert_allclose(out, g["test_out"], rtol=0, atol=5e-3)
    net.close()


# -- specialised kernels ------------------------------------------------------

@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C4F"])
def test_specialised_kernels_bit_identical_to_generic(name):
    """The BASELINE nets train and evaluate with compile-time specialised
    kernels; the generic interpreter must give the same bits."""
    from paper_1102_0183_b200.configs import spec_for
    spec = spec_for(name)
    first = spec.layers[0]
    n = 24 if name in ("C1", "C2") else (3 if name == "C4F" else 6)
    data = ck.make_glyph_dataset(n, spec.n_classes, first.out_width, seed=4,
                                 channels=first.out_maps)
    cfg = ck.TrainConfig(epochs=1, eta0=1e-3, seed=1)
    fast = ck.NetworkState(spec, 3)
    slow = ck.NetworkState(spec, 3)
    slow.set_specialized(False)
    assert fast.kernel_info() == f"specialised:Spec_{name}"
    assert slow.kernel_info() == "generic"
    m_fast = ck.train_epoch(fast, data, cfg, 0)
    m_slow = ck.train_epoch(slow, data, cfg, 0)
    assert m_fast == m_slow
    np.testing.assert_array_equal(fast.flat_parameters(), slow.flat_parameters())
    p_fast, o_fast = ck.predict_batch(fast, data, outputs=True)
    p_slow, o_slow = ck.predict_batch(slow, data, outputs=True)
    np.testing.assert_array_equal(p_fast, p_slow)
    np.testing.assert_array_equal(o_fast, o_slow)
    fast.close()
    slow.close()


PREPASS_NETS = {
    "C3": None,
    "hat5_sobel": "input 2x16x16; imgproc hat5,sobel; conv 4M k5x5 s0x0 rand3; maxpool 3x3; "
                  "fc 6N; output 4",
    "odd": "input 1x15x15; imgproc hat3; conv 3M k3x3 s0x0; maxpool 2x2; fc 5N; output 3",
}


@pytest.mark.parametrize("name", list(PREPASS_NETS))
@pytest.mark.parametrize("kernel", ["strip", "lanes"])
def test_contrast_prepass_bit_identical(name, kernel):
    """Training launches of nets with an image-processing layer compute it for
    every visited image in a batched prepass (ck_net.cu: the strip kernel, or
    the lane kernel with CKB200_PRE_LANES=1) and skip the per-image phase 0;
    the result must equal the per-image path bit for bit (CKB200_NO_PRE=1
    disables the prepass)."""
    import os
    import warnings
    from paper_1102_0183_b200.configs import spec_for
    if PREPASS_NETS[name] is None:
        spec = spec_for(name)
    else:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            spec = ck.parse_architecture(PREPASS_NETS[name])
    first = spec.layers[0]
    data = ck.make_glyph_dataset(6, spec.n_classes, first.out_width, seed=8,
                                 channels=first.out_maps)
    cfg = ck.TrainConfig(epochs=1, eta0=1e-3, seed=2)
    a = ck.NetworkState(spec, 3)
    b = ck.NetworkState(spec, 3)
    os.environ["CKB200_NO_PRE"] = "1"
    try:
        m_b = ck.train_epoch(b, data, cfg, 0)
    finally:
        del os.environ["CKB200_NO_PRE"]
    if kernel == "lanes":
        os.environ["CKB200_PRE_LANES"] = "1"
    try:
        m_a = ck.train_epoch(a, data, cfg, 0)
    finally:
        os.environ.pop("CKB200_PRE_LANES", None)
    assert m_a == m_b
    np.testing.assert_array_equal(a.flat_parameters(), b.flat_parameters())
    a.close()
    b.close()


@pytest.mark.parametrize("name", ["C3", "C4F"])
def test_epoch_launch_equals_single_steps(name):
    """The epoch launch takes the throughput paths (the contrast prepass, the
    source-pass conv of full tables too big to stage, pooled-only work); the
    per-sample train_step takes the readback paths.  Same arithmetic: the
    weights after the same visits are bit-identical."""
    from paper_1102_0183_b200.configs import spec_for
    spec = spec_for(name)
    first = spec.layers[0]
    data = ck.make_glyph_dataset(3, spec.n_classes, first.out_width, seed=9,
                                 channels=first.out_maps)
    cfg = ck.TrainConfig(epochs=1, eta0=1e-3, shuffle=False)
    a = ck.NetworkState(spec, 4)
    b = ck.NetworkState(spec, 4)
    ck.train_epoch(a, data, cfg, 0)
    for i in range(len(data)):
        b.train_step(data.images[i], ck.targets_for(int(data.labels[i]), spec.n_classes), 1e-3)
    np.testing.assert_array_equal(a.flat_parameters(), b.flat_parameters())
    a.close()
    b.close()
