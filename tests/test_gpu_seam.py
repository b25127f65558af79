"""The operator seam end to end: every arithmetic step of the reference's
NetworkState.train_step (network.py:163-282) has a device entry point --
the six convkit.kernels (kernels.py:70-180), the contrast layer and the FC-side
operators the reference runs inline in numpy (fc_forward / fc_backward /
act_deriv_mul / sgd_update / output_deltas).

  * each FC-side operator against numpy on the reference's expressions;
  * a network walk built ONLY from seam calls reproduces the reference's own
    train_step (tests/golden/nets.npz, made by importing convkit) with the
    tolerances of tests/test_gpu_parity.py;
  * the reference's own convkit.NetworkState, with convkit.kernels pointed at
    the seam (the swap INTEGRATION.md §1 documents), trains bit-identically to
    the unmodified reference -- run wherever convkit can be imported
    (baseline/_ref, installed by the one offline pip install).
"""

from __future__ import annotations

import os
import sys
import tempfile
import warnings

import numpy as np
import pytest

from tests.conftest import ROOT, has_cuda

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]

import paper_1102_0183_b200 as ck  # noqa: E402
from paper_1102_0183_b200 import kernels as gk  # noqa: E402
from oracle import oracle  # noqa: E402

RTOL = 2e-6
F32 = np.float32


def _act(a):
    return (F32(1.7159) * np.tanh(F32(0.6666) * a)).astype(F32)


def _deriv(a):
    t = np.tanh(F32(0.6666) * a)
    return (F32(1.7159 * 0.6666) * (F32(1.0) - t * t)).astype(F32)


@pytest.mark.parametrize("n_in,n_out", [(1, 1), (17, 5), (540, 150), (1200, 300), (150, 10)])
def test_fc_forward_matches_numpy(n_in, n_out):
    rng = np.random.default_rng(n_in * 1000 + n_out)
    x = rng.uniform(-1, 1, n_in).astype(F32)
    W = rng.uniform(-0.05, 0.05, (n_in, n_out)).astype(F32)
    b = rng.uniform(-0.05, 0.05, n_out).astype(F32)
    a = np.zeros(n_out, F32)
    y = np.zeros(n_out, F32)
    gk.fc_forward(x, W, b, a, y)
    want_a = (x.astype(np.float64) @ W.astype(np.float64)).astype(F32) + b
    np.testing.assert_allclose(a, want_a, rtol=RTOL, atol=1e-7)
    np.testing.assert_allclose(y, _act(a), rtol=RTOL, atol=1e-7)


def test_fc_backward_and_update_match_numpy():
    rng = np.random.default_rng(3)
    n_in, n_out = 300, 10
    x = rng.uniform(-1, 1, n_in).astype(F32)
    W = rng.uniform(-0.05, 0.05, (n_in, n_out)).astype(F32)
    b = rng.uniform(-0.05, 0.05, n_out).astype(F32)
    d = rng.uniform(-1, 1, n_out).astype(F32)
    xg = np.zeros(n_in, F32)
    gw = np.zeros_like(W)
    gb = np.zeros_like(b)
    W0, b0 = W.copy(), b.copy()
    gk.fc_backward(x, W, b, d, xg, gw, gb, eta=0.0)
    np.testing.assert_array_equal(W, W0)                      # eta 0: no update
    np.testing.assert_array_equal(gw, np.outer(x, d))         # f32 products: exact
    np.testing.assert_array_equal(gb, d)
    np.testing.assert_allclose(xg, (W0.astype(np.float64) @ d).astype(F32), rtol=RTOL, atol=1e-7)
    eta = 2e-3
    gk.fc_backward(x, W, b, d, eta=eta)
    np.testing.assert_array_equal(W, W0 - eta * np.outer(x, d))   # network.py:271 bits
    np.testing.assert_array_equal(b, b0 - eta * d)
    with pytest.raises(ck.ConfigError):
        gk.fc_backward(x, W, b, d, eta=-1.0)


def test_act_deriv_sgd_and_output_deltas():
    rng = np.random.default_rng(5)
    a = rng.uniform(-3, 3, (3, 7, 32)).astype(F32)
    d = rng.uniform(-1, 1, a.shape).astype(F32)
    want = d.copy()
    want[:, :5, :11] *= _deriv(a[:, :5, :11])
    got = d.copy()
    gk.act_deriv_mul(a, got, width=11, height=5)                # padding untouched
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=1e-8)
    np.testing.assert_array_equal(got[:, 5:, :], d[:, 5:, :])
    np.testing.assert_array_equal(got[:, :, 11:], d[:, :, 11:])
    p = rng.uniform(-1, 1, 1001).astype(F32)
    g = rng.uniform(-1, 1, 1001).astype(F32)
    want = p - 1e-3 * g
    gk.sgd_update(p, g, 1e-3)
    np.testing.assert_array_equal(p, want)
    with pytest.raises(ck.ConfigError):
        gk.sgd_update(p, g, 0.0)
    y = rng.uniform(-1.7, 1.7, 10).astype(F32)
    ao = rng.uniform(-2, 2, 10).astype(F32)
    t = oracle.targets_for(3, 10)
    delta = np.zeros(10, F32)
    loss = gk.output_deltas(y, t, ao, delta)
    np.testing.assert_allclose(delta, oracle.output_deltas(y, t, ao), rtol=RTOL, atol=1e-8)
    assert loss == pytest.approx(oracle.sample_loss(y, t), rel=1e-12)
    # the reference's known answer (test_backprop.py:51-53): y=0, t=1, a=0
    one = np.zeros(1, F32)
    gk.output_deltas(np.zeros(1, F32), np.ones(1), np.zeros(1, F32), one)
    assert one[0] == pytest.approx(-1.7159 * 0.6666, rel=1e-6)


class SeamWalk(oracle.OracleNet):
    """network.py's forward/backward/apply_gradients with EVERY arithmetic
    step routed through the seam (no numpy arithmetic left)."""

    def forward(self, channels):
        first = self.layers[0]
        first.y[:] = channels
        prev = first
        for L in self.layers[1:]:
            if L.kind == "image_processing":
                c = prev.y.shape[0]
                L.y[:c] = prev.y
                L.y[c:] = gk.contrast(prev.y, L.coeffs)
            elif L.kind == "convolutional":
                t = L.table
                gk.conv_fwd(prev.y, prev.y.shape[2], L.arena, t._fwd_offsets, t._fwd_srcs,
                            t._fwd_widx, t.bias_offset, t.kx, t.ky, L.skip[0], L.skip[1],
                            L.a, L.y, L.y.shape[2], L.y.shape[1])
            elif L.kind == "max_pooling":
                gk.maxpool_fwd(prev.y, L.region[0], L.region[1], L.y, L.y.shape[2],
                               L.y.shape[1], L.arg_r, L.arg_c)
            else:
                L.x[:] = prev.y.ravel()
                gk.fc_forward(L.x, L.weights, L.bias, L.a, L.y)
            prev = L
        return self.layers[-1].y

    def backward(self, targets):
        layers = self.layers
        k = len(layers) - 1
        out = layers[k]
        self.loss = gk.output_deltas(out.y, targets, out.a, out.delta)
        while layers[k].kind in ("fully_connected", "output"):
            fc = layers[k]
            xgrad = np.zeros(fc.x.shape, F32)
            gk.fc_backward(fc.x, fc.weights, fc.bias, fc.delta, xgrad, fc.grad_w, fc.grad_b)
            k -= 1
            below = layers[k]
            if below.delta is None:
                return
            below.delta[:] = xgrad.reshape(below.delta.shape)
            if below.kind in ("fully_connected", "output", "convolutional"):
                gk.act_deriv_mul(below.a, below.delta)
        while k >= 1:
            L, prev = layers[k], layers[k - 1]
            if L.kind == "convolutional":
                t = L.table
                dh, dw = L.delta.shape[1], L.delta.shape[2]
                gk.weight_grad(L.delta, dw, dh, prev.y, t._pair_dest, t._pair_src,
                               t.pair_offsets, t.kx, t.ky, L.skip[0], L.skip[1], L.grad)
                gk.bias_grad(L.delta, dw, dh, t.bias_offset, L.grad)
                if prev.delta is None:
                    return
                gk.pull_bwd(L.delta, dw, dh, L.arena, t._bwd_offsets, t._bwd_dests,
                            t._bwd_widx, t.kx, t.ky, L.skip[0], L.skip[1], prev.delta,
                            prev.delta.shape[2], prev.delta.shape[1])
            else:
                if prev.delta is None:
                    return
                prev.delta[:] = 0
                gk.maxpool_bwd(L.delta, L.delta.shape[2], L.delta.shape[1], L.arg_r,
                               L.arg_c, prev.delta)
            if prev.kind == "convolutional":
                gk.act_deriv_mul(prev.a, prev.delta)
            k -= 1

    def apply_gradients(self, eta):
        for L in self.layers:
            if L.kind == "convolutional":
                gk.sgd_update(L.arena, L.grad, eta)
            elif L.kind in ("fully_connected", "output"):
                gk.sgd_update(L.weights, L.grad_w, eta)
                gk.sgd_update(L.bias, L.grad_b, eta)

    def train_step(self, channels, targets, eta):
        self.forward(channels)
        self.backward(targets)
        if eta > 0:
            self.apply_gradients(eta)
        return self.loss


def _spec(arch):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return ck.parse_architecture(str(arch))


@pytest.mark.parametrize("name", ["tiny", "imgproc", "poolpool", "convconv", "fconly"])
def test_seam_only_walk_matches_reference_step(golden, name):
    g = golden("nets")
    p = f"{name}_"
    spec = _spec(g[p + "arch"])
    net = SeamWalk(spec, int(g[p + "seed"]))
    np.testing.assert_array_equal(net.flat_parameters(), g[p + "params0"])
    x = ck.byte_lut()[g[p + "images_u8"]]
    labels = g[p + "labels"]
    loss = net.train_step(x[0], oracle.targets_for(int(labels[0]), spec.n_classes), 1e-2)
    assert loss == pytest.approx(float(g[p + "loss0"]), rel=1e-6)
    for idx, L in enumerate(net.layers):
        q = f"{p}s0_L{idx}_"
        if L.kind in ("input", "image_processing"):
            np.testing.assert_array_equal(L.y, g[q + "y"], err_msg=q)
        elif L.kind == "convolutional":
            np.testing.assert_array_equal(L.a, g[q + "a"], err_msg=q + "a")
            np.testing.assert_array_equal(L.y, g[q + "y"], err_msg=q + "y")
        elif L.kind == "max_pooling":
            np.testing.assert_array_equal(L.arg_r, g[q + "arg_r"], err_msg=q)
            np.testing.assert_array_equal(L.arg_c, g[q + "arg_c"], err_msg=q)
        else:
            np.testing.assert_allclose(L.a, g[q + "a"], rtol=RTOL, atol=1e-8, err_msg=q)
            np.testing.assert_allclose(L.y, g[q + "y"], rtol=RTOL, atol=1e-8, err_msg=q)
    np.testing.assert_allclose(net.flat_parameters(), g[p + "params1"], rtol=0, atol=1e-6)
    for i in range(1, 31):
        net.train_step(x[i], oracle.targets_for(int(labels[i]), spec.n_classes), 1e-2)
    np.testing.assert_allclose(net.flat_parameters(), g[p + "params31"], rtol=0, atol=1e-5)
    np.testing.assert_array_equal([net.predict(x[i]) for i in range(31)], g[p + "pred31"])


def _convkit():
    """The reference package from baseline/_ref (or an installed one)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "convkit")) and ref not in sys.path:
        sys.path.append(ref)
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="ck_numba_"))
    try:
        import convkit
        from convkit import kernels  # noqa: F401  (numba)
    except Exception as e:       # pragma: no cover - depends on the box
        pytest.skip(f"reference package not importable: {e}")
    return convkit


@pytest.mark.parametrize("arch", [
    "input 1x13x13; conv 3M k3x3 s1x1; maxpool 2x2; conv 4M k3x3 s0x0; fc 8N; output 3",
    "input 1x29x29; conv 20M k4x4 s0x0; maxpool 2x2; conv 40M k5x5 s0x0; maxpool 3x3; "
    "fc 150N; output 10",
    "input 1x12x12; conv 4M k3x3 s0x0; conv 5M k2x2 s1x1 rand2; fc 7N; fc 6N; output 3",
], ids=["tiny", "C1", "convconv"])
def test_convkit_network_state_through_seam(arch):
    """the reference's own NetworkState with its
    convkit.kernels pointed at the sm_100a seam trains bit-identically."""
    convkit = _convkit()
    from convkit import kernels as rk
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        spec = convkit.parse_architecture(arch)
    c, w = spec.layers[0].out_maps, spec.layers[0].out_width
    data = ck.make_glyph_dataset(6, spec.n_classes, w, seed=2, channels=c)
    plain = convkit.NetworkState(spec, 3, dtype=F32)
    via = convkit.NetworkState(spec, 3, dtype=F32)
    targets = [convkit.targets_for(int(lb), spec.n_classes) for lb in data.labels]
    want = [plain.train_step(data.images[i], targets[i], 1e-2) for i in range(6)]
    want_pred = [plain.predict(data.images[i]) for i in range(6)]
    saved = {n: getattr(rk, n) for n in gk.SEAM}
    launches0 = ck._lib.kernel_launches()
    try:
        for n in gk.SEAM:
            setattr(rk, n, getattr(gk, n))
        got = [via.train_step(data.images[i], targets[i], 1e-2) for i in range(6)]
        got_pred = [via.predict(data.images[i]) for i in range(6)]
    finally:
        for n, f in saved.items():
            setattr(rk, n, f)
    assert ck._lib.kernel_launches() > launches0          # the seam really ran
    assert got == want
    assert got_pred == want_pred
    for (_, _, a), (_, _, b) in zip(via.parameters(), plain.parameters()):
        np.testing.assert_array_equal(a, b)
