"""Pin the CPU oracle against the reference's own outputs.

tests/golden/*.npz were produced by running convkit itself (float32) in the
build container (tests/golden/make_golden.py).  The oracle must reproduce
them: bit-exact for the six kernels and every conv / pool buffer; the FC
layers go through numpy/OpenBLAS exactly as in the reference, so they are
bit-exact on the same host and within a few ulp on another CPU.
"""

from __future__ import annotations

import hashlib
import warnings

import numpy as np
import pytest

from oracle import oracle
from paper_1102_0183_b200 import parse_architecture
from paper_1102_0183_b200.data import byte_lut

FC_RTOL = 2e-6     # OpenBLAS sgemv blocking / numpy tanh differ across host ISAs
FC_ATOL = 1e-7


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def spec_of(arch):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return parse_architecture(str(arch))


def case(g, k, name):
    return g[f"k{k}_{name}"]


@pytest.mark.parametrize("k", range(24))
def test_kernels_match_reference(golden, k):
    g = golden("kernels")
    (n_src, n_dest, kx, ky, sx, sy, W, H, ow, oh, px, py, pw, ph) = case(g, k, "geom").tolist()
    src = case(g, k, "src")
    a = np.zeros_like(case(g, k, "a"))
    y = np.zeros_like(a)
    oracle.conv_fwd(src, W, case(g, k, "arena"), case(g, k, "fwd_offsets"),
                    case(g, k, "fwd_srcs"), case(g, k, "fwd_widx"), case(g, k, "bias_offset"),
                    kx, ky, sx, sy, a, y, ow, oh)
    np.testing.assert_array_equal(a, case(g, k, "a"))
    np.testing.assert_array_equal(y, case(g, k, "y"))

    pull = np.zeros_like(case(g, k, "pull"))
    oracle.pull_bwd(case(g, k, "delta"), ow, oh, case(g, k, "arena"), case(g, k, "bwd_offsets"),
                    case(g, k, "bwd_dests"), case(g, k, "bwd_widx"), kx, ky, sx, sy, pull, W, H)
    np.testing.assert_array_equal(pull, case(g, k, "pull"))

    grad = np.zeros_like(case(g, k, "grad"))
    oracle.weight_grad(case(g, k, "delta"), ow, oh, src, case(g, k, "pair_dest"),
                       case(g, k, "pair_src"), case(g, k, "pair_offsets"), kx, ky, sx, sy, grad)
    oracle.bias_grad(case(g, k, "delta"), ow, oh, case(g, k, "bias_offset"), grad)
    np.testing.assert_array_equal(grad, case(g, k, "grad"))

    pout = np.zeros_like(case(g, k, "pout"))
    ar = np.zeros_like(case(g, k, "arg_r"))
    ac = np.zeros_like(ar)
    oracle.maxpool_fwd(case(g, k, "psrc"), px, py, pout, pw, ph, ar, ac)
    np.testing.assert_array_equal(pout, case(g, k, "pout"))
    np.testing.assert_array_equal(ar, case(g, k, "arg_r"))
    np.testing.assert_array_equal(ac, case(g, k, "arg_c"))
    back = np.zeros_like(case(g, k, "pback"))
    oracle.maxpool_bwd(case(g, k, "pdelta"), pw, ph, ar, ac, back)
    np.testing.assert_array_equal(back, case(g, k, "pback"))


def test_kernels_thread_count_invariant(golden):
    g = golden("kernels")
    k = 3
    (n_src, n_dest, kx, ky, sx, sy, W, H, ow, oh, *_rest) = case(g, k, "geom").tolist()
    outs = []
    for threads in (1, 4):
        oracle.set_threads(threads)
        pull = np.zeros_like(case(g, k, "pull"))
        oracle.pull_bwd(case(g, k, "delta"), ow, oh, case(g, k, "arena"),
                        case(g, k, "bwd_offsets"), case(g, k, "bwd_dests"),
                        case(g, k, "bwd_widx"), kx, ky, sx, sy, pull, W, H)
        outs.append(pull)
    oracle.set_threads(1)
    np.testing.assert_array_equal(outs[0], outs[1])


NET_NAMES = ("tiny", "imgproc", "poolpool", "convconv", "fconly")


def _compare_layers(net, g, prefix, exact_fc):
    for idx, L in enumerate(net.layers):
        p = f"{prefix}L{idx}_"
        if L.kind in ("input", "image_processing"):
            np.testing.assert_array_equal(L.y, g[p + "y"], err_msg=p + "y")
        elif L.kind == "convolutional":
            for name in ("a", "y", "delta", "grad"):
                np.testing.assert_array_equal(getattr(L, name), g[p + name], err_msg=p + name)
        elif L.kind == "max_pooling":
            for name in ("y", "delta", "arg_r", "arg_c"):
                np.testing.assert_array_equal(getattr(L, name), g[p + name], err_msg=p + name)
        else:
            for name in ("a", "y", "delta", "grad_w", "grad_b"):
                got, want = getattr(L, name), g[p + name]
                if exact_fc:
                    np.testing.assert_array_equal(got, want, err_msg=p + name)
                else:
                    np.testing.assert_allclose(got, want, rtol=FC_RTOL, atol=FC_ATOL,
                                               err_msg=p + name)


@pytest.mark.parametrize("name", NET_NAMES)
def test_oracle_net_one_step_matches_reference(golden, name):
    g = golden("nets")
    p = f"{name}_"
    spec = spec_of(g[p + "arch"])
    net = oracle.OracleNet(spec, int(g[p + "seed"]))
    np.testing.assert_array_equal(net.flat_parameters(), g[p + "params0"])
    imgs = g[p + "images_u8"]
    labels = g[p + "labels"]
    x = byte_lut()[imgs]
    n_cls = spec.n_classes
    loss = net.train_step(x[0], oracle.targets_for(int(labels[0]), n_cls), 1e-2)
    assert loss == pytest.approx(float(g[p + "loss0"]), rel=1e-12)
    _compare_layers(net, g, p + "s0_", exact_fc=False)
    np.testing.assert_allclose(net.flat_parameters(), g[p + "params1"], rtol=0, atol=1e-7)


@pytest.mark.parametrize("name", NET_NAMES)
def test_oracle_net_online_run_matches_reference(golden, name):
    g = golden("nets")
    p = f"{name}_"
    spec = spec_of(g[p + "arch"])
    net = oracle.OracleNet(spec, int(g[p + "seed"]), params=g[p + "params1"])
    imgs, labels = g[p + "images_u8"], g[p + "labels"]
    x = byte_lut()[imgs]
    losses = [net.train_step(x[i], oracle.targets_for(int(labels[i]), spec.n_classes), 1e-2)
              for i in range(1, 31)]
    np.testing.assert_allclose(losses, g[p + "losses"], rtol=1e-6)
    np.testing.assert_allclose(net.flat_parameters(), g[p + "params31"], rtol=0, atol=2e-6)
    pred = [net.predict(x[i]) for i in range(31)]
    np.testing.assert_array_equal(pred, g[p + "pred31"])


@pytest.mark.parametrize("cfg", ("C1", "C2", "C3", "C4", "C4F"))
def test_oracle_configs_match_reference(golden, cfg):
    g = golden("configs")
    p = f"{cfg}_"
    spec = spec_of(g[p + "arch"])
    net = oracle.OracleNet(spec, 0)
    assert sha(net.flat_parameters()) == str(g[p + "params0_digest"])
    for idx, L in enumerate(net.layers):
        if L.kind == "convolutional":
            t = L.table
            assert sha(t._fwd_offsets) + sha(t._fwd_srcs) + sha(t._fwd_widx) == \
                str(g[p + f"L{idx}_fwd_digest"])
            assert sha(t._bwd_offsets) + sha(t._bwd_dests) + sha(t._bwd_widx) == \
                str(g[p + f"L{idx}_bwd_digest"])
    x = byte_lut()[g[p + "image_u8"]]
    t = oracle.targets_for(int(g[p + "label"]), spec.n_classes)
    loss = net.train_step(x, t, 1e-3)
    assert loss == pytest.approx(float(g[p + "loss"]), rel=1e-6)
    for idx, L in enumerate(net.layers):
        q = p + f"L{idx}_"
        if L.kind == "convolutional":
            assert sha(L.a) == str(g[q + "a_digest"]), f"{q} a"
            assert sha(L.y) == str(g[q + "y_digest"]), f"{q} y"
            np.testing.assert_allclose(L.delta.ravel()[g[q + "sel"]], g[q + "delta_sub"],
                                       rtol=1e-5, atol=1e-9)
            np.testing.assert_allclose(L.grad[g[q + "gsel"]], g[q + "grad_sub"],
                                       rtol=1e-5, atol=1e-9)
        elif L.kind == "max_pooling":
            np.testing.assert_array_equal(L.arg_r, g[q + "arg_r"])
            np.testing.assert_array_equal(L.arg_c, g[q + "arg_c"])
        elif L.kind == "image_processing":
            assert sha(L.y) == str(g[q + "y_digest"])
        elif L.kind in ("fully_connected", "output"):
            for name in ("a", "y", "delta"):
                np.testing.assert_allclose(getattr(L, name), g[q + name], rtol=FC_RTOL,
                                           atol=FC_ATOL)
    np.testing.assert_allclose(net.flat_parameters()[g[p + "psel"]], g[p + "params1_sub"],
                               rtol=0, atol=1e-7)
