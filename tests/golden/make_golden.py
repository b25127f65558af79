"""Generate golden fixtures by running the REFERENCE (convkit) in float32.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nbcache \
        python tests/golden/make_golden.py

Writes, next to this script:
  kernels.npz   per-kernel cases on random pitched geometries (kernels.py)
  nets.npz      small architectures: one full train_step with every layer
                buffer, then a 30-step online run (network.py / training.py)
  configs.npz   the BASELINE configs C1-C4: table / init / one-step digests
                plus dense FC buffers
  c2_traj.npz   deep-MNIST C2: 1000 online steps, weight subsamples after
                steps 1/10/100/1000, per-step losses (BASELINE configs[1])
  traj_<C>.npz  C3 / C4 / C4': multi-step online trajectories (weights after
                steps 1/10/half/all, losses, test labels and outputs)
  deform.npz    augment.sample_params / deform_channels on C1/C3/C4-shaped
                glyphs under several DeformationConfigs, and one deformed
                online epoch of a small net (training.py:140-144)
Large arrays are stored as sha256 digests of their float32 bytes plus
seeded subsamples so the fixtures stay small.
"""

from __future__ import annotations

import hashlib
import os
import sys
import warnings

import numpy as np

import convkit as ck
from convkit import kernels
from convkit.synth import make_glyph_images

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from cases import DEFORM_CFGS, DEFORM_SHAPES  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
F32 = np.float32

SMALL_NETS = {
    "tiny": "input 1x13x13; conv 3M k3x3 s1x1; maxpool 2x2; conv 4M k3x3 s0x0; fc 8N; output 3",
    "imgproc": "input 2x16x16; imgproc hat5,sobel; conv 4M k5x5 s0x0 rand3; maxpool 3x3; fc 6N; output 4",
    "poolpool": "input 1x20x20; maxpool 2x2; conv 3M k3x3 s0x0; maxpool 2x2; maxpool 2x2; output 5",
    "convconv": "input 1x12x12; conv 4M k3x3 s0x0; conv 5M k2x2 s1x1 rand2; fc 7N; fc 6N; output 3",
    "fconly": "input 1x6x6; fc 9N; output 4",
}

CONFIGS = {
    "C1": "input 1x29x29; conv 20M k4x4 s0x0; maxpool 2x2; conv 40M k5x5 s0x0; maxpool 3x3; fc 150N; output 10",
    "C2": "input 1x29x29; conv 40M k4x4 s0x0; maxpool 2x2; conv 60M k5x5 s0x0; maxpool 3x3; fc 150N; output 10",
    "C3": "input 2x48x48; imgproc hat21; conv 50M k5x5 s0x0; maxpool 2x2; conv 50M k5x5 s0x0; maxpool 4x4; fc 300N; output 6",
    "C4": "input 3x32x32; conv 300M k3x3 s0x0; maxpool 2x2; conv 300M k2x2 s0x0 rand30; maxpool 2x2; conv 300M k3x3 s0x0 rand30; maxpool 2x2; fc 300N; output 10",
    # C4' (SURVEY §8d stress case): the same net with full connection tables
    # (topology.py:126-130 build_full_table)
    "C4F": "input 3x32x32; conv 300M k3x3 s0x0; maxpool 2x2; conv 300M k2x2 s0x0; maxpool 2x2; conv 300M k3x3 s0x0; maxpool 2x2; fc 300N; output 10",
}

# multi-step online trajectories of the larger BASELINE nets (VERDICT r1:
# C2 alone had one): (init seed, online steps, distinct train images, test images)
TRAJ = {"C3": (7, 200, 100, 60), "C4": (7, 200, 100, 60), "C4F": (7, 100, 50, 40)}


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


def glyph_images(n, n_classes, size, channels, seed, split="train"):
    """(n, C, size, size) uint8 + labels; channel c from seed+c."""
    chans = []
    labels = None
    for c in range(channels):
        img, lab = make_glyph_images(n, n_classes, size, seed + c, split)
        chans.append(img)
        labels = lab
    return np.stack(chans, axis=1), labels


def pitched(rng, maps, h, w, quantum=32):
    pitch = ((w + quantum - 1) // quantum) * quantum
    a = np.zeros((maps, h, pitch), F32)
    a[:, :, :w] = rng.uniform(-1, 1, (maps, h, w))
    return a


def kernel_cases(seed=11, n_cases=24):
    rng = np.random.default_rng(seed)
    out = {}
    for case in range(n_cases):
        n_src = int(rng.integers(1, 5))
        n_dest = int(rng.integers(1, 5))
        kx, ky = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        sx, sy = int(rng.integers(0, 3)), int(rng.integers(0, 3))
        W = int(rng.integers(kx, kx + 14))
        H = int(rng.integers(ky, ky + 14))
        ow = ck.output_map_size(W, kx, sx)
        oh = ck.output_map_size(H, ky, sy)
        if rng.uniform() < 0.5:
            table = ck.build_full_table(n_src, n_dest, (kx, ky))
        else:
            deg = int(rng.integers(1, n_src + 1))
            deg = max(deg, -(-n_src // n_dest))
            table = ck.build_random_table(n_src, n_dest, deg, [seed, case], (kx, ky))
        arena = rng.uniform(-0.5, 0.5, table.arena_size).astype(F32)
        src = pitched(rng, n_src, H, W)
        a = ck.new_stack(n_dest, ow, oh, dtype=F32).data
        y = np.zeros_like(a)
        kernels.conv_fwd.serial(src, W, arena, table._fwd_offsets, table._fwd_srcs,
                                table._fwd_widx, table.bias_offset, kx, ky, sx, sy,
                                a, y, ow, oh)
        delta = np.zeros_like(a)
        delta[:, :, :ow] = rng.uniform(-1, 1, (n_dest, oh, ow))
        pull = ck.new_stack(n_src, W, H, dtype=F32).data
        kernels.pull_bwd.serial(delta, ow, oh, arena, table._bwd_offsets, table._bwd_dests,
                                table._bwd_widx, kx, ky, sx, sy, pull, W, H)
        g = np.zeros_like(arena)
        kernels.weight_grad.serial(delta, ow, oh, src, table._pair_dest, table._pair_src,
                                   table.pair_offsets, kx, ky, sx, sy, g)
        kernels.bias_grad.serial(delta, ow, oh, table.bias_offset, g)
        px, py = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        px, py = min(px, W), min(py, H)
        pw, ph = W // px, H // py
        # quantised values create exact ties, exercising the first-in-scan rule
        psrc = np.round(pitched(rng, n_src, H, W) * 2) / 2
        pout = ck.new_stack(n_src, pw, ph, dtype=F32).data
        arg_r = np.zeros((n_src, ph, pw), np.int64)
        arg_c = np.zeros_like(arg_r)
        kernels.maxpool_fwd.serial(psrc, px, py, pout, pw, ph, arg_r, arg_c)
        pdelta = np.zeros_like(pout)
        pdelta[:, :, :pw] = rng.uniform(-1, 1, (n_src, ph, pw))
        back = np.zeros_like(psrc)
        kernels.maxpool_bwd.serial(pdelta, pw, ph, arg_r, arg_c, back)
        p = f"k{case}_"
        out.update({
            p + "geom": np.array([n_src, n_dest, kx, ky, sx, sy, W, H, ow, oh, px, py, pw, ph]),
            p + "fwd_offsets": table._fwd_offsets, p + "fwd_srcs": table._fwd_srcs,
            p + "fwd_widx": table._fwd_widx, p + "bias_offset": table.bias_offset,
            p + "bwd_offsets": table._bwd_offsets, p + "bwd_dests": table._bwd_dests,
            p + "bwd_widx": table._bwd_widx, p + "pair_dest": table._pair_dest,
            p + "pair_src": table._pair_src, p + "pair_offsets": table.pair_offsets,
            p + "arena": arena, p + "src": src, p + "a": a, p + "y": y, p + "delta": delta,
            p + "pull": pull, p + "grad": g, p + "psrc": psrc, p + "pout": pout,
            p + "arg_r": arg_r, p + "arg_c": arg_c, p + "pdelta": pdelta, p + "pback": back,
        })
    out["n_cases"] = np.array(n_cases)
    return out


def dump_layers(net, prefix, out):
    for idx, layer in enumerate(net.layers):
        p = f"{prefix}L{idx}_"
        kind = layer.kind
        if kind in ("input", "image_processing"):
            out[p + "y"] = layer.y.view.copy()
        elif kind == "convolutional":
            out[p + "a"] = layer.a.view.copy()
            out[p + "y"] = layer.y.view.copy()
            out[p + "delta"] = layer.delta.view.copy()
            out[p + "grad"] = layer.grad.copy()
        elif kind == "max_pooling":
            out[p + "y"] = layer.y.view.copy()
            out[p + "delta"] = layer.delta.view.copy()
            out[p + "arg_r"] = layer.arg_r.copy()
            out[p + "arg_c"] = layer.arg_c.copy()
        else:
            out[p + "a"] = layer.a.copy()
            out[p + "y"] = layer.y.copy()
            out[p + "delta"] = layer.delta.copy()
            out[p + "grad_w"] = layer.grad_w.copy()
            out[p + "grad_b"] = layer.grad_b.copy()


def flat_params(net):
    return np.concatenate([a.ravel() for _, _, a in net.parameters()]).astype(F32)


def small_nets():
    out = {}
    for name, arch in SMALL_NETS.items():
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            spec = ck.parse_architecture(arch)
        c, w, h = spec.layers[0].out_maps, spec.layers[0].out_width, spec.layers[0].out_height
        n_cls = spec.n_classes
        seed = 5
        net = ck.NetworkState(spec, seed, dtype=F32)
        imgs, labels = glyph_images(31, n_cls, w, c, seed=3)
        labels = labels % n_cls
        x = ck.from_bytes(imgs, labels, n_cls, "train", F32).images
        p = f"{name}_"
        out[p + "arch"] = np.array(arch)
        out[p + "seed"] = np.array(seed)
        out[p + "images_u8"] = imgs
        out[p + "labels"] = labels
        out[p + "params0"] = flat_params(net)
        t = ck.targets_for(int(labels[0]), n_cls)
        loss = net.train_step(x[0], t, 1e-2)
        out[p + "loss0"] = np.array(loss)
        dump_layers(net, p + "s0_", out)
        out[p + "params1"] = flat_params(net)
        losses = []
        for i in range(1, 31):
            losses.append(net.train_step(x[i], ck.targets_for(int(labels[i]), n_cls), 1e-2))
        out[p + "losses"] = np.array(losses)
        out[p + "params31"] = flat_params(net)
        out[p + "pred31"] = np.array([net.predict(x[i]) for i in range(31)])
    return out


def configs():
    out = {}
    rng = np.random.default_rng(99)
    for name, arch in CONFIGS.items():
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            spec = ck.parse_architecture(arch)
        c, w, h = spec.layers[0].out_maps, spec.layers[0].out_width, spec.layers[0].out_height
        n_cls = spec.n_classes
        net = ck.NetworkState(spec, 0, dtype=F32)
        p = f"{name}_"
        out[p + "arch"] = np.array(arch)
        for idx, layer in enumerate(net.layers):
            if layer.kind == "convolutional":
                t = layer.table
                out[p + f"L{idx}_fwd_digest"] = np.array(
                    digest(t._fwd_offsets) + digest(t._fwd_srcs) + digest(t._fwd_widx))
                out[p + f"L{idx}_bwd_digest"] = np.array(
                    digest(t._bwd_offsets) + digest(t._bwd_dests) + digest(t._bwd_widx))
        params0 = flat_params(net)
        out[p + "params0_digest"] = np.array(digest(params0))
        imgs, labels = glyph_images(1, n_cls, w, c, seed=1)
        x = ck.from_bytes(imgs, labels, n_cls, "train", F32).images[0]
        out[p + "image_u8"] = imgs[0]
        out[p + "label"] = labels[0]
        loss = net.train_step(x, ck.targets_for(int(labels[0]), n_cls), 1e-3)
        out[p + "loss"] = np.array(loss)
        for idx, layer in enumerate(net.layers):
            q = p + f"L{idx}_"
            if layer.kind == "convolutional":
                out[q + "a_digest"] = np.array(digest(layer.a.view.copy()))
                out[q + "y_digest"] = np.array(digest(layer.y.view.copy()))
                sel = rng.choice(layer.a.view.size, size=min(512, layer.a.view.size), replace=False)
                out[q + "sel"] = sel
                out[q + "a_sub"] = layer.a.view.ravel()[sel]
                out[q + "delta_sub"] = layer.delta.view.ravel()[sel]
                gsel = rng.choice(layer.grad.size, size=min(512, layer.grad.size), replace=False)
                out[q + "gsel"] = gsel
                out[q + "grad_sub"] = layer.grad[gsel]
            elif layer.kind == "max_pooling":
                out[q + "arg_r"] = layer.arg_r.copy()
                out[q + "arg_c"] = layer.arg_c.copy()
            elif layer.kind == "image_processing":
                out[q + "y_digest"] = np.array(digest(layer.y.view.copy()))
            elif layer.kind in ("fully_connected", "output"):
                out[q + "a"] = layer.a.copy()
                out[q + "y"] = layer.y.copy()
                out[q + "delta"] = layer.delta.copy()
        params1 = flat_params(net)
        out[p + "params1_digest"] = np.array(digest(params1))
        sel = rng.choice(params1.size, size=4096, replace=False)
        out[p + "psel"] = sel
        out[p + "params1_sub"] = params1[sel]
    return out


def c2_trajectory(steps=1000, n_images=200):
    spec = ck.parse_architecture(CONFIGS["C2"])
    net = ck.NetworkState(spec, 7, dtype=F32)
    imgs, labels = glyph_images(n_images, 10, 29, 1, seed=1)
    x = ck.from_bytes(imgs, labels, 10, "train", F32).images
    test_u8, test_lab = glyph_images(100, 10, 29, 1, seed=1, split="test")
    xt = ck.from_bytes(test_u8, test_lab, 10, "test", F32).images
    rng = np.random.default_rng(2024)
    out = {"images_u8": imgs, "labels": labels, "test_u8": test_u8, "test_labels": test_lab}
    sel = rng.choice(net.count_parameters(), size=8192, replace=False)
    out["psel"] = sel
    losses = []
    checkpoints = (1, 10, 100, steps)
    for step in range(1, steps + 1):
        i = (step - 1) % n_images
        losses.append(net.train_step(x[i], ck.targets_for(int(labels[i]), 10), 1e-3))
        if step in checkpoints:
            flat = flat_params(net)
            out[f"params_sub_{step}"] = flat[sel]
            out[f"params_digest_{step}"] = np.array(digest(flat))
            offs = 0
            for idx, name, arr in net.parameters():
                out[f"maxabs_{step}_L{idx}_{name}"] = np.array(np.abs(arr).max())
                offs += arr.size
    out["losses"] = np.array(losses)
    out["test_pred"] = np.array([net.predict(xt[i]) for i in range(len(xt))])
    out["test_out"] = np.stack([net.forward(xt[i]).copy() for i in range(len(xt))])
    return out




def trajectory(name, seed, steps, n_images, n_test):
    """`steps` online steps of config `name` (network.py:275-282), images
    visited cyclically without shuffling; weight subsamples + digests after
    steps 1/10/steps/2/steps, per-step losses, test labels and outputs."""
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        spec = ck.parse_architecture(CONFIGS[name])
    c, w = spec.layers[0].out_maps, spec.layers[0].out_width
    n_cls = spec.n_classes
    net = ck.NetworkState(spec, seed, dtype=F32)
    imgs, labels = glyph_images(n_images, n_cls, w, c, seed=1)
    x = ck.from_bytes(imgs, labels, n_cls, "train", F32).images
    test_u8, test_lab = glyph_images(n_test, n_cls, w, c, seed=1, split="test")
    xt = ck.from_bytes(test_u8, test_lab, n_cls, "test", F32).images
    rng = np.random.default_rng(2025)
    out = {"arch": np.array(CONFIGS[name]), "seed": np.array(seed), "steps": np.array(steps),
           "images_u8": imgs, "labels": labels, "test_u8": test_u8, "test_labels": test_lab}
    sel = rng.choice(net.count_parameters(), size=8192, replace=False)
    out["psel"] = sel
    checkpoints = (1, 10, steps // 2, steps)
    out["checkpoints"] = np.array(checkpoints)
    losses = []
    for step in range(1, steps + 1):
        i = (step - 1) % n_images
        losses.append(net.train_step(x[i], ck.targets_for(int(labels[i]), n_cls), 1e-3))
        if step in checkpoints:
            flat = flat_params(net)
            out[f"params_sub_{step}"] = flat[sel]
            out[f"params_digest_{step}"] = np.array(digest(flat))
    out["losses"] = np.array(losses)
    out["test_pred"] = np.array([net.predict(xt[i]) for i in range(len(xt))])
    out["test_out"] = np.stack([net.forward(xt[i]).copy() for i in range(len(xt))])
    return out


def deform_cases(n_images=6, seed=5, epoch=2):
    from convkit import augment
    out = {}
    for shp, (c, size) in DEFORM_SHAPES.items():
        imgs, labels = glyph_images(n_images, 10, size, c, seed=3)
        x = ck.from_bytes(imgs, labels, 10, "train", F32).images
        out[f"{shp}_u8"] = imgs
        for name, kw in DEFORM_CFGS.items():
            cfg = augment.DeformationConfig(**kw)
            prm, defd = [], []
            for i in range(n_images):
                p = augment.sample_params(cfg, [seed, epoch, i])
                prm.append([p.translate[0], p.translate[1], p.rotate, p.scale[0], p.scale[1],
                            p.shear_h, p.elastic_alpha, float(p.seed)])
                defd.append(augment.deform_channels(x[i], p))
            out[f"{shp}_{name}_params"] = np.array(prm)
            out[f"{shp}_{name}_out"] = np.stack(defd).astype(F32)
    # one deformed online epoch of the tiny net (train_epoch with deformation)
    spec = ck.parse_architecture(SMALL_NETS["tiny"])
    net = ck.NetworkState(spec, 4, dtype=F32)
    imgs, labels = glyph_images(24, 3, 13, 1, seed=9)
    data = ck.from_bytes(imgs, labels, 3, "train", F32)
    cfg = ck.TrainConfig(epochs=1, eta0=1e-2, seed=seed,
                         deformation=augment.DeformationConfig(**DEFORM_CFGS["all"]))
    from convkit import training
    out["epoch_u8"] = imgs
    out["epoch_labels"] = labels
    out["epoch_loss"] = np.array(training.train_epoch(net, data, cfg, 1))
    out["epoch_params"] = flat_params(net)
    return out


def main(which=("kernels", "nets", "configs", "c2", "deform", "traj")):
    # results are bit-identical for every worker count (kernels.py:1-10)
    kernels.set_workers(int(os.environ.get("CK_GOLDEN_WORKERS", "1")))
    if "kernels" in which:
        np.savez_compressed(os.path.join(HERE, "kernels.npz"), **kernel_cases())
        print("kernels.npz written")
    if "nets" in which:
        np.savez_compressed(os.path.join(HERE, "nets.npz"), **small_nets())
        print("nets.npz written")
    if "configs" in which:
        np.savez_compressed(os.path.join(HERE, "configs.npz"), **configs())
        print("configs.npz written")
    if "c2" in which:
        np.savez_compressed(os.path.join(HERE, "c2_traj.npz"), **c2_trajectory())
        print("c2_traj.npz written")
    if "deform" in which:
        np.savez_compressed(os.path.join(HERE, "deform.npz"), **deform_cases())
        print("deform.npz written")
    if "traj" in which:
        for name, (seed, steps, n_images, n_test) in TRAJ.items():
            np.savez_compressed(os.path.join(HERE, f"traj_{name}.npz"),
                                **trajectory(name, seed, steps, n_images, n_test))
            print(f"traj_{name}.npz written")


if __name__ == "__main__":
    main(tuple(sys.argv[1:]) or ("kernels", "nets", "configs", "c2", "deform", "traj"))
