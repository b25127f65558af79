"""The BASELINE configurations and their algorithmic work.

``ARCH`` holds the reference-grammar architecture strings of C1..C4 (C5 is a
committee of C1 nets).  ``work_per_image`` counts the algorithmic FLOPs the
roofline figures use: 2 per multiply-accumulate of every conv forward,
weight-gradient and delta-pull (pull only where the layer below keeps deltas,
network.py:245-246), 2 per FC MAC forward and 4 backward (xgrad + outer),
plus 2 per updated parameter; activation functions are not counted.  The
contrast layer's MACs are reported separately.
"""

from __future__ import annotations

import warnings

from .arch import parse_architecture
from .network import _padded_bank
from .topology import NetworkSpec, build_full_table, build_random_table

ARCH = {
    "C1": ("input 1x29x29; conv 20M k4x4 s0x0; maxpool 2x2; conv 40M k5x5 s0x0; "
           "maxpool 3x3; fc 150N; output 10"),
    "C2": ("input 1x29x29; conv 40M k4x4 s0x0; maxpool 2x2; conv 60M k5x5 s0x0; "
           "maxpool 3x3; fc 150N; output 10"),
    "C3": ("input 2x48x48; imgproc hat21; conv 50M k5x5 s0x0; maxpool 2x2; "
           "conv 50M k5x5 s0x0; maxpool 4x4; fc 300N; output 6"),
    "C4": ("input 3x32x32; conv 300M k3x3 s0x0; maxpool 2x2; conv 300M k2x2 s0x0 rand30; "
           "maxpool 2x2; conv 300M k3x3 s0x0 rand30; maxpool 2x2; fc 300N; output 10"),
    "C4F": ("input 3x32x32; conv 300M k3x3 s0x0; maxpool 2x2; conv 300M k2x2 s0x0; "
            "maxpool 2x2; conv 300M k3x3 s0x0; maxpool 2x2; fc 300N; output 10"),
}

DESCRIPTION = {
    "C1": "MNIST-shaped 1x29x29-20C4-MP2-40C5-MP3-150N-10N",
    "C2": "deep MNIST 1x29x29-40C4-MP2-60C5-MP3-150N-10N",
    "C3": "NORB-shaped 2x48x48-hat21-50C5-MP2-50C5-MP4-300N-6N",
    "C4": "CIFAR10-shaped 3x32x32-300C3-MP2-300C2(rand30)-MP2-300C3(rand30)-MP2-300N-10N",
    "C4F": "CIFAR10-shaped, full connection tables",
}


def spec_for(name: str) -> NetworkSpec:
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")        # pool truncation warnings (C3, C4)
        return parse_architecture(ARCH[name])


def work_per_image(spec: NetworkSpec, table_seed: int = 0x7AB1E) -> dict:
    """Algorithmic FLOPs per image: train, forward (= eval) and contrast."""
    fwd = bwd = upd = contrast = 0
    has_delta = False
    for idx, ls in enumerate(spec.layers):
        prev = spec.layers[idx - 1] if idx else None
        if ls.kind == "image_processing":
            bank, fh, fw = _padded_bank(ls.filters)
            # unpadded taps: what the reference correlates
            from .filters import expand_selection, filter_coefficients
            taps = sum(filter_coefficients(n).size for n in expand_selection(ls.filters))
            contrast += 2 * taps * prev.out_maps * ls.out_height * ls.out_width
            has_delta = False
        elif ls.kind == "convolutional":
            if ls.connectivity == "random":
                t = build_random_table(prev.out_maps, ls.maps, ls.in_degree,
                                       [table_seed, idx], ls.kernel)
            else:
                t = build_full_table(prev.out_maps, ls.maps, ls.kernel)
            macs = t.n_pairs * ls.out_width * ls.out_height * t.kx * t.ky
            fwd += 2 * macs
            bwd += 2 * macs + (2 * macs if has_delta else 0)
            upd += 2 * t.arena_size
            has_delta = True
        elif ls.kind == "max_pooling":
            pass
        elif ls.kind in ("fully_connected", "output"):
            n_in = (prev.out_maps * prev.out_width * prev.out_height
                    if prev.is_spatial else prev.neurons)
            fwd += 2 * n_in * ls.neurons
            bwd += 4 * n_in * ls.neurons
            upd += 2 * (n_in * ls.neurons + ls.neurons)
            has_delta = True
        else:
            has_delta = False
    return {"train": fwd + bwd + upd, "forward": fwd, "contrast": contrast}
