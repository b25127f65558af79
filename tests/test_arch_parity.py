"""The architecture parser keeps the reference's interface (convkit
arch.py:3-185): on every stanza below both parsers either resolve the same
geometry with the same warnings or raise the same exception type with the
same message.  Needs the reference package (baseline/_ref or /root/reference);
skipped where it is absent."""

from __future__ import annotations

import warnings

import pytest

import paper_1102_0183_b200 as ck
from tests.conftest import reference_convkit

CASES = [
    "input 1x29x29; conv 20M k4x4 s0x0; maxpool 2x2; conv 40M k5x5 s0x0; maxpool 3x3; "
    "fc 150N; output 10",
    "input 2x48x48; imgproc hat21; conv 50M k5x5 s0x0; maxpool 2x2; conv 50M k5x5 s0x0; "
    "maxpool 4x4; fc 300N; output 6",
    "input 3x32x32; conv 300M k3x3 s0x0; maxpool 2x2; conv 300M k2x2 s0x0 rand30; maxpool 2x2; "
    "conv 300M k3x3 s0x0 rand30; maxpool 2x2; fc 300N; output 10",
    "input 2x16x16; imgproc hat5,sobel,scharr; conv 4M k5x5 s1x1 rand3; maxpool 3x3; fc 6N; output 4",
    "# comment only\ninput 1x6x6  # trailing\n\nfc 9N;;output 4",
    "input 1x6x6; fc 9N; output 4; lr=0.001",
    "input 1x12x12; conv 4M k3x3 s0x0; conv 5M k2x2 s1x1 rand2; fc 7N; fc 6N; output 3",
    "input 1x20x20; maxpool 2x2; conv 3M k3x3 s0x0; maxpool 2x2; maxpool 2x2; output 5",
    # errors
    "", "fc 3N; output 2", "input 1x8x8; fc 3N", "input 1x8x8; input 1x8x8; output 2",
    "input 0x8x8; output 2", "input 1x8x8; bogus 3; output 2", "input 1x8x8; conv 3 k2x2 s0x0; output 2",
    "input 1x8x8; conv 3M k2x2; output 2", "input 1x8x8; conv 3M k2x2 s0x0 rand; output 2",
    "input 1x8x8; conv 3M k2x2 s0x0 rand1 extra; output 2", "input 1x8x8; conv 3M K2x2 s0x0; output 2",
    "input 1x8x8; imgproc hat4; output 2", "input 1x8x8; imgproc blur; output 2",
    "input 1x8x8; imgproc hat5,; output 2", "input 1x8x8; imgproc hat5 sobel; output 2",
    "input 1x8x8; imgproc hat9; output 2", "input 1x8x8; fc 3N; imgproc sobel; output 2",
    "input 1x8x8; conv 2M k3x3 s0x0; imgproc sobel; output 2",
    "input 1x8x8; conv 2M k9x9 s0x0; output 2", "input 1x8x8; conv 2M k3x3 s1x1; output 2",
    "input 1x9x9; conv 2M k3x3 s1x1; output 2", "input 4x8x8; conv 2M k3x3 s0x0 rand1; output 2",
    "input 4x8x8; conv 2M k3x3 s0x0 rand5; output 2", "input 4x8x8; conv 2M k3x3 s0x0 rand0; output 2",
    "input 1x8x8; maxpool 3x3; output 2", "input 1x8x8; maxpool 9x1; output 2",
    "input 1x8x8; maxpool 0x2; output 2", "input 1x8x8; fc 4N; maxpool 2x2; output 2",
    "input 1x8x8; fc 4N; conv 2M k2x2 s0x0; output 2", "input 1x8x8; output 2; fc 3N; output 2",
    "input 1x8x8; fc 0N; output 2", "input 1x8x8; output 0", "input 1x8x8; fc 3n; output 2",
    "input 1x8x8x; output 2", "input 1x8; output 2", "input 1x8x8; maxpool 2x2x2; output 2",
    "input 1x8x8; conv 1M k1x1 s7x7; output 2", "input 1x2x2; maxpool 2x2; maxpool 1x1; output 1",
]


def _outcome(mod, text, experiment):
    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always")
        try:
            if experiment:
                spec, cfg = mod.parse_experiment(text)
            else:
                spec, cfg = mod.parse_architecture(text), {}
        except Exception as exc:           # noqa: BLE001 - compared by type name + text
            return ("error", type(exc).__name__, str(exc))
    geo = [(l.kind, l.out_maps, l.out_width, l.out_height, l.connectivity, l.in_degree,
            tuple(l.filters), tuple(l.kernel), tuple(l.skip), tuple(l.pool), l.neurons)
           for l in spec.layers]
    msgs = [(type(w.message).__name__, str(w.message)) for w in caught]
    return ("ok", geo, cfg, msgs)


@pytest.mark.parametrize("text", CASES)
@pytest.mark.parametrize("experiment", [False, True])
def test_parser_matches_reference(text, experiment):
    ref = reference_convkit()
    if ref is None:
        pytest.skip("reference package not available")
    assert _outcome(ck, text, experiment) == _outcome(ref, text, experiment)
