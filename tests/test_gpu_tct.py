"""Tensor-core training variant: opt-in, outside the
bit-exact contract.  Its stated tolerance, against the exact engine on the
same visits from the same weights:

  * per-image losses within 1e-4 relative, weights within 2e-4 absolute after
    a short online run (the fp16 hi/lo split GEMMs are ~f32-accurate; their
    sums are not in the reference's order, and max-pool ties / near-ties can
    route a delta to a different winner);
  * predicted test labels agree on >= 99% of images.
"""

from __future__ import annotations

import numpy as np
import pytest

from tests.conftest import has_cuda

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]

import paper_1102_0183_b200 as ck  # noqa: E402
from paper_1102_0183_b200.configs import spec_for  # noqa: E402


@pytest.mark.parametrize("name,n", [("C1", 40), ("C4F", 12), ("C4", 12)])
def test_tc_training_tracks_exact_engine(name, n):
    spec = spec_for(name)
    first = spec.layers[0]
    data = ck.make_glyph_dataset(n, spec.n_classes, first.out_width, seed=2,
                                 channels=first.out_maps)
    test = ck.make_glyph_dataset(200, spec.n_classes, first.out_width, seed=2, split="test",
                                 channels=first.out_maps)
    cfg = ck.TrainConfig(epochs=1, eta0=1e-3, seed=1)
    exact = ck.NetworkState(spec, 5)
    tc = ck.NetworkState(spec, 5)
    m_exact = ck.train_epoch(exact, data, cfg, 0)
    m_tc = ck.train_epoch(tc, data, cfg, 0, engine="tc")
    assert m_tc == pytest.approx(m_exact, rel=1e-4)
    diff = np.abs(tc.flat_parameters() - exact.flat_parameters()).max()
    assert diff <= 2e-4, diff
    agree = np.mean(ck.predict_batch(tc, test) == ck.predict_batch(exact, test))
    assert agree >= 0.99, agree
    exact.close()
    tc.close()
