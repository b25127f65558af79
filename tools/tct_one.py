"""Two C4' visits on the tensor-core training path (ncu target)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1102_0183_b200 as ck  # noqa: E402
from paper_1102_0183_b200.configs import spec_for  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "C4F"
spec = spec_for(name)
f = spec.layers[0]
data = ck.make_glyph_dataset(2, spec.n_classes, f.out_width, seed=2, channels=f.out_maps)
net = ck.NetworkState(spec, 5)
ck.train_epoch(net, data, ck.TrainConfig(epochs=1, eta0=1e-3), 0, engine="tc")
