"""One C1 train_epoch launch (100 images) for an ncu capture."""
import os, sys, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1102_0183_b200 as ck
arch = sys.argv[1] if len(sys.argv) > 1 else "C1"
A = {"C1": "input 1x29x29; conv 20M k4x4 s0x0; maxpool 2x2; conv 40M k5x5 s0x0; maxpool 3x3; fc 150N; output 10",
     "C4": "input 3x32x32; conv 300M k3x3 s0x0; maxpool 2x2; conv 300M k2x2 s0x0 rand30; maxpool 2x2; conv 300M k3x3 s0x0 rand30; maxpool 2x2; fc 300N; output 10"}[arch]
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    spec = ck.parse_architecture(A)
c, w = spec.layers[0].out_maps, spec.layers[0].out_width
data = ck.make_glyph_dataset(100, spec.n_classes, w, seed=1, channels=c)
net = ck.NetworkState(spec, 0)
cfg = ck.TrainConfig(epochs=1, eta0=1e-3)
ck.train_epoch(net, data, cfg, 0)
import torch; torch.cuda.synchronize()
print("done")
