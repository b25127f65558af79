"""One train_epoch launch for an ncu capture.
usage: python tools/ncu_one.py [CONFIG] [IMGS] [kind,ctas,threads]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1102_0183_b200 as ck  # noqa: E402
from paper_1102_0183_b200.configs import spec_for  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100
team = tuple(int(v) for v in sys.argv[3].split(",")) if len(sys.argv) > 3 else None
spec = spec_for(name)
c, w = spec.layers[0].out_maps, spec.layers[0].out_width
data = ck.make_glyph_dataset(n, spec.n_classes, w, seed=1, channels=c)
net = ck.NetworkState(spec, 0, team=team)
cfg = ck.TrainConfig(epochs=1, eta0=1e-3)
ck.train_epoch(net, data.limit(4), cfg, 0)
ck.train_epoch(net, data, cfg, 0)
import torch  # noqa: E402
torch.cuda.synchronize()
print("done")
