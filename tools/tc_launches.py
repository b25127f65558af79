"""One TC-path evaluation of 10k images per config (for an ncu launch list).
usage: python tools/tc_launches.py C2 [passes]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1102_0183_b200 as ck  # noqa: E402
from paper_1102_0183_b200 import training  # noqa: E402
from paper_1102_0183_b200.configs import spec_for  # noqa: E402
from paper_1102_0183_b200.device import DeviceDataset  # noqa: E402

cfg = sys.argv[1]
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 3
spec = spec_for(cfg)
first = spec.layers[0]
data = ck.make_glyph_dataset(10_000, spec.n_classes, first.out_width, seed=1, split="test",
                             channels=first.out_maps)
net = ck.NetworkState(spec, 0, device=0)
dd = DeviceDataset(data, 0)
pred = torch.empty(10_000, dtype=torch.int32, device="cuda")
training.eval_range_async(net, dd, 0, 10_000, pred, engine="tc", passes=passes)
torch.cuda.synchronize()
