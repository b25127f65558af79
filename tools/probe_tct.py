"""Tensor-core training vs the exact engine: per-image time, agreement.
usage: python tools/probe_tct.py [C4F C4 C1]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1102_0183_b200 as ck  # noqa: E402
from paper_1102_0183_b200.configs import spec_for  # noqa: E402

for name in sys.argv[1:] or ["C4F", "C4", "C1"]:
    spec = spec_for(name)
    f = spec.layers[0]
    data = ck.make_glyph_dataset(64, spec.n_classes, f.out_width, seed=2, channels=f.out_maps)
    cfg = ck.TrainConfig(epochs=1, eta0=1e-3, seed=1)
    res = {}
    for eng in ("exact", "tc"):
        net = ck.NetworkState(spec, 5)
        ck.train_epoch(net, data.limit(8), cfg, 0, engine=eng)   # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m = ck.train_epoch(net, data, cfg, 1, engine=eng)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        res[eng] = (len(data) / el, m, net.flat_parameters())
        net.close()
    d = np.abs(res["tc"][2] - res["exact"][2]).max()
    print(f"{name}: exact {res['exact'][0]:.0f} img/s  tc {res['tc'][0]:.0f} img/s  "
          f"loss {res['exact'][1]:.6f} vs {res['tc'][1]:.6f}  max|dw| {d:.2e}", flush=True)
