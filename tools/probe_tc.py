"""Eval throughput: bit-exact SIMT path vs tensor-core path, 10k images.
usage: python tools/probe_tc.py [C1 C2 C3 C4]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1102_0183_b200 as ck  # noqa: E402
from paper_1102_0183_b200 import training  # noqa: E402
from paper_1102_0183_b200.configs import spec_for, work_per_image  # noqa: E402
from paper_1102_0183_b200.device import DeviceDataset  # noqa: E402

N = 10_000
for cfg in sys.argv[1:] or ["C1", "C2", "C3", "C4", "C4F"]:
    spec = spec_for(cfg)
    first = spec.layers[0]
    data = ck.make_glyph_dataset(N, spec.n_classes, first.out_width, seed=1, split="test",
                                 channels=first.out_maps)
    net = ck.NetworkState(spec, 0, device=0)
    train = ck.make_glyph_dataset(1000, spec.n_classes, first.out_width, seed=1,
                                  channels=first.out_maps)
    ck.train_epoch(net, train, ck.TrainConfig(epochs=1, eta0=1e-3), 0)   # trained weights
    dd = DeviceDataset(data, 0)
    outs = {}
    pred = torch.empty(N, dtype=torch.int32, device="cuda")
    res = {}
    for eng, passes in (("exact", 3), ("tc", 3), ("tc", 1)):
        for _ in range(2):
            training.eval_range_async(net, dd, 0, N, pred, engine=eng, passes=passes)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        reps = 20
        for _ in range(reps):
            training.eval_range_async(net, dd, 0, N, pred, engine=eng, passes=passes)
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e) / reps
        key = f"{eng}{passes if eng == 'tc' else ''}"
        res[key] = (N / ms * 1e3, pred.cpu().numpy().copy())
        out = torch.empty((N, net.n_classes), dtype=torch.float32, device="cuda")
        training.eval_range_async(net, dd, 0, N, pred, outputs=out, engine=eng, passes=passes)
        outs[key] = out.cpu().numpy()
    ex = res["exact"][1]
    w = work_per_image(spec)["forward"]
    line = " ".join(f"{k}={v[0]:,.0f} img/s ({v[0] * w / 1e12:.1f} TF/s, agree {np.mean(v[1] == ex):.4f})"
                    for k, v in res.items())
    err = {k: float(np.abs(v - outs["exact"]).max()) for k, v in outs.items() if k != "exact"}
    print(cfg, line, "max|dout|", err, flush=True)
    net.close()
