"""Stage-by-stage check of train_epoch / exact eval / TC eval (debug aid).
usage: python tools/dbg_eval.py [configs...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1102_0183_b200 as ck  # noqa: E402
from paper_1102_0183_b200 import training  # noqa: E402
from paper_1102_0183_b200.configs import spec_for  # noqa: E402
from paper_1102_0183_b200.device import DeviceDataset  # noqa: E402

N = int(os.environ.get("DBG_N", "10000"))
for cfg in sys.argv[1:] or ["C1", "C3"]:
    spec = spec_for(cfg)
    first = spec.layers[0]
    net = ck.NetworkState(spec, 0, device=0)
    train = ck.make_glyph_dataset(1000, spec.n_classes, first.out_width, seed=1,
                                  channels=first.out_maps)
    ck.train_epoch(net, train, ck.TrainConfig(epochs=1, eta0=1e-3), 0)
    torch.cuda.synchronize()
    print(cfg, "train ok", flush=True)
    data = ck.make_glyph_dataset(N, spec.n_classes, first.out_width, seed=1, split="test",
                                 channels=first.out_maps)
    dd = DeviceDataset(data, 0)
    pred = torch.empty(N, dtype=torch.int32, device="cuda")
    engines = [(e[:-1] if e[-1].isdigit() else e, int(e[-1]) if e[-1].isdigit() else 3)
               for e in os.environ.get("DBG_ENGINES", "exact,tc3,tc1").split(",")]
    for eng, passes in engines:
        training.eval_range_async(net, dd, 0, N, pred, engine=eng, passes=passes)
        torch.cuda.synchronize()
        print(cfg, eng, passes, "ok", flush=True)
    net.close()
