"""Batched-evaluation throughput per config (development aid).
usage: python tools/probe_eval.py [CONFIGS] [N]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1102_0183_b200 as ck  # noqa: E402
from paper_1102_0183_b200 import training  # noqa: E402
from paper_1102_0183_b200.configs import spec_for, work_per_image  # noqa: E402
from paper_1102_0183_b200.device import DeviceDataset  # noqa: E402

names = (sys.argv[1] if len(sys.argv) > 1 else "C1,C2,C3,C4").split(",")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
for name in names:
    spec = spec_for(name)
    f = spec.layers[0]
    data = ck.make_glyph_dataset(n, spec.n_classes, f.out_width, seed=1, channels=f.out_maps)
    dd = DeviceDataset(data, 0)
    for generic in (False, True):
        net = ck.NetworkState(spec, 0)
        net.set_specialized(not generic)
        pred = torch.empty(n, dtype=torch.int32, device="cuda")
        for _ in range(3):
            training.eval_range_async(net, dd, 0, n, pred)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            training.eval_range_async(net, dd, 0, n, pred)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 5
        fl = work_per_image(spec)["forward"]
        print(f"{name} eval [{'generic' if generic else net.kernel_info()}]: {n / ms * 1e3:,.0f} img/s "
              f"({fl * n / ms / 1e9:.2f} TFLOP/s)", flush=True)
        net.close()
