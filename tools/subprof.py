"""Sub-phase timers of the training kernel (development aid).
usage: python tools/subprof.py CONFIG [ranks] [kind,ctas,threads]
Prints, per phase, the ns between consecutive recorded points of thread 0 of
each listed team rank for the last image of a short epoch (point 0 = phase
start, 30 = ops done, 31 = barrier exit)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1102_0183_b200 as ck  # noqa: E402
from paper_1102_0183_b200 import _lib  # noqa: E402
from paper_1102_0183_b200.configs import spec_for  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
ranks = [int(r) for r in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0]
team = tuple(int(v) for v in sys.argv[3].split(",")) if len(sys.argv) > 3 else None
spec = spec_for(name)
c, w = spec.layers[0].out_maps, spec.layers[0].out_width
data = ck.make_glyph_dataset(40, spec.n_classes, w, seed=1, channels=c)
net = ck.NetworkState(spec, 0, team=team)
cfg = ck.TrainConfig(epochs=1, eta0=1e-3)
ck.train_epoch(net, data, cfg, 0)
prog = net.describe_program(0).strip().splitlines()
buf = torch.zeros(32 * 64, dtype=torch.int64, device="cuda")
for rank in ranks:
    buf.zero_()
    _lib.call("ck_debug_subprof", buf.data_ptr(), rank)
    ck.train_epoch(net, data, cfg, 0)
    torch.cuda.synchronize()
    _lib.call("ck_debug_subprof", None, 0)
    b = buf.cpu().numpy().reshape(64, 32)
    print(f"== {name} rank {rank}")
    for ph, line in enumerate(prog):
        row = b[ph]
        pts = [(i, int(row[i])) for i in range(28) if row[i]] + \
              [(i, int(row[i])) for i in (30, 31) if row[i]]
        if not pts:
            continue
        t0 = pts[0][1]
        segs = " ".join(f"{i}:{(t - t0) / 1e3:.2f}" for i, t in pts[1:])
        clk = ""
        if row[28] and row[29] and row[30] and row[0]:
            clk = f" | SM clock {(row[29] - row[28]) / max(1, row[30] - row[0]):.2f} GHz"
        print(f"  {line[:60]:60s} | {segs}{clk}")
