"""Quick device timing probe (development aid, not the bench contract).

    python tools/probe.py [--imgs 2000]

Times one online epoch chunk of C1..C4 for several team shapes, the
committee launch, and batched evaluation, with CUDA events.
"""

from __future__ import annotations

import argparse
import os
import sys
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1102_0183_b200 as ck  # noqa: E402

ARCH = {
    "C1": "input 1x29x29; conv 20M k4x4 s0x0; maxpool 2x2; conv 40M k5x5 s0x0; maxpool 3x3; fc 150N; output 10",
    "C2": "input 1x29x29; conv 40M k4x4 s0x0; maxpool 2x2; conv 60M k5x5 s0x0; maxpool 3x3; fc 150N; output 10",
    "C3": "input 2x48x48; imgproc hat21; conv 50M k5x5 s0x0; maxpool 2x2; conv 50M k5x5 s0x0; maxpool 4x4; fc 300N; output 6",
    "C4": "input 3x32x32; conv 300M k3x3 s0x0; maxpool 2x2; conv 300M k2x2 s0x0 rand30; maxpool 2x2; conv 300M k3x3 s0x0 rand30; maxpool 2x2; fc 300N; output 10",
}


def timed(fn, reps=1):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--imgs", type=int, default=2000)
    ap.add_argument("--configs", default="C1,C2,C3,C4")
    ap.add_argument("--teams", default="1,16,512;1,8,512;2,148,512;2,74,512")
    ap.add_argument("--generic", action="store_true", help="force the generic kernel")
    args = ap.parse_args()
    for name in args.configs.split(","):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            spec = ck.parse_architecture(ARCH[name])
        c, w = spec.layers[0].out_maps, spec.layers[0].out_width
        n = args.imgs if name in ("C1", "C2") else max(200, args.imgs // 10)
        data = ck.make_glyph_dataset(n, spec.n_classes, w, seed=1, channels=c)
        cfg = ck.TrainConfig(epochs=1, eta0=1e-3, seed=0)
        teams = [tuple(int(v) for v in t.split(",")) for t in args.teams.split(";")]
        for team in teams:
            try:
                net = ck.NetworkState(spec, 0, team=team)
                if args.generic:
                    net.set_specialized(False)
                ck.train_epoch(net, data.limit(50), cfg, 0)
                ms = timed(lambda: ck.train_epoch(net, data, cfg, 0))
                print(f"{name} [{net.kernel_info()}] train team={team}: {ms:.2f} ms / {n} imgs -> "
                      f"{n / ms * 1e3:.0f} img/s ({ms / n * 1e3:.2f} us/img)", flush=True)
                net.close()
            except Exception as exc:  # keep probing other shapes
                print(f"{name} team={team} failed: {exc}", flush=True)
        for team in ((1, 16, 512), (2, 148, 512)):
            net = ck.NetworkState(spec, 0, team=team)
            if args.generic:
                net.set_specialized(False)
            if team[0] == 1:
                print(net.describe_program(0), flush=True)
            work, bar = ck.training.profile_phases(net, data.limit(200))
            print(f"{name} team={team} work ns:", work.tolist(), "sum", int(work.sum()),
                  "| barrier ns:", bar.tolist(), "sum", int(bar.sum()), flush=True)
        ck.predict_batch(net, data.limit(10))
        ms = timed(lambda: ck.predict_batch(net, data))
        print(f"{name} eval: {ms:.2f} ms / {n} -> {n / ms * 1e3:.0f} img/s", flush=True)
        if name in ("C1", "C2"):
            for k in (2, 4, 8):
                nets = [ck.NetworkState(spec, s) for s in range(k)]
                ck.train_committee_epoch(nets, data.limit(20), cfg, 0)
                ms = timed(lambda: ck.train_committee_epoch(nets, data, cfg, 0))
                print(f"{name} committee x{k} [{nets[0].kernel_info()}]: {ms:.2f} ms -> "
                      f"{k * n / ms * 1e3:.0f} img/s total",
                      flush=True)
                for nn in nets:
                    nn.close()
        net.close()


if __name__ == "__main__":
    main()
