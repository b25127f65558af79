import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1102_0183_b200 as ck
from paper_1102_0183_b200.configs import spec_for
for name in sys.argv[1:]:
    spec = spec_for(name)
    c, w = spec.layers[0].out_maps, spec.layers[0].out_width
    data = ck.make_glyph_dataset(500, spec.n_classes, w, seed=1, channels=c)
    net = ck.NetworkState(spec, 0, device=0)
    work, bar = ck.training.profile_phases(net, data)
    print(name, net.kernel_info())
    print(net.describe_program(0))
    for i, (a, b) in enumerate(zip(work, bar)):
        print(f"  phase {i}: work {a/1e3:6.2f} us  barrier {b/1e3:5.2f} us")
    print(f"  total {(work.sum()+bar.sum())/1e3:.2f} us")
