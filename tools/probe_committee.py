import sys, ctypes as C
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1102_0183_b200 as ck
from paper_1102_0183_b200 import _lib
from paper_1102_0183_b200.configs import spec_for
from paper_1102_0183_b200.device import DeviceDataset
spec = spec_for("C1")
data = ck.make_glyph_dataset(2000, 10, 29, seed=1)
dd = DeviceDataset(data, 0)
order = torch.from_numpy(np.random.default_rng(0).permutation(2000).astype(np.int32)).cuda()
for team in [None, (1, 16, 512), (2, 18, 512), (2, 16, 512), (2, 12, 512)]:
    nets = [ck.NetworkState(spec, s, device=0) for s in range(8)]
    if team:
        for n in nets: n.set_team(*team)
    handles = (C.c_void_p * 8)(*[n.handle.value for n in nets])
    def step():
        _lib.call("ck_committee_train_epoch", handles, 8, dd.images_ptr, dd.lut_ptr, dd.labels.data_ptr(), order.data_ptr(), 2000, 1e-3, None, torch.cuda.current_stream().cuda_stream)
    step(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); step(); step(); e.record(); e.synchronize()
    print(team, nets[0].kernel_info(), f"{8*4000/(s.elapsed_time(e)/1e3):,.0f} img/s total")
    for n in nets: n.close()
