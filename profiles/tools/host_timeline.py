"""Dev tool: CUPTI timeline (torch.profiler / kineto) of one host-buffer
btg_forward and btg_adjoint at configs[1]: every kernel and memcpy with its
stream, start and duration relative to the call, to see what the host pipeline
leaves exposed. Usage on the GPU box: python profiles/tools/host_timeline.py"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2407_13066_b200 import _lib  # noqa: E402

cfg = dict(bench.CONFIGS[os.environ.get("CFG", "B")], precision=int(os.environ.get("PREC", "64")))
nt, nd, nm = cfg["nt"], cfg["nd"], cfg["nm"]
op = bench.build_operator(cfg, 0, seed=1000)
hm = torch.empty((nm, nt), dtype=torch.float64, pin_memory=True).uniform_(-1, 1)
hd = torch.empty((nd, nt), dtype=torch.float64, pin_memory=True).uniform_(-1, 1)
hm_np, hd_np = hm.numpy(), hd.numpy()
out_d = torch.empty((nd, nt), dtype=torch.float64, pin_memory=True).numpy()
out_m = torch.empty((nm, nt), dtype=torch.float64, pin_memory=True).numpy()
L = _lib.load()
op._bind_stream(None)


def fwd():
    _lib.check(L.btg_forward(op._h, hm_np.ctypes.data, hm_np.size, out_d.ctypes.data, out_d.size, 1, 0))


def adj():
    _lib.check(L.btg_adjoint(op._h, hd_np.ctypes.data, hd_np.size, out_m.ctypes.data, out_m.size, 1, 0))


for _ in range(3):
    fwd()
    adj()
torch.cuda.synchronize()
for name, fn in (("forward", fwd), ("adjoint", adj)):
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        fn()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    cpu = [e for e in prof.events() if e.device_type != torch.autograd.DeviceType.CUDA]
    t0 = min(e.time_range.start for e in evs)
    t1 = max(e.time_range.end for e in evs)
    print(f"== {name}: device span {(t1 - t0) / 1e3:.3f} ms, {len(evs)} device events")
    for e in sorted(evs, key=lambda e: e.time_range.start):
        print(f"  {(e.time_range.start - t0) / 1e3:8.3f} +{(e.time_range.end - e.time_range.start) / 1e3:7.3f} ms"
              f"  ch{getattr(e, 'device_resource_id', '?')}  {e.name[:70]}")
