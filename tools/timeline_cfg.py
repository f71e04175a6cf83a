"""Device timeline (CUPTI through torch.profiler) of a few bench steps of one
config, with the bench's L2 flush before each step: per-kernel start/end
relative to the step's first kernel. Run under gpurun: python tools/timeline_cfg.py <config index>"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
dev = torch.device("cuda:0")
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
fbuf = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
st = torch.cuda.Stream()
wl = bench.Workload(bench.CONFIGS[idx], dev)
with torch.cuda.stream(st):
    for i in range(5):
        wl.run(st)
    st.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(6):
            fbuf.fill_(float(i))
            wl.run(st)
        st.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t_prev_end = None
for e in evs:
    s, t = e.time_range.start, e.time_range.end
    gap = "" if t_prev_end is None else f"gap {s - t_prev_end:7.2f}"
    print(f"{e.name[:60]:60s} start {s:12.2f} dur {t - s:8.2f} us {gap}")
    t_prev_end = t
