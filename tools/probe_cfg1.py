"""Where cfg1's ~20 us per step goes (fp32 attention B1 H1 S1024 D64): step time
with and without the bench's L2 flush, per reference segment count S, and with a
write-then-read flush (no dirty lines left for the step's loads to evict).
Run under gpurun."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

dev = torch.device("cuda:0")
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
fbuf = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
st = torch.cuda.Stream()
for segs in [int(x) for x in (sys.argv[1:] or ["8"])]:
    cfg = dict(bench.CONFIGS[0], segments=segs)
    wl = bench.Workload(cfg, dev)
    print(f"S={segs}: plan {wl.plan.info}")
    for mode in ["none", "write", "write+read"]:
        ts = []
        with torch.cuda.stream(st):
            for i in range(60):
                if mode != "none":
                    fbuf.fill_(float(i))
                if mode == "write+read":
                    fbuf.sum()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(st)
                wl.run(st)
                e1.record(st)
                st.synchronize()
                if i >= 10:
                    ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        print(f"  flush {mode:10s}: median {ts[len(ts) // 2]:.1f} us, min {ts[0]:.1f}")
