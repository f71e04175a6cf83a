"""Per-rank work of the strong-sharded configs at G = 1, 2, 4, 8, timed alone
on one B200: cfg2 / cfg4 / cfg5 / cfg6 / cfg8 shard with no
collective, so the time of the largest rank share bounds the G-GPU step and
T(1) / T(G) is the scaling the sharding allows (a projection for the 8-GPU
box the driver did not run; NCCL / launch skew not included).

  python tools/project_scaling.py [config indices] > profiles/rNN_scaling_projection.json
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def time_share(cfg, steps=20, warmup=5):
    dev = torch.device("cuda:0")
    st = torch.cuda.Stream()
    wl = bench.Workload(cfg, dev)
    with torch.cuda.stream(st):
        for _ in range(warmup):
            wl.run(st)
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            wl.run(st)
        e1.record(st)
        st.synchronize()
    ms = e0.elapsed_time(e1) / steps
    del wl
    torch.cuda.empty_cache()
    return ms


def main():
    idx = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "3", "4", "5", "7"])]
    out = {"what": "largest rank share of the strong-sharded config timed alone on one B200 (per-rank work at G GPUs)",
           "results": {}}
    for i in idx:
        cfg = bench.CONFIGS[i]
        row = {}
        for g in (1, 2, 4, 8):
            # the largest share (shard_units gives the first ranks the extra unit)
            share = bench.local_config(cfg, 0, g, "strong")
            ms = time_share(share)
            row[g] = {"ms": round(ms, 4), "share": {k: share[k] for k in ("B", "H", "M", "Skv") if k in share}}
        t1 = row[1]["ms"]
        for g in (2, 4, 8):
            row[g]["projected_speedup"] = round(t1 / row[g]["ms"], 2)
        out["results"][cfg["name"].split(":")[0]] = row
        print(cfg["name"].split(":")[0], {g: (row[g]["ms"], row[g].get("projected_speedup")) for g in row},
              file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
