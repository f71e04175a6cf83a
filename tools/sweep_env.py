"""Tuning sweep on the GPU box: runs bench.py for one config under several
environment settings (e.g. RF_GEMM_GROUP) and prints one JSON line per run,
optionally with the ncu DRAM bytes of the dominant kernel's launch.

  python tools/sweep_env.py --config 3 --var RF_GEMM_GROUP --values 4,-4,-8 [--ncu quant_gemm]
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench(cfg, env, steps):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", str(cfg), "--also", "",
                          "--no-cpu-baseline", "--no-parity", "--steps", str(steps), "--warmup", "5"],
                         capture_output=True, text=True, env=env, timeout=900)
    line = [x for x in out.stdout.splitlines() if x.startswith("{")]
    if not line:
        return {"error": out.stderr[-2000:]}
    d = json.loads(line[-1])
    return {"value": d["value"], "ms": d["ms_per_step"], "frac": d["roofline"]["frac"],
            "sm_mhz": (d.get("clocks") or {}).get("sm_mhz")}


def ncu_dram(cfg, env, kernel):
    rep = os.path.join(ROOT, "gpurun_out", "sweep_tmp")
    subprocess.run(["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                    "--clock-control", "none", "-k", f"regex:{kernel}", "-s", "3", "-c", "1", "--csv",
                    "--log-file", rep + ".csv", sys.executable, os.path.join(ROOT, "bench.py"),
                    "--config", str(cfg), "--also", "", "--no-cpu-baseline", "--no-parity", "--steps", "2",
                    "--warmup", "3", "--no-graph"], capture_output=True, text=True, env=env, timeout=900)
    try:
        rows = list(csv.reader(io.StringIO(open(rep + ".csv").read().split("\n", 0)[0])))
    except OSError:
        return None
    hdr = None
    vals = {}
    for r in rows:
        if "Metric Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            vals[r[hdr.index("Metric Name")]] = r[hdr.index("Metric Value")]
    return vals


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--var", required=True)
    ap.add_argument("--values", required=True)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--repeat", type=int, default=2)
    ap.add_argument("--ncu", default="")
    a = ap.parse_args()
    for rep in range(a.repeat):
        for v in a.values.split(","):
            env = dict(os.environ)
            if v != "default":
                env[a.var] = v
            r = {"config": a.config, a.var: v, "rep": rep, **bench(a.config, env, a.steps)}
            if a.ncu and rep == 0:
                r["ncu"] = ncu_dram(a.config, env, a.ncu)
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
