"""Run on the GPU box (gpurun): one `ncu --set full` capture of the dominant
kernel of every BASELINE config plus the launch list of the default bench,
summarised as JSON into gpurun_out/ (copy the summaries into profiles/).

  python tools/profile_all.py --tag r1 [--configs 0,1,2,3,4]
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KERNELS = {0: "attn_tf32_kernel", 1: "attn_sm100_kernel", 2: "attn_decode_kernel",
           3: "quant_gemm", 4: "rms_gemm", 5: "rms_gemm", 6: "router_kernel", 7: "mla_decode"}
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals) if h in METRICS}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--configs", default="0,1,2,3,4,5,6,7")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    summary, traffic = {}, {}
    for c in [int(x) for x in a.configs.split(",")]:
        rep = os.path.join(ROOT, "gpurun_out", f"{a.tag}_cfg{c}")
        cmd = ["ncu", "--set", "full", "--clock-control", "none", "--import-source", "on",
               "-k", f"regex:{KERNELS[c]}", "-s", "3", "-c", "1", "-f", "-o", rep,
               sys.executable, os.path.join(ROOT, "bench.py"), "--config", str(c), "--steps", "2",
               "--warmup", "3", "--no-cpu-baseline", "--no-parity", "--also", ""]
        subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        try:
            m = raw(rep + ".ncu-rep")
        except Exception as e:  # noqa: BLE001
            summary[f"cfg{c + 1}"] = {"error": str(e)}
            continue
        summary[f"cfg{c + 1}"] = {"kernel": KERNELS[c], **{k: v for k, v in m.items()}}
        unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(m["dram__bytes_read.sum"][0]) * unit[m["dram__bytes_read.sum"][1]]
        wr = float(m["dram__bytes_write.sum"][0]) * unit[m["dram__bytes_write.sum"][1]]
        traffic[f"cfg{c + 1}"] = rd + wr
    # launch list of the default bench (cold-cache, serialised: shares, not absolutes)
    lcsv = os.path.join(ROOT, "gpurun_out", f"{a.tag}_launches_cfg2.csv")
    subprocess.run(["ncu", "--metrics", "gpu__time_duration.sum", "--clock-control", "none",
                    "-c", "60", "--csv", "--log-file", lcsv, sys.executable,
                    os.path.join(ROOT, "bench.py"), "--steps", "5", "--warmup", "3",
                    "--no-cpu-baseline", "--no-parity", "--also", ""], capture_output=True, timeout=900)
    json.dump(summary, open(os.path.join(ROOT, "gpurun_out", f"{a.tag}_ncu_summary.json"), "w"),
              indent=1)
    json.dump({k: int(v) for k, v in traffic.items()},
              open(os.path.join(ROOT, "gpurun_out", f"{a.tag}_traffic.json"), "w"), indent=1)
    print(json.dumps(traffic))


if __name__ == "__main__":
    main()
