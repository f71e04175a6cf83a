"""Benchmark of the fused cascaded-reduction hot path (driver contract).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

A "step" is one pass of the fused loop (rf_run) over one batch of synthetic
input of a BASELINE.json configuration. Default workload = configs[1]
(bf16 MHA prefill B8 H32 S4096 D128, non-causal) — the config the metric is
quoted on that fits one GPU. Multi-GPU (torchrun, NCCL): every rank runs the
same per-GPU workload on its own (b,h) units (batch/head sharding needs no
data-path collective) -> "scaling": "weak"; the timed region is bracketed by
barriers, and the time is the max over ranks.

`--impl reference` times the reference's own CPU fused loop
(oracle/_ref/ref_driver, built from /root/reference/proj/src: run_incremental
per row on all host threads) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused-op TFLOP/s & % roofline at 1/2/4/8 B200 vs CPU ref (cores stated)"
REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")

# BASELINE.json configs (index = position in BASELINE.json "configs").
CONFIGS = {
    0: dict(name="cfg1: single-head safe-softmax->GEMM attention fp32 S1024 D64 B1",
            pattern="attention", B=1, H=1, Sq=1024, Skv=1024, D=64, dtype="f32", segments=8),
    1: dict(name="cfg2: MHA prefill bf16 B8 H32 S4096 D128 (non-causal)",
            pattern="attention", B=8, H=32, Sq=4096, Skv=4096, D=128, dtype="bf16", segments=1),
    2: dict(name="cfg3: decode bf16 B64 H32 Sq1 Skv32768 D128 split-KV",
            pattern="attention", B=64, H=32, Sq=1, Skv=32768, D=128, dtype="bf16", segments=8),
    3: dict(name="cfg4: per-token absmax FP8 quant + GEMM M=K=N=8192",
            pattern="quant", M=8192, K=8192, N=8192, dtype="bf16"),
    4: dict(name="cfg5: RMSNorm stats + GEMM T16384 K4096 N11008",
            pattern="rms", M=16384, K=4096, N=11008, dtype="bf16"),
    # not a BASELINE.json config: the north_star's LayerNorm variant of cfg5
    5: dict(name="cfg6: LayerNorm stats + GEMM T16384 K4096 N11008 (extra, north_star)",
            pattern="ln", M=16384, K=4096, N=11008, dtype="bf16"),
    # not a BASELINE.json config: SURVEY §8 f1, the paper's MoE routing R8
    # (PAPER.md:1583-1590): router GEMM 2048 x 4096 -> 128 experts + top-8
    6: dict(name="cfg7: MoE router R8 s2048 hd4096 en128 top8 (extra, SURVEY f1)",
            pattern="router", M=2048, K=4096, N=128, topk=8, dtype="bf16"),
    # not a BASELINE.json config: SURVEY §8 f4, the paper's MLA decode L3
    # (PAPER.md:1559-1567): bs 32, 128 heads, kv 4096, latent 512 + rope 64
    7: dict(name="cfg8: MLA decode L3 bs32 hn128 kv4096 hd512+64 (extra, SURVEY f4)",
            pattern="mla", B=32, Skv=4096, dtype="bf16", segments=1),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def fp8_peak():
    """Dense e4m3 peak measured on this pool's B200 (tools/measure_fp8_peak.py)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            v = json.load(f).get("fp8_tflops")
        if v:
            return float(v)
    except OSError:
        pass
    try:
        with open(os.path.join(ROOT, "profiles", "r1c_fp8_peak.json")) as f:
            return float(json.load(f)["fp8_tflops"])
    except (OSError, KeyError, ValueError):
        return None


def work_of(cfg):
    """Algorithmic FLOPs and bytes per step."""
    if cfg["pattern"] == "mla":  # S = q K^T (576) + P V (512) per head; cache read once
        B, S = cfg["B"], cfg["Skv"]
        return 2.0 * B * 128 * S * (576 + 512), 2 * B * S * 576 + 2 * B * 128 * (576 + 512) + 8 * B * 128
    if cfg["pattern"] == "attention":
        B, H, Sq, Skv, D = cfg["B"], cfg["H"], cfg["Sq"], cfg["Skv"], cfg["D"]
        es = 4 if cfg["dtype"] == "f32" else 2
        flops = 4.0 * B * H * Sq * Skv * D
        bytes_ = es * B * H * (2 * Sq * D + 2 * Skv * D) + 8 * B * H * Sq
        return flops, bytes_
    M, K, N = cfg["M"], cfg["K"], cfg["N"]
    flops = 2.0 * M * N * K
    if cfg["pattern"] == "router":  # X once, packed W once, d1/d2 + top-k records
        return flops, 2 * M * K + 2 * N * K + 8 * M + 8 * M * cfg["topk"]
    if cfg["pattern"] == "quant":
        bytes_ = 2 * M * K + N * K + 4 * M * N + 4 * M
    elif cfg["pattern"] == "ln":  # d3 and d4 both written (bf16), d1/d2 f32
        bytes_ = 2 * M * K + 2 * N * K + 4 * N + 4 * M * N + 8 * M
    else:
        bytes_ = 2 * M * K + 2 * N * K + 2 * M * N + 4 * M
    return flops, bytes_


def bound_of(cfg):
    if cfg["pattern"] == "attention" and cfg["Sq"] == 1:
        return "hbm"
    if cfg["pattern"] == "router":  # 2 * en FLOP per byte of X: far below the ridge
        return "hbm"
    if cfg["pattern"] == "mla":  # ~240 FLOP/B: at the ridge; the cache stream bounds it
        return "hbm"
    return "tensor"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        if not shutil.which("nvidia-smi"):
            return
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        self.proc = subprocess.Popen(
            ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
             "--format=csv,noheader,nounits", "-lms", "20"],
            stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        time.sleep(0.3)

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.1)
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        # "under load": samples at or above the median (idle gaps at start/end excluded)
        med = statistics.median(sm) if sm else None
        loaded = [x for x in sm if med is None or x >= 0.8 * med]
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def cpu_reference(cfg, budget_s=12.0, threads=None):
    """The reference's CPU fused loop on the host cores (bounded sample)."""
    if not os.path.exists(REF_DRIVER):
        return None
    threads = threads or os.cpu_count() or 1
    if cfg["pattern"] == "mla":
        args = ["attention", str(cfg["Skv"]), "512", "100000000", str(threads), "1"]
        sample = (f"rows = (b, head) cascades of kv={cfg['Skv']}, V width 512 (the reference's "
                  f"attention cascade; its P row is a 512-wide dot, the 64 rope columns not counted)")
    elif cfg["pattern"] == "attention":
        segs = cfg.get("segments", 1) if cfg["Sq"] == 1 else 1
        args = ["attention", str(cfg["Skv"]), str(cfg["D"]), "100000000", str(threads), str(segs)]
        sample = f"rows = (b,h,query) cascades of kv={cfg['Skv']}, hd={cfg['D']}"
    elif cfg["pattern"] == "router":
        args = ["router", str(cfg["K"]), str(cfg["N"]), "100000000", str(threads), str(cfg["topk"])]
        sample = (f"rows = tokens: router GEMM hd={cfg['K']} -> en={cfg['N']} (fp64) + the "
                  f"moe_routing cascade (top-{cfg['topk']})")
    elif cfg["pattern"] == "quant":
        args = ["quant", str(cfg["K"]), str(cfg["N"]), str(threads), str(threads), "1"]
        sample = f"rows = tokens of K={cfg['K']}, N={cfg['N']}"
    else:
        args = [cfg["pattern"], str(cfg["K"]), str(cfg["N"]), str(threads), str(threads), "1"]
        sample = f"rows = tokens of K={cfg['K']}, N={cfg['N']}"
    out = subprocess.run([REF_DRIVER, "bench"] + args + [f"{budget_s}"], capture_output=True,
                         text=True, timeout=600)
    if out.returncode != 0:
        return None
    r = json.loads(out.stdout.strip().splitlines()[-1])
    return {
        "value": r["flop_per_s"] / 1e12,
        "unit": "TFLOP/s",
        "cores": r["threads"],
        "kind": "reference",
        "sample": f"{r['rows']} {sample} through redfuse run_incremental"
                  f"{' / run_multisegment' if r['segments'] > 1 else ''} "
                  f"(oracle/_ref/ref_driver, {r['s_per_row_thread']:.3f} s/row/thread, "
                  f"{r['wall_s']:.1f} s wall)",
        "rows_per_s": r["rows_per_s"],
    }


def dist_setup(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


class Workload:
    """Plan + device/host buffers for one BASELINE config (plan-time work, e.g.
    weight packing, happens here — outside every timed region)."""

    def __init__(self, cfg, dev, world=1):
        import torch

        from paper_2603_10026_b200 import Desc, Plan
        from paper_2603_10026_b200 import _native as N

        g = torch.Generator(device=dev)
        g.manual_seed(1234)
        rnd = lambda *shape: torch.rand(*shape, device=dev, generator=g)  # noqa: E731
        self.cfg = cfg
        pat = cfg["pattern"]
        if pat == "mla":
            B, S = cfg["B"], cfg["Skv"]
            q = (rnd(B, 128, 576) * 2 - 1).bfloat16()
            kv = (rnd(B, S, 576) * 2 - 1).bfloat16()
            self.plan = Plan(Desc(N.RF_PATTERN_MLA_DECODE, "bf16", rows=1, len=S, free_len=512, batch=B,
                                  heads=128, segments=cfg.get("segments", 1), softmax_scale=576 ** -0.5,
                                  producer_len=576, device=dev.index))
            self.inputs = [q, kv]
            m = torch.empty(B, 128, device=dev)
            self.outputs = [m, torch.empty_like(m), torch.empty(B, 128, 512, dtype=torch.bfloat16, device=dev)]
            self.step_inputs = [0, 1]
            self.data = "synthetic (q, cache ~ U(-1,1) bf16; cache rows [c_kv 512 | k_rope 64])"
        elif pat == "attention":
            dt = torch.float32 if cfg["dtype"] == "f32" else torch.bfloat16
            B, H, Sq, Skv, D = cfg["B"], cfg["H"], cfg["Sq"], cfg["Skv"], cfg["D"]
            q = ((rnd(B, H, Sq, D) * 2 - 1) / D ** 0.5).to(dt)
            k = (rnd(B, H, Skv, D) * 2 - 1).to(dt)
            v = (rnd(B, H, Skv, D) * 2 - 1).to(dt)
            self.plan = Plan(Desc(N.RF_PATTERN_ATTENTION, cfg["dtype"], rows=Sq, len=Skv,
                                  free_len=D, batch=B, heads=H, segments=cfg.get("segments", 1),
                                  device=dev.index))
            self.inputs = [q, k, v]
            m = torch.empty(B, H, Sq, device=dev)
            self.outputs = [m, torch.empty_like(m), torch.empty_like(q)]
            self.step_inputs = [0, 1, 2]  # all inputs are per-step data
            self.data = "synthetic (uniform, make_attention distributions; q pre-scaled by 1/sqrt(D))"
            # split-KV decode over G GPUs: this rank's K/V are its shard of a
            # G x Skv sequence (weak scaling); partials are all-gathered (NCCL)
            # and merged in slice order inside every step
            self.split_kv = Sq == 1 and world > 1
            self.segments_global = cfg.get("segments", 1) * world
        else:
            M, K, Nn = cfg["M"], cfg["K"], cfg["N"]
            if pat == "router":
                a = (rnd(M, K) * 2 - 1).bfloat16()
                self.plan = Plan(Desc(N.RF_PATTERN_MOE_ROUTER, "bf16", rows=M, len=Nn,
                                      free_len=cfg["topk"], producer_len=K, device=dev.index))
                w = (rnd(K, Nn) * 2 - 1) / K ** 0.5
                wp = self.plan.pack_weight(w)
                del w
                self.outputs = [torch.empty(M, device=dev), torch.empty(M, device=dev),
                                torch.empty(M, cfg["topk"], 2, dtype=torch.int32, device=dev)]
                self.data = "synthetic (x ~ U(-1,1) bf16, router w ~ U(-1,1)/sqrt(hd) packed bf16)"
            elif pat == "quant":
                a = (rnd(M, K) * 4 - 2).bfloat16()  # make_quant_gemm: a ~ U(-2, 2)
                self.plan = Plan(Desc(N.RF_PATTERN_QUANT_GEMM_E4M3, "bf16", rows=M, len=K,
                                      free_len=Nn, device=dev.index))
                w = rnd(K, Nn) * 2 - 1  # w ~ U(-1, 1)
                wp = self.plan.pack_weight(w)
                del w
                self.outputs = [torch.empty(M, device=dev), torch.empty(M, Nn, device=dev)]
                self.data = "synthetic (make_quant_gemm distributions: a~U(-2,2), w~U(-1,1) packed e4m3)"
            elif pat == "ln":
                a = (rnd(M, K) * 2 - 1).bfloat16()
                self.plan = Plan(Desc(N.RF_PATTERN_LAYERNORM_GEMM, "bf16", rows=M, len=K,
                                      free_len=Nn, eps=1e-5, device=dev.index))
                w = rnd(K, Nn) * 2 - 1
                gam = rnd(K) * 2 - 1
                wp = self.plan.pack_weight(w, gam)
                del w
                self.outputs = [torch.empty(M, device=dev), torch.empty(M, device=dev),
                                torch.empty(M, Nn, dtype=torch.bfloat16, device=dev),
                                torch.empty(M, Nn, dtype=torch.bfloat16, device=dev)]
                self.data = "synthetic (DSL wrap_spec convention: x, g, w ~ U(-1,1); g folded into bf16 W)"
            else:
                a = (rnd(M, K) * 2 - 1).bfloat16()
                self.plan = Plan(Desc(N.RF_PATTERN_RMSNORM_GEMM, "bf16", rows=M, len=K,
                                      free_len=Nn, eps=1e-6, device=dev.index))
                w = rnd(K, Nn) * 2 - 1
                gam = rnd(K) * 2 - 1
                wp = self.plan.pack_weight(w, gam)
                del w
                self.outputs = [torch.empty(M, device=dev),
                                torch.empty(M, Nn, dtype=torch.bfloat16, device=dev)]
                self.data = "synthetic (DSL wrap_spec convention: x, g, w ~ U(-1,1); g folded into bf16 W)"
            self.inputs = [a, wp]
            self.step_inputs = [0]  # the packed weight is plan-time resident
        torch.cuda.synchronize()

    def run(self, stream):
        if getattr(self, "split_kv", False):
            from paper_2603_10026_b200.distributed import split_kv_decode

            q, k, v = self.inputs
            split_kv_decode(q, k, v, self.segments_global, stream=stream)
        else:
            self.plan.run(self.inputs, self.outputs, stream)

    def host_buffers(self):
        import torch

        hin = [x.cpu().pin_memory() if i in self.step_inputs else x
               for i, x in enumerate(self.inputs)]
        hout = [torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in self.outputs]
        return hin, hout


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_setup(args)
    dev = torch.device("cuda", torch.cuda.current_device())
    wl = Workload(cfg, dev, world)
    plan = wl.plan
    stream = torch.cuda.Stream(device=dev)
    flops, nbytes = work_of(cfg)

    def barrier():
        if world > 1:
            dist.barrier()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            wl.run(stream)
        stream.synchronize()
        # Inputs smaller than L2 (cfg1) would stay L2-resident across steps:
        # then L2 is flushed (a 2x-L2 buffer write) before every step, outside
        # the per-step events. Larger inputs: G consecutive steps are
        # captured once as a CUDA graph and replayed K/G times, so host launch
        # cost stays off the device timeline; every step's kernels still run.
        # The split-KV multi-GPU step (NCCL all-gather) runs eagerly.
        l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
        in_bytes = sum(wl.inputs[i].numel() * wl.inputs[i].element_size() for i in wl.step_inputs)
        flush = in_bytes < l2_bytes
        graphed = not args.no_graph and not getattr(wl, "split_kv", False)
        G = 1 if flush else max(g for g in range(1, 21) if args.steps % g == 0) if graphed else 1
        step = lambda: wl.run(stream)  # noqa: E731
        if graphed:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream, capture_error_mode="thread_local"):
                for _ in range(G):
                    wl.run(stream)
            step = graph.replay
            step()
            stream.synchronize()
        flush_buf = torch.empty(2 * l2_bytes // 4, dtype=torch.float32, device=dev) if flush else None
        barrier()
        torch.cuda.synchronize()
        clocks = ClockSampler(dev.index)
        clocks.start()
        nrep = args.steps // G
        ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(nrep)]
        ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(nrep)]
        for i in range(nrep):
            if flush:
                flush_buf.fill_(float(i))
            ev0[i].record(stream)
            step()
            ev1[i].record(stream)
        stream.synchronize()
        torch.cuda.synchronize()
        barrier()
        clk = clocks.stop()
    per_step = [ev0[i].elapsed_time(ev1[i]) / G for i in range(nrep)]
    total_ms = sum(per_step) * G
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = flops * world * args.steps / (total_ms * 1e-3) / 1e12

    # ---- end-to-end through the C-ABI host path (pinned host buffers) ----
    hin, hout = wl.host_buffers()
    for _ in range(2):
        plan.run_host(hin, hout)
    barrier()
    e2e_steps = max(3, min(args.steps, 10))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        plan.run_host(hin, hout)
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item())
    h2d = sum(hin[i].numel() * hin[i].element_size() for i in wl.step_inputs)
    d2h = sum(x.numel() * x.element_size() for x in hout)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    pk, pk_src = peaks()
    bound = bound_of(cfg)
    kern_ms = statistics.mean(per_step)
    if bound == "hbm":
        achieved = nbytes / (kern_ms * 1e-3) / 1e9
        peak, unit, psrc = pk["hbm_gbs"], "GB/s", f"{pk_src} hbm_gbs (MEASURED_PEAKS.json)"
    elif cfg["dtype"] == "f32":
        # fp32 SIMT FMA peak: 148 SMs x 128 lanes x 2 FLOP x max SM clock
        peak = 148 * 128 * 2 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        achieved = flops / (kern_ms * 1e-3) / 1e12
        unit, psrc, bound = "TFLOP/s", "fp32 SIMT FMA peak at max SM clock (no tensor cores on this path)", "compute"
    else:
        achieved = flops / (kern_ms * 1e-3) / 1e12
        unit = "TFLOP/s"
        if cfg["pattern"] == "quant":
            fp8 = fp8_peak()
            if fp8:
                peak = fp8
                psrc = ("measured e4m3 cuBLASLt peak (torch._scaled_mm 16384^3, "
                        "profiles/r1c_fp8_peak.json; MEASURED_PEAKS.json has no FP8 entry)")
            else:
                peak = 2 * pk["bf16_tflops"]
                psrc = f"2 x {pk_src} bf16 burst (dense FP8 = 2x BF16 tensor rate on sm_100)"
        else:
            peak = pk["bf16_tflops"]
            psrc = f"{pk_src} bf16 burst (MEASURED_PEAKS.json)"
    traffic = None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        traffic = json.load(open(prof)).get(cfg["name"].split(":")[0])
    par = (f"split-KV over {world} GPUs: local partials + NCCL all-gather + slice-ordered merge"
           if getattr(wl, "split_kv", False)
           else f"batch/head (or token) shards x{world}, no data-path collective")
    conf = {"workload": cfg["name"], "kernel": plan.info["kernel"], "parallelism": par,
            "launch": f"CUDA graph of {G} step(s), replayed {args.steps // G}x" if graphed else "eager launches",
            "l2": (f"step inputs {in_bytes / 1e6:.1f} MB < {l2_bytes / 1e6:.0f} MB L2: L2 flushed "
                   f"({2 * l2_bytes / 1e6:.0f} MB write) before every step, outside the timed events"
                   if flush else f"step inputs {in_bytes / 1e6:.0f} MB > {l2_bytes / 1e6:.0f} MB L2, no flush")}
    conf.update({k: v for k, v in cfg.items() if k not in ("name", "pattern", "dtype")})
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": {"quant": "e4m3 (bf16 in)", "rms": "bf16", "ln": "bf16", "router": "bf16", "mla": "bf16"}.get(cfg["pattern"], cfg["dtype"]),
        "data": wl.data,
        "config": conf,
        "roofline": {"bound": bound, "achieved": round(achieved, 2), "peak": round(peak, 1),
                     "unit": unit, "frac": round(achieved / peak, 4), "traffic": traffic,
                     "peak_source": psrc,
                     "algorithmic": {"flops": flops, "bytes": nbytes}},
        "e2e": {"value": round(flops * e2e_steps / e2e_s / 1e12, 3), "unit": "TFLOP/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": "rf_run_host (C-ABI, pinned host buffers, chunked H2D/compute/D2H)"},
        "gpu_launches": args.steps * plan.launches_per_run,
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_reference(cfg)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    flops, _ = work_of(cfg)
    t0 = time.perf_counter()
    vals = []
    cb = None
    step_budget = min(5.0, max(0.5, 40.0 / args.steps))
    for _ in range(args.warmup):
        cpu_reference(cfg, budget_s=0.5)
    for _ in range(args.steps):
        cb = cpu_reference(cfg, budget_s=step_budget)
        if cb is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_driver not built"}))
            return
        vals.append(cb["value"])
    value = statistics.median(vals)
    cb["value"] = value
    print(json.dumps({
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "TFLOP/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": flops / (value * 1e12) * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (" + {
            "attention": "the reference's own make_attention generator",
            "quant": "the reference's own make_quant_gemm generator",
            "rms": "the reference's DSL input generator for the RMSNorm->GEMM cascade",
            "ln": "the reference's DSL input generator for the LayerNorm->GEMM cascade",
            "router": "x, w ~ U(-1,1); scores through make_moe_routing's cascade",
            "mla": "the reference's own make_attention generator at hd 512",
        }[cfg["pattern"]] + ")",
        "config": {"workload": cfg["name"]},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t0,
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=1, help="index into BASELINE.json configs")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch each step eagerly")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
