"""Benchmark of the fused cascaded-reduction hot path (driver contract).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1] [--also 0,2,...]
                  [--impl ours|reference] [--scaling strong|weak] [--dist-backend nccl|gloo]

A "step" is one pass of the fused loop (rf_run) over one batch of synthetic
input of a BASELINE.json configuration. Default workload = configs[1]
(bf16 MHA prefill B8 H32 S4096 D128, non-causal) — the config the metric is
quoted on that fits one GPU; the other configs (`--also`, default all) are
measured in the same run and reported under `other_configs`.

Multi-GPU (one process per GPU; `--gpus N` starts the N ranks itself when no
torchrun environment is present): by default every config is split over the
ranks as BASELINE/SURVEY §8e state it ("scaling": "strong") — prefill by (b,h)
units, decode by KV range (split-KV: partials, NCCL all-gather and the
slice-ordered merge inside every step), the GEMM patterns by token tiles, MLA
by batch; cfg1 runs replicas. `--scaling weak` gives every rank the whole
config. The timed region is bracketed by barriers and the time is the max
over ranks; `value` is the whole job's FLOPs / that time.

After the timed region the outputs the timed steps wrote are checked on
sampled rows against the oracle (tests/bench_parity.py; reported as `parity`,
never timed). `--impl reference` times the reference's own CPU fused loop
(oracle/_ref/ref_driver, built from /root/reference/proj/src: run_incremental
per row on all host threads) on a bounded sample of the same workload. Those
two legs and `cpu_baseline` are the only places this file touches oracle/.
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
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows),
                "note": ("nvidia-smi clock counters refresh every ~100 ms, longer than short timed windows; "
                         "under sw_power_cap the device-side clock of the tensor-bound kernels is lower "
                         "(cfg2: profiles/r2g_attn_effective_clock.txt, tools/attn_clock.py)")}


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
        "rows": r["rows"],
    }


GRAN = {"quant": 128, "rms": 128, "ln": 256, "router": 128}  # row tile of the GEMM kernels


def parallelism(cfg, world, scaling):
    """How the config is split over `world` GPUs (rank-independent text; the
    reference arm prints the same config dict)."""
    pat = cfg["pattern"]
    if world == 1:
        return "1 GPU"
    if scaling == "weak":
        return f"weak: every one of {world} ranks runs the whole config on its own data"
    if pat == "attention" and cfg["dtype"] == "f32":
        return f"replicas: cfg1 is too small to shard (SURVEY §8e); {world} independent replicas"
    if pat == "attention" and cfg["Sq"] == 1:
        return (f"split-KV: rank r owns keys [r*Skv/{world}, (r+1)*Skv/{world}) of every (b,h); "
                f"local partials, NCCL all-gather, slice-ordered merge inside every step")
    if pat == "attention":
        return f"batch/head: B*H (b,h) units split {world} ways, no data-path collective"
    if pat == "mla":
        return f"batch: B split {world} ways (heads share a batch's cache), no collective"
    return f"tokens: M split {world} ways in {GRAN[pat]}-row tiles, W replicated, no collective"


def scaling_label(cfg, world, scaling):
    if scaling == "weak" or (cfg["pattern"] == "attention" and cfg["dtype"] == "f32"):
        return "weak"
    return "strong"


def local_config(cfg, rank, world, scaling):
    """This rank's share of the config: a dict with the same keys
    plus `split_kv` / `segments_global` for the split-KV decode."""
    from paper_2603_10026_b200.distributed import shard_units

    c = dict(cfg)
    c["split_kv"] = False
    if world == 1 or scaling_label(cfg, world, scaling) == "weak":
        return c
    pat = cfg["pattern"]
    if pat == "attention" and cfg["Sq"] == 1:
        if cfg["Skv"] % world:
            raise SystemExit(f"Skv {cfg['Skv']} does not split over {world} GPUs")
        c["Skv"] = cfg["Skv"] // world
        c["split_kv"] = True
        seg = max(cfg.get("segments", 1), world)
        c["segments_global"] = seg + (-seg) % world
    elif pat == "attention":
        b0, b1 = shard_units(cfg["B"] * cfg["H"], rank, world)
        c["B"], c["H"] = 1, b1 - b0
    elif pat == "mla":
        b0, b1 = shard_units(cfg["B"], rank, world)
        c["B"] = b1 - b0
    else:
        g = GRAN[pat]
        t0, t1 = shard_units(cfg["M"] // g, rank, world)
        c["M"] = (t1 - t0) * g
    if min(c.get("B", 1), c.get("H", 1), c.get("M", 1)) < 1:
        raise SystemExit(f"{cfg['name']}: nothing left to shard onto rank {rank} of {world}")
    return c


class Dist:
    """One process per GPU (torchrun env); NCCL, or gloo for a one-GPU
    multi-rank smoke run (--dist-backend gloo)."""

    def __init__(self, backend):
        import torch

        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.backend = backend
        if torch.cuda.is_available():
            torch.cuda.set_device(self.local % torch.cuda.device_count())
            self.dev = torch.device("cuda", torch.cuda.current_device())
        else:  # host-logic tests (gloo on CPU); every GPU leg needs a device
            self.dev = torch.device("cpu")
        if self.world > 1:
            import torch.distributed as dist

            if backend == "nccl":
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group("gloo")

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist

            dist.barrier()

    def max(self, x):
        """Max over ranks of a host float."""
        if self.world == 1:
            return x
        import torch
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64,
                         device=self.dev if self.backend == "nccl" else "cpu")  # gloo: host tensors
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def gather_objects(self, obj):
        if self.world == 1:
            return [obj]
        import torch.distributed as dist

        out = [None] * self.world
        dist.all_gather_object(out, obj)
        return out

    def gather_seq(self, t):
        """All-gather [rows, S_local, D] shards along the sequence axis, rank
        order = slice order."""
        if self.world == 1:
            return t
        import torch
        import torch.distributed as dist

        src = t.contiguous() if self.backend == "nccl" else t.contiguous().cpu()
        parts = [torch.empty_like(src) for _ in range(self.world)]
        dist.all_gather(parts, src)
        return torch.cat(parts, dim=1).to(t.device)

    def close(self):
        if self.world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


class Workload:
    """Plan + device buffers of this rank's share of a config. Plan-time work
    (weight packing) happens here, outside every timed region. Per-step data
    (activations, Q/K/V, caches) is drawn per rank (a distinct shard of one
    global problem); static weights and the decode query are identical on
    every rank."""

    def __init__(self, cfg, dev, rank=0, stream=None):
        import torch

        from paper_2603_10026_b200 import Desc, Plan
        from paper_2603_10026_b200 import _native as N

        g = torch.Generator(device=dev)
        g.manual_seed(1234 + 7919 * rank)
        gs = torch.Generator(device=dev)  # shared (replicated) tensors
        gs.manual_seed(99)
        rnd = lambda *shape, gen=g: torch.rand(*shape, device=dev, generator=gen)  # noqa: E731
        self.local = cfg
        self.split_kv = cfg.get("split_kv", False)
        pat = cfg["pattern"]
        if pat == "mla":
            B, S = cfg["B"], cfg["Skv"]
            q = (rnd(B, 128, 576) * 2 - 1).bfloat16()
            kv = (rnd(B, S, 576) * 2 - 1).bfloat16()
            self.desc = Desc(N.RF_PATTERN_MLA_DECODE, "bf16", rows=1, len=S, free_len=512, batch=B,
                             heads=128, segments=cfg.get("segments", 1), softmax_scale=576 ** -0.5,
                             producer_len=576, device=dev.index)
            self.inputs = [q, kv]
            m = torch.empty(B, 128, device=dev)
            self.outputs = [m, torch.empty_like(m), torch.empty(B, 128, 512, dtype=torch.bfloat16, device=dev)]
            self.step_inputs = [0, 1]
            self.data = "synthetic (q, cache ~ U(-1,1) bf16; cache rows [c_kv 512 | k_rope 64])"
        elif pat == "attention":
            dt = torch.float32 if cfg["dtype"] == "f32" else torch.bfloat16
            B, H, Sq, Skv, D = cfg["B"], cfg["H"], cfg["Sq"], cfg["Skv"], cfg["D"]
            q = ((rnd(B, H, Sq, D, gen=gs if self.split_kv else g) * 2 - 1) / D ** 0.5).to(dt)
            k = (rnd(B, H, Skv, D) * 2 - 1).to(dt)
            v = (rnd(B, H, Skv, D) * 2 - 1).to(dt)
            segs = (cfg["segments_global"] // int(os.environ.get("WORLD_SIZE", "1"))
                    if self.split_kv else cfg.get("segments", 1))
            self.desc = Desc(N.RF_PATTERN_ATTENTION, cfg["dtype"], rows=Sq, len=Skv, free_len=D,
                             batch=B, heads=H, segments=segs, device=dev.index)
            self.inputs = [q, k, v]
            m = torch.empty(B, H, Sq, device=dev)
            self.outputs = [m, torch.empty_like(m), torch.empty_like(q)]
            self.step_inputs = [0, 1, 2]
            self.data = "synthetic (uniform, make_attention distributions; q pre-scaled by 1/sqrt(D))"
        else:
            M, K, Nn = cfg["M"], cfg["K"], cfg["N"]
            if pat == "router":
                a = (rnd(M, K) * 2 - 1).bfloat16()
                self.desc = Desc(N.RF_PATTERN_MOE_ROUTER, "bf16", rows=M, len=Nn, free_len=cfg["topk"],
                                 producer_len=K, device=dev.index)
                w = (rnd(K, Nn, gen=gs) * 2 - 1) / K ** 0.5
                self.outputs = [torch.empty(M, device=dev), torch.empty(M, device=dev),
                                torch.empty(M, cfg["topk"], 2, dtype=torch.int32, device=dev)]
                self.data = "synthetic (x ~ U(-1,1) bf16, router w ~ U(-1,1)/sqrt(hd) packed bf16)"
                gam = None
            elif pat == "quant":
                a = (rnd(M, K) * 4 - 2).bfloat16()  # make_quant_gemm: a ~ U(-2, 2)
                self.desc = Desc(N.RF_PATTERN_QUANT_GEMM_E4M3, "bf16", rows=M, len=K, free_len=Nn,
                                 device=dev.index)
                w = rnd(K, Nn, gen=gs) * 2 - 1  # w ~ U(-1, 1)
                self.outputs = [torch.empty(M, device=dev), torch.empty(M, Nn, device=dev)]
                self.data = "synthetic (make_quant_gemm distributions: a~U(-2,2), w~U(-1,1) packed e4m3)"
                gam = None
            else:
                a = (rnd(M, K) * 2 - 1).bfloat16()
                ln = pat == "ln"
                self.desc = Desc(N.RF_PATTERN_LAYERNORM_GEMM if ln else N.RF_PATTERN_RMSNORM_GEMM, "bf16",
                                 rows=M, len=K, free_len=Nn, eps=1e-5 if ln else 1e-6, device=dev.index)
                w = rnd(K, Nn, gen=gs) * 2 - 1
                gam = rnd(K, gen=gs) * 2 - 1
                d1 = torch.empty(M, device=dev)
                self.outputs = ([d1, torch.empty_like(d1)] if ln else [d1]) + \
                    [torch.empty(M, Nn, dtype=torch.bfloat16, device=dev) for _ in range(2 if ln else 1)]
                self.data = "synthetic (DSL wrap_spec convention: x, g, w ~ U(-1,1); g folded into bf16 W)"
            self.plan = Plan(self.desc)
            wp = self.plan.pack_weight(w, gam)
            del w
            self.inputs = [a, wp]
            self.step_inputs = [0]  # the packed weight is plan-time resident
        if not hasattr(self, "plan"):
            self.plan = Plan(self.desc)
        torch.cuda.synchronize()

    def run(self, stream):
        if self.split_kv:
            from paper_2603_10026_b200.distributed import split_kv_decode

            q, k, v = self.inputs
            self.outputs = list(split_kv_decode(q, k, v, self.local["segments_global"], stream=stream))
        else:
            self.plan.run_unchecked(self.inputs, self.outputs, stream)

    def step_bytes(self):
        return sum(self.inputs[i].numel() * self.inputs[i].element_size() for i in self.step_inputs)

    def launches(self, world):
        if self.split_kv:  # partials kernel + merge kernel (+ the NCCL all-gather)
            return 2
        return self.plan.launches_per_run

    def host_buffers(self):
        import torch

        hin = [x.cpu().pin_memory() if i in self.step_inputs else x
               for i, x in enumerate(self.inputs)]
        hout = [torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in self.outputs]
        return hin, hout

    def run_host(self, hin, hout, stream):
        """One end-to-end call from pinned host memory: the C-ABI rf_run_host,
        or for split-KV the public split_kv_decode between the copies."""
        import torch

        if not self.split_kv:
            self.plan.run_host(hin, hout)
            return
        with torch.cuda.stream(stream):
            dq, dk, dv = (x.to(self.inputs[0].device, non_blocking=True) for x in hin)
            from paper_2603_10026_b200.distributed import split_kv_decode

            out = split_kv_decode(dq, dk, dv, self.local["segments_global"], stream=stream)
            for h, d in zip(hout, out):
                h.copy_(d, non_blocking=True)
        stream.synchronize()


def measure(cfg, args, D, steps, warmup, want_cpu, cpu_budget):
    """Times one config on this rank (all ranks call it) and returns rank 0's
    dict (None elsewhere)."""
    import torch

    scaling = args.scaling
    lcfg = local_config(cfg, D.rank, D.world, scaling)
    stream = torch.cuda.Stream(device=D.dev)
    wl = Workload(lcfg, D.dev, D.rank, stream)
    plan = wl.plan
    flops_total, _ = work_of(cfg)
    lflops, lbytes = work_of(lcfg)
    label = scaling_label(cfg, D.world, scaling)
    job_flops = flops_total * (D.world if label == "weak" else 1)

    with torch.cuda.stream(stream):
        for _ in range(warmup):
            wl.run(stream)
        stream.synchronize()
        # Inputs smaller than L2 would stay L2-resident across steps: then L2
        # is flushed (a 2x-L2 buffer write) before every step, outside the
        # per-step events. Larger inputs: G consecutive steps are captured once
        # as a CUDA graph and replayed K/G times, so host launch cost stays off
        # the device timeline; every step's kernels still run. The split-KV
        # step (NCCL all-gather) runs eagerly.
        l2_bytes = torch.cuda.get_device_properties(D.dev).L2_cache_size
        in_bytes = wl.step_bytes()
        flush = in_bytes < l2_bytes
        graphed = not args.no_graph and not wl.split_kv
        G = 1 if (flush or not graphed) else max(g for g in range(1, 21) if steps % g == 0)
        step = lambda: wl.run(stream)  # noqa: E731
        if graphed:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream, capture_error_mode="thread_local"):
                for _ in range(G):
                    wl.run(stream)
            step = graph.replay
            step()
            stream.synchronize()
        flush_buf = torch.empty(2 * l2_bytes // 4, dtype=torch.float32, device=D.dev) if flush else None
        D.barrier()
        torch.cuda.synchronize()
        clocks = ClockSampler(D.dev.index)
        clocks.start()
        nrep = steps // G
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
        D.barrier()
        clk = clocks.stop()
    per_step = [ev0[i].elapsed_time(ev1[i]) / G for i in range(nrep)]
    total_ms = D.max(sum(per_step) * G)
    ms_per_step = total_ms / steps
    value = job_flops * steps / (total_ms * 1e-3) / 1e12

    # ---- parity of the buffers the timed steps wrote (checker; untimed) ----
    parity = None
    if not args.no_parity:
        from tests import bench_parity

        try:
            mine = bench_parity.check(wl, gather_rows=D.gather_seq)
        except Exception as e:  # a checker failure is reported, never hidden
            mine = {"pass": False, "error": f"{type(e).__name__}: {e}"}
        allp = D.gather_objects(mine)
        parity = allp[0] if D.world == 1 else merge_parity(allp)

    # ---- end-to-end through the public API from pinned host buffers ----
    hin, hout = wl.host_buffers()
    e2e_steps = max(3, min(steps, 10)) if in_bytes < 4e9 else 3
    for _ in range(2):
        wl.run_host(hin, hout, stream)
    D.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        wl.run_host(hin, hout, stream)
    e2e_s = D.max(time.perf_counter() - t0)
    h2d = sum(hin[i].numel() * hin[i].element_size() for i in wl.step_inputs)
    d2h = sum(x.numel() * x.element_size() for x in hout)
    kernel = plan.info["kernel"]
    launches = wl.launches(D.world)
    del hin, hout
    if D.rank != 0:
        return None

    pk, pk_src = peaks()
    bound = bound_of(cfg)
    kern_ms = statistics.mean(per_step)  # rank 0's own step (its share of the config)
    if bound == "hbm":
        achieved = lbytes / (kern_ms * 1e-3) / 1e9
        peak, unit, psrc = pk["hbm_gbs"], "GB/s", f"{pk_src} hbm_gbs (MEASURED_PEAKS.json)"
    elif cfg["dtype"] == "f32":
        # fp32 SIMT FMA peak: 148 SMs x 128 lanes x 2 FLOP x max SM clock
        peak = 148 * 128 * 2 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        achieved = lflops / (kern_ms * 1e-3) / 1e12
        unit, bound = "TFLOP/s", "compute"
        psrc = "fp32 SIMT FMA peak at max SM clock (no tensor cores on this path)"
        if "tf32" in kernel:
            # fp32-accurate products as 3xTF32 tcgen05 MMAs: the tensor rate for
            # tf32 is half the bf16 rate, and every product costs three MMAs
            simt_peak, peak, bound = peak, pk["bf16_tflops"] / 6, "tensor"
            psrc = (f"{pk_src} bf16 burst / 2 (tf32 rate) / 3 (3xTF32 passes); the fp32 SIMT FMA peak "
                    f"{simt_peak:.1f} TFLOP/s is roofline.fp32_simt_peak. Latency-bound at this size "
                    "(1 MB problem, L2 flushed): neither peak is approachable")
    else:
        achieved = lflops / (kern_ms * 1e-3) / 1e12
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
    if os.path.exists(prof) and D.world == 1:
        traffic = json.load(open(prof)).get(cfg["name"].split(":")[0])
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "TFLOP/s",
        "n_gpus": D.world,
        "steps": steps,
        "warmup": warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": label,
        "vs_baseline": None,
        "dtype": {"quant": "e4m3 (bf16 in)", "rms": "bf16", "ln": "bf16", "router": "bf16",
                  "mla": "bf16"}.get(cfg["pattern"], cfg["dtype"]),
        "data": wl.data,
        "config": config_dict(cfg, D.world, scaling),
        "impl_detail": {
            "kernel": kernel,
            "launch": (f"CUDA graph of {G} step(s), replayed {steps // G}x" if graphed
                       else "eager launches (NCCL all-gather inside the step)"),
            "l2": (f"step inputs {in_bytes / 1e6:.1f} MB/rank < {l2_bytes / 1e6:.0f} MB L2: L2 flushed "
                   f"({2 * l2_bytes / 1e6:.0f} MB write) before every step, outside the timed events"
                   if flush else f"step inputs {in_bytes / 1e6:.0f} MB/rank > {l2_bytes / 1e6:.0f} MB L2, no flush"),
            "rank0_share": {k: lcfg[k] for k in ("B", "H", "M", "Skv") if k in lcfg},
            "dist_backend": D.backend if D.world > 1 else None,
        },
        "roofline": {"bound": bound, "achieved": round(achieved, 2), "peak": round(peak, 1),
                     "unit": unit, "frac": round(achieved / peak, 4), "traffic": traffic,
                     "peak_source": psrc,
                     "algorithmic": {"flops": lflops, "bytes": lbytes,
                                     "per": "rank 0's launch (its share of the config)"},
                     **({"fp32_simt_peak": round(simt_peak, 1), "frac_vs_fp32_simt": round(achieved / simt_peak, 4)}
                        if cfg["dtype"] == "f32" and "tf32" in kernel else {})},
        "e2e": {"value": round(job_flops * e2e_steps / e2e_s / 1e12, 3), "unit": "TFLOP/s",
                "h2d_bytes_per_step": h2d * D.world, "d2h_bytes_per_step": d2h * D.world,
                "path": ("split_kv_decode between pinned-host copies (partials + all-gather + merge)"
                         if wl.split_kv else
                         "rf_run_host (C-ABI, pinned host buffers, chunked H2D/compute/D2H)")},
        "gpu_launches": steps * launches,
        "clocks": clk,
        "parity": parity,
    }
    if want_cpu and D.world == 1:
        line["cpu_baseline"] = cpu_reference(cfg, budget_s=cpu_budget)
    return line


def merge_parity(parts):
    out = dict(parts[0])
    out["rows_checked"] = sum(p.get("rows_checked", 0) for p in parts)
    out["pass"] = all(p.get("pass", False) for p in parts)
    errs = {}
    for p in parts:
        for k, v in (p.get("max_scaled_err") or {}).items():
            if v is not None:
                errs[k] = max(errs.get(k, 0.0), v)
    out["max_scaled_err"] = errs
    out["ranks"] = len(parts)
    return out


def config_dict(cfg, world, scaling):
    conf = {"workload": cfg["name"], "parallelism": parallelism(cfg, world, scaling)}
    conf.update({k: v for k, v in cfg.items() if k not in ("name", "pattern")})
    return conf


def compact(line):
    keep = ("value", "unit", "ms_per_step", "scaling", "dtype", "roofline", "e2e", "parity",
            "gpu_launches", "clocks", "cpu_baseline", "steps", "warmup")
    out = {k: line[k] for k in keep if k in line}
    out["workload"] = line["config"]["workload"]
    out["kernel"] = line["impl_detail"]["kernel"]
    out["l2"] = line["impl_detail"]["l2"]
    return out


def run_ours(args):
    import gc

    import torch

    D = Dist(args.dist_backend)
    line = measure(CONFIGS[args.config], args, D, args.steps, args.warmup,
                   not args.no_cpu_baseline, 12.0)
    also = []
    for idx in args.also:
        if idx == args.config:
            continue
        gc.collect()
        torch.cuda.empty_cache()
        steps = min(args.steps, 20)
        r = measure(CONFIGS[idx], args, D, steps, 3, not args.no_cpu_baseline, 3.0)
        if D.rank == 0:
            also.append(compact(r))
    if D.rank == 0:
        if also:
            line["other_configs"] = also
        print(json.dumps(line), flush=True)
    D.close()


def run_reference(args):
    """The reference's own CPU fused loop (oracle/_ref/ref_driver: redfuse
    run_incremental per row on all host threads), rank 0 only; each step is a
    bounded sample of the config, and the per-step time is the time the
    sampled rows' rate implies for the whole config (extrapolated)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    flops, _ = work_of(cfg)
    t0 = time.perf_counter()
    vals, rows = [], 0
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
        rows += cb.get("rows", 0)
    value = statistics.median(vals)
    cb["value"] = value
    print(json.dumps({
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": flops / (value * 1e12) * 1e3,
        "ms_per_step_is": "extrapolated: the whole config at the sampled rows' rate",
        "extrapolated_from_rows": rows,
        "higher_is_better": True,
        "scaling": scaling_label(cfg, world, args.scaling),
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
        "config": config_dict(cfg, world, args.scaling),
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t0,
    }), flush=True)


def relaunch(args):
    """`--gpus N` without a torchrun environment: start N ranks here."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=1, help="index into CONFIGS (BASELINE.json order)")
    ap.add_argument("--also", default="0,2,3,4,5,6,7",
                    help="other CONFIGS indices measured in the same run and reported under "
                         "other_configs ('' = none)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config is split over the ranks (SURVEY §8e); "
                         "weak: every rank runs the whole config")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: several ranks may share one GPU (smoke runs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch each step eagerly")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    args.also = [int(x) for x in args.also.split(",") if x.strip()]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
