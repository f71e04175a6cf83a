"""The drop-in check (oracle/dropin_check.cpp): the reference's own workloads
through the reference executors AND the reference-side CUDA binding
(integration/redfuse_cuda.cpp), compared with the reference's own
compare_reports (values and load counters)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_check")


@pytest.mark.gpu
def test_reference_workloads_through_cuda_binding():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_check not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    bad = [x for x in lines if x.get("pass") is False or x.get("not_fusable") is False]
    assert r.returncode == 0 and not bad, (r.stdout[-3000:], r.stderr[-2000:])
    assert lines[-1]["failures"] == 0
    fp32 = [x for x in lines if x.get("gate") == "max_rel 1.0e-05"]
    assert len(fp32) >= 20 and all(x["input_load_delta"] == 0 for x in fp32)


VERIFY = os.path.join(ROOT, "oracle", "_ref", "redfuse-verify")
BUILTINS = ["safe_softmax", "attention", "moe_routing", "quant_gemm", "sum_sum", "variance",
            "moment_of_inertia"]


def _verify(args):
    if not os.path.exists(VERIFY):
        pytest.skip("oracle/_ref/redfuse-verify not built (needs /root/reference at build time)")
    r = subprocess.run([VERIFY, "verify", "--json", "--seeds", "2"] + args, capture_output=True,
                       text=True, timeout=600)
    return r.returncode, json.loads(r.stdout) if r.stdout.strip().startswith("{") else None, r


@pytest.mark.gpu
@pytest.mark.parametrize("name", BUILTINS)
def test_cli_verify_cuda_mode_on_every_builtin(name):
    """the reference CLI's verify loop with cuda modes — every
    reference builtin runs on librf_cuda and passes its gate."""
    rc, j, r = _verify(["--workload", name])
    assert rc == 0, (r.stdout[-3000:], r.stderr[-2000:])
    modes = {m["mode"]: m for m in j["modes"]}
    assert j["version"] == 1 and j["pass"] is True
    assert all(m["pass"] for m in j["modes"]) and {"cuda", "cuda-multi:4"} <= set(modes)
    assert modes["cuda"]["gpu"]["pattern"]


@pytest.mark.gpu
def test_cli_verify_dsl_specs(tmp_path):
    """--spec DSL cascades routed through the pattern matcher (RMSNorm / LayerNorm
    -> GEMM) and a cascade with no kernel (exit code 2, like NotFusable)."""
    sig = "sqrt(d2 * INVK - d1 * INVK * d1 * INVK + EPS)"
    specs = {
        "rms": "cascade rms\ninput x len 256\ninput g len 256\ninput w len 256 free 48\n"
               "const INVK = 0.00390625\nconst EPS = 1e-6\nreduce 1 op sum\n    x[l] * x[l]\n"
               "reduce 2 op sum free 48\n    x[l] * g[l] / sqrt(d1 * INVK + EPS) * w[l, f]\n",
        "ln": "cascade ln\ninput x len 256\ninput g len 256\ninput w len 256 free 48\n"
              "const INVK = 0.00390625\nconst EPS = 1e-5\nreduce 1 op sum\n    x[l]\n"
              "reduce 2 op sum\n    x[l] * x[l]\nreduce 3 op sum free 48\n"
              f"    x[l] * g[l] * w[l, f] / {sig}\nreduce 4 op sum free 48\n"
              f"    d1 * INVK * g[l] * w[l, f] / {sig}\n",
    }
    for nm, text in specs.items():
        f = tmp_path / f"{nm}.cascade"
        f.write_text(text)
        rc, j, r = _verify(["--spec", str(f), "--modes", "incremental,cuda"])
        assert rc == 0 and j["pass"], (nm, r.stdout[-3000:], r.stderr[-2000:])
    f = tmp_path / "prod.cascade"
    f.write_text("cascade prod_chain\ninput x len 64\nreduce 1 op prod\n    x[l]\n"
                 "reduce 2 op sum\n    x[l] / d1\n")
    rc, j, r = _verify(["--spec", str(f), "--modes", "incremental,cuda"])
    assert rc == 2 and j["modes"][1]["pass"] is False


@pytest.mark.gpu
@pytest.mark.parametrize("name,levels", [("safe_softmax", "1024,32,4,1"), ("attention", "256,16,4,1"),
                                         ("sum_sum", "1024,32,8,1"), ("variance", "8192,16,4,1"),
                                         ("quant_gemm", "512,4,1")])
def test_cli_verify_cuda_fused_mode(name, levels):
    """The reference CLI's fused@k next to cuda-fused@k (run_fused on librf_cuda,
    simulator.cpp:485-559) at every level k of a 3- or 2-level tree."""
    depth = len(levels.split(",")) - 1
    modes = ",".join([f"fused@{k}" for k in range(1, depth + 1)] +
                     [f"cuda-fused@{k}" for k in range(1, depth + 1)])
    rc, j, r = _verify(["--workload", name, "--levels", levels, "--modes", modes])
    assert rc == 0, (r.stdout[-3000:], r.stderr[-2000:])
    got = {m["mode"]: m for m in j["modes"]}
    assert all(m["pass"] for m in j["modes"]) and set(got) == set(modes.split(","))
