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
