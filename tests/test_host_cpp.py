"""The C++ host layer (include/rf_host.hpp) — the drop-in mirror of the
reference's C++ operator API — exercised by tests/cpp/test_host.cpp, written
after the reference's tests/test_simulator.cpp."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_host")


def _run(mode):
    if not os.path.exists(BIN):
        import __graft_entry__

        __graft_entry__.build()
    r = subprocess.run([BIN, mode], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout


def test_host_layer_cpu():
    """DSL parsing, pattern matching (NotFusable), shape/segmentation errors,
    compare_reports — no device needed."""
    _run("cpu")


@pytest.mark.gpu
def test_host_layer_gpu():
    """run_incremental / run_multisegment through librf_cuda on reference-shaped
    TensorStores (softmax, attention, quant 896 known answer, DomainError, RMS)."""
    _run("gpu")
