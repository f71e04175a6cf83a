"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/rf_cuda.h declares, and fails loudly (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "rf_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rf_[a-z_]+)\s*\(", src)))


def test_header_declares_expected_entry_points():
    syms = _declared_symbols()
    for s in ["rf_plan_create", "rf_run", "rf_run_host", "rf_merge_partials", "rf_pack_weight",
              "rf_plan_destroy", "rf_status_string", "rf_check_domain"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2603_10026_b200 import _native as N

    h = ctypes.CDLL(N.LIB_PATH)
    for s in _declared_symbols():
        assert hasattr(h, s), s
    assert set(_declared_symbols()) == set(N.SIGNATURES)


def test_abi_version_and_status_strings():
    from paper_2603_10026_b200 import _native as N

    L = N.lib()
    assert L.rf_abi_version() == N.ABI_VERSION == 4
    assert b"ShapeMismatch" in L.rf_status_string(N.RF_ERR_SHAPE)
    assert b"IncompatibleSegmentation" in L.rf_status_string(N.RF_ERR_SEGMENTATION)
    assert b"DomainError" in L.rf_status_string(N.RF_ERR_DOMAIN)


def test_segmentation_checked_before_device():
    """IncompatibleSegmentation (simulator.cpp:668-671) is a descriptor error."""
    from paper_2603_10026_b200 import Desc, IncompatibleSegmentation, Plan, _native as N

    with pytest.raises(IncompatibleSegmentation):
        Plan(Desc(N.RF_PATTERN_ATTENTION, "f32", rows=4, len=6, free_len=64, segments=4))


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_10026_b200 import CudaError, Desc, Plan, _native as N

    with pytest.raises(CudaError):
        Plan(Desc(N.RF_PATTERN_ATTENTION, "f32", rows=4, len=8, free_len=64))


def test_null_arguments_are_rejected():
    from paper_2603_10026_b200 import _native as N

    L = N.lib()
    assert L.rf_plan_create(None, None) == N.RF_ERR_ARG
    assert L.rf_run(None, None, None) == N.RF_ERR_ARG
