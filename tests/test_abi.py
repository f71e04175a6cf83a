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
    assert L.rf_abi_version() == N.ABI_VERSION == 5
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


def test_fused_tree_is_validated_before_device():
    """run_fused's tree (validate_tree, cascade.cpp:37-66) and fuse level
    (simulator.cpp:491-493) are descriptor errors (ABI v5)."""
    from paper_2603_10026_b200 import Desc, Plan, ShapeMismatch, _native as N

    def mk(tree, k, segments=1):
        return Desc(N.RF_PATTERN_SAFE_SOFTMAX, "f32", rows=2, len=64, segments=segments,
                    fuse_level=k, tree=tuple(tree))

    with pytest.raises(ShapeMismatch):
        Plan(mk((3, 1), 1))           # 3 does not divide 64
    with pytest.raises(ShapeMismatch):
        Plan(mk((8, 2), 1))           # last level must be 1
    with pytest.raises(ShapeMismatch):
        Plan(mk((8, 3, 1), 1))        # 3 does not divide 8
    with pytest.raises(ShapeMismatch):
        Plan(mk((64, 1), 1))          # NotDecreasing: levels [64, 64, 1]
    with pytest.raises(ValueError):
        Plan(mk((8, 1), 3))           # k > depth
    with pytest.raises(ValueError):
        Plan(mk((8, 1), 1, segments=2))  # the tree gives the segments


def test_desc_layout_matches_header():
    """The ctypes rf_desc mirrors include/rf_cuda.h field for field (ABI v5)."""
    from paper_2603_10026_b200 import _native as N

    src = open(os.path.join(ROOT, "include", "rf_cuda.h")).read()
    body = src[src.index("typedef struct rf_desc {"):src.index("} rf_desc;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"\b(int32_t|int64_t|double)\s+(\w+)(\[\d+\])?;", body)
    assert [f[1] for f in fields] == [f[0] for f in N.rf_desc._fields_]
    # sizes and offsets as the C compiler lays the header out
    import subprocess
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        c = os.path.join(td, "l.c")
        with open(c, "w") as f:
            f.write('#include <stddef.h>\n#include <stdio.h>\n#include "rf_cuda.h"\nint main(void){'
                    'printf("%zu %zu %zu", sizeof(rf_desc), offsetof(rf_desc, stat_len), '
                    'offsetof(rf_desc, tree));return 0;}')
        r = subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", os.path.join(td, "l")],
                           capture_output=True, text=True)
        if r.returncode != 0:
            pytest.skip("no C compiler: " + r.stderr[-200:])
        size, off_stat, off_tree = map(int, subprocess.run([os.path.join(td, "l")], capture_output=True,
                                                         text=True).stdout.split())
    assert ctypes.sizeof(N.rf_desc) == size
    assert N.rf_desc.stat_len.offset == off_stat and N.rf_desc.tree.offset == off_tree
