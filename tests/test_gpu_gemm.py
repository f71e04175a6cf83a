"""GPU parity of the GEMM-shaped fused cascades (gemm_sm100.cu):
RMSNorm statistics -> GEMM and per-token absmax -> e4m3 -> GEMM, against the
oracle evaluated on the same rounded inputs (tolerance 2e-2, north_star), and
against the reference's own golden fixtures (tests/golden/)."""
import numpy as np
import pytest

from tests import oracle as O

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _err(a, b):
    return O.scaled_max_err(np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64))[0]


def _rms_run(x, g, w, eps=1e-6):
    import torch
    from paper_2603_10026_b200 import rmsnorm_gemm, rmsnorm_gemm_plan

    T, K = x.shape
    N = w.shape[1]
    p = rmsnorm_gemm_plan(T, K, N, eps)
    assert "tcgen05" in p.info["kernel"]
    wp = p.pack_weight(torch.tensor(w, dtype=torch.float32).cuda(),
                       torch.tensor(g, dtype=torch.float32).cuda())
    xd = torch.tensor(x).to(torch.bfloat16).cuda()
    ss, y = rmsnorm_gemm(xd, wp, eps)
    torch.cuda.synchronize()
    return ss.double().cpu().numpy(), y.double().cpu().numpy(), wp.double().cpu().numpy()


@pytest.mark.parametrize("shape", [(128, 64, 256), (256, 512, 512), (384, 1024, 768)])
def test_rmsnorm_gemm_vs_oracle(shape):
    T, K, N = shape
    rng = np.random.default_rng(T + K + N)
    x = O.round_bf16(rng.uniform(-1, 1, (T, K)))
    g = rng.uniform(-1, 1, K)
    w = rng.uniform(-1, 1, (K, N))
    ss, y, wp = _rms_run(x, g, w)
    # same rounded inputs: x in bf16, W' = bf16(g w) (the packed operand)
    d1, yr = O.rmsnorm_gemm(x, np.ones(K), wp.T)
    assert _err(ss, d1) < 1e-5
    assert _err(y, yr) < TOL
    # deviation from the real-arithmetic oracle (unrounded g, w) is the bf16
    # rounding of W' = g w itself: reported, loosely bounded, not the gate
    _, yreal = O.rmsnorm_gemm(x, g, w)
    assert _err(y, yreal) < 0.15


@pytest.mark.parametrize("name", O.golden_names("rmsnorm_gemm_"))
def test_rmsnorm_gemm_against_reference_goldens(name):
    """The reference engine's own run_unfused / run_incremental results, with
    the golden row embedded in a tile-aligned problem (zero padding)."""
    gd = O.load_golden(name)
    K, N = gd["in.w"].shape
    x = np.zeros((128, K))
    x[0] = gd["in.x"]
    w = np.zeros((K, 256))
    w[:, :N] = gd["in.w"]
    ss, y, wp = _rms_run(x, gd["in.g"], w)
    # gate: the oracle (pinned to these goldens by test_oracle_golden) on the
    # same bf16-rounded operands the kernel consumed
    xr = O.round_bf16(x[:1])
    d1r, yr = O.rmsnorm_gemm(xr, np.ones(K), wp.T)
    assert _err(ss[:1], d1r) < 1e-5
    assert _err(y[0, :N], yr[0, :N]) < TOL
    # the reference's own unrounded results: within bf16 input-rounding error
    assert _err(ss[:1], gd["oracle.d1"]) < 1e-2
    assert _err(y[0, :N], gd["oracle.d2"]) < 0.1
    assert _err(y[0, :N], gd["incremental.d2"]) < 0.1
    assert np.all(y[1:] == 0)


def test_rmsnorm_gemm_unsupported_shape_raises():
    from paper_2603_10026_b200 import UnsupportedPattern, rmsnorm_gemm_plan

    with pytest.raises(UnsupportedPattern):
        rmsnorm_gemm_plan(100, 64, 256)
