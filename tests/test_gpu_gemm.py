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


@pytest.mark.parametrize("shape", [(128, 64, 256), (256, 512, 512), (384, 1024, 768),
                                   (512, 4096, 512)])
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


# --------------------------------------------------------------- layernorm --


def _ln_run(x, g, w, eps=1e-5, with_d4=True):
    import torch
    from paper_2603_10026_b200 import layernorm_gemm, layernorm_gemm_plan

    T, K = x.shape
    N = w.shape[1]
    p = layernorm_gemm_plan(T, K, N, eps)
    assert "layernorm" in p.info["kernel"]
    raw = p.pack_weight(torch.tensor(w, dtype=torch.float32).cuda(),
                        torch.tensor(g, dtype=torch.float32).cuda())
    wp = raw[: 2 * N * K].view(torch.bfloat16).view(N, K)
    colsum = raw[2 * N * K:].view(torch.float32)
    xd = torch.tensor(x).to(torch.bfloat16).cuda()
    d1, d2, d3, d4 = layernorm_gemm(xd, raw, N, eps, with_d4=with_d4)
    torch.cuda.synchronize()
    f = lambda t: None if t is None else t.double().cpu().numpy()  # noqa: E731
    return f(d1), f(d2), f(d3), f(d4), f(wp), f(colsum)


@pytest.mark.parametrize("shape", [(256, 64, 256), (256, 512, 512), (512, 1024, 768),
                                   (768, 4096, 512)])
@pytest.mark.parametrize("offset", [0.0, 1.5])
def test_layernorm_gemm_vs_oracle(shape, offset):
    T, K, N = shape
    rng = np.random.default_rng(T + K + N)
    x = O.round_bf16(rng.uniform(-1, 1, (T, K)) + offset)
    g = rng.uniform(-1, 1, K)
    w = rng.uniform(-1, 1, (K, N))
    d1, d2, d3, d4, wp, colsum = _ln_run(x, g, w)
    # the packed operand: W' = bf16(g w) and its exact f32 column sums
    assert np.abs(colsum - wp.sum(axis=1)).max() < 1e-4 * max(1.0, np.abs(colsum).max())
    r1, r2, r3, r4 = O.layernorm_gemm(x, np.ones(K), wp.T)
    assert _err(d1, r1) < 1e-5
    assert _err(d2, r2) < 1e-5
    assert _err(d3, r3) < TOL
    assert _err(d4, r4) < TOL
    # the normalised product d3 - d4, RMS-relative (bf16 outputs cancel)
    diff, ref = d3 - d4, r3 - r4
    assert np.sqrt(np.mean((diff - ref) ** 2)) < TOL * np.sqrt(np.mean(ref ** 2))


def test_layernorm_gemm_d4_optional():
    rng = np.random.default_rng(5)
    T, K, N = 256, 128, 256
    x = O.round_bf16(rng.uniform(-1, 1, (T, K)))
    g, w = rng.uniform(-1, 1, K), rng.uniform(-1, 1, (K, N))
    a1, a2, a3, a4, _, _ = _ln_run(x, g, w, with_d4=True)
    b1, b2, b3, b4, _, _ = _ln_run(x, g, w, with_d4=False)
    assert b4 is None
    assert np.array_equal(a1, b1) and np.array_equal(a2, b2) and np.array_equal(a3, b3)


@pytest.mark.parametrize("name", O.golden_names("layernorm_gemm_"))
def test_layernorm_gemm_against_reference_goldens(name):
    gd = O.load_golden(name)
    K, N = gd["in.w"].shape
    x = np.zeros((256, K))
    x[0] = gd["in.x"]
    w = np.zeros((K, 256))
    w[:, :N] = gd["in.w"]
    d1, d2, d3, d4, wp, _ = _ln_run(x, gd["in.g"], w)
    xr = O.round_bf16(x[:1])
    r1, r2, r3, r4 = O.layernorm_gemm(xr, np.ones(K), wp.T)
    assert _err(d1[:1], r1) < 1e-5 and _err(d2[:1], r2) < 1e-5
    assert _err(d3[0, :N], r3[0, :N]) < TOL
    assert _err(d4[0, :N], r4[0, :N]) < TOL
    for tag in ["oracle", "incremental", "multi2"]:
        assert _err(d1[:1], gd[f"{tag}.d1"]) < 1e-2
        assert _err(d2[:1], gd[f"{tag}.d2"]) < 1e-2
        assert _err(d3[0, :N], gd[f"{tag}.d3"]) < 0.1
        assert _err(d4[0, :N], gd[f"{tag}.d4"]) < 0.1
    assert np.all(d3[1:] == 0) and np.all(d4[1:] == 0)


def test_layernorm_gemm_unsupported_shape_raises():
    from paper_2603_10026_b200 import UnsupportedPattern, layernorm_gemm_plan

    with pytest.raises(UnsupportedPattern):
        layernorm_gemm_plan(128, 64, 256)  # the LN kernel is the 2-SM M=256 tile


# ------------------------------------------------------------------- quant --

def _quant_run(a, w, fmax=448.0):
    import torch
    from paper_2603_10026_b200 import quant_gemm, quant_gemm_plan

    M, K = a.shape
    N = w.shape[1]
    p = quant_gemm_plan(M, K, N, fmax)
    assert "tcgen05" in p.info["kernel"]
    wp = p.pack_weight(torch.tensor(w, dtype=torch.float32).cuda())
    ad = torch.tensor(a).to(torch.bfloat16).cuda()
    amax, c = quant_gemm(ad, wp, fmax, check_domain=False)
    torch.cuda.synchronize()
    w8 = wp.view(torch.float8_e4m3fn).double().cpu().numpy().T  # [K, N] static e4m3 weight
    return amax.double().cpu().numpy(), c.double().cpu().numpy(), w8, p


@pytest.mark.parametrize("shape", [(128, 128, 512), (256, 1024, 1024), (128, 2048, 512)])
def test_quant_gemm_vs_oracle(shape):
    M, K, N = shape
    rng = np.random.default_rng(M + K + N)
    a = O.round_bf16(rng.uniform(-2, 2, (M, K)))
    w = rng.uniform(-1, 1, (K, N))
    amax, c, w8, _ = _quant_run(a, w)
    assert np.array_equal(w8, O.round_e4m3(w))  # packing = RNE satfinite e4m3
    d1, cr = O.quant_gemm_e4m3(a, w8, tile_k=128)  # same rounded inputs, kernel's scheme
    assert _err(amax, d1) == 0.0  # absmax is exact
    assert _err(c, cr) < TOL
    assert _err(c, cr) < 1e-3  # same quantisation decisions: only fp32 accumulation differs
    # deviation from the unrounded real-arithmetic reference (reported, not the gate)
    _, creal = O.quant_gemm(a, w)
    rel = np.sqrt(np.mean((c - creal) ** 2)) / np.sqrt(np.mean(creal ** 2))
    assert rel < 0.06


@pytest.mark.parametrize("M", [128, 256])  # 1-SM and 2-SM (cta_group::2) kernels
def test_quant_gemm_rescale_path(M):
    """Magnitudes growing along K force ref (power of two >= running absmax) to
    change on many tiles: the in-loop accumulator correction ref'/ref runs."""
    K, N = 1024, 512
    rng = np.random.default_rng(3)
    grow = 2.0 ** (np.arange(K) // 128)  # x2 per tile
    a = O.round_bf16(rng.uniform(-1, 1, (M, K)) * grow)
    w = rng.uniform(-1, 1, (K, N))
    amax, c, w8, _ = _quant_run(a, w)
    d1, cr = O.quant_gemm_e4m3(a, w8, tile_k=128)
    assert _err(amax, d1) == 0.0
    assert _err(c, cr) < 1e-3


@pytest.mark.parametrize("M", [128, 256])
def test_quant_gemm_known_answer_and_domain_error(M):
    """test_simulator.cpp:53-68: a=[1], w=[[2]] -> d1 = 1, d2 = 896 (padded to a
    tile); an all-zero row is the reference's DomainError (0/0) at finalize."""
    import torch
    from paper_2603_10026_b200 import DomainError

    a = np.zeros((M, 128))
    a[0, 0] = 1.0
    a[1, :] = 0.0  # all-zero row
    a[2:, :] = 0.5
    w = np.zeros((128, 512))
    w[0, 0] = 2.0
    amax, c, _, p = _quant_run(a, w)
    assert amax[0] == 1.0 and c[0, 0] == 896.0
    assert amax[1] == 0.0 and np.isnan(c[1]).all()
    with pytest.raises(DomainError):
        p.check_domain(torch.cuda.current_stream())
    p.check_domain(torch.cuda.current_stream())  # flag cleared


@pytest.mark.parametrize("name", O.golden_names("quant_gemm_"))
def test_quant_gemm_against_reference_goldens(name):
    gd = O.load_golden(name)
    K, N = gd["in.w"].shape
    Kp = -(-K // 128) * 128
    a = np.zeros((128, Kp))
    a[0, :K] = gd["in.a"]
    w = np.zeros((Kp, 512))
    w[:K, :N] = gd["in.w"]
    amax, c, w8, _ = _quant_run(O.round_bf16(a), w)
    d1, cr = O.quant_gemm_e4m3(O.round_bf16(a[:1]), w8, tile_k=128)
    assert _err(amax[:1], d1) == 0.0
    assert _err(c[0], cr[0]) < 1e-3
    # the reference's unrounded result: within FP8 input-rounding error
    rel = np.sqrt(np.mean((c[0, :N] - gd["oracle.d2"]) ** 2)) / np.sqrt(np.mean(gd["oracle.d2"] ** 2))
    assert rel < 0.06
    assert abs(amax[0] - gd["oracle.d1"][0]) <= 2e-2 * gd["oracle.d1"][0]
