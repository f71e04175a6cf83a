"""The C oracle (oracle/rf_oracle.c) pinned against fixtures produced by the
reference itself (oracle/ref_driver.cpp -> tests/golden/). CPU only."""
import numpy as np
import pytest

from tests import oracle as O

TOL = 1e-12  # restatement vs reference, both float64


def _err(a, b):
    return O.scaled_max_err(a, b)[0]


@pytest.mark.parametrize("name", O.golden_names("attention_"))
def test_attention_oracle_and_streaming_match_reference(name):
    g = O.load_golden(name)
    q, k, v, p = g["in.Q"], g["in.K"], g["in.V"], g["in.P"]
    kv, hd = k.shape
    m, l, o = O.attention(q.reshape(1, 1, hd), k.reshape(1, kv, hd), v.reshape(1, kv, hd))
    assert _err(m, g["oracle.d1"]) < TOL
    assert _err(l, g["oracle.d2"]) < TOL
    assert _err(o.ravel(), g["oracle.d3"]) < TOL
    # run_incremental and run_multisegment semantics
    mi, li, oi = O.attention_incremental(p.reshape(1, kv), v.reshape(1, kv, hd), 1)
    assert _err(mi, g["incremental.d1"]) < TOL
    assert _err(li, g["incremental.d2"]) < TOL
    assert _err(oi.ravel(), g["incremental.d3"]) < TOL
    for key in g:
        if key.startswith("multi") and key.endswith(".d3"):
            s = int(key[len("multi"):-3])
            ms, ls, os_ = O.attention_incremental(p.reshape(1, kv), v.reshape(1, kv, hd), s)
            assert _err(ms, g[f"multi{s}.d1"]) < TOL
            assert _err(ls, g[f"multi{s}.d2"]) < TOL
            assert _err(os_.ravel(), g[f"multi{s}.d3"]) < TOL


@pytest.mark.parametrize("name", O.golden_names("attention_"))
def test_attention_closed_form_matches_reference(name):
    """The numpy closed form used for MLA (K and V of different widths)."""
    g = O.load_golden(name)
    p, v = g["in.P"], g["in.V"]
    kv, hd = v.shape
    m, l, o = O.attention_closed_form(p.reshape(1, kv), v.reshape(1, kv, hd))
    assert _err(m, g["oracle.d1"]) < TOL
    assert _err(l, g["oracle.d2"]) < TOL
    assert _err(o.ravel(), g["oracle.d3"]) < TOL


def test_attention_incremental_rejects_bad_segmentation():
    p = np.zeros((1, 6))
    v = np.zeros((1, 6, 2))
    with pytest.raises(ValueError):
        O.attention_incremental(p, v, 4)


@pytest.mark.parametrize("name", O.golden_names("safe_softmax_"))
def test_softmax_oracle_matches_reference(name):
    g = O.load_golden(name)
    d1, d2 = O.safe_softmax(g["in.x"].reshape(1, -1))
    for tag in ["oracle", "incremental", "multi2", "multi4", "multi8"]:
        assert _err(d1, g[f"{tag}.d1"]) < TOL
        assert _err(d2, g[f"{tag}.d2"]) < TOL


@pytest.mark.parametrize("name", O.golden_names("quant_gemm_"))
def test_quant_oracle_matches_reference(name):
    g = O.load_golden(name)
    a, w = g["in.a"], g["in.w"]
    d1, c = O.quant_gemm(a.reshape(1, -1), w)
    for tag in ["oracle", "incremental", "multi2", "multi4", "multi8"]:
        assert _err(d1, g[f"{tag}.d1"]) < TOL
        assert _err(c.ravel(), g[f"{tag}.d2"]) < 1e-10


@pytest.mark.parametrize("name", O.golden_names("rmsnorm_gemm_"))
def test_rmsnorm_oracle_matches_reference_engine(name):
    g = O.load_golden(name)
    x, gg, w = g["in.x"], g["in.g"], g["in.w"]
    d1, y = O.rmsnorm_gemm(x.reshape(1, -1), gg, w)
    assert _err(d1, g["oracle.d1"]) < TOL
    assert _err(y.ravel(), g["oracle.d2"]) < 1e-10
    assert _err(y.ravel(), g["incremental.d2"]) < 1e-10
    di, yi = O.rmsnorm_gemm_incremental(x, gg, w)
    assert _err(np.array([di]), g["incremental.d1"]) < TOL
    assert _err(yi, g["incremental.d2"]) < 1e-12


@pytest.mark.parametrize("name", O.golden_names("layernorm_gemm_"))
def test_layernorm_oracle_matches_reference_engine(name):
    g = O.load_golden(name)
    x, gg, w = g["in.x"], g["in.g"], g["in.w"]
    d1, d2, d3, d4 = O.layernorm_gemm(x.reshape(1, -1), gg, w)
    for tag in ["oracle", "incremental", "multi2", "multi4"]:
        assert _err(d1, g[f"{tag}.d1"]) < TOL, tag
        assert _err(d2, g[f"{tag}.d2"]) < TOL, tag
        assert _err(d3.ravel(), g[f"{tag}.d3"]) < 1e-10, tag
        assert _err(d4.ravel(), g[f"{tag}.d4"]) < 1e-10, tag
    i1, i2, i3, i4 = O.layernorm_gemm_incremental(x, gg, w)
    assert _err(np.array([i1, i2]), np.concatenate([g["incremental.d1"], g["incremental.d2"]])) < TOL
    assert _err(i3, g["incremental.d3"]) < 1e-12
    assert _err(i4, g["incremental.d4"]) < 1e-12
    # the normalised product: d3 - d4 == ((x - mean) / sigma * g) @ W
    K = x.size
    mu = x.mean()
    sig = np.sqrt((x * x).mean() - mu * mu + 1e-5)
    ref = ((x - mu) / sig * gg) @ w
    assert np.abs((d3 - d4).ravel() - ref).max() < 1e-9 * max(1.0, np.abs(ref).max())


def test_moe_routing_oracle_matches_reference():
    g = O.load_golden("moe_routing_128x8_s100")
    d1, d2, tv, ti = O.moe_routing(g["in.s"].reshape(1, -1), 8)
    for tag in ["oracle", "incremental", "multi2", "multi4"]:
        assert _err(d1, g[f"{tag}.d1"]) < TOL
        assert _err(d2, g[f"{tag}.d2"]) < TOL
        np.testing.assert_array_equal(ti.ravel(), g[f"{tag}.d3.topk_idx"].astype(np.int64))
        assert _err(tv.ravel(), g[f"{tag}.d3.topk_val"]) == 0.0


def test_moe_topk_ties_lowest_index():
    # test_simulator.cpp:254-271: g = {0.3,0.9,0.9,-1,0.5,2,0.1,0.9}, top-3
    s = np.array([[0.3, 0.9, 0.9, -1.0, 0.5, 2.0, 0.1, 0.9]])
    _, _, tv, ti = O.moe_routing(s, 3)
    assert ti.tolist() == [[6, 2, 3]]
    assert tv.tolist() == [[2.0, 0.9, 0.9]]


def test_known_answers_from_reference_tests():
    # test_simulator.cpp:39-51 softmax [1,2,3]
    d1, d2 = O.safe_softmax(np.array([[1.0, 2.0, 3.0]]))
    assert d1[0] == 3.0
    assert abs(d2[0] - (np.exp(-2) + np.exp(-1) + 1)) < 1e-12
    # test_simulator.cpp:53-68 quant a=[1], w=[[2]] -> m=1, c=896
    d1, c = O.quant_gemm(np.array([[1.0]]), np.array([[2.0]]))
    assert d1[0] == 1.0 and c[0, 0] == 896.0
    # test_workloads.cpp:66-73 constant vector: m = 0.75, t = n
    d1, d2 = O.safe_softmax(np.full((1, 8), 0.75))
    assert d1[0] == 0.75 and d2[0] == 8.0


def test_merge_is_multisegment():
    rng = np.random.default_rng(0)
    p = rng.uniform(-2, 2, (3, 64))
    v = rng.uniform(-1, 1, (3, 64, 8))
    m4, l4, o4 = O.attention_incremental(p, v, 4)
    parts = [O.attention_incremental(p[:, s * 16:(s + 1) * 16], v[:, s * 16:(s + 1) * 16], 1)
             for s in range(4)]
    pm = np.stack([x[0] for x in parts])
    pl = np.stack([x[1] for x in parts])
    po = np.stack([x[2] for x in parts])
    m, l, o = O.attention_merge(pm, pl, po)
    assert _err(m, m4) == 0 and _err(l, l4) < 1e-15 and _err(o, o4) < 1e-15


def test_e4m3_rounding_grid():
    vals = np.array([0.0, 1.0, 1.0625, 1.1875, 448.0, 480.0, 1e6, -3.3, 2.0 ** -9, 2.0 ** -10,
                     0.0017, 17.0, 19.0, np.nan])
    r = O.round_e4m3(vals)
    assert r[0] == 0 and r[1] == 1.0
    assert r[2] == 1.0          # tie 1.0625 -> even (1.0)
    assert r[3] == 1.25         # tie 1.1875 -> even mantissa (1.25)
    assert r[4] == 448.0 and r[5] == 448.0 and r[6] == 448.0  # satfinite
    assert r[7] == -3.25
    assert r[8] == 2.0 ** -9 and r[9] == 0.0  # smallest subnormal, tie to even 0
    assert r[11] == 16.0 and r[12] == 20.0    # 17 ties to 16, 19 -> 20 (quantum 2)
    assert np.isnan(r[13])


def test_bf16_rounding():
    r = O.round_bf16(np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, -2.5]))
    assert r.tolist() == [1.0, 1.0, 1.0 + 2 ** -7, -2.5]


def test_quant_e4m3_restatement_close_to_real_oracle():
    rng = np.random.default_rng(1)
    a = rng.uniform(-2, 2, (4, 512))
    w = O.round_e4m3(rng.uniform(-1, 1, (512, 64)))
    d1r, cr = O.quant_gemm(a, w)
    d1q, cq = O.quant_gemm_e4m3(a, w, tile_k=128)
    assert np.abs(d1r - d1q).max() < 1e-6  # f32 absmax
    # e4m3 rounding alone: a few percent RMS of the scale of c
    rel = np.sqrt(np.mean((cr - cq) ** 2)) / np.sqrt(np.mean(cr ** 2))
    assert rel < 0.05


def test_quant_zero_row_is_domain_nan():
    d1, c = O.quant_gemm_e4m3(np.zeros((1, 128)), np.ones((128, 4)))
    assert d1[0] == 0 and np.isnan(c).all()


@pytest.mark.parametrize("name", O.golden_names("variance_"))
def test_variance_oracle_matches_reference(name):
    g = O.load_golden(name)
    d1, d2 = O.variance(g["in.x"].reshape(1, -1))
    for tag in ["oracle", "incremental", "multi2", "multi8"]:
        assert _err(d1, g[f"{tag}.d1"]) < TOL, tag
        assert _err(d2, g[f"{tag}.d2"]) < TOL, tag


@pytest.mark.parametrize("name", O.golden_names("sum_sum_"))
def test_sum_sum_oracle_matches_reference(name):
    g = O.load_golden(name)
    d1, d2 = O.sum_sum(g["in.x1"].reshape(1, -1), g["in.x2"].reshape(1, -1), 10.0, 1e-12)
    for tag in ["oracle", "incremental", "multi2", "multi8"]:
        assert _err(d1, g[f"{tag}.d1"]) < TOL, tag
        assert _err(d2, g[f"{tag}.d2"]) < TOL, tag


def test_moments_oracle_matches_reference():
    g = O.load_golden("moment_of_inertia_1024_s100")
    d1, d2, d3 = O.moments(g["in.mass"].reshape(1, -1), g["in.pos"].reshape(1, 1024, 3))
    for tag in ["oracle", "incremental", "multi2", "multi8"]:
        assert _err(d1, g[f"{tag}.d1"]) < TOL, tag
        assert _err(d2.ravel(), g[f"{tag}.d2"]) < TOL, tag
        assert _err(d3.ravel(), g[f"{tag}.d3"]) < TOL, tag


# ---------------------------------------------------------------- run_fused --
# Fusion at level k (simulator.cpp:485-559): the reference's own fused@k
# reports (ref_driver golden: "fused_<levels[1..K]>_k<k>") against the C
# restatement rfo_fused_row, and against the oracle (equal in exact arithmetic).

def _fused_cases(prefix):
    out = []
    for name in O.golden_names(prefix):
        g = O.load_golden(name)
        for key in g:
            if key.startswith("fused_") and key.endswith(".d1"):
                tag, k = key[len("fused_"):-3].rsplit("_k", 1)
                out.append((name, tag, int(k)))
    return out


FUSED = (_fused_cases("safe_softmax_") + _fused_cases("attention_") + _fused_cases("variance_")
         + _fused_cases("sum_sum_"))


def test_fused_goldens_exist():
    assert len(FUSED) >= 30
    assert {n.split("_")[0] for n, _, _ in FUSED} >= {"safe", "attention", "variance", "sum"}


@pytest.mark.parametrize("name,tag,k", FUSED)
def test_fused_restatement_matches_reference(name, tag, k):
    g = O.load_golden(name)
    pre = f"fused_{tag}_k{k}"
    if name.startswith("attention_"):
        p, v = g["in.P"], g["in.V"]
        levels = [p.size] + [int(x) for x in tag.split("-")]
        d1, d2, d3 = O.fused("attention", p.reshape(1, -1), v.reshape(1, *v.shape), levels, k)
        assert _err(d3.ravel(), g[pre + ".d3"]) < TOL
        assert _err(d3.ravel(), g["oracle.d3"]) < 1e-10
    elif name.startswith("sum_sum_"):
        x1, x2 = g["in.x1"], g["in.x2"]
        levels = [x1.size] + [int(x) for x in tag.split("-")]
        d1, d2 = O.fused("sum_sum", x1.reshape(1, -1), x2.reshape(1, -1), levels, k, 10.0, 1e-12)
    else:
        pat = "safe_softmax" if name.startswith("safe_softmax_") else "variance"
        x = g["in.x"]
        levels = [x.size] + [int(t) for t in tag.split("-")]
        d1, d2 = O.fused(pat, x.reshape(1, -1), None, levels, k)
    assert _err(d1, g[pre + ".d1"]) < TOL
    assert _err(d2, g[pre + ".d2"]) < TOL
    assert _err(d2, g["oracle.d2"]) < 1e-10


def test_fused_restatement_rejects_bad_tree():
    x = np.zeros((1, 8))
    with pytest.raises(ValueError):
        O.fused("safe_softmax", x, None, [8, 3, 1], 1)
    with pytest.raises(ValueError):
        O.fused("safe_softmax", x, None, [8, 2, 1], 3)
