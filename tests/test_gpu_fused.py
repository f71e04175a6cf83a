"""GPU parity of run_fused — fusion at level k, the reference's NON-incremental
executor (proj/src/simulator.cpp:485-559) — on librf_cuda
(ABI v5: rf_desc.fuse_level / tree). Each level-1 segment is buffered on chip
and evaluated with its own dependency values; the segment states are then
corrected and folded in segment order.

Checked against the reference's own fused@k reports (tests/golden,
"fused_<levels>_k<k>") and the C restatement rfo_fused_row (pinned to those
reports at 1e-12 by tests/test_oracle_golden.py). Gates: 1e-5 scaled for the
fp32 paths, 2e-2 for bf16 operands (north_star)."""
import numpy as np
import pytest

from tests import oracle as O

pytestmark = pytest.mark.gpu
TOL32 = 1e-5


def _err(a, b):
    return O.scaled_max_err(np.asarray(a, dtype=np.float64).ravel(), np.asarray(b, dtype=np.float64).ravel())[0]


def _cases(prefix):
    out = []
    for name in O.golden_names(prefix):
        g = O.load_golden(name)
        for key in g:
            if key.startswith("fused_") and key.endswith(".d1"):
                tag, k = key[len("fused_"):-3].rsplit("_k", 1)
                out.append((name, tuple(int(x) for x in tag.split("-")), int(k)))
    return out


ROWS = _cases("safe_softmax_") + _cases("variance_") + _cases("sum_sum_")


@pytest.mark.parametrize("name,tree,k", ROWS)
def test_fused_rows_vs_reference_goldens(name, tree, k):
    import torch
    import paper_2603_10026_b200 as rf

    g = O.load_golden(name)
    pre = "fused_" + "-".join(map(str, tree)) + f"_k{k}"
    if name.startswith("sum_sum_"):
        x1 = torch.tensor(g["in.x1"], dtype=torch.float32).reshape(1, -1).cuda()
        x2 = torch.tensor(g["in.x2"], dtype=torch.float32).reshape(1, -1).cuda()
        d1, d2 = rf.sum_sum(x1, x2, 10.0, 1e-12, tree=tree, fuse_level=k)
    else:
        x = torch.tensor(g["in.x"], dtype=torch.float32).reshape(1, -1).cuda()
        op = rf.safe_softmax if name.startswith("safe_softmax_") else rf.variance
        d1, d2 = op(x, tree=tree, fuse_level=k)
    torch.cuda.synchronize()
    assert _err(d1.cpu(), g[pre + ".d1"]) < TOL32
    assert _err(d2.cpu(), g[pre + ".d2"]) < TOL32


@pytest.mark.parametrize("pattern", ["safe_softmax", "variance", "sum_sum"])
@pytest.mark.parametrize("tree,k", [((64, 8, 1), 1), ((64, 8, 1), 2), ((64, 8, 1), 3), ((4, 1), 1),
                                    ((2048, 1), 2), ((1,), 1)])
def test_fused_rows_batched_vs_restatement(pattern, tree, k):
    """Many rows per launch, segments from 2 to 1024 elements (one warp's
    register buffer), including one segment per row (tree (1,))."""
    import torch
    import paper_2603_10026_b200 as rf

    n = 4096 if tree != (1,) else 1024
    rows = 37
    rng = np.random.default_rng(len(tree) * 10 + k)
    a = rng.uniform(-2, 2, (rows, n)).astype(np.float32)
    b = rng.uniform(-1, 1, (rows, n)).astype(np.float32)
    levels = [n] + list(tree)
    if pattern == "sum_sum":
        d1, d2 = rf.sum_sum(torch.tensor(a).cuda(), torch.tensor(b).cuda(), 10.0, 1e-12, tree=tree, fuse_level=k)
        w1, w2 = O.fused("sum_sum", a, b, levels, k, 10.0, 1e-12)
    else:
        op = rf.safe_softmax if pattern == "safe_softmax" else rf.variance
        d1, d2 = op(torch.tensor(a).cuda(), tree=tree, fuse_level=k)
        w1, w2 = O.fused(pattern, a, None, levels, k)
    torch.cuda.synchronize()
    assert _err(d1.cpu(), w1) < TOL32
    assert _err(d2.cpu(), w2) < TOL32


def _attn_from_p(p, v):
    """The host layer's trick (include/rf_host.hpp): q = e_0 and K[l] = (P[l], 0, ...)
    make Q K^T = P exactly; one (b, h) row per cascade row."""
    rows, L0 = p.shape
    D = v.shape[2]
    q = np.zeros((1, rows, 1, D), np.float32)
    q[..., 0] = 1.0
    k = np.zeros((1, rows, L0, D), np.float32)
    k[..., 0] = p
    return q, k, v.reshape(1, rows, L0, D).astype(np.float32)


@pytest.mark.parametrize("name,tree,k", _cases("attention_"))
def test_fused_attention_fp32_vs_reference_goldens(name, tree, k):
    import torch
    import paper_2603_10026_b200 as rf

    g = O.load_golden(name)
    p, v = g["in.P"], g["in.V"]
    kv, hd = v.shape
    q, kk, vv = _attn_from_p(p.reshape(1, kv), v.reshape(1, kv, hd))
    m, l, o = rf.attention(torch.tensor(q).cuda(), torch.tensor(kk).cuda(), torch.tensor(vv).cuda(),
                           tree=tree, fuse_level=k)
    torch.cuda.synchronize()
    pre = "fused_" + "-".join(map(str, tree)) + f"_k{k}"
    assert _err(m.cpu(), g[pre + ".d1"]) < TOL32
    assert _err(l.cpu(), g[pre + ".d2"]) < TOL32
    assert _err(o.cpu(), g[pre + ".d3"]) < TOL32


@pytest.mark.parametrize("tree,k", [((4, 1), 1), ((16, 4, 1), 2), ((16, 4, 1), 3), ((128, 1), 1)])
def test_fused_attention_fp32_batched(tree, k):
    """B2 H3 Sq100 Skv256 D64: segments of 64 keys (one fp32 tile) down to 2."""
    import torch
    import paper_2603_10026_b200 as rf

    B, H, Sq, Skv, D = 2, 3, 100, 256, 64
    rng = np.random.default_rng(k + len(tree))
    q = (rng.uniform(-1, 1, (B, H, Sq, D)) / 8).astype(np.float32)
    kk = rng.uniform(-1, 1, (B, H, Skv, D)).astype(np.float32)
    v = rng.uniform(-1, 1, (B, H, Skv, D)).astype(np.float32)
    m, l, o = rf.attention(torch.tensor(q).cuda(), torch.tensor(kk).cuda(), torch.tensor(v).cuda(),
                           tree=tree, fuse_level=k)
    torch.cuda.synchronize()
    p = np.einsum("bhqd,bhkd->bhqk", q.astype(np.float64), kk.astype(np.float64)).reshape(-1, Skv)
    vr = np.repeat(v.reshape(B * H, 1, Skv, D), Sq, axis=1).reshape(-1, Skv, D)
    w1, w2, w3 = O.fused("attention", p, vr, [Skv] + list(tree), k)
    assert _err(m.cpu(), w1) < TOL32
    assert _err(l.cpu(), w2) < TOL32
    assert _err(o.cpu().reshape(-1, D), w3) < TOL32


@pytest.mark.parametrize("tree,k", [((4, 1), 1), ((4, 2, 1), 2)])
def test_fused_attention_bf16_tcgen05(tree, k):
    """bf16 prefill on tcgen05: one 128-key tile per level-1 segment."""
    import torch
    import paper_2603_10026_b200 as rf
    from paper_2603_10026_b200 import Desc, Plan, _native as N

    B, H, Sq, Skv, D = 1, 2, 256, 512, 128
    info = Plan(Desc(N.RF_PATTERN_ATTENTION, "bf16", rows=Sq, len=Skv, free_len=D, batch=B, heads=H,
                     fuse_level=k, tree=tree)).info
    assert "tcgen05" in info["kernel"] and info["fuse_level"] == k and info["slices_launched"] == 4
    rng = np.random.default_rng(7)
    q = torch.tensor(rng.uniform(-1, 1, (B, H, Sq, D)) / np.sqrt(D)).bfloat16()
    kk = torch.tensor(rng.uniform(-1, 1, (B, H, Skv, D))).bfloat16()
    v = torch.tensor(rng.uniform(-1, 1, (B, H, Skv, D))).bfloat16()
    m, l, o = rf.attention(q.cuda(), kk.cuda(), v.cuda(), tree=tree, fuse_level=k)
    torch.cuda.synchronize()
    f = lambda t: t.double().numpy()
    rm, rl, ro = O.attention(f(q).reshape(B * H, Sq, D), f(kk).reshape(B * H, Skv, D), f(v).reshape(B * H, Skv, D))
    assert _err(m.cpu(), rm) < 1e-5
    assert _err(l.cpu(), rl) < 1e-3
    assert _err(o.float().cpu(), ro) < 2e-2


def test_fused_segment_longer_than_on_chip_buffer_is_not_fusable():
    """Non-incremental fusion is only feasible for short segments
    (PAPER.md:1127-1135): longer ones are rejected, never run incrementally."""
    from paper_2603_10026_b200 import Desc, Plan, UnsupportedPattern, _native as N

    with pytest.raises(UnsupportedPattern):  # 2048 > one warp's 1024-element buffer
        Plan(Desc(N.RF_PATTERN_SAFE_SOFTMAX, "f32", rows=4, len=4096, fuse_level=1, tree=(2, 1)))
    with pytest.raises(UnsupportedPattern):  # 128 keys > the 64-key fp32 tile
        Plan(Desc(N.RF_PATTERN_ATTENTION, "f32", rows=1, len=256, free_len=64, fuse_level=1, tree=(2, 1)))
    with pytest.raises(UnsupportedPattern):  # 256 keys > one 128-key tcgen05 tile
        Plan(Desc(N.RF_PATTERN_ATTENTION, "bf16", rows=256, len=512, free_len=128, fuse_level=1, tree=(2, 1)))
    with pytest.raises(UnsupportedPattern):  # quant: one 128-wide K tile per segment
        Plan(Desc(N.RF_PATTERN_QUANT_GEMM_E4M3, "bf16", rows=256, len=512, free_len=512, fuse_level=1,
                  tree=(2, 1)))
    with pytest.raises(UnsupportedPattern):  # no non-incremental kernel
        Plan(Desc(N.RF_PATTERN_MOE_ROUTING, "f32", rows=4, len=64, free_len=2, fuse_level=1, tree=(4, 1)))


@pytest.mark.parametrize("tree", [(8, 1), (2, 1)])
def test_fused_rmsnorm_gemm(tree):
    """The accumulator carries H' = 1 and each segment's 1/sigma is applied to
    the segment's sum: the non-incremental form for whole 64-wide K tiles."""
    import torch
    from paper_2603_10026_b200 import Desc, Plan, _native as N

    M, K, N_ = 256, 512, 512
    rng = np.random.default_rng(len(tree) + tree[0])
    x = O.round_bf16(rng.uniform(-1, 2, (M, K)))
    p = Plan(Desc(N.RF_PATTERN_RMSNORM_GEMM, "bf16", rows=M, len=K, free_len=N_, fuse_level=1, tree=tree))
    assert p.info["fuse_level"] == 1 and p.info["slices_launched"] == tree[0]
    wp = p.pack_weight(torch.tensor(rng.uniform(-1, 1, (K, N_)), dtype=torch.float32).cuda(),
                       torch.tensor(rng.uniform(-1, 1, K), dtype=torch.float32).cuda())
    ss, y = torch.empty(M, device="cuda"), torch.empty(M, N_, dtype=torch.bfloat16, device="cuda")
    p.run([torch.tensor(x).bfloat16().cuda(), wp], [ss, y])
    torch.cuda.synchronize()
    d1, yr = O.rmsnorm_gemm(x, np.ones(K), wp.double().cpu().numpy().T)
    assert _err(ss.cpu(), d1) < 1e-5 and _err(y.float().cpu(), yr) < 2e-2


def test_fused_quant_gemm_one_tile_segments():
    """Each level-1 segment is one 128-wide K tile quantised with ITS OWN
    absmax (taken over the whole tile before any element is quantised); the
    segment states fold as c = sum_s c_s m_s / max_s m_s."""
    import torch
    from paper_2603_10026_b200 import Desc, Plan, _native as N

    M, K, N_ = 256, 512, 512
    S = K // 128
    rng = np.random.default_rng(3)
    a = O.round_bf16(rng.uniform(-2, 2, (M, K)) * np.linspace(0.1, 1.0, K)[None])
    p = Plan(Desc(N.RF_PATTERN_QUANT_GEMM_E4M3, "bf16", rows=M, len=K, free_len=N_, fuse_level=1, tree=(S, 1)))
    wp = p.pack_weight(torch.tensor(rng.uniform(-1, 1, (K, N_)), dtype=torch.float32).cuda())
    amax, c = torch.empty(M, device="cuda"), torch.empty(M, N_, device="cuda")
    p.run([torch.tensor(a).bfloat16().cuda(), wp], [amax, c])
    torch.cuda.synchronize()
    w8 = wp.view(torch.float8_e4m3fn).double().cpu().numpy().T
    parts = [O.quant_gemm_e4m3(a[:, s * 128:(s + 1) * 128], w8[s * 128:(s + 1) * 128], 448.0, 128) for s in range(S)]
    m = np.max([d for d, _ in parts], axis=0)
    want = sum(cs * ds[:, None] for ds, cs in parts) / m[:, None]
    assert _err(amax.cpu(), m) == 0.0
    assert _err(c.cpu(), want) < 1e-3
