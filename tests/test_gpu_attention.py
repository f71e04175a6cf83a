"""GPU parity: librf_cuda attention kernels vs the oracle (oracle/rf_oracle.c,
pinned to the reference) on identical inputs. Tolerances (north_star):
fp32 path <= 1e-5 scaled error; bf16 <= 2e-2 against the oracle evaluated on
the same bf16-rounded inputs."""
import numpy as np
import pytest

from tests import oracle as O

pytestmark = pytest.mark.gpu


def _inputs(B, H, Sq, Skv, D, seed, dtype):
    import torch

    g = torch.Generator().manual_seed(seed)
    # make_attention's distributions (workloads.cpp:78-99): q pre-scaled by 1/sqrt(hd)
    q = (torch.rand(B, H, Sq, D, generator=g, dtype=torch.float64) * 2 - 1) / np.sqrt(D)
    k = torch.rand(B, H, Skv, D, generator=g, dtype=torch.float64) * 2 - 1
    v = torch.rand(B, H, Skv, D, generator=g, dtype=torch.float64) * 2 - 1
    q, k, v = (t.to(dtype) for t in (q, k, v))
    return q, k, v


def _check(q, k, v, m, l, o, tol):
    B, H, Sq, D = q.shape
    Skv = k.shape[2]
    f = lambda t: t.double().cpu().numpy()  # the same (rounded) inputs the kernel saw
    rm, rl, ro = O.attention(f(q).reshape(B * H, Sq, D), f(k).reshape(B * H, Skv, D),
                             f(v).reshape(B * H, Skv, D))
    em = O.scaled_max_err(f(m).ravel(), rm.ravel())[0]
    el = O.scaled_max_err(f(l).ravel(), rl.ravel())[0]
    eo = O.scaled_max_err(f(o).ravel(), ro.ravel())[0]
    assert em <= tol and el <= tol and eo <= tol, (em, el, eo)
    return em, el, eo


@pytest.mark.parametrize("segments", [1, 2, 4, 8])
def test_fp32_config1_vs_oracle(segments):
    """BASELINE config 1: B1 H1 S1024 D64 fp32, all 1,024 rows, <= 1e-5."""
    import torch
    from paper_2603_10026_b200 import attention

    q, k, v = _inputs(1, 1, 1024, 1024, 64, 42, torch.float32)
    m, l, o = attention(q.cuda(), k.cuda(), v.cuda(), segments=segments)
    torch.cuda.synchronize()
    _check(q, k, v, m, l, o, 1e-5)


@pytest.mark.parametrize("shape", [(2, 3, 37, 129, 32), (1, 2, 5, 3, 16), (1, 1, 64, 512, 128),
                                   (1, 1, 1, 1, 64)])
def test_fp32_ragged_shapes(shape):
    import torch
    from paper_2603_10026_b200 import attention

    B, H, Sq, Skv, D = shape
    q, k, v = _inputs(B, H, Sq, Skv, D, 7, torch.float32)
    m, l, o = attention(q.cuda(), k.cuda(), v.cuda())
    torch.cuda.synchronize()
    _check(q, k, v, m, l, o, 1e-5)


@pytest.mark.parametrize("shape,segments", [((2, 3, 100, 512, 128), 4), ((1, 2, 64, 96, 64), 2),
                                            ((1, 1, 200, 1024, 64), 8), ((3, 1, 17, 64, 128), 1),
                                            ((1, 1, 64, 1024, 16), 32)])
def test_fp32_sub_slices(shape, segments):
    """Reference slices cut into sub-slices by the plan to fill the GPU, folded
    by the merge kernel: ragged rows, slices shorter than a KV tile, D = 64 /
    128, and run_incremental (segments = 1) on a small grid."""
    import torch
    from paper_2603_10026_b200 import Desc, Plan
    from paper_2603_10026_b200 import _native as N

    B, H, Sq, Skv, D = shape
    q, k, v = _inputs(B, H, Sq, Skv, D, 11, torch.float32)
    plan = Plan(Desc(N.RF_PATTERN_ATTENTION, "f32", rows=Sq, len=Skv, free_len=D, batch=B,
                     heads=H, segments=segments))
    m = torch.empty(B, H, Sq, device="cuda")
    l, o = torch.empty_like(m), torch.empty(B, H, Sq, D, device="cuda")
    plan.run([q.cuda(), k.cuda(), v.cuda()], [m, l, o])
    torch.cuda.synchronize()
    _check(q, k, v, m, l, o, 1e-5)


@pytest.mark.parametrize("name", O.golden_names("attention_"))
def test_fp32_against_reference_goldens(name):
    """The reference's own fixtures (its generator, oracle and executors)."""
    import torch
    from paper_2603_10026_b200 import attention

    g = O.load_golden(name)
    kv, hd = g["in.K"].shape
    q = torch.tensor(g["in.Q"], dtype=torch.float32).reshape(1, 1, 1, hd).cuda()
    k = torch.tensor(g["in.K"], dtype=torch.float32).reshape(1, 1, kv, hd).cuda()
    v = torch.tensor(g["in.V"], dtype=torch.float32).reshape(1, 1, kv, hd).cuda()
    for seg, tag in [(1, "incremental"), (2, "multi2"), (4, "multi4")]:
        m, l, o = attention(q, k, v, segments=seg)
        torch.cuda.synchronize()
        assert O.scaled_max_err(m.double().cpu().numpy().ravel(), g[f"{tag}.d1"])[0] <= 1e-5
        assert O.scaled_max_err(l.double().cpu().numpy().ravel(), g[f"{tag}.d2"])[0] <= 1e-5
        assert O.scaled_max_err(o.double().cpu().numpy().ravel(), g[f"{tag}.d3"])[0] <= 1e-5


def test_partials_and_merge_match_multisegment():
    """rf_run_partials over slice ranges + rf_merge_partials == run_multisegment."""
    import torch
    from paper_2603_10026_b200 import Desc, Plan, _native as N

    B, H, Sq, Skv, D, S = 1, 2, 64, 1024, 64, 8
    q, k, v = _inputs(B, H, Sq, Skv, D, 3, torch.float32)
    q, k, v = q.cuda(), k.cuda(), v.cuda()
    p = Plan(Desc(N.RF_PATTERN_ATTENTION, "f32", rows=Sq, len=Skv, free_len=D, batch=B, heads=H,
                  segments=S))
    rows = B * H * Sq
    pm = torch.empty(S, rows, device="cuda")
    pl = torch.empty(S, rows, device="cuda")
    po = torch.empty(S, rows, D, device="cuda")
    # two "shards" of 4 slices each, like two GPUs owning halves of the KV axis
    p.run_partials([q, k, v], 0, pm[:4], pl[:4], po[:4])
    p.run_partials([q, k, v], 4, pm[4:], pl[4:], po[4:])
    m = torch.empty(B, H, Sq, device="cuda")
    l = torch.empty_like(m)
    o = torch.empty_like(q)
    p.merge_partials(pm, pl, po, [m, l, o])
    torch.cuda.synchronize()
    _check(q.cpu(), k.cpu(), v.cpu(), m, l, o, 1e-5)
    # the partials themselves are the reference's per-slice states
    pr = (q.double() @ k.double().transpose(-1, -2)).reshape(rows, Skv).cpu().numpy()
    vr = v.double().cpu().numpy().reshape(B * H, 1, Skv, D).repeat(Sq, 1).reshape(rows, Skv, D)
    for s in range(S):
        sl = slice(s * 128, (s + 1) * 128)
        rm, rl, ro = O.attention_incremental(pr[:, sl], vr[:, sl], 1)
        assert O.scaled_max_err(pm[s].double().cpu().numpy(), rm)[0] <= 1e-5
        assert O.scaled_max_err(pl[s].double().cpu().numpy(), rl)[0] <= 1e-5
        assert O.scaled_max_err(po[s].double().cpu().numpy(), ro)[0] <= 1e-5


def test_run_host_matches_device_path():
    import torch
    from paper_2603_10026_b200 import Desc, Plan, _native as N

    B, H, Sq, Skv, D = 2, 4, 128, 256, 64
    q, k, v = _inputs(B, H, Sq, Skv, D, 11, torch.float32)
    p = Plan(Desc(N.RF_PATTERN_ATTENTION, "f32", rows=Sq, len=Skv, free_len=D, batch=B, heads=H))
    hq, hk, hv = (t.pin_memory() for t in (q, k, v))
    m = torch.empty(B, H, Sq).pin_memory()
    l = torch.empty(B, H, Sq).pin_memory()
    o = torch.empty(B, H, Sq, D).pin_memory()
    p.run_host([hq, hk, hv], [m, l, o])
    _check(q, k, v, m, l, o, 1e-5)


def test_segmentation_error():
    import torch
    from paper_2603_10026_b200 import IncompatibleSegmentation, attention

    q, k, v = _inputs(1, 1, 4, 6, 16, 0, torch.float32)
    with pytest.raises(IncompatibleSegmentation):
        attention(q.cuda(), k.cuda(), v.cuda(), segments=4)


def test_safe_softmax_vs_goldens_and_oracle():
    import torch
    from paper_2603_10026_b200 import safe_softmax

    for name in O.golden_names("safe_softmax_"):
        g = O.load_golden(name)
        x = torch.tensor(g["in.x"], dtype=torch.float32).reshape(1, -1).cuda()
        d1, d2 = safe_softmax(x)
        torch.cuda.synchronize()
        assert O.scaled_max_err(d1.double().cpu().numpy(), g["incremental.d1"])[0] <= 1e-5
        assert O.scaled_max_err(d2.double().cpu().numpy(), g["incremental.d2"])[0] <= 1e-5
    x = (torch.rand(333, 5000) * 4 - 2).cuda()
    d1, d2 = safe_softmax(x)
    r1, r2 = O.safe_softmax(x.double().cpu().numpy())
    assert O.scaled_max_err(d1.double().cpu().numpy(), r1)[0] <= 1e-5
    assert O.scaled_max_err(d2.double().cpu().numpy(), r2)[0] <= 1e-5
    # known answer (test_simulator.cpp:39-51)
    d1, d2 = safe_softmax(torch.tensor([[1.0, 2.0, 3.0]], device="cuda"))
    assert d1.item() == 3.0
    assert abs(d2.item() - (np.exp(-2) + np.exp(-1) + 1)) < 1e-6


def _plan_run(shape, segments, seed, simt=False):
    import os

    import torch
    from paper_2603_10026_b200 import Desc, Plan
    from paper_2603_10026_b200 import _native as N

    B, H, Sq, Skv, D = shape
    q, k, v = _inputs(B, H, Sq, Skv, D, seed, torch.float32)
    if simt:
        os.environ["RF_ATTN_F32_SIMT"] = "1"
    try:
        plan = Plan(Desc(N.RF_PATTERN_ATTENTION, "f32", rows=Sq, len=Skv, free_len=D, batch=B,
                         heads=H, segments=segments))
    finally:
        os.environ.pop("RF_ATTN_F32_SIMT", None)
    m = torch.empty(B, H, Sq, device="cuda")
    l, o = torch.empty_like(m), torch.empty(B, H, Sq, D, device="cuda")
    plan.run([q.cuda(), k.cuda(), v.cuda()], [m, l, o])
    torch.cuda.synchronize()
    return plan, (q, k, v), (m, l, o)


@pytest.mark.parametrize("shape,segments,nsplit", [
    ((1, 1, 1024, 1024, 64), 8, 8),    # cfg1: one 128-key tile per CTA, cluster of 8
    ((1, 1, 1024, 1024, 64), 1, 8),    # run_incremental cut into 8 sub-slices
    ((1, 1, 256, 2048, 64), 2, 8),     # 256-key slices: two tiles per CTA (running-max rescale of O in TMEM)
    ((2, 3, 128, 1024, 64), 1, 8),     # several (b, h)
    ((5, 8, 128, 512, 64), 1, 4),      # a 4-CTA cluster (the grid fills the GPU at 4 sub-slices)
    ((4, 37, 128, 256, 64), 1, 1),     # grid already fills the GPU: one slice, no fold
    ((2, 3, 200, 512, 64), 1, 4),      # ragged row tiles (Sq % 128 != 0) across heads
    ((1, 1, 1000, 1024, 64), 8, 8),    # ragged cfg1-like shape
])
def test_fp32_tcgen05_tf32x3(shape, segments, nsplit):
    """The fp32 path on tcgen05 (3xTF32, attn_tf32.cu) with the slice fold in
    the kernel's cluster: plan choice, sub-slicing and <= 1e-5 against the
    oracle, on shapes with one and several KV tiles per slice."""
    plan, (q, k, v), (m, l, o) = _plan_run(shape, segments, 23)
    assert "tf32" in plan.info["kernel"] and plan.info["segments"] == segments
    assert plan.info["slices_launched"] == nsplit and plan.info["launches_per_run"] == 1
    _check(q, k, v, m, l, o, 1e-5)


def test_fp32_tcgen05_matches_simt_path():
    """Same inputs through the tcgen05 kernel and the SIMT paper-form kernel
    (+ merge): both within the fp32 gate of the oracle and of each other."""
    shape = (1, 1, 1024, 1024, 64)
    p1, inp, out_t = _plan_run(shape, 8, 5)
    p2, _, out_s = _plan_run(shape, 8, 5, simt=True)
    assert "tf32" in p1.info["kernel"] and "SIMT" in p2.info["kernel"]
    for a, b in zip(out_t, out_s):
        e = O.scaled_max_err(a.double().cpu().numpy().ravel(), b.double().cpu().numpy().ravel())[0]
        assert e <= 2e-6, e
    _check(*inp, *out_t, 1e-5)
