"""Boundary robustness on the device: undersized / misplaced buffers raise the
reference's ShapeMismatch (check_shapes, proj/src/simulator.cpp:235-245)
instead of reaching a kernel; concurrent streams get separate plans (their
split workspaces never alias); bad dtypes are rejected; the entry points
leave the caller's current device alone; a zero absmax row raises
DomainError through the Python quant_gemm as in the reference."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_undersized_and_misplaced_buffers_raise_shape_mismatch():
    from paper_2603_10026_b200 import Desc, Plan, ShapeMismatch, _native as N

    p = Plan(Desc(N.RF_PATTERN_ATTENTION, "bf16", rows=128, len=256, free_len=128, batch=1, heads=2))
    q = torch.zeros(1, 2, 128, 128, dtype=torch.bfloat16, device="cuda")
    k = torch.zeros(1, 2, 256, 128, dtype=torch.bfloat16, device="cuda")
    m = torch.empty(1, 2, 128, device="cuda")
    o = torch.empty_like(q)
    p.run([q, k, k.clone()], [m, torch.empty_like(m), o])  # well-formed: runs
    with pytest.raises(ShapeMismatch):
        p.run([q, k[:, :, :128], k], [m, torch.empty_like(m), o])  # K too short
    with pytest.raises(ShapeMismatch):
        p.run([q, k, k], [m[:, :1], torch.empty_like(m), o])  # d1 too short
    with pytest.raises(ShapeMismatch):
        p.run([q.cpu(), k, k], [m, torch.empty_like(m), o])  # host tensor on the device path
    with pytest.raises(ShapeMismatch):
        p.run([q, k.transpose(2, 3), k], [m, torch.empty_like(m), o])  # strided view
    with pytest.raises(ShapeMismatch):
        p.run([q, k], [m, torch.empty_like(m), o])  # V missing
    with pytest.raises(ShapeMismatch):
        p.run_host([q, k, k], [m.cpu(), m.cpu(), o.cpu()])  # device input on the host path


def test_io_bytes_match_the_documented_layouts():
    from paper_2603_10026_b200 import Desc, Plan, _native as N

    p = Plan(Desc(N.RF_PATTERN_RMSNORM_GEMM, "bf16", rows=256, len=512, free_len=512))
    assert p.in_bytes == (2 * 256 * 512, 2 * 512 * 512, 0, 0)
    assert p.out_bytes == (4 * 256, 2 * 256 * 512, 0, 0)


def test_streams_get_separate_plans():
    from paper_2603_10026_b200 import _native as N
    from paper_2603_10026_b200.executors import Desc, plan

    d = Desc(N.RF_PATTERN_ATTENTION, "bf16", rows=1, len=8192, free_len=128, batch=2, heads=4,
             segments=8)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    assert plan(d, s1) is plan(d, s1)
    assert plan(d, s1) is not plan(d, s2)


def test_concurrent_split_kv_on_two_streams_do_not_share_workspace():
    from paper_2603_10026_b200 import attention

    torch.manual_seed(1)
    B, H, S, D = 2, 4, 8192, 128
    xs = [((torch.rand(B, H, 1, D, device="cuda") * 2 - 1) / D ** 0.5).bfloat16() for _ in range(2)]
    ks = [(torch.rand(B, H, S, D, device="cuda") * 2 - 1).bfloat16() for _ in range(2)]
    want = [attention(xs[i], ks[i], ks[i], segments=8) for i in range(2)]
    torch.cuda.synchronize()
    s = [torch.cuda.Stream(), torch.cuda.Stream()]
    got = [None, None]
    for _ in range(3):
        for i in range(2):
            with torch.cuda.stream(s[i]):
                got[i] = attention(xs[i], ks[i], ks[i], segments=8, stream=s[i])
    torch.cuda.synchronize()
    for i in range(2):
        for g, w in zip(got[i], want[i]):
            assert torch.equal(g, w)


def test_quant_gemm_rejects_float32_activations_and_raises_domain_error():
    from paper_2603_10026_b200 import DomainError, ShapeMismatch, quant_gemm, quant_gemm_plan

    M, K, Nn = 128, 256, 512
    p = quant_gemm_plan(M, K, Nn)
    wp = p.pack_weight(torch.rand(K, Nn, device="cuda") * 2 - 1)
    with pytest.raises(ShapeMismatch):
        quant_gemm(torch.rand(M, K, device="cuda"), wp)
    a = (torch.rand(M, K, device="cuda") * 2 - 1).bfloat16()
    quant_gemm(a, wp)
    a[5].zero_()
    with pytest.raises(DomainError):
        quant_gemm(a, wp)


def test_entry_points_keep_the_callers_device():
    from paper_2603_10026_b200 import attention

    dev = torch.cuda.current_device()
    q = torch.zeros(1, 1, 128, 64, device="cuda")
    attention(q, q, q)
    assert torch.cuda.current_device() == dev
