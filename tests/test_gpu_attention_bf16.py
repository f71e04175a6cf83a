"""GPU parity of the bf16 attention kernels — tcgen05 prefill (attn_sm100.cu)
and split-KV decode (attn_decode.cu) — against the oracle evaluated on the
same bf16-rounded inputs (tolerance 2e-2 scaled, north_star)."""
import numpy as np
import pytest

from tests import oracle as O
from tests.test_gpu_attention import _check, _inputs

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _run(B, H, Sq, Skv, D, segments=1, seed=0, expect=None):
    import torch
    from paper_2603_10026_b200 import Desc, Plan, _native as N

    q, k, v = _inputs(B, H, Sq, Skv, D, seed, torch.bfloat16)
    p = Plan(Desc(N.RF_PATTERN_ATTENTION, "bf16", rows=Sq, len=Skv, free_len=D, batch=B, heads=H,
                  segments=segments))
    if expect:
        assert expect in p.info["kernel"], p.info
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    m = torch.empty(B, H, Sq, device="cuda")
    l = torch.empty_like(m)
    o = torch.empty_like(qd)
    p.run([qd, kd, vd], [m, l, o])
    torch.cuda.synchronize()
    return _check(q, k, v, m, l, o, TOL), (m, l, o)


@pytest.mark.parametrize("D", [128, 64])
@pytest.mark.parametrize("shape", [(1, 2, 256, 128), (1, 2, 512, 1024), (2, 1, 256, 4096)])
def test_tcgen05_prefill_vs_oracle(D, shape):
    B, H, Sq, Skv = shape
    errs, _ = _run(B, H, Sq, Skv, D, expect="tcgen05")
    assert max(errs) < TOL


@pytest.mark.parametrize("segments", [2, 4])
def test_tcgen05_prefill_multisegment(segments):
    errs, _ = _run(1, 2, 256, 1024, 128, segments=segments, expect="tcgen05")
    assert max(errs) < TOL


@pytest.mark.parametrize("B,H,Sq,Skv,segments,D", [(2, 64, 512, 256, 1, 128), (1, 100, 512, 512, 2, 128),
                                                   (3, 50, 256, 384, 1, 64), (1, 160, 256, 128, 1, 128)])
def test_tcgen05_persistent_multi_unit(B, H, Sq, Skv, segments, D):
    """More work units than SMs: each persistent CTA walks several units, so
    barrier phases, the Q reload after the last S, and the o_empty hand-off of
    the epilogue to the next unit are all exercised (and so are units whose
    KV slice has 2-4 tiles)."""
    errs, _ = _run(B, H, Sq, Skv, D, segments=segments, seed=B + H, expect="tcgen05")
    assert max(errs) < TOL


def test_tcgen05_stats_are_tight():
    """d1 is an exact max of fp32 logits; d2 accumulates fp32 exps: both far
    tighter than the bf16 tolerance."""
    (em, el, eo), _ = _run(1, 4, 256, 2048, 128, seed=5, expect="tcgen05")
    assert em < 1e-5 and el < 1e-3 and eo < 1e-2


def test_tcgen05_large_logits_rescale_path():
    """Growing logits force exp(d1'-d1) != 1 on many tiles (correction warpgroup)."""
    import torch
    from paper_2603_10026_b200 import attention

    B, H, Sq, Skv, D = 1, 2, 256, 2048, 128
    q, k, v = _inputs(B, H, Sq, Skv, D, 9, torch.float64)
    ramp = torch.linspace(0.0, 8.0, Skv, dtype=torch.float64).view(1, 1, Skv, 1)
    k = k * (1 + ramp)  # later keys have larger logits -> max increases along the loop
    q, k, v = (t.to(torch.bfloat16) for t in (q, k, v))
    m, l, o = attention(q.cuda(), k.cuda(), v.cuda())
    torch.cuda.synchronize()
    _check(q, k, v, m, l, o, TOL)


@pytest.mark.parametrize("segments", [1, 4, 8])
def test_decode_split_kv(segments):
    errs, _ = _run(2, 4, 1, 8192, 128, segments=segments, expect="decode")
    assert max(errs) < TOL


def test_decode_odd_slice_uses_generic_path():
    errs, _ = _run(1, 2, 1, 96, 128, segments=1)
    assert max(errs) < TOL


def test_bf16_ragged_prefill_generic_path():
    errs, _ = _run(1, 2, 100, 300, 64)
    assert max(errs) < TOL


@pytest.mark.parametrize("dtype_name,shape,S", [("bf16", (2, 4, 1, 8192, 128), 8),
                                                 ("f32", (1, 2, 64, 1024, 64), 4)])
def test_split_kv_shards_merge_equals_multisegment(dtype_name, shape, S):
    """Two KV shards (as two GPUs would hold them): rf_run_partials on each
    local shard, concatenation in rank = slice order (what the NCCL all-gather
    produces), rf_merge_partials == single-device run_multisegment(S)."""
    import torch
    from paper_2603_10026_b200 import Desc, Plan, _native as N
    from paper_2603_10026_b200.distributed import kv_shard, split_kv_decode

    dt = torch.bfloat16 if dtype_name == "bf16" else torch.float32
    B, H, Sq, Skv, D = shape
    q, k, v = _inputs(B, H, Sq, Skv, D, 21, dt)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    G = 2
    parts = []
    for r in range(G):
        kv0, kv1, s0, local = kv_shard(r, G, Skv, S)
        p = Plan(Desc(N.RF_PATTERN_ATTENTION, dtype_name, rows=Sq, len=kv1 - kv0, free_len=D,
                      batch=B, heads=H, segments=local))
        rows = B * H * Sq
        pm = torch.empty(local, rows, device="cuda")
        pl = torch.empty_like(pm)
        po = torch.empty(local, rows, D, device="cuda")
        p.run_partials([qd, kd[:, :, kv0:kv1].contiguous(), vd[:, :, kv0:kv1].contiguous()], 0,
                       pm, pl, po)
        parts.append((pm, pl, po))
    pm = torch.cat([x[0] for x in parts])
    pl = torch.cat([x[1] for x in parts])
    po = torch.cat([x[2] for x in parts])
    m = torch.empty(B, H, Sq, device="cuda")
    l = torch.empty_like(m)
    o = torch.empty_like(qd)
    p.merge_partials(pm, pl, po, [m, l, o])
    torch.cuda.synchronize()
    tol = 2e-2 if dt == torch.bfloat16 else 1e-5
    _check(q, k, v, m, l, o, tol)
    # the single-rank path of split_kv_decode (no process group) is the same plan
    m1, l1, o1 = split_kv_decode(qd, kd, vd, S)
    torch.cuda.synchronize()
    _check(q, k, v, m1, l1, o1, tol)
