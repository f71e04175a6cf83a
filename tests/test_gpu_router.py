"""GPU parity of the MoE router (router.cu): the router GEMM s = X W on tcgen05
(split-K, deterministic split-ordered sums) feeding the routing cascade of
make_moe_routing (proj/src/workloads.cpp:124-169). Shapes: the paper's routing
table R1-R8 (s = 2048 tokens, hd, en experts, top-k).

Parity is checked at the cascade boundary the reference itself draws (the GEMM
is a producer outside the cascade, proj/src/scalar_ir.cpp:483-491):
  * scores vs the fp64 oracle on the same bf16-rounded X and W (<= 1e-5 scaled);
  * the routing outputs vs the oracle run on the kernel's own scores: d1 exact,
    d2 <= 1e-5, top-k values and indices bit-exact (north_star);
  * the routing vs the oracle on the fp64 scores: indices may differ only where
    the oracle's k-th and (k+1)-th scores are closer than the GEMM error."""
import numpy as np
import pytest

from tests import oracle as O

pytestmark = pytest.mark.gpu

R = {  # name: (tokens, hd, experts, top-k)
    "R1": (2048, 768, 128, 1), "R2": (2048, 1024, 128, 1), "R3": (2048, 4096, 128, 1),
    "R4": (2048, 2560, 64, 6), "R5": (2048, 8192, 64, 8), "R6": (2048, 2048, 64, 6),
    "R7": (2048, 2048, 128, 8), "R8": (2048, 4096, 128, 8),
}


def _run(tokens, hd, experts, k, seed):
    import torch
    from paper_2603_10026_b200 import moe_router, moe_router_plan

    g = torch.Generator().manual_seed(seed)
    x = (torch.rand(tokens, hd, generator=g) * 2 - 1).bfloat16()
    w = (torch.rand(hd, experts, generator=g) * 2 - 1) / hd ** 0.5
    p = moe_router_plan(tokens, hd, experts, k)
    wp = p.pack_weight(w.cuda())
    d1, d2, tv, ti, sc = moe_router(x.cuda(), wp, k, with_scores=True)
    torch.cuda.synchronize()
    xs = x.double().numpy()
    ws = w.bfloat16().double().numpy()
    return (xs @ ws, d1.double().cpu().numpy(), d2.double().cpu().numpy(),
            tv.double().cpu().numpy(), ti.cpu().numpy(), sc.double().cpu().numpy())


@pytest.mark.parametrize("name", sorted(R))
def test_router_paper_shapes(name):
    tokens, hd, experts, k = R[name]
    ref, d1, d2, tv, ti, sc = _run(tokens, hd, experts, k, seed=int(name[1:]))
    # producer: the router GEMM (fp32 accumulation of bf16 products)
    assert O.scaled_max_err(sc.ravel(), ref.ravel())[0] <= 1e-5
    # cascade on the kernel's own scores: bit-exact indices and values
    r1, r2, rv, ri = O.moe_routing(sc, k)
    assert O.scaled_max_err(d1, r1)[0] == 0.0
    assert O.scaled_max_err(d2, r2)[0] <= 1e-5
    np.testing.assert_array_equal(ti, ri)
    np.testing.assert_array_equal(tv, rv)
    # against the fp64 scores: index differences only at near-ties
    _, _, fv, fi = O.moe_routing(ref, k)
    srt = -np.sort(-ref, axis=1)
    gap = srt[:, k - 1] - (srt[:, k] if k < experts else -np.inf)
    bad = np.any(ti != fi, axis=1)
    assert np.all(gap[bad] < 1e-4), gap[bad]


@pytest.mark.parametrize("tokens,hd,experts,k", [
    (1000, 512, 32, 2), (300, 256, 256, 8), (128, 64, 64, 1),
    # split-K with the L2 exchange on a ragged last row tile (1000 = 7 x 128 + 104; 4 splits), 256 experts
    # over 8 splits with a 2-token last tile (some split CTAs own no live token), 32 experts
    (1000, 2048, 64, 4), (130, 4096, 256, 8), (200, 1024, 32, 3)])
def test_router_ragged_and_expert_counts(tokens, hd, experts, k):
    ref, d1, d2, tv, ti, sc = _run(tokens, hd, experts, k, seed=tokens + hd)
    assert O.scaled_max_err(sc.ravel(), ref.ravel())[0] <= 1e-5
    r1, r2, rv, ri = O.moe_routing(sc, k)
    assert O.scaled_max_err(d1, r1)[0] == 0.0
    assert O.scaled_max_err(d2, r2)[0] <= 1e-5
    np.testing.assert_array_equal(ti, ri)


def test_router_host_path_and_launches():
    import torch
    from paper_2603_10026_b200 import moe_router, moe_router_plan

    tokens, hd, experts, k = 1024, 1024, 128, 4
    x = (torch.rand(tokens, hd) * 2 - 1).bfloat16()
    w = (torch.rand(hd, experts) * 2 - 1) / hd ** 0.5
    p = moe_router_plan(tokens, hd, experts, k)
    assert p.launches_per_run == 1 and "router" in p.info["kernel"]
    wp = p.pack_weight(w.cuda())
    d1, d2, tv, ti = moe_router(x.cuda(), wp, k)
    h1 = torch.empty(tokens).pin_memory()
    h2 = torch.empty(tokens).pin_memory()
    hr = torch.empty(tokens, k, 2, dtype=torch.int32).pin_memory()
    p.run_host([x.pin_memory(), wp], [h1, h2, hr, None])
    torch.cuda.synchronize()
    assert torch.equal(h1, d1.cpu()) and torch.equal(h2, d2.cpu())
    assert torch.equal(hr[..., 1], ti.cpu())


def test_router_unsupported_shapes():
    from paper_2603_10026_b200 import UnsupportedPattern, moe_router_plan

    with pytest.raises(UnsupportedPattern):
        moe_router_plan(128, 100, 64, 2)  # hd % 64
    with pytest.raises(UnsupportedPattern):
        moe_router_plan(128, 128, 48, 2)  # experts
    with pytest.raises(UnsupportedPattern):
        moe_router_plan(128, 128, 64, 9)  # K' > 8


def test_router_counters_across_launches():
    """The split exchange's arrival counters (plan workspace, never reset): repeated device runs of one
    plan interleaved with host-path runs (16 chunks: other row-tile counters, one row tile per launch)
    give bit-identical scores and routes every time."""
    import torch
    from paper_2603_10026_b200 import moe_router, moe_router_plan

    tokens, hd, experts, k = 2048, 4096, 128, 8  # R8: 16 row tiles x 8 splits
    g = torch.Generator().manual_seed(5)
    x = (torch.rand(tokens, hd, generator=g) * 2 - 1).bfloat16()
    w = (torch.rand(hd, experts, generator=g) * 2 - 1) / hd ** 0.5
    p = moe_router_plan(tokens, hd, experts, k)
    assert p.launches_per_run == 1
    wp = p.pack_weight(w.cuda())
    xd = x.cuda()
    ref = moe_router(xd, wp, k, with_scores=True)
    h1 = torch.empty(tokens).pin_memory()
    h2 = torch.empty(tokens).pin_memory()
    hr = torch.empty(tokens, k, 2, dtype=torch.int32).pin_memory()
    for i in range(40):
        got = moe_router(xd, wp, k, with_scores=True)
        for a, b in zip(got, ref):
            assert torch.equal(a, b), i
        if i % 8 == 0:
            p.run_host([x.pin_memory(), wp], [h1, h2, hr, None])
            torch.cuda.synchronize()
            assert torch.equal(h1, ref[0].cpu()) and torch.equal(hr[..., 1], ref[3].cpu())
