"""GPU parity of the MoE routing cascade (moe.cu): softmax statistics + top-k
with bit-exact indices (ties to the lowest index), against the oracle
(pinned to the reference's goldens) on the same float32 inputs. Shapes follow
the paper's routing table R1-R8 (2048 tokens, 64/128
experts, top-1..8)."""
import numpy as np
import pytest

from tests import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("experts,k", [(128, 1), (64, 6), (64, 8), (128, 8), (100, 3), (7, 4), (300, 5), (256, 8)])
def test_moe_routing_vs_oracle(experts, k):
    import torch
    from paper_2603_10026_b200 import moe_routing

    rng = np.random.default_rng(experts * 10 + k)
    s = rng.uniform(-2, 2, (2048, experts)).astype(np.float32)
    s[::7, 3] = s[::7, 5]  # exact ties -> lowest index first
    d1, d2, tv, ti = moe_routing(torch.tensor(s).cuda(), k)
    torch.cuda.synchronize()
    r1, r2, rv, ri = O.moe_routing(s.astype(np.float64), k)
    kk = min(k, experts)
    assert O.scaled_max_err(d1.double().cpu().numpy(), r1)[0] == 0.0  # exact max
    assert O.scaled_max_err(d2.double().cpu().numpy(), r2)[0] < 1e-5
    np.testing.assert_array_equal(ti.cpu().numpy()[:, :kk], ri[:, :kk])  # bit-exact indices
    np.testing.assert_array_equal(tv.double().cpu().numpy()[:, :kk], rv[:, :kk])
    if kk < k:
        assert (ti.cpu().numpy()[:, kk:] == 0).all()


def test_moe_routing_reference_golden_and_ties():
    import torch
    from paper_2603_10026_b200 import moe_routing

    g = O.load_golden("moe_routing_128x8_s100")
    s = torch.tensor(g["in.s"], dtype=torch.float32).reshape(1, -1).cuda()
    d1, d2, tv, ti = moe_routing(s, 8)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(ti.cpu().numpy().ravel(), g["incremental.d3.topk_idx"].astype(np.int64))
    assert O.scaled_max_err(d1.double().cpu().numpy(), g["oracle.d1"])[0] < 1e-6
    assert O.scaled_max_err(d2.double().cpu().numpy(), g["oracle.d2"])[0] < 1e-5
    # test_simulator.cpp:254-271
    s = torch.tensor([[0.3, 0.9, 0.9, -1.0, 0.5, 2.0, 0.1, 0.9]], device="cuda")
    _, _, tv, ti = moe_routing(s, 3)
    assert ti.cpu().tolist() == [[6, 2, 3]]


@pytest.mark.parametrize("experts,k", [(128, 8), (256, 8), (64, 5), (200, 7)])
def test_moe_routing_heavy_ties(experts, k):
    """Scores on a 4-level grid (+0/-0 included): every round's argmax is a tie
    across lanes and within a lane's experts; indices must follow (value desc,
    index asc) exactly (topk_merge, proj/src/simulator.cpp:80-88)."""
    import torch
    from paper_2603_10026_b200 import moe_routing

    g = torch.Generator().manual_seed(experts * 31 + k)
    levels = torch.tensor([-1.0, -0.0, 0.0, 0.5])
    s = levels[torch.randint(0, 4, (257, experts), generator=g)]
    _, _, tv, ti = moe_routing(s.cuda(), k)
    torch.cuda.synchronize()
    sv = s.numpy().astype(np.float64) + 0.0  # -0 == +0
    want = np.argsort(-sv, axis=1, kind="stable")[:, :k] + 1
    np.testing.assert_array_equal(ti.cpu().numpy(), want)
