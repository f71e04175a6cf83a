"""Parity at the exact shapes bench.py times:
every BASELINE config and the extras cfg6-cfg8 at full size, plus the
per-rank shares the strong-scaling split gives ranks 0 and G-1 at G = 8.
The workloads are bench.py's own (same generators, plans, packing) and the
checks are tests/bench_parity.py's sampled-row oracle comparisons: GEMMs with
several rasterisation N groups and an N tail (cfg5: 43 N tiles = 5 groups of
8 + 3), FP8 with K = 8192 (64 K tiles of running-ref updates), decode at
Skv = 32768 with the bench's split choice, prefill over all 256 (b,h) units."""
import gc
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu


def _run(cfg, rank=0, world=1):
    import torch

    import bench
    from tests import bench_parity

    lcfg = bench.local_config(cfg, rank, world, "strong")
    lcfg["split_kv"] = False  # one process: run the rank's share through rf_run
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    wl = bench.Workload(lcfg, dev, rank, stream)
    with torch.cuda.stream(stream):
        wl.run(stream)
    stream.synchronize()
    res = bench_parity.check(wl)
    del wl
    gc.collect()
    torch.cuda.empty_cache()
    return res


@pytest.mark.parametrize("idx", [0, 1, 2, 3, 4, 5, 6, 7])
def test_full_config_parity(idx):
    import bench

    res = _run(bench.CONFIGS[idx])
    assert res["pass"], res
    assert res["rows_checked"] >= {0: 1024, 1: 256, 2: 64, 3: 64, 4: 64, 5: 64, 6: 2048, 7: 512}[idx]


@pytest.mark.parametrize("idx", [1, 3, 4, 5, 6, 7])
@pytest.mark.parametrize("rank", [0, 7])
def test_g8_rank_share_parity(idx, rank):
    """The small-M / few-unit shards of the 8-GPU split (cfg4: 1,024 rows)."""
    import bench

    res = _run(bench.CONFIGS[idx], rank, 8)
    assert res["pass"], res


def test_decode_local_kv_share_partials_merge_equals_full():
    """Split-KV share of rank r at G = 4: partials of its KV range folded with
    the other ranks' (computed here in one process) equal single-GPU
    run_multisegment(8) — the cross-GPU merge's slice order."""
    import torch

    from paper_2603_10026_b200 import _native as N
    from paper_2603_10026_b200 import attention
    from paper_2603_10026_b200.executors import Desc, plan

    torch.manual_seed(0)
    B, H, Skv, D, G = 4, 8, 32768, 128, 4
    q = ((torch.rand(B, H, 1, D, device="cuda") * 2 - 1) / D ** 0.5).bfloat16()
    k = (torch.rand(B, H, Skv, D, device="cuda") * 2 - 1).bfloat16()
    v = (torch.rand(B, H, Skv, D, device="cuda") * 2 - 1).bfloat16()
    m, l, o = attention(q, k, v, segments=8)
    pm, pl, po = [], [], []
    for r in range(G):  # rank r's KV share, as split_kv_decode hands it to rf_run_partials
        ks = k[:, :, r * Skv // G:(r + 1) * Skv // G].contiguous()
        vs = v[:, :, r * Skv // G:(r + 1) * Skv // G].contiguous()
        p = plan(Desc(N.RF_PATTERN_ATTENTION, "bf16", rows=1, len=Skv // G, free_len=D, batch=B,
                      heads=H, segments=8 // G))
        a = torch.empty(8 // G, B * H, device="cuda")
        b = torch.empty_like(a)
        c = torch.empty(8 // G, B * H, D, device="cuda")
        p.run_partials([q, ks, vs], 0, a, b, c)
        pm.append(a)
        pl.append(b)
        po.append(c)
    full = plan(Desc(N.RF_PATTERN_ATTENTION, "bf16", rows=1, len=Skv, free_len=D, batch=B, heads=H,
                     segments=8))
    m2, l2, o2 = torch.empty_like(m), torch.empty_like(l), torch.empty_like(o)
    full.merge_partials(torch.cat(pm), torch.cat(pl), torch.cat(po), [m2, l2, o2])
    torch.cuda.synchronize()
    assert torch.equal(m, m2)
    assert (l - l2).abs().max().item() <= 1e-5 * l.abs().max().item()
    assert (o.float() - o2.float()).abs().max().item() <= 2e-2
