"""The N>1 path on CPU: world_size-2 gloo process group driving the real
split-KV plumbing of paper_2603_10026_b200/distributed.py (shard bookkeeping,
all-gather in rank = slice order, slice-ordered merge), with the oracle
standing in for the kernels (no GPU here). The merged result must equal the
single-process run_multisegment(S) restatement."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_10026_b200.distributed import kv_shard, shard_units, split_kv_decode
from paper_2603_10026_b200.executors import IncompatibleSegmentation


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(B=2, H=3, Sq=2, Skv=64, D=8, seed=0):
    g = torch.Generator().manual_seed(seed)
    q = (torch.rand(B, H, Sq, D, generator=g, dtype=torch.float64) * 2 - 1) / np.sqrt(D)
    k = torch.rand(B, H, Skv, D, generator=g, dtype=torch.float64) * 2 - 1
    v = torch.rand(B, H, Skv, D, generator=g, dtype=torch.float64) * 2 - 1
    return q, k, v


def _oracle_partials(q, k, v, pm, pl, po):
    from tests import oracle as O

    B, H, Sq, D = q.shape
    local = pm.shape[0]
    skv = k.shape[2]
    sl = skv // local
    p = torch.einsum("bhqd,bhkd->bhqk", q, k).reshape(B * H * Sq, skv).numpy()
    vv = v.reshape(B * H, 1, skv, D).expand(B * H, Sq, skv, D).reshape(B * H * Sq, skv, D).numpy()
    for s in range(local):
        m, l, o = O.attention_incremental(p[:, s * sl:(s + 1) * sl], vv[:, s * sl:(s + 1) * sl], 1)
        pm[s] = torch.from_numpy(m)
        pl[s] = torch.from_numpy(l)
        po[s] = torch.from_numpy(o)


def _oracle_merge(pm, pl, po, outs):
    from tests import oracle as O

    m, l, o = O.attention_merge(pm.double().numpy(), pl.double().numpy(), po.double().numpy())
    outs[0].copy_(torch.from_numpy(m).reshape(outs[0].shape))
    outs[1].copy_(torch.from_numpy(l).reshape(outs[1].shape))
    outs[2].copy_(torch.from_numpy(o).reshape(outs[2].shape))


def _worker(rank, world, port, S, q_ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q, k, v = _problem()
        kv0, kv1, s0, local = kv_shard(rank, world, k.shape[2], S)
        assert s0 == rank * local
        m, l, o = split_kv_decode(q, k[:, :, kv0:kv1].contiguous(), v[:, :, kv0:kv1].contiguous(),
                                  S, partials_fn=_oracle_partials, merge_fn=_oracle_merge)
        q_ret.put((rank, m.numpy(), l.numpy(), o.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("S", [2, 4, 8])
def test_split_kv_over_two_ranks_equals_multisegment(S):
    from tests import oracle as O

    ctx = mp.get_context("spawn")
    qret = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, S, qret)) for r in range(2)]
    for p in procs:
        p.start()
    res = [qret.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    q, k, v = _problem()
    B, H, Sq, D = q.shape
    P = torch.einsum("bhqd,bhkd->bhqk", q, k).reshape(B * H * Sq, -1).numpy()
    V = v.reshape(B * H, 1, -1, D).expand(B * H, Sq, -1, D).reshape(B * H * Sq, -1, D).numpy()
    rm, rl, ro = O.attention_incremental(P, V, S)  # single-process run_multisegment(S)
    for rank, m, l, o in res:  # every rank holds the merged result
        assert O.scaled_max_err(m.ravel(), rm)[0] < 1e-6
        assert O.scaled_max_err(l.ravel(), rl)[0] < 1e-6
        assert O.scaled_max_err(o.reshape(-1, D), ro)[0] < 1e-6


def test_shard_bookkeeping():
    assert [shard_units(10, r, 4) for r in range(4)] == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert kv_shard(1, 2, 32768, 8) == (16384, 32768, 4, 4)
    with pytest.raises(IncompatibleSegmentation):
        kv_shard(0, 2, 96, 5)  # S does not divide L0
    with pytest.raises(IncompatibleSegmentation):
        kv_shard(0, 4, 96, 6)  # S not divisible by G
