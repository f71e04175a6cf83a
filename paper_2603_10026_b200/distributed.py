"""Multi-GPU layer: batch/head (or token) sharding and the split-KV partial
(m, l, O) merge over NVLink (SURVEY §8 e).

* Batch/head-sharded workloads (attention prefill, the GEMM patterns) need no
  collective: every rank runs its own units (`shard_units`).
* Split-KV decode shards the reduce axis: rank r owns KV positions
  [r*Skv/G, (r+1)*Skv/G) of every (b,h) — slices [r*S/G, (r+1)*S/G) of the
  reference's Multi-Segment strategy (run_multisegment,
  proj/src/simulator.cpp:660-687). Each rank streams its slices into partial
  states, the partials are all-gathered (NCCL over NVLink; about
  B*H*(D+2)*4 bytes per slice), and every rank folds them in global slice
  order with rf_merge_partials — the reference's incr_push_child order, so
  the result equals single-GPU run_multisegment(S).

The collective and the slice bookkeeping are independent of the compute, so
tests can drive the same code with gloo on CPU (tests/test_multigpu_gloo.py).
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

from .executors import IncompatibleSegmentation


def shard_units(units: int, rank: int, world: int) -> Tuple[int, int]:
    """[begin, end) of the independent units (b,h pairs or token rows) owned by
    `rank` — contiguous, balanced to within one unit."""
    base, extra = divmod(units, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def kv_shard(rank: int, world: int, skv: int, segments: int) -> Tuple[int, int, int, int]:
    """KV range and slices of `rank` in a `segments`-way split over `world`
    GPUs: (kv_begin, kv_end, slice_begin, local_slices). The reference's
    constraint S | Skv (simulator.cpp:668-671) plus G | S."""
    if segments < 1 or skv % segments:
        raise IncompatibleSegmentation(f"{segments} segments do not divide L0 = {skv}")
    if segments % world:
        raise IncompatibleSegmentation(f"{segments} segments do not split over {world} GPUs")
    local = segments // world
    slice_len = skv // segments
    s0 = rank * local
    return s0 * slice_len, (s0 + local) * slice_len, s0, local


def gather_partials(m, l, o, group=None):
    """All-gather local partials [S_local, rows(, D)] into [S, rows(, D)] in rank
    (= global slice) order. NCCL for CUDA tensors, gloo for CPU tensors."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if world == 1:
        return m, l, o
    # gloo has no CUDA all_gather: stage through host memory (the CPU test
    # path and the one-GPU multi-rank smoke run); NCCL gathers in place.
    host = dist.get_backend(group) == "gloo" and m.is_cuda
    out = []
    for t in (m, l, o):
        src = t.contiguous().cpu() if host else t.contiguous()
        parts = [torch.empty_like(src) for _ in range(world)]
        dist.all_gather(parts, src, group=group)
        cat = torch.cat(parts, dim=0)
        out.append(cat.to(t.device) if host else cat)
    return tuple(out)


def split_kv_decode(q, k_local, v_local, segments: int, group=None, stream=None,
                    partials_fn: Optional[Callable] = None, merge_fn: Optional[Callable] = None):
    """Split-KV attention across the ranks of `group`.

    q: [B,H,Sq,D] (replicated); k_local/v_local: [B,H,Skv/G,D] — this rank's KV
    shard. `segments` is the global S (G | S). Returns the merged (d1, d2, d3)
    on every rank. partials_fn / merge_fn default to the librf_cuda kernels
    (rf_run_partials / rf_merge_partials); tests may inject others.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    # the kernels read dense [B,H,S,D] buffers: a strided view (e.g.
    # k[:, :, a:b]) must be materialised, never passed as a raw pointer
    q, k_local, v_local = q.contiguous(), k_local.contiguous(), v_local.contiguous()
    B, H, Sq, D = q.shape
    skv_local = k_local.shape[2]
    if segments % world:
        raise IncompatibleSegmentation(f"{segments} segments do not split over {world} GPUs")
    local = segments // world
    if skv_local % local:
        raise IncompatibleSegmentation(f"{local} local segments do not divide {skv_local}")
    rows = B * H * Sq
    if partials_fn is None or merge_fn is None:
        from . import _native as N
        from .executors import Desc, plan

        dt = "bf16" if q.dtype == torch.bfloat16 else "f32"
        p = plan(Desc(N.RF_PATTERN_ATTENTION, dt, rows=Sq, len=skv_local, free_len=D, batch=B,
                      heads=H, segments=local, device=q.device.index or 0), stream)

        def partials_fn(q, k, v, pm, pl, po):  # noqa: F811
            p.run_partials([q, k, v], 0, pm, pl, po, stream)

        def merge_fn(pm, pl, po, outs):  # noqa: F811
            p.merge_partials(pm, pl, po, outs, stream)

    dev = q.device
    pm = torch.empty(local, rows, dtype=torch.float32, device=dev)
    pl = torch.empty_like(pm)
    po = torch.empty(local, rows, D, dtype=torch.float32, device=dev)
    partials_fn(q, k_local, v_local, pm, pl, po)
    if world > 1:
        # the collective runs on torch's current stream: order it after the
        # partials kernel (on `stream`), and the merge (on `stream`) after it
        cur = torch.cuda.current_stream(dev) if q.is_cuda else None
        if cur is not None and stream is not None:
            cur.wait_stream(stream)
        pm, pl, po = gather_partials(pm, pl, po, group)
        if cur is not None and stream is not None:
            stream.wait_stream(cur)
    m = torch.empty(B, H, Sq, dtype=torch.float32, device=dev)
    l = torch.empty_like(m)
    o = torch.empty_like(q)
    merge_fn(pm, pl, po, [m, l, o])
    return m, l, o
