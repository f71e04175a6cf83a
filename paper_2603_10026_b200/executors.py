"""Batched fused-loop executors over librf_cuda (the C-ABI, include/rf_cuda.h).

This is the Python mirror of the host plan layer: it builds rf_desc
descriptors, owns rf_plan handles, and maps rf_status codes back onto the
reference's exception types:

  ShapeMismatch             proj/include/redfuse/simulator.hpp:17-19
  IncompatibleSegmentation  proj/include/redfuse/simulator.hpp:21-23
  DomainError               proj/include/redfuse/expr.hpp:29-31

Tensors are torch tensors used purely as device memory (PyTorch is plumbing:
allocation, streams, torch.distributed); every computation runs in a
librf_cuda kernel. There is no CPU fallback — without the library or an
sm_100 device the calls raise.
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass
from typing import Optional, Sequence

from . import _native as N


class RedfuseError(RuntimeError):
    pass


class ShapeMismatch(RedfuseError):
    """redfuse::ShapeMismatch (simulator.hpp:17-19)."""


class IncompatibleSegmentation(RedfuseError):
    """redfuse::IncompatibleSegmentation (simulator.hpp:21-23)."""


class DomainError(RedfuseError):
    """redfuse::DomainError (expr.hpp:29-31): a fault at finalize, e.g. 0/0."""


class UnsupportedPattern(RedfuseError):
    """No librf_cuda kernel implements this pattern / dtype / shape."""


class CudaError(RedfuseError):
    pass


_EXC = {
    N.RF_ERR_SHAPE: ShapeMismatch,
    N.RF_ERR_SEGMENTATION: IncompatibleSegmentation,
    N.RF_ERR_DOMAIN: DomainError,
    N.RF_ERR_UNSUPPORTED: UnsupportedPattern,
    N.RF_ERR_CUDA: CudaError,
    N.RF_ERR_ARG: ValueError,
}


def check(status: int) -> None:
    if status != N.RF_OK:
        exc = _EXC.get(status, RedfuseError)
        raise exc(f"{N.lib().rf_status_string(status).decode()}: {N.last_error()}")


def _ptr(t) -> Optional[int]:
    return None if t is None else int(t.data_ptr())


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        import torch

        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


_DT = {"f32": N.RF_F32, "bf16": N.RF_BF16, "e4m3": N.RF_E4M3}


@dataclass(frozen=True)
class Desc:
    pattern: int
    dtype: str
    rows: int
    len: int
    free_len: int = 0
    batch: int = 1
    heads: int = 1
    segments: int = 1
    fmax: float = 448.0
    eps: float = 1e-6
    softmax_scale: float = 1.0
    offset: float = 0.0
    device: int = 0
    producer_len: int = 0  # MOE_ROUTER: hd (the router GEMM's reduce axis)
    stat_len: int = 0  # RMSNORM / LAYERNORM: K of the statistics' means (0 = len)
    # run_fused (simulator.cpp:485-559): fusion level k >= 1 over the tree
    # levels[1..K] (L0 = len implicit); 0 = the incremental executors
    fuse_level: int = 0
    tree: tuple = ()

    def to_c(self) -> N.rf_desc:
        d = N.rf_desc()
        d.pattern = self.pattern
        d.dtype = _DT[self.dtype]
        d.batch, d.heads, d.rows = self.batch, self.heads, self.rows
        d.len, d.free_len, d.segments = self.len, self.free_len, self.segments
        d.fmax, d.eps, d.softmax_scale = self.fmax, self.eps, self.softmax_scale
        d.offset = self.offset
        d.tile_rows = d.tile_stream = 0
        d.device = self.device
        d.producer_len = self.producer_len
        d.stat_len = self.stat_len
        d.fuse_level = self.fuse_level
        d.tree_depth = len(self.tree)
        for i, w in enumerate(tuple(self.tree)[:8]):
            d.tree[i] = int(w)
        return d


class Plan:
    """An immutable rf_plan (kernel + tiles + persistent workspace)."""

    def __init__(self, desc: Desc):
        self.desc = desc
        self._h = ctypes.c_void_p()
        c = desc.to_c()
        check(N.lib().rf_plan_create(ctypes.byref(c), ctypes.byref(self._h)))
        buf = ctypes.create_string_buffer(1024)
        check(N.lib().rf_plan_describe(self._h, buf, 1024))
        self.info = json.loads(buf.value.decode())
        self.launches_per_run = int(N.lib().rf_plan_launches_per_run(self._h))
        ib, ob = (ctypes.c_size_t * 4)(), (ctypes.c_size_t * 4)()
        check(N.lib().rf_plan_io_bytes(self._h, ib, ob))
        self.in_bytes, self.out_bytes = tuple(ib), tuple(ob)

    def close(self):
        if self._h:
            N.lib().rf_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _io(inputs: Sequence, outputs: Sequence) -> N.rf_io:
        io = N.rf_io()
        for i, t in enumerate(inputs):
            io.in_[i] = t if isinstance(t, int) else _ptr(t)
        for i, t in enumerate(outputs):
            io.d[i] = _ptr(t)
        return io

    def _check_io(self, inputs: Sequence, outputs: Sequence, host: bool) -> None:
        """ShapeMismatch (check_shapes, proj/src/simulator.cpp:235-245) for any
        buffer whose size, layout or placement disagrees with the plan — the
        kernels take raw pointers and would otherwise read out of bounds."""
        dev = self.desc.device
        for kind, ts, need in (("in", inputs, self.in_bytes), ("d", outputs, self.out_bytes)):
            _require(len(ts) <= 4, f"at most 4 {kind} buffers")
            for i, t in enumerate(ts):
                if t is None or isinstance(t, int) or need[i] == 0:
                    continue
                name = f"{kind}[{i}]" if kind == "in" else f"d{i + 1}"
                got = t.numel() * t.element_size()
                _require(got == need[i], f"{name}: {got} bytes, the plan needs {need[i]}")
                _require(t.is_contiguous(), f"{name} must be contiguous")
                # the packed weight stays device-resident on the host path too
                want_cuda = not host or (kind == "in" and i == 1 and _packed(self) > 0)
                if want_cuda:
                    _require(t.is_cuda and (t.device.index or 0) == dev,
                             f"{name} must be on cuda:{dev}")
                else:
                    _require(not t.is_cuda, f"{name} must be a host tensor for run_host")
            for i in range(len(ts), 4):
                if need[i] and not (kind == "d" and i == 3):
                    raise ShapeMismatch(f"missing {kind} buffer {i}")

    def run(self, inputs: Sequence, outputs: Sequence, stream=None) -> None:
        self._check_io(inputs, outputs, host=False)
        io = self._io(inputs, outputs)
        check(N.lib().rf_run(self._h, ctypes.byref(io), _stream_ptr(stream)))

    def run_unchecked(self, inputs: Sequence, outputs: Sequence, stream=None) -> None:
        """rf_run without the Python-side buffer checks (callers that validated
        their buffers once, e.g. a CUDA-graph capture loop)."""
        io = self._io(inputs, outputs)
        check(N.lib().rf_run(self._h, ctypes.byref(io), _stream_ptr(stream)))

    def run_host(self, inputs: Sequence, outputs: Sequence) -> None:
        """Host (pinned) buffers in and out; copies happen inside the call."""
        self._check_io(inputs, outputs, host=True)
        io = self._io(inputs, outputs)
        check(N.lib().rf_run_host(self._h, ctypes.byref(io)))

    def run_partials(self, inputs: Sequence, slice_begin: int, m, l, o, stream=None) -> None:
        io = self._io(inputs, [])
        p = N.rf_partials(_ptr(m), _ptr(l), _ptr(o), int(m.shape[0]))
        check(N.lib().rf_run_partials(self._h, ctypes.byref(io), slice_begin, ctypes.byref(p),
                                      _stream_ptr(stream)))

    def merge_partials(self, m, l, o, outputs: Sequence, stream=None) -> None:
        io = self._io([], outputs)
        p = N.rf_partials(_ptr(m), _ptr(l), _ptr(o), int(m.shape[0]))
        check(N.lib().rf_merge_partials(self._h, ctypes.byref(p), ctypes.byref(io),
                                        _stream_ptr(stream)))

    def pack_weight(self, w, g=None, stream=None):
        import torch

        k, n = self.desc.len, self.desc.free_len
        if self.desc.pattern == N.RF_PATTERN_MOE_ROUTER:
            k, n = self.desc.producer_len, self.desc.len  # w [hd, experts]
        if tuple(w.shape) != (k, n) or w.dtype != torch.float32:
            raise ShapeMismatch(f"w must be float32 [{k}, {n}] (reduce-axis major)")
        nbytes = int(N.lib().rf_packed_bytes(self._h))
        if nbytes == 0:
            raise UnsupportedPattern("pattern has no packed weight")
        raw = torch.empty(nbytes, dtype=torch.uint8, device=w.device)
        check(N.lib().rf_pack_weight(self._h, _ptr(w.contiguous()), _ptr(g), _ptr(raw),
                                     _stream_ptr(stream)))
        if self.desc.pattern == N.RF_PATTERN_QUANT_GEMM_E4M3:
            return raw.view(n, k)
        if self.desc.pattern in (N.RF_PATTERN_RMSNORM_GEMM, N.RF_PATTERN_MOE_ROUTER):
            return raw.view(torch.bfloat16).view(n, k)
        # layernorm: bf16 [N, K] (g folded) followed by N f32 column sums; the
        # returned tensor is the whole buffer (rf_run reads both parts)
        return raw

    def check_domain(self, stream=None) -> None:
        check(N.lib().rf_check_domain(self._h, _stream_ptr(stream)))


def _packed(p: "Plan") -> int:
    return int(N.lib().rf_packed_bytes(p._h))


_plans: dict = {}


def plan(desc: Desc, stream=None) -> Plan:
    """The cached plan for (desc, stream). A plan owns its split workspace, so
    calls on different streams get different plans and never share it
    (rf_cuda.h: one plan per stream for concurrent execution)."""
    key = (desc, _stream_ptr(stream) if stream is not None or _cuda_ok() else 0)
    p = _plans.get(key)
    if p is None:
        p = _plans[key] = Plan(desc)
    return p


def _cuda_ok() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


# ----------------------------------------------------------- batched ops ---


def _require(cond: bool, msg: str):
    if not cond:
        raise ShapeMismatch(msg)


def attention(q, k, v, segments: int = 1, softmax_scale: float = 1.0, stream=None,
              tree: tuple = (), fuse_level: int = 0):
    """Fused safe-softmax -> GEMM attention over every (b, h, query) row.

    q: [B,H,Sq,D], k/v: [B,H,Skv,D] (float32 or bfloat16, contiguous, cuda).
    Returns (d1 = m [B,H,Sq] f32, d2 = l [B,H,Sq] f32, d3 = O [B,H,Sq,D]).
    fuse_level k >= 1 with tree = TreeConfig.levels[1..K]: run_fused
    (simulator.cpp:485-559), each level-1 segment one on-chip KV tile.
    """
    import torch

    _require(q.dim() == 4 and k.shape == v.shape and k.dim() == 4, "q/k/v must be 4-D")
    B, H, Sq, D = q.shape
    _require(k.shape[0] == B and k.shape[1] == H and k.shape[3] == D, "k/v shape mismatch")
    _require(q.dtype == k.dtype == v.dtype, "q/k/v dtype mismatch")
    dt = {torch.float32: "f32", torch.bfloat16: "bf16"}.get(q.dtype)
    if dt is None:
        raise UnsupportedPattern(f"attention: dtype {q.dtype}")
    p = plan(Desc(N.RF_PATTERN_ATTENTION, dt, rows=Sq, len=k.shape[2], free_len=D, batch=B,
                  heads=H, segments=segments, softmax_scale=softmax_scale,
                  device=q.device.index or 0, fuse_level=fuse_level, tree=tuple(tree)), stream)
    m = torch.empty((B, H, Sq), dtype=torch.float32, device=q.device)
    l = torch.empty_like(m)
    o = torch.empty_like(q)
    p.run([q.contiguous(), k.contiguous(), v.contiguous()], [m, l, o], stream)
    return m, l, o


def safe_softmax(x, stream=None, tree: tuple = (), fuse_level: int = 0):
    """d1 = max, d2 = sum exp(x - d1) per row of x [rows, n] (float32).
    fuse_level k >= 1 with tree = TreeConfig.levels[1..K]: run_fused."""
    import torch

    _require(x.dim() == 2 and x.dtype == torch.float32, "x must be float32 [rows, n]")
    p = plan(Desc(N.RF_PATTERN_SAFE_SOFTMAX, "f32", rows=x.shape[0], len=x.shape[1],
                  device=x.device.index or 0, fuse_level=fuse_level, tree=tuple(tree)), stream)
    d1 = torch.empty(x.shape[0], dtype=torch.float32, device=x.device)
    d2 = torch.empty_like(d1)
    p.run([x.contiguous()], [d1, d2], stream)
    return d1, d2


def quant_gemm_plan(m: int, k: int, n: int, fmax: float = 448.0, device: int = 0,
                    stream=None) -> Plan:
    return plan(Desc(N.RF_PATTERN_QUANT_GEMM_E4M3, "bf16", rows=m, len=k, free_len=n,
                     fmax=fmax, device=device), stream)


def quant_gemm(a, w_packed, fmax: float = 448.0, stream=None, check_domain: bool = True):
    """Per-token absmax -> e4m3 quantise -> GEMM. a: [M,K] bf16; w_packed from
    Plan.pack_weight. Returns (d1 = amax [M] f32, d2 = C [M,N] f32).
    check_domain: raise DomainError, as the reference does at finalize
    (simulator.cpp:611-621), when a row's absmax is 0 (synchronises the
    stream; pass False inside graphs / timed loops and call
    Plan.check_domain later)."""
    import torch

    _require(a.dim() == 2 and a.dtype == torch.bfloat16, "a must be bfloat16 [M, K]")
    M, K = a.shape
    _require(w_packed.dim() == 2 and w_packed.shape[1] == K, "w_packed must be [N, K]")
    Nn = w_packed.shape[0]
    p = quant_gemm_plan(M, K, Nn, fmax, a.device.index or 0, stream)
    amax = torch.empty(M, dtype=torch.float32, device=a.device)
    c = torch.empty((M, Nn), dtype=torch.float32, device=a.device)
    p.run([a.contiguous(), w_packed], [amax, c], stream)
    if check_domain:
        p.check_domain(stream)
    return amax, c


def rmsnorm_gemm_plan(t: int, k: int, n: int, eps: float = 1e-6, device: int = 0,
                      stream=None) -> Plan:
    return plan(Desc(N.RF_PATTERN_RMSNORM_GEMM, "bf16", rows=t, len=k, free_len=n, eps=eps,
                     device=device), stream)


def rmsnorm_gemm(x, w_packed, eps: float = 1e-6, stream=None):
    """RMSNorm statistics fused with the following GEMM. x: [T,K] bf16;
    w_packed from Plan.pack_weight (g folded). Returns (d1 = sum x^2 [T] f32,
    d2 = Y [T,N] bf16)."""
    import torch

    _require(x.dim() == 2 and x.dtype == torch.bfloat16, "x must be bfloat16 [T, K]")
    T, K = x.shape
    _require(w_packed.dim() == 2 and w_packed.shape[1] == K, "w_packed must be [N, K]")
    Nn = w_packed.shape[0]
    p = rmsnorm_gemm_plan(T, K, Nn, eps, x.device.index or 0, stream)
    ss = torch.empty(T, dtype=torch.float32, device=x.device)
    y = torch.empty((T, Nn), dtype=torch.bfloat16, device=x.device)
    p.run([x.contiguous(), w_packed], [ss, y], stream)
    return ss, y


def layernorm_gemm_plan(t: int, k: int, n: int, eps: float = 1e-5, device: int = 0,
                        stream=None) -> Plan:
    return plan(Desc(N.RF_PATTERN_LAYERNORM_GEMM, "bf16", rows=t, len=k, free_len=n, eps=eps,
                     device=device), stream)


def layernorm_gemm(x, w_packed, n: int, eps: float = 1e-5, with_d4: bool = True, stream=None):
    """LayerNorm statistics fused with the following GEMM (the 4-reduction
    cascade d1 = sum x, d2 = sum x^2, d3 = (x*g) @ W / sigma,
    d4 = mean * colsum(g*W) / sigma; normalised output = d3 - d4).
    x: [T,K] bf16; w_packed from Plan.pack_weight (raw bytes). Returns
    (d1 [T] f32, d2 [T] f32, d3 [T,N] bf16, d4 [T,N] bf16 or None)."""
    import torch

    _require(x.dim() == 2 and x.dtype == torch.bfloat16, "x must be bfloat16 [T, K]")
    T, K = x.shape
    p = layernorm_gemm_plan(T, K, n, eps, x.device.index or 0, stream)
    _require(w_packed.numel() * w_packed.element_size() == N.lib().rf_packed_bytes(p._h),
             "w_packed size does not match the plan")
    d1 = torch.empty(T, dtype=torch.float32, device=x.device)
    d2 = torch.empty_like(d1)
    d3 = torch.empty((T, n), dtype=torch.bfloat16, device=x.device)
    d4 = torch.empty_like(d3) if with_d4 else None
    p.run([x.contiguous(), w_packed], [d1, d2, d3, d4], stream)
    return d1, d2, d3, d4


def moe_routing(logits, k: int, stream=None):
    """MoE routing cascade per token row: d1 = max, d2 = sum exp(s - d1) and the
    top-k experts (ties to the lowest index). logits: [rows, experts] float32.
    Returns (d1 [rows], d2 [rows], values [rows, k] f32, indices [rows, k] int32,
    1-based like the reference's OutputVal.topk; 0 marks an empty slot)."""
    import torch

    _require(logits.dim() == 2 and logits.dtype == torch.float32, "logits must be float32 [rows, experts]")
    rows, experts = logits.shape
    p = plan(Desc(N.RF_PATTERN_MOE_ROUTING, "f32", rows=rows, len=experts, free_len=k,
                  device=logits.device.index or 0), stream)
    d1 = torch.empty(rows, dtype=torch.float32, device=logits.device)
    d2 = torch.empty_like(d1)
    rec = torch.empty(rows, k, 2, dtype=torch.int32, device=logits.device)
    p.run([logits.contiguous()], [d1, d2, rec], stream)
    return d1, d2, rec[..., 0].view(torch.float32), rec[..., 1]


def moe_router_plan(tokens: int, hd: int, experts: int, k: int, device: int = 0,
                    stream=None) -> Plan:
    return plan(Desc(N.RF_PATTERN_MOE_ROUTER, "bf16", rows=tokens, len=experts, free_len=k,
                     producer_len=hd, device=device), stream)


def moe_router(x, w_packed, k: int, with_scores: bool = False, stream=None):
    """MoE router: scores s = x W (router GEMM on tcgen05) and the routing
    cascade over them (d1 = max s, d2 = sum exp(s - d1), top-k experts, ties to
    the lowest index). x: [tokens, hd] bf16; w_packed: Plan.pack_weight of
    w [hd, experts] float32. Returns (d1, d2, values, indices[, scores])."""
    import torch

    _require(x.dim() == 2 and x.dtype == torch.bfloat16, "x must be bfloat16 [tokens, hd]")
    tokens, hd = x.shape
    _require(w_packed.dim() == 2 and w_packed.shape[1] == hd, "w_packed must be [experts, hd]")
    experts = w_packed.shape[0]
    p = moe_router_plan(tokens, hd, experts, k, x.device.index or 0, stream)
    d1 = torch.empty(tokens, dtype=torch.float32, device=x.device)
    d2 = torch.empty_like(d1)
    rec = torch.empty(tokens, k, 2, dtype=torch.int32, device=x.device)
    sc = torch.empty(tokens, experts, dtype=torch.float32, device=x.device) if with_scores else None
    p.run([x.contiguous(), w_packed], [d1, d2, rec, sc], stream)
    out = (d1, d2, rec[..., 0].view(torch.float32), rec[..., 1])
    return out + (sc,) if with_scores else out


def mla_decode(q, cache, segments: int = 1, softmax_scale: float = 1.0, stream=None):
    """MLA decode (absorbed multi-latent attention): the attention cascade with
    P = scale * q . cache^T over the 576-wide cache rows [c_kv | k_rope] and
    V = c_kv (their first 512 columns). q: [B, 128, 576] bf16, cache:
    [B, Skv, 576] bf16. Returns (m [B,128], l [B,128], O [B,128,512] bf16)."""
    import torch

    _require(q.dim() == 3 and cache.dim() == 3 and q.dtype == cache.dtype == torch.bfloat16,
             "q [B,128,576] and cache [B,Skv,576] must be bfloat16")
    B, hn, dqk = q.shape
    _require(cache.shape[0] == B and cache.shape[2] == dqk, "cache must be [B, Skv, q.shape[2]]")
    skv = cache.shape[1]
    p = plan(Desc(N.RF_PATTERN_MLA_DECODE, "bf16", rows=1, len=skv, free_len=512, batch=B, heads=hn,
                  segments=segments, softmax_scale=softmax_scale, producer_len=dqk,
                  device=q.device.index or 0), stream)
    m = torch.empty(B, hn, dtype=torch.float32, device=q.device)
    l = torch.empty_like(m)
    o = torch.empty(B, hn, 512, dtype=torch.bfloat16, device=q.device)
    p.run([q.contiguous(), cache.contiguous()], [m, l, o], stream)
    return m, l, o


def _rows_f32(name, *ts):
    import torch

    for t in ts:
        _require(t.dtype == torch.float32 and t.is_cuda, f"{name}: float32 cuda tensors")
    return [t.contiguous() for t in ts]


def variance(x, segments: int = 1, stream=None, tree: tuple = (), fuse_level: int = 0):
    """make_variance per row: d1 = sum x, d2 = sum x^2. x: [rows, n] float32.
    fuse_level k >= 1 with tree = TreeConfig.levels[1..K]: run_fused."""
    import torch

    _require(x.dim() == 2, "x must be [rows, n]")
    (x,) = _rows_f32("variance", x)
    p = plan(Desc(N.RF_PATTERN_VARIANCE, "f32", rows=x.shape[0], len=x.shape[1],
                  segments=segments, device=x.device.index or 0, fuse_level=fuse_level,
                  tree=tuple(tree)), stream)
    d1 = torch.empty(x.shape[0], dtype=torch.float32, device=x.device)
    d2 = torch.empty_like(d1)
    p.run([x], [d1, d2], stream)
    return d1, d2


def sum_sum(x1, x2, offset: float = 10.0, eps: float = 1e-12, segments: int = 1, stream=None,
            tree: tuple = (), fuse_level: int = 0):
    """make_sum_sum per row: d1 = sum x1^2, d2 = sum x1 x2 / sqrt(max(d1 - offset, eps)).
    fuse_level k >= 1 with tree = TreeConfig.levels[1..K]: run_fused."""
    import torch

    _require(x1.dim() == 2 and x1.shape == x2.shape, "x1, x2 must be [rows, n]")
    x1, x2 = _rows_f32("sum_sum", x1, x2)
    p = plan(Desc(N.RF_PATTERN_SUM_SUM, "f32", rows=x1.shape[0], len=x1.shape[1], eps=eps,
                  offset=offset, segments=segments, device=x1.device.index or 0,
                  fuse_level=fuse_level, tree=tuple(tree)), stream)
    d1 = torch.empty(x1.shape[0], dtype=torch.float32, device=x1.device)
    d2 = torch.empty_like(d1)
    p.run([x1, x2], [d1, d2], stream)
    return d1, d2


def moments(mass, pos, segments: int = 1, stream=None):
    """moment_of_inertia per row: d1 = sum m, d2[f] = sum m p_f, d3[f] = sum m p_f^2.
    mass: [rows, n], pos: [rows, n, F] (F <= 8) float32."""
    import torch

    _require(mass.dim() == 2 and pos.dim() == 3 and pos.shape[:2] == mass.shape,
             "mass [rows, n], pos [rows, n, F]")
    mass, pos = _rows_f32("moments", mass, pos)
    rows, n, F = pos.shape
    p = plan(Desc(N.RF_PATTERN_MOMENTS, "f32", rows=rows, len=n, free_len=F, segments=segments,
                  device=mass.device.index or 0), stream)
    d1 = torch.empty(rows, dtype=torch.float32, device=mass.device)
    d2 = torch.empty(rows, F, dtype=torch.float32, device=mass.device)
    d3 = torch.empty_like(d2)
    p.run([mass, pos], [d1, d2, d3], stream)
    return d1, d2, d3
