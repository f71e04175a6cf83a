"""The smallest parity shape of every librf_cuda kernel, run once each, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

Every case also checks its result loosely against a torch fp32 reference so
a sanitizer run cannot pass on garbage. Prints one line per case.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_10026_b200 import (attention, layernorm_gemm, layernorm_gemm_plan, mla_decode,  # noqa: E402
                                   moe_router, moe_router_plan, moe_routing, moments, quant_gemm,
                                   quant_gemm_plan, rmsnorm_gemm, rmsnorm_gemm_plan, safe_softmax,
                                   sum_sum, variance)


def _attn_ref(q, k, v, scale=1.0):
    s = scale * q.float() @ k.float().transpose(-1, -2)
    return torch.softmax(s, -1) @ v.float()


def _close(got, want, tol):
    e = ((got.float() - want.float()).abs().max() / (1 + want.float().abs().max())).item()
    assert e < tol, e
    return e


def attn_f32():
    q = (torch.rand(1, 1, 64, 64, device="cuda") * 2 - 1) / 8
    k, v = (torch.rand(2, 1, 1, 256, 64, device="cuda") * 2 - 1)
    _, _, o = attention(q, k, v, segments=2)
    return _close(o, _attn_ref(q, k, v), 1e-4)


def attn_tf32():
    """fp32 on tcgen05 (3xTF32), a 4-CTA cluster with the in-cluster fold."""
    q = (torch.rand(1, 1, 128, 64, device="cuda") * 2 - 1) / 8
    k, v = (torch.rand(2, 1, 1, 512, 64, device="cuda") * 2 - 1)
    _, _, o = attention(q, k, v, segments=4)
    return _close(o, _attn_ref(q, k, v), 1e-5)


def attn_bf16():
    q = ((torch.rand(1, 2, 256, 128, device="cuda") * 2 - 1) / 11).bfloat16()
    k, v = (torch.rand(2, 1, 2, 256, 128, device="cuda") * 2 - 1).bfloat16()
    _, _, o = attention(q, k, v)
    return _close(o, _attn_ref(q, k, v), 2e-2)


def decode():
    q = ((torch.rand(1, 2, 1, 128, device="cuda") * 2 - 1) / 11).bfloat16()
    k, v = (torch.rand(2, 1, 2, 2048, 128, device="cuda") * 2 - 1).bfloat16()
    _, _, o = attention(q, k, v, segments=2)
    return _close(o, _attn_ref(q, k, v), 2e-2)


def softmax():
    x = torch.randn(8, 1000, device="cuda")
    m, l = safe_softmax(x)
    return _close(l, torch.exp(x - x.max(1, keepdim=True).values).sum(1), 1e-5)


def _w(k, n):
    return torch.rand(k, n, device="cuda") * 2 - 1


def quant(m=128):
    K, N = 256, 512
    p = quant_gemm_plan(m, K, N)
    w = _w(K, N)
    wp = p.pack_weight(w)
    a = (torch.rand(m, K, device="cuda") * 4 - 2).bfloat16()
    d1, c = quant_gemm(a, wp)
    ref = (448.0 * a.float() / d1[:, None]) @ wp.view(torch.float8_e4m3fn).float().t()
    return _close(c, ref, 8e-2)


def quant_2sm():
    return quant(256)


def rms(m=128):
    K, N = 128, 256
    p = rmsnorm_gemm_plan(m, K, N)
    w, g = _w(K, N), torch.rand(K, device="cuda")
    wp = p.pack_weight(w, g)
    x = (torch.rand(m, K, device="cuda") * 2 - 1).bfloat16()
    d1, y = rmsnorm_gemm(x, wp)
    ref = (x.float() / torch.sqrt(d1[:, None] / K + 1e-6)) @ wp.float().t()
    return _close(y, ref, 2e-2)


def rms_2sm():
    return rms(256)


def layernorm():
    M, K, N = 256, 128, 256
    p = layernorm_gemm_plan(M, K, N)
    w, g = _w(K, N), torch.rand(K, device="cuda")
    wp = p.pack_weight(w, g)
    x = (torch.rand(M, K, device="cuda") * 2 - 1).bfloat16()
    d1, d2, d3, d4 = layernorm_gemm(x, wp, N)
    mean = d1 / K
    sig = torch.sqrt(d2 / K - mean * mean + 1e-5)
    wt = wp[:2 * N * K].view(torch.bfloat16).view(N, K).float()
    ref = ((x.float() - mean[:, None]) / sig[:, None]) @ wt.t()
    return _close(d3.float() - d4.float(), ref, 2e-2)


def routing():
    s = torch.randn(64, 128, device="cuda")
    d1, d2, vals, idx = moe_routing(s, 8)
    ref = torch.topk(s, 8, dim=1)
    assert torch.equal(idx.long() - 1, ref.indices)
    return 0.0


def router():
    """2 row tiles x 2 K splits: the split CTAs exchange partials through L2 (arrival counter)."""
    T, hd, E = 256, 1024, 64
    p = moe_router_plan(T, hd, E, 4)
    w = _w(hd, E) / hd ** 0.5
    wp = p.pack_weight(w)
    x = (torch.rand(T, hd, device="cuda") * 2 - 1).bfloat16()
    d1, d2, vals, idx, sc = moe_router(x, wp, 4, with_scores=True)
    return _close(sc, x.float() @ wp.float().t(), 1e-4)


def mla():
    """One batch over 4 CTA pairs: the in-kernel fold of the cut batch (arrival counters)."""
    q = ((torch.rand(1, 128, 576, device="cuda") * 2 - 1)).bfloat16()
    kv = (torch.rand(1, 512, 576, device="cuda") * 2 - 1).bfloat16()
    m, l, o = mla_decode(q, kv, segments=2, softmax_scale=576 ** -0.5)
    ref = _attn_ref(q, kv, kv[..., :512], 576 ** -0.5)
    return _close(o, ref, 2e-2)


def rowstats():
    x = torch.randn(16, 5000, device="cuda")
    d1, d2 = variance(x)
    _close(d2, (x.double() ** 2).sum(1), 1e-5)
    d1, d2 = sum_sum(x, x)
    mass, pos = torch.rand(4, 300, device="cuda"), torch.randn(4, 300, 3, device="cuda")
    m1, m2, m3 = moments(mass, pos)
    return _close(m2, (mass[..., None] * pos).sum(1), 1e-4)


CASES = [attn_f32, attn_tf32, attn_bf16, decode, softmax, quant, quant_2sm, rms, rms_2sm, layernorm, routing, router,
         mla, rowstats]


def main():
    want = set(sys.argv[1:])
    for c in CASES:
        if want and c.__name__ not in want:
            continue
        e = c()
        torch.cuda.synchronize()
        print(f"case {c.__name__}: ok (err {e:.2e})", flush=True)


if __name__ == "__main__":
    main()
