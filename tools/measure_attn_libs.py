"""Library reference points for the cfg2 attention shape (not product code).

Times, at BASELINE configs[1] (B8 H32 S4096 D128 bf16, non-causal), the
attention kernels that ship in this image as libraries: FlashAttention-4
(vllm.vllm_flash_attn.cute, CuTe DSL sm100) and torch SDPA's cuDNN backend.
These say how far the hand-written kernel is from the state of the art on the
same box; they are not part of the bench contract.

  python tools/measure_attn_libs.py > profiles/rNN_attn_libs.json
"""
import json
import sys

import torch


def timeit(fn, iters=30, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    B, H, S, D = 8, 32, 4096, 128
    flops = 4.0 * B * H * S * S * D
    out = {"shape": dict(B=B, H=H, S=S, D=D, causal=False), "results": {}}
    q = (torch.rand(B, S, H, D, device="cuda") * 2 - 1).bfloat16()
    k = (torch.rand(B, S, H, D, device="cuda") * 2 - 1).bfloat16()
    v = (torch.rand(B, S, H, D, device="cuda") * 2 - 1).bfloat16()
    try:
        from vllm.vllm_flash_attn.cute.interface import flash_attn_func

        fn = lambda: flash_attn_func(q, k, v, softmax_scale=1.0, causal=False)
        ms = timeit(fn)
        out["results"]["fa4_cute"] = {"ms": ms, "tflops": flops / ms / 1e9}
    except Exception as ex:  # noqa: BLE001
        out["results"]["fa4_cute"] = {"error": repr(ex)[:300]}
    try:
        from torch.nn.attention import SDPBackend, sdpa_kernel

        qt, kt, vt = (t.transpose(1, 2).contiguous() for t in (q, k, v))
        with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
            fn = lambda: torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, scale=1.0)
            ms = timeit(fn)
        out["results"]["cudnn_sdpa"] = {"ms": ms, "tflops": flops / ms / 1e9}
    except Exception as ex:  # noqa: BLE001
        out["results"]["cudnn_sdpa"] = {"error": repr(ex)[:300]}
    json.dump(out, sys.stdout)
    print()


if __name__ == "__main__":
    main()
