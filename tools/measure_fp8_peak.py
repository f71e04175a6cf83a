"""Measure the dense FP8 (e4m3) tensor peak on this B200 with cuBLASLt via
torch._scaled_mm — the roofline denominator for the quant GEMM (cfg4), which
MEASURED_PEAKS.json does not carry. Prints one JSON line."""
import json

import torch


def main():
    dev = torch.device("cuda", 0)
    best = {}
    for n in (8192, 16384):
        a = torch.randn(n, n, device=dev).to(torch.float8_e4m3fn)
        b = torch.randn(n, n, device=dev).to(torch.float8_e4m3fn).t()  # column-major B
        one = torch.ones((), device=dev)
        for _ in range(5):
            torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iters = 50 if n == 8192 else 10
        s.record()
        for _ in range(iters):
            torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / iters
        best[str(n)] = 2.0 * n ** 3 / (ms * 1e-3) / 1e12
    print(json.dumps({"fp8_e4m3_tflops_cublaslt": best,
                      "fp8_tflops": max(best.values()),
                      "method": "torch._scaled_mm e4m3 x e4m3 -> bf16, CUDA events, after warm-up"}))


if __name__ == "__main__":
    main()
