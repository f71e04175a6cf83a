"""Timeline of the MoE router (cfg7 shape, L2 flushed before the call) from a
build with -DRF_ROUTER_TRACE. Usage (GPU box):
  python tools/trace_router.py <traced librf_cuda.so>
Build: nvcc ... -DRF_ROUTER_TRACE (see the librf_cuda Makefile flags) into a
separate .so. Per CTA: start / warp 0's partials summed / first K tile landed / last K tile
landed / accumulator ready / partial slices written / row tile's counter met /
slice routed."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2603_10026_b200._native as N

N.LIB_PATH = os.path.abspath(sys.argv[1])
from paper_2603_10026_b200 import moe_router, moe_router_plan  # noqa: E402

lib = ctypes.CDLL(N.LIB_PATH)
T, HD, EN, K = 2048, 4096, 128, 8
x = (torch.rand(T, HD, device="cuda") * 2 - 1).bfloat16()
w = (torch.rand(HD, EN) * 2 - 1) / HD ** 0.5
wp = moe_router_plan(T, HD, EN, K).pack_weight(w.cuda())
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.fill_(1)
    torch.cuda.synchronize()
    moe_router(x, wp, K)
torch.cuda.synchronize()
g = (ctypes.c_ulonglong * (8 * 1024))()
r = (ctypes.c_ulonglong * 3072)()
assert lib.rf_router_trace_read(g, r) == 0
g, r = list(g), list(r)
n = 128
t0 = min(g[8 * i] for i in range(n) if g[8 * i])
q = lambda v: [round((x - t0) / 1000, 2) for x in (v[0], v[len(v) // 4], v[len(v) // 2], v[3 * len(v) // 4], v[-1])]  # noqa: E731
for j, name in enumerate(["start", "summed (warp 0)", "tile0 landed", "last tile landed", "acc ready",
                          "partials written", "counter met", "routed"]):
    v = sorted(g[8 * i + j] for i in range(n) if g[8 * i + j])
    print(f"gemm {name:16s} (min/q1/med/q3/max us):", q(v))
