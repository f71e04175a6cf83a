"""Effective SM clock during the cfg2 attention kernel (CTA 0's clock64 vs
%globaltimer per launch, RF_ATTN_TRACE build in librf_probe.so) over n
back-to-back launches: shows the power cap's clock, which nvidia-smi's
~100 ms counters smear. Run under gpurun."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
h = ctypes.CDLL(os.path.join(ROOT, "paper_2603_10026_b200", "librf_probe.so"))
B, H, S, D = 8, 32, 4096, 128
n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
q = ((torch.rand(B, H, S, D, device="cuda") * 2 - 1) / D ** 0.5).bfloat16()
k = (torch.rand(B, H, S, D, device="cuda") * 2 - 1).bfloat16()
v = (torch.rand(B, H, S, D, device="cuda") * 2 - 1).bfloat16()
o = torch.empty_like(q)
m = torch.empty(B, H, S, device="cuda")
l = torch.empty_like(m)
out = (ctypes.c_double * 64)()
rc = h.rf_probe_attn_clock(*(ctypes.c_void_p(t.data_ptr()) for t in (q, k, v, o, m, l)),
                           ctypes.c_longlong(B * H), ctypes.c_longlong(S), ctypes.c_int(n), out)
assert rc == 0, rc
mhz = list(out)[:min(n, 64)]
print("launch: effective MHz of CTA 0")
for i in range(0, len(mhz), 5):
    print(i, " ".join(f"{x:7.1f}" for x in mhz[i:i + 5]))
