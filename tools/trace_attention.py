"""Timeline of one CTA of the tcgen05 attention kernel (cfg2 shape, full GPU
load) from the RF_ATTN_TRACE build in librf_probe.so. Run under gpurun.
Prints per-tile cycle stamps relative to the first S ready:
  softmax k: S ready / max done / P stored / P released,  MMA: PV0, S0', PV1 issue."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
h = ctypes.CDLL(os.path.join(ROOT, "paper_2603_10026_b200", os.environ.get("RF_PROBE_LIB", "librf_probe.so")))
h.rf_probe_attn_trace.restype = ctypes.c_int
B, H, S, D = 8, 32, 4096, 128
q = ((torch.rand(B, H, S, D, device="cuda") * 2 - 1) / D ** 0.5).bfloat16()
k = (torch.rand(B, H, S, D, device="cuda") * 2 - 1).bfloat16()
v = (torch.rand(B, H, S, D, device="cuda") * 2 - 1).bfloat16()
o = torch.empty_like(q)
m = torch.empty(B, H, S, device="cuda")
l = torch.empty_like(m)
buf = (ctypes.c_longlong * 4096)()
for _ in range(3):
    rc = h.rf_probe_attn_trace(*(ctypes.c_void_p(t.data_ptr()) for t in (q, k, v, o, m, l)),
                               ctypes.c_longlong(B * H), ctypes.c_longlong(S), buf)
assert rc == 0, rc
t = list(buf)
t0 = t[0]
n = S // 128
print("tile | sm0: Srdy maxd Pst Prel | sm1: Srdy maxd Pst Prel | mma: PV0 S0' PV1")
for i in range(n):
    a = [t[4 * i + j] - t0 for j in (0, 3, 1, 2)]
    b = [t[512 + 4 * i + j] - t0 for j in (0, 3, 1, 2)]
    c = [t[1024 + 4 * i + j] - t0 for j in range(3)]
    print(f"{i:3d} | {a} | {b} | {c}")
per = [(t[4 * (i + 1)] - t[4 * i]) for i in range(n - 1)]
print("cycles per tile (softmax0 S-ready to S-ready):", sorted(per)[len(per) // 2])
sm = [t[4 * i + 2] - t[4 * i] for i in range(n)]
print("softmax0 busy per tile (S ready -> P released):", sorted(sm)[len(sm) // 2])
# units of CTA 0: start (S_0 ready) / end (last P released), cycles relative to unit 0's start
us = [(t[2048 + 2 * u], t[2048 + 2 * u + 1]) for u in range(32) if t[2048 + 2 * u]]
print("CTA 0 units: duration, gap to the next unit's first S (cycles)")
for u, (a, b) in enumerate(us):
    gap = us[u + 1][0] - b if u + 1 < len(us) else 0
    print(f"  unit {u:2d}: start {a - us[0][0]:9d} dur {b - a:7d} gap {gap:6d}")

# ---- the 2-SM (CTA pair) kernel: first cluster ----
h.rf_probe_attn2_trace.restype = ctypes.c_int
for _ in range(3):
    rc = h.rf_probe_attn2_trace(*(ctypes.c_void_p(t.data_ptr()) for t in (q, k, v, o, m, l)),
                                ctypes.c_longlong(B * H), ctypes.c_longlong(S), buf)
assert rc == 0, rc
t = list(buf)
t0 = t[2048]
print("2-SM: tile | S issue, PV issue | CTA0 Srdy maxd Prel | CTA1 Srdy maxd Prel | peer P relay")
for i in range(n):
    mm = [t[2048 + 4 * i + j] - t0 for j in range(2)]
    a = [t[4 * i + j] - t0 for j in range(3)]
    b = [t[1024 + 4 * i + j] - t0 for j in range(3)]
    print(f"{i:3d} | {mm} | {a} | {b} | {t[3072 + i] - t0}")
per = [(t[4 * (i + 1)] - t[4 * i]) for i in range(n - 1)]
print("2-SM cycles per tile (CTA0 S-ready to S-ready):", sorted(per)[len(per) // 2])
sm = [t[4 * i + 2] - t[4 * i] for i in range(n)]
print("2-SM softmax busy per tile:", sorted(sm)[len(sm) // 2])
