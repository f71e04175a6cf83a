"""Timeline of the first and last CTA pair of mla_decode (cfg8 shape) from a
build with -DRF_MLA_TRACE. Usage (GPU box):
  python tools/trace_mla.py <traced librf_cuda.so> [noflush]
Columns per tile, microseconds from the kernel's first stamp:
  K0 / K8: first / last K stage load issued, V0: first V stage issued,
  S: S MMAs issued (all K stages landed), Pin: P ready (MMA warp), PV: P V issued,
  Srdy: softmax sees S, Prel: softmax released P."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2603_10026_b200._native as N

N.LIB_PATH = os.path.abspath(sys.argv[1])
from paper_2603_10026_b200 import mla_decode  # noqa: E402

lib = ctypes.CDLL(N.LIB_PATH)
B, SKV = 32, 4096
q = (torch.rand(B, 128, 576, device="cuda") * 2 - 1).bfloat16()
kv = (torch.rand(B, SKV, 576, device="cuda") * 2 - 1).bfloat16()
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
NOFLUSH = "noflush" in sys.argv[2:]  # the bench does not flush for cfg8 (160 MB of inputs > L2)
for _ in range(3):
    if not NOFLUSH:
        flush.fill_(1)
    mla_decode(q, kv, segments=4, softmax_scale=576 ** -0.5)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (2 * 2 * 64 * 8))()
assert lib.rf_mla_trace_read(buf) == 0
t = list(buf)


def at(c, x, i, j):
    return t[((c * 2 + x) * 64 + i) * 8 + j]


t0 = min(at(c, x, 63, 0) for c in range(2) for x in range(2))
us = lambda v: round((v - t0) / 1000, 2) if v else None  # noqa: E731
for c in range(2):
    print(f"cluster {'first' if c == 0 else 'last'}: start {us(at(c, 0, 63, 0))} / {us(at(c, 1, 63, 0))}"
          f"  end {us(at(c, 0, 63, 1))} / {us(at(c, 1, 63, 1))}  setup done {us(at(c, 0, 63, 2))}"
          f"  (barriers {us(at(c, 0, 63, 6))}, TMEM allocated {us(at(c, 0, 63, 7))})"
          f"  first Q issue {us(at(c, 0, 63, 3))}  (TMA warp: elected {us(at(c, 0, 63, 4))},"
          f" tensor maps prefetched {us(at(c, 0, 63, 5))})")
    print(" tile |   K0    K8    V0 |    S    Pin    PV | Srdy0  Prel0 | Srdy1  Prel1")
    for i in range(16):
        print(f" {i:4d} | {us(at(c, 0, i, 0))} {us(at(c, 0, i, 7))} {us(at(c, 0, i, 1))} | "
              f"{us(at(c, 0, i, 2))} {us(at(c, 0, i, 3))} {us(at(c, 0, i, 4))} | "
              f"{us(at(c, 0, i, 5))} {us(at(c, 0, i, 6))} | {us(at(c, 1, i, 5))} {us(at(c, 1, i, 6))}")

fb = (ctypes.c_ulonglong * (1024 * 3))()
if hasattr(lib, "rf_mla_fold_trace_read") and lib.rf_mla_fold_trace_read(fb) == 0:
    f = list(fb)
    n = 148  # in-kernel fold: one entry per decode CTA (y * 2 + x) that folded a cut batch
    st = sorted(us(f[3 * i]) for i in range(n) if f[3 * i])
    go = sorted(us(f[3 * i + 1]) for i in range(n) if f[3 * i + 1])
    en = sorted(us(f[3 * i + 2]) for i in range(n) if f[3 * i + 2])
    q = lambda v: [v[0], v[len(v) // 4], v[len(v) // 2], v[3 * len(v) // 4], v[-1]] if v else None  # noqa: E731
    print("fold (in-kernel): started (min/q1/med/q3/max)", q(st))
    print("                  counter met", q(go))
    print("                  done       ", q(en))

eb = (ctypes.c_ulonglong * 256)()
if hasattr(lib, "rf_mla_end_trace_read") and lib.rf_mla_end_trace_read(eb) == 0:
    e = sorted(us(v) for v in list(eb)[:148] if v)
    print("decode CTAs end (min/q1/med/q3/max):", [e[0], e[len(e) // 4], e[len(e) // 2], e[3 * len(e) // 4], e[-1]])
