"""globaltimer timeline of the fp32 tcgen05 attention kernel (cfg1 shape,
RF_TF32_TRACE build librf_tf32trace.so), with the bench's L2 flush before the
traced launch. Events per CTA (ns after the earliest CTA start): start, Q split,
K/V split, S done, softmax done, PV done, partial stored, cluster barrier, fold
end. Run under gpurun."""
import ctypes
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
h = ctypes.CDLL(os.path.join(ROOT, "paper_2603_10026_b200", "librf_tf32trace.so"))
S, D, NS = 1024, 64, 8
q = ((torch.rand(S, D, device="cuda") * 2 - 1) / 8).contiguous()
k = torch.rand(S, D, device="cuda") * 2 - 1
v = torch.rand(S, D, device="cuda") * 2 - 1
o = torch.empty(S, D, device="cuda")
m = torch.empty(S, device="cuda")
l = torch.empty(S, device="cuda")
pm = torch.empty(NS, S, device="cuda")
pl = torch.empty(NS, S, device="cuda")
po = torch.empty(NS, S, D, device="cuda")
l2 = torch.cuda.get_device_properties(0).L2_cache_size
flush = torch.empty(2 * l2 // 4, device="cuda")
buf = (ctypes.c_ulonglong * (512 * 16))()
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
for it in range(3):
    flush.fill_(float(it))
    torch.cuda.synchronize()
    rc = h.rf_probe_tf32_trace(P(q), P(k), P(v), P(o), P(m), P(l), P(pm), P(pl), P(po), ctypes.c_longlong(S),
                               ctypes.c_longlong(S), ctypes.c_int(NS), ctypes.c_float(1.0), buf)
    assert rc == 0, rc
t = [list(buf[i * 16:(i + 1) * 16]) for i in range(64)]
t0 = min(x[0] for x in t)
names = ["start", "Q split", "K/V split", "S done", "softmax", "PV done", "stored", "cluster bar", "fold end"]
print("event        " + "".join(f"{n:>12s}" for n in names))
for label, f in [("min", min), ("median", lambda xs: sorted(xs)[len(xs) // 2]), ("max", max)]:
    print(f"{label:12s} " + "".join(f"{f([x[e] - t0 for x in t]) / 1e3:12.2f}" for e in range(9)) + "  us")
