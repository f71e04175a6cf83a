"""clock64 timeline of one CTA pair leader of the 2-SM FP8 quant GEMM (cfg4,
full-GPU load) from the RF_QNT_TRACE build (librf_qtrace.so). Run under gpurun.
Per K step t: MMA warp W landed / A8 ready (issue), quantiser A landed /
A8 slot free / A8 written, TMA abf slot free / W slot free."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
h = ctypes.CDLL(os.path.join(ROOT, "paper_2603_10026_b200", "librf_qtrace.so"))
sys.path.insert(0, ROOT)
from paper_2603_10026_b200 import quant_gemm_plan  # noqa: E402

M = N = K = 8192
p = quant_gemm_plan(M, K, N)
wp = p.pack_weight(torch.rand(K, N, device="cuda") * 2 - 1)
a = (torch.rand(M, K, device="cuda") * 4 - 2).bfloat16()
d1 = torch.empty(M, device="cuda")
c = torch.empty(M, N, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
buf = (ctypes.c_longlong * 8192)()
for cta in [int(x) for x in (sys.argv[1:] or ["0", "300", "700"])]:
    for _ in range(2):
        rc = h.rf_probe_qnt_trace(*(ctypes.c_void_p(t.data_ptr()) for t in (a, wp, d1, c, flag)),
                                  ctypes.c_longlong(M), ctypes.c_longlong(N), ctypes.c_longlong(K),
                                  ctypes.c_int(cta), buf)
        assert rc == 0, rc
    full = list(buf)
    tr = [full[:4096], full[4096:]]  # leader, peer
    # origin of each CTA: clock64 right after the pair's first cluster barrier
    # (event 7 slot 3); older builds without it fall back to the kernel start.
    org = [x[7 * 64 + 3] or x[7 * 64 + 2] for x in tr]
    print(f"== pair of CTA {cta} (times in cycles after the pair's first cluster barrier)")
    for rk, t in enumerate(tr):
        rel = lambda v, o=org[rk]: v - o if v else -1  # noqa: E731
        print(f"-- {'leader' if rk == 0 else 'peer'}: acc_full {rel(t[7 * 64])}, epilogue end {rel(t[7 * 64 + 1])}")
        print("  t |  W_land  A8_rdy |  A_land  A8_free  A8_done | abf_free  w_free")
        for i in range(64):
            ev = [rel(t[e * 64 + i]) for e in range(7)]
            if i < 6 or i % 8 == 0 or i > 60:
                print(f"{i:3d} | {ev[0]:7d} {ev[1]:7d} | {ev[2]:7d} {ev[3]:7d} {ev[4]:7d} | {ev[5]:7d} {ev[6]:7d}")
        qbusy = sorted(t[4 * 64 + i] - max(t[2 * 64 + i], t[3 * 64 + i]) for i in range(8, 63))
        print(f"  median quantiser busy per step (ready -> A8 written): {qbusy[len(qbusy) // 2]}")
    t = tr[0]
    issue = [t[64 + i] for i in range(64)]
    d = sorted(issue[i + 1] - issue[i] for i in range(8, 63))
    wait_a8 = sorted(t[64 + i] - t[i] for i in range(8, 63))
    peer_lag = sorted((tr[1][4 * 64 + i] - org[1]) - (tr[0][4 * 64 + i] - org[0]) for i in range(8, 63))
    print(f"  median cycles per K step (MMA issue to issue): {d[len(d) // 2]}")
    print(f"  median MMA wait for A8 after W landed: {wait_a8[len(wait_a8) // 2]}")
    print(f"  median peer A8_done minus leader A8_done: {peer_lag[len(peer_lag) // 2]}")
