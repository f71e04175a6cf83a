"""TEST INFRASTRUCTURE: post-timing parity of bench.py's timed outputs.

bench.py calls `check(workload)` AFTER its timed region, on the very device
buffers the timed steps wrote: sampled rows of every benchmarked config are
recomputed by the oracle (tests/oracle.py over oracle/rf_oracle.c, pinned to
the reference's goldens) on the same rounded inputs, and compared with the
reference's own metric (compare_reports, proj/src/simulator.cpp:691-752:
|x-y| / (1 + max(|x|, |y|))). Nothing here is timed or shipped; it is the
checker, like tests/.

Samples (VERDICT r1 "next" 1): cfg1 all 1,024 rows; prefill 256 (b,h,q)
rows spread over b, h and q; decode 64 (b,h) rows; GEMM patterns 64 tokens
spread over every 128-row tile band, every output column (so every N group
and the N tail of the rasterisation); router every token; MLA 4 batches x 128
heads.
"""
from __future__ import annotations

import numpy as np

from . import oracle as O

TOL = {"f32": 1e-5, "bf16": 2e-2}  # north_star tolerances (compare_reports metric)


def _np(t):
    import torch

    return t.detach().to(torch.float64).cpu().numpy()


def _err(got, want):
    return float(O.scaled_max_err(np.asarray(got, dtype=np.float64).ravel(),
                                  np.asarray(want, dtype=np.float64).ravel())[0])


def _spread(n, k):
    """k indices spread over [0, n) (first and last included), deduplicated."""
    if k >= n:
        return np.arange(n)
    return np.unique(np.linspace(0, n - 1, k).round().astype(np.int64))


def _result(errs, rows, tol, oracle, extra=None):
    out = {"rows_checked": int(rows), "tol": tol,
           "max_scaled_err": {k: (None if v is None else float(f"{v:.3e}")) for k, v in errs.items()},
           "oracle": oracle}
    gated = [v for k, v in errs.items() if v is not None and not k.startswith("vs_")]
    out["pass"] = bool(all(v <= tol for v in gated))
    if extra:
        out.update(extra)
    return out


def attention_rows(q, k, v, m, l, o, bh_idx, q_idx, scale=1.0):
    """Oracle (m, l, O) of the sampled (bh, query) rows of [BH, S, D] tensors;
    returns the max scaled error of d1, d2, d3."""
    import torch

    B = q.shape[0] * q.shape[1]
    qf = q.reshape(B, q.shape[2], q.shape[3])
    kf = k.reshape(B, k.shape[2], k.shape[3])
    vf = v.reshape(B, v.shape[2], v.shape[3])
    mf, lf = m.reshape(B, -1), l.reshape(B, -1)
    of = o.reshape(B, o.shape[2], o.shape[3])
    e = {"d1": 0.0, "d2": 0.0, "d3": 0.0}
    rows = 0
    qi = torch.as_tensor(q_idx, device=q.device)
    for b in bh_idx:
        b = int(b)
        kk, vv = _np(kf[b]), _np(vf[b])
        qq = _np(qf[b].index_select(0, qi))
        p = scale * qq @ kk.T  # P = q K^T in fp64 (workloads.cpp:86-93)
        rm, rl, ro = O.attention_closed_form(p, vv[None])
        gm, gl = _np(mf[b].index_select(0, qi)), _np(lf[b].index_select(0, qi))
        go = _np(of[b].index_select(0, qi))
        e["d1"] = max(e["d1"], _err(gm, rm))
        e["d2"] = max(e["d2"], _err(gl, rl))
        e["d3"] = max(e["d3"], _err(go, ro))
        rows += len(q_idx)
    return e, rows


def check_attention(wl):
    q, k, v = wl.inputs
    m, l, o = wl.outputs
    cfg = wl.local
    tol = TOL[cfg["dtype"]]
    BH, Sq = q.shape[0] * q.shape[1], q.shape[2]
    if cfg["dtype"] == "f32":  # cfg1: every row
        bh, qi = np.arange(BH), np.arange(Sq)
    elif Sq == 1:  # decode: 64 (b,h) rows
        bh, qi = _spread(BH, 64), np.arange(1)
    else:  # prefill: 16 (b,h) pairs x 16 queries = 256 rows
        bh, qi = _spread(BH, 16), _spread(Sq, 16)
    e, rows = attention_rows(q, k, v, m, l, o, bh, qi)
    return _result(e, rows, tol, "closed form of make_attention's oracle (workloads.cpp:101-118), "
                                 "fp64 on the same rounded inputs")


def check_split_kv(wl, gather_rows):
    """Split-KV across ranks: the merged rows need the whole KV sequence of the
    sampled (b,h) rows; `gather_rows(t, idx)` all-gathers this rank's KV
    shard of those rows along the sequence axis (rank = slice order)."""
    import torch

    q, k, v = wl.inputs
    m, l, o = wl.outputs
    BH = q.shape[0] * q.shape[1]
    bh = _spread(BH, 64)
    idx = torch.as_tensor(bh, device=q.device)
    kf = k.reshape(BH, k.shape[2], k.shape[3]).index_select(0, idx)
    vf = v.reshape(BH, v.shape[2], v.shape[3]).index_select(0, idx)
    kg, vg = gather_rows(kf), gather_rows(vf)  # [64, Skv, D]
    qf = q.reshape(BH, 1, 1, q.shape[3]).index_select(0, idx)
    e, rows = attention_rows(qf, kg[:, None], vg[:, None],
                             m.reshape(BH, 1, 1).index_select(0, idx),
                             l.reshape(BH, 1, 1).index_select(0, idx),
                             o.reshape(BH, 1, 1, o.shape[3]).index_select(0, idx),
                             np.arange(len(bh)), np.arange(1))
    return _result(e, rows, TOL["bf16"], "closed form of make_attention's oracle over the "
                                         "all-gathered KV of the sampled rows (fp64)")


def _token_sample(M, n=64, band=128):
    """n tokens over every `band`-row tile band (first/last rows included)."""
    bands = max(1, M // band)
    per = max(1, n // min(bands, n))
    picks = []
    for b in _spread(bands, min(bands, n)):
        lo = b * band
        picks.extend(lo + _spread(min(band, M - lo), per))
    return np.unique(np.asarray(picks, dtype=np.int64))


def check_quant(wl):
    """cfg4: gated against the kernel's FP8 scheme restated in C
    (rfo_quant_gemm_e4m3: running absmax, power-of-two H', e4m3 RNE per K tile,
    in-loop ref'/ref correction) AND cross-checked with an independent torch
    float8_e4m3fn emulation of the same scheme; the deviations from the
    real-arithmetic reference (make_quant_gemm, no rounding) and from the
    true-running-amax e4m3 variant are reported, not gated."""
    import torch

    a, wp = wl.inputs
    d1, c = wl.outputs
    M = a.shape[0]
    rows = _token_sample(M)
    idx = torch.as_tensor(rows, device=a.device)
    A = _np(a.index_select(0, idx))
    W = wp.view(torch.float8_e4m3fn).to(torch.float64).t().contiguous().cpu().numpy()  # [K, N]
    fmax = wl.desc.fmax
    r1, rc = O.quant_gemm_e4m3(A, W, fmax, 128)
    g1, gc = _np(d1.index_select(0, idx)), _np(c.index_select(0, idx))
    t1, tc = O.quant_gemm_e4m3_torch(A, W, fmax, 128, pow2=True)
    _, uc = O.quant_gemm(A, W, fmax)
    _, ac = O.quant_gemm_e4m3_torch(A, W, fmax, 128, pow2=False)
    def rms(x, y):  # RMS relative error: the max scaled error of outputs that
        # differ by ~1 % of their norm is dominated by elements near zero
        return float(f"{np.sqrt(np.mean((x - y) ** 2) / np.mean(y ** 2)):.3e}")

    errs = {"d1": _err(g1, r1), "d2": _err(gc, rc), "vs_torch_emulation_d2": _err(gc, tc)}
    return _result(errs, len(rows), TOL["bf16"],
                   "rfo_quant_gemm_e4m3 (C restatement of the kernel's e4m3 scheme on the same "
                   "bf16 A / e4m3 W), cross-checked by an independent torch float8_e4m3fn "
                   "emulation; rms_rel_* = not gated",
                   {"oracle_pair_agreement_d2": float(f"{_err(rc, tc):.3e}"),
                    "rms_rel_vs_true_amax_e4m3": rms(gc, ac),
                    "rms_rel_vs_unrounded_reference": rms(gc, uc),
                    "rms_rel_true_amax_vs_unrounded_reference": rms(ac, uc)})


def check_rms(wl, ln=False):
    import torch

    a, wp = wl.inputs
    M, K = a.shape
    N = wl.local["N"]
    rows = _token_sample(M, band=256 if ln else 128)
    idx = torch.as_tensor(rows, device=a.device)
    X = _np(a.index_select(0, idx))
    Wt = wp[:2 * N * K].view(torch.bfloat16).view(N, K) if ln else wp
    W = Wt.to(torch.float64).t().contiguous().cpu().numpy()  # [K, N] = bf16(g * w)
    g = np.ones(K)
    eps = wl.desc.eps
    if ln:
        d1, d2, d3, d4 = wl.outputs
        r1, r2, r3, r4 = O.layernorm_gemm(X, g, W, eps)
        errs = {"d1": _err(_np(d1.index_select(0, idx)), r1),
                "d2": _err(_np(d2.index_select(0, idx)), r2),
                "d3": _err(_np(d3.index_select(0, idx)), r3),
                "d4": _err(_np(d4.index_select(0, idx)), r4)}
    else:
        d1, y = wl.outputs
        r1, ry = O.rmsnorm_gemm(X, g, W, eps)
        errs = {"d1": _err(_np(d1.index_select(0, idx)), r1),
                "d2": _err(_np(y.index_select(0, idx)), ry)}
    return _result(errs, len(rows), TOL["bf16"],
                   ("rfo_layernorm_gemm" if ln else "rfo_rmsnorm_gemm") +
                   " (fp64, same bf16 X and bf16(g*W) operands)")


def check_router(wl):
    """Every token: d1/d2 against fp64 scores of the same bf16 operands;
    top-k indices bit-exact against the routing oracle evaluated on the
    kernel's own scores (the scores are re-produced once, untimed)."""
    import torch

    x, wp = wl.inputs
    d1, d2, rec = wl.outputs
    M, E, k = x.shape[0], wp.shape[0], rec.shape[1]
    sc = torch.empty(M, E, dtype=torch.float32, device=x.device)
    chk = [torch.empty_like(d1), torch.empty_like(d2), torch.empty_like(rec), sc]
    wl.plan.run([x, wp], chk)
    torch.cuda.synchronize()
    s64 = _np(x) @ _np(wp).T
    r1, r2, _, _ = O.moe_routing(s64, k)
    k1, k2, kv, ki = O.moe_routing(_np(sc), k)
    gi = rec[..., 1].cpu().numpy().astype(np.int64)
    gv = rec[..., 0].contiguous().view(torch.float32).cpu().numpy()
    mism = int((gi != ki).sum())
    errs = {"d1": _err(_np(d1), r1), "d2": _err(_np(d2), r2), "d3_values": _err(gv, kv),
            "scores": _err(_np(sc), s64)}
    out = _result(errs, M, 1e-5, "fp64 X W for d1/d2/scores; make_moe_routing oracle on the "
                                 "kernel's scores for the top-k (indices bit-exact)",
                  {"topk_index_mismatches": mism})
    out["pass"] = out["pass"] and mism == 0 and bool(np.array_equal(_np(chk[2]), _np(rec)))
    return out


def check_mla(wl):
    import torch

    q, kv = wl.inputs
    m, l, o = wl.outputs
    B = q.shape[0]
    e = {"d1": 0.0, "d2": 0.0, "d3": 0.0}
    bs = _spread(B, 4)
    for b in bs:
        b = int(b)
        qq, cc = _np(q[b]), _np(kv[b])
        p = wl.desc.softmax_scale * qq @ cc.T
        rm, rl, ro = O.attention_closed_form(p, cc[None, :, :512])
        e["d1"] = max(e["d1"], _err(_np(m[b]), rm))
        e["d2"] = max(e["d2"], _err(_np(l[b]), rl))
        e["d3"] = max(e["d3"], _err(_np(o[b]), ro))
    return _result(e, len(bs) * q.shape[1], TOL["bf16"],
                   "closed form of the attention cascade over the latent cache (fp64)")


def check(wl, gather_rows=None):
    pat = wl.local["pattern"]
    if pat == "attention":
        if wl.split_kv:
            return check_split_kv(wl, gather_rows)
        return check_attention(wl)
    if pat == "quant":
        return check_quant(wl)
    if pat in ("rms", "ln"):
        return check_rms(wl, ln=pat == "ln")
    if pat == "router":
        return check_router(wl)
    if pat == "mla":
        return check_mla(wl)
    raise ValueError(pat)
