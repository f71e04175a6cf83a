"""TEST INFRASTRUCTURE: numpy wrappers over the C oracle (oracle/rf_oracle.c,
built into oracle/_ref/librf_oracle.so) and the golden-fixture reader.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use this."""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_ref", "librf_oracle.so")
GOLDEN = os.path.join(ROOT, "tests", "golden")

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            import subprocess

            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True,
                           capture_output=True)
        _lib = ctypes.CDLL(ORACLE_SO)
        D = ctypes.POINTER(ctypes.c_double)
        I = ctypes.c_int64
        sig = {
            "rfo_round_bf16": (ctypes.c_float, [ctypes.c_float]),
            "rfo_round_e4m3": (ctypes.c_float, [ctypes.c_float]),
            "rfo_round_bf16_array": (None, [D, D, I]),
            "rfo_round_e4m3_array": (None, [D, D, I]),
            "rfo_safe_softmax": (None, [D, I, I, D, D]),
            "rfo_attention": (None, [D, D, D, I, I, I, I, ctypes.c_double, D, D, D, ctypes.c_int]),
            "rfo_attention_incremental": (ctypes.c_int, [D, D, I, I, I, I, D, D, D]),
            "rfo_attention_merge": (None, [D, D, D, I, I, I, D, D, D]),
            "rfo_quant_gemm": (None, [D, D, I, I, I, ctypes.c_double, D, D, ctypes.c_int]),
            "rfo_quant_gemm_e4m3": (None, [D, D, I, I, I, ctypes.c_double, I, D, D, ctypes.c_int]),
            "rfo_rmsnorm_gemm": (None, [D, D, D, I, I, I, ctypes.c_double, D, D, ctypes.c_int]),
            "rfo_rmsnorm_gemm_incremental": (None, [D, D, D, I, I, ctypes.c_double, D, D]),
            "rfo_layernorm_gemm": (None, [D, D, D, I, I, I, ctypes.c_double, D, D, D, D,
                                          ctypes.c_int]),
            "rfo_variance": (None, [D, I, I, D, D]),
            "rfo_sum_sum": (None, [D, D, I, I, ctypes.c_double, ctypes.c_double, D, D]),
            "rfo_moments": (None, [D, D, I, I, I, D, D, D]),
            "rfo_layernorm_gemm_incremental": (None, [D, D, D, I, I, ctypes.c_double, D, D, D, D]),
            "rfo_moe_routing": (None, [D, I, I, I, D, D, D, ctypes.POINTER(ctypes.c_int64)]),
            "rfo_scaled_max_err": (ctypes.c_double, [D, D, I, ctypes.POINTER(ctypes.c_int64)]),
            "rfo_fused_row": (ctypes.c_int, [ctypes.c_int, D, D, I, ctypes.POINTER(ctypes.c_int64),
                                             ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                             D, D, D]),
        }
        for n, (r, a) in sig.items():
            f = getattr(_lib, n)
            f.restype = r
            f.argtypes = a
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


THREADS = max(1, min(32, os.cpu_count() or 1))


def round_bf16(a):
    a = _f64(a)
    out = np.empty_like(a)
    lib().rfo_round_bf16_array(_p(a), _p(out), a.size)
    return out


def round_e4m3(a):
    a = _f64(a)
    out = np.empty_like(a)
    lib().rfo_round_e4m3_array(_p(a), _p(out), a.size)
    return out


def safe_softmax(x):
    x = _f64(x)
    rows, n = x.shape
    d1, d2 = np.empty(rows), np.empty(rows)
    lib().rfo_safe_softmax(_p(x), rows, n, _p(d1), _p(d2))
    return d1, d2


def attention(q, k, v, scale=1.0):
    """q [BH,Sq,D], k/v [BH,Skv,D] -> m, l [BH,Sq], o [BH,Sq,D] (oracle form)."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    bh, sq, d = q.shape
    skv = k.shape[1]
    m, l = np.empty((bh, sq)), np.empty((bh, sq))
    o = np.empty((bh, sq, d))
    lib().rfo_attention(_p(q), _p(k), _p(v), bh, sq, skv, d, scale, _p(m), _p(l), _p(o), THREADS)
    return m, l, o


def attention_closed_form(p, v):
    """The attention cascade's oracle lambda (make_attention, workloads.cpp:101-118)
    on precomputed scores: p [rows, kv], v [rows or 1, kv, Dv] -> m, l [rows],
    o [rows, Dv]: m = max p, l = sum e^(p-m), o = sum e^(p-m)/l v. numpy fp64;
    pinned against the C oracle by tests/test_oracle_golden.py. Lets K and V
    differ in width (MLA: K = [c_kv | k_rope] 576 wide, V = c_kv 512 wide)."""
    p = np.asarray(p, dtype=np.float64)
    m = p.max(axis=1)
    e = np.exp(p - m[:, None])
    l = e.sum(axis=1)
    o = np.einsum("rk,rkd->rd", e, np.broadcast_to(v, (p.shape[0],) + v.shape[1:])) / l[:, None]
    return m, l, o


def attention_incremental(p, v, segments=1):
    """p [rows, kv], v [rows, kv, D] -> m, l, o (run_incremental/multisegment semantics)."""
    p, v = _f64(p), _f64(v)
    rows, kv = p.shape
    d = v.shape[2]
    m, l = np.empty(rows), np.empty(rows)
    o = np.empty((rows, d))
    rc = lib().rfo_attention_incremental(_p(p), _p(v), rows, kv, d, segments, _p(m), _p(l), _p(o))
    if rc == -2:
        raise ValueError("IncompatibleSegmentation")
    return m, l, o


def attention_merge(pm, pl, po):
    pm, pl, po = _f64(pm), _f64(pl), _f64(po)
    s, rows = pm.shape
    d = po.shape[2]
    m, l = np.empty(rows), np.empty(rows)
    o = np.empty((rows, d))
    lib().rfo_attention_merge(_p(pm), _p(pl), _p(po), s, rows, d, _p(m), _p(l), _p(o))
    return m, l, o


def quant_gemm(a, w, fmax=448.0):
    a, w = _f64(a), _f64(w)
    M, K = a.shape
    Nn = w.shape[1]
    d1, c = np.empty(M), np.empty((M, Nn))
    lib().rfo_quant_gemm(_p(a), _p(w), M, K, Nn, fmax, _p(d1), _p(c), THREADS)
    return d1, c


def quant_gemm_e4m3(a, w, fmax=448.0, tile_k=128):
    a, w = _f64(a), _f64(w)
    M, K = a.shape
    Nn = w.shape[1]
    d1, c = np.empty(M), np.empty((M, Nn))
    lib().rfo_quant_gemm_e4m3(_p(a), _p(w), M, K, Nn, fmax, tile_k, _p(d1), _p(c), THREADS)
    return d1, c


def quant_gemm_e4m3_torch(a, w, fmax=448.0, tile_k=128, pow2=True):
    """Independent emulation (torch float8_e4m3fn casts, not rf_oracle.c) of
    the single-loop FP8 quant GEMM over K tiles of `tile_k`:
      m_t   = running max |a| (fp32, as the kernel keeps it)
      ref_t = 2^ceil(log2 m_t)  (pow2=True: the kernel's H' proxy)
              m_t               (pow2=False: SURVEY §7.3's true running amax)
      q     = e4m3(fp32(a * (fmax / ref_t)))          (RNE, |q| <= fmax)
      acc   = acc * (ref_{t-1} / ref_t) + q . w       (Eq.17 correction d1'/d1)
      c     = acc * ref_T / m_T                       (finalize_root retarget)
    The real-arithmetic reference (make_quant_gemm, workloads.cpp:192-207) is
    c = sum (fmax a / m_T) w; both forms equal it without the rounding."""
    import torch

    A = torch.as_tensor(_f64(a)).to(torch.float32)
    W = torch.as_tensor(_f64(w))
    M, K = A.shape
    acc = torch.zeros(M, W.shape[1], dtype=torch.float64)
    amax = torch.zeros(M, dtype=torch.float32)
    ref = torch.zeros(M, dtype=torch.float32)
    for l0 in range(0, K, tile_k):
        blk = A[:, l0:l0 + tile_k]
        amax = torch.maximum(amax, blk.abs().amax(dim=1))
        if pow2:
            mant, ex = torch.frexp(amax)
            nref = torch.where(mant == 0.5, torch.ldexp(torch.ones_like(amax), ex - 1),
                               torch.ldexp(torch.ones_like(amax), ex))
        else:
            nref = amax.clone()
        if l0 > 0:
            corr = torch.where((ref > 0) & (nref != ref), ref.double() / nref.double(),
                               torch.ones_like(ref, dtype=torch.float64))
            acc *= corr[:, None]
        ref = nref
        scale = torch.where(ref > 0, torch.full_like(ref, float(fmax)) / ref, torch.zeros_like(ref))[:, None]
        qv = (blk * scale).to(torch.float8_e4m3fn).to(torch.float64)
        acc += qv @ W[l0:l0 + tile_k]
    fin = ref.double() / amax.double()
    return amax.double().numpy(), (acc * fin[:, None]).numpy()


def rmsnorm_gemm(x, g, w, eps=1e-6):
    x, g, w = _f64(x), _f64(g), _f64(w)
    T, K = x.shape
    Nn = w.shape[1]
    d1, y = np.empty(T), np.empty((T, Nn))
    lib().rfo_rmsnorm_gemm(_p(x), _p(g), _p(w), T, K, Nn, eps, _p(d1), _p(y), THREADS)
    return d1, y


def rmsnorm_gemm_incremental(x, g, w, eps=1e-6):
    x, g, w = _f64(x), _f64(g), _f64(w)
    K = x.shape[0]
    Nn = w.shape[1]
    d1 = np.empty(1)
    y = np.empty(Nn)
    lib().rfo_rmsnorm_gemm_incremental(_p(x), _p(g), _p(w), K, Nn, eps, _p(d1), _p(y))
    return d1[0], y


def layernorm_gemm(x, g, w, eps=1e-5):
    """(d1 = sum x, d2 = sum x^2, d3, d4) with LayerNorm(x*g) @ W = d3 - d4."""
    x, g, w = _f64(x), _f64(g), _f64(w)
    T, K = x.shape
    Nn = w.shape[1]
    d1, d2 = np.empty(T), np.empty(T)
    d3, d4 = np.empty((T, Nn)), np.empty((T, Nn))
    lib().rfo_layernorm_gemm(_p(x), _p(g), _p(w), T, K, Nn, eps, _p(d1), _p(d2), _p(d3), _p(d4),
                             THREADS)
    return d1, d2, d3, d4


def layernorm_gemm_incremental(x, g, w, eps=1e-5):
    x, g, w = _f64(x), _f64(g), _f64(w)
    K = x.shape[0]
    Nn = w.shape[1]
    d1, d2 = np.empty(1), np.empty(1)
    d3, d4 = np.empty(Nn), np.empty(Nn)
    lib().rfo_layernorm_gemm_incremental(_p(x), _p(g), _p(w), K, Nn, eps, _p(d1), _p(d2),
                                         _p(d3), _p(d4))
    return d1[0], d2[0], d3, d4


def variance(x):
    x = _f64(x)
    rows, n = x.shape
    d1, d2 = np.empty(rows), np.empty(rows)
    lib().rfo_variance(_p(x), rows, n, _p(d1), _p(d2))
    return d1, d2


def sum_sum(x1, x2, c=10.0, eps=1e-12):
    x1, x2 = _f64(x1), _f64(x2)
    rows, n = x1.shape
    d1, d2 = np.empty(rows), np.empty(rows)
    lib().rfo_sum_sum(_p(x1), _p(x2), rows, n, c, eps, _p(d1), _p(d2))
    return d1, d2


def moments(mass, pos):
    mass, pos = _f64(mass), _f64(pos)
    rows, n, F = pos.shape
    d1, d2, d3 = np.empty(rows), np.empty((rows, F)), np.empty((rows, F))
    lib().rfo_moments(_p(mass), _p(pos), rows, n, F, _p(d1), _p(d2), _p(d3))
    return d1, d2, d3


def moe_routing(s, k):
    s = _f64(s)
    rows, e = s.shape
    d1, d2 = np.empty(rows), np.empty(rows)
    tv = np.empty((rows, k))
    ti = np.zeros((rows, k), dtype=np.int64)
    lib().rfo_moe_routing(_p(s), rows, e, k, _p(d1), _p(d2), _p(tv),
                          ti.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    return d1, d2, tv, ti


FUSED_PATTERNS = {"safe_softmax": 1, "attention": 2, "variance": 7, "sum_sum": 8}


def fused(pattern, a, b=None, levels=(), k=1, c=10.0, eps=1e-12):
    """run_fused (simulator.cpp:485-559) per row: a [rows, L0] (softmax x,
    attention P, variance x, sum_sum x1), b = attention V [rows, L0, hd] or
    sum_sum x2 [rows, L0]; levels = TreeConfig.levels (L0 first, 1 last).
    Returns d1, d2 [rows] (+ d3 [rows, hd] for attention)."""
    pat = FUSED_PATTERNS[pattern]
    a = _f64(a)
    rows, L0 = a.shape
    lv = np.asarray(levels, dtype=np.int64)
    assert lv[0] == L0
    hd = b.shape[2] if pat == 2 else 0
    b = _f64(b) if b is not None else np.zeros(1)
    d1, d2 = np.empty(rows), np.empty(rows)
    d3 = np.zeros((rows, max(hd, 1)))
    for r in range(rows):
        br = b[r] if pat in (2, 8) else b
        o1, o2 = np.zeros(1), np.zeros(1)
        rc = lib().rfo_fused_row(pat, _p(np.ascontiguousarray(a[r])), _p(np.ascontiguousarray(br)), hd,
                                 lv.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), len(lv) - 1, k, c, eps,
                                 _p(o1), _p(o2), _p(d3[r]))
        if rc != 0:
            raise ValueError("bad tree / fuse level")
        d1[r], d2[r] = o1[0], o2[0]
    return (d1, d2, d3) if pat == 2 else (d1, d2)


def scaled_max_err(x, y):
    """compare_reports' metric (simulator.cpp:717-721): max |x-y|/(1+max(|x|,|y|))."""
    x, y = _f64(x).ravel(), _f64(y).ravel()
    assert x.shape == y.shape
    w = ctypes.c_int64(-1)
    e = lib().rfo_scaled_max_err(_p(x), _p(y), x.size, ctypes.byref(w))
    return e, w.value


def load_golden(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        man = json.load(f)
    blob = np.fromfile(os.path.join(GOLDEN, name + ".f64"), dtype="<f8")
    out = {}
    for a in man["arrays"]:
        out[a["name"]] = blob[a["offset"]:a["offset"] + a["count"]].reshape(a["shape"])
    out["_meta"] = man["meta"]
    return out


def golden_names(prefix=""):
    return sorted(f[:-5] for f in os.listdir(GOLDEN) if f.endswith(".json") and f.startswith(prefix))
