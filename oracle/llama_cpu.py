"""ORACLE — TEST INFRASTRUCTURE ONLY (parity unpinned by the reference: the reference has no
neural model).

A plain numpy fp32 restatement of the Llama-architecture verify/draft forward the GPU path
runs (RMSNorm → QKV → rotate-half RoPE with llama3 frequency scaling → causal GQA attention →
O-proj → RMSNorm → SwiGLU MLP → final norm → LM head). Used (a) as the CPU "port" baseline
timed in bench.py's cpu_baseline / --impl reference legs on a bounded sample, and (b) as an
independent CPU check of small shapes.
"""
import math
import os
import time

import numpy as np

SHAPES = {
    "llama3-8b": dict(layers=32, d=4096, nq=32, nkv=8, hd=128, ffn=14336, vocab=128256, theta=500000.0,
                      factor=8.0),
    "llama3.2-1b": dict(layers=16, d=2048, nq=32, nkv=8, hd=64, ffn=8192, vocab=128256, theta=500000.0,
                        factor=32.0),
    "tiny": dict(layers=2, d=256, nq=4, nkv=2, hd=64, ffn=512, vocab=1000, theta=10000.0, factor=0.0),
}


def inv_freq(s):
    hd = s["hd"]
    out = np.empty(hd // 2, dtype=np.float64)
    for i in range(hd // 2):
        inv = 1.0 / (s["theta"] ** (2.0 * i / hd))
        if s["factor"] > 0:
            factor, lo, hi, old = s["factor"], 1.0, 4.0, 8192.0
            wl = 2 * math.pi / inv
            if wl > old / lo:
                inv = inv / factor
            elif wl >= old / hi:
                sm = (old / wl - lo) / (hi - lo)
                inv = (1 - sm) * inv / factor + sm * inv
        out[i] = inv
    return out.astype(np.float32)


def rms(x, w, eps=1e-5):
    return x * (1.0 / np.sqrt((x * x).mean(-1, keepdims=True) + eps)) * w


def rope(x, pos, inv):
    hd = x.shape[-1]
    ang = pos[:, None].astype(np.float32) * inv[None, :]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    a, b = x[..., :hd // 2], x[..., hd // 2:]
    return np.concatenate([a * c - b * s, b * c + a * s], axis=-1)


def layer_forward(x, pos, kv_k, kv_v, W, s, inv):
    """One decoder layer for T new rows at positions `pos` appended after cached K/V
    (kv_k/kv_v [ctx, nkv, hd]); returns (x, k_all, v_all)."""
    nq, nkv, hd = s["nq"], s["nkv"], s["hd"]
    T = x.shape[0]
    xn = rms(x, W["an"])
    qkv = xn @ W["wqkv"].T
    q = rope(qkv[:, :nq * hd].reshape(T, nq, hd), pos, inv)
    k = rope(qkv[:, nq * hd:(nq + nkv) * hd].reshape(T, nkv, hd), pos, inv)
    v = qkv[:, (nq + nkv) * hd:].reshape(T, nkv, hd)
    K = np.concatenate([kv_k, k], 0)
    Vv = np.concatenate([kv_v, v], 0)
    S = K.shape[0]
    G = nq // nkv
    Kr, Vr = np.repeat(K, G, axis=1), np.repeat(Vv, G, axis=1)
    att = np.einsum("thd,shd->hts", q, Kr) / math.sqrt(hd)
    start = S - T
    mask = np.arange(S)[None, :] > (start + np.arange(T))[:, None]
    att = np.where(mask[None], -np.inf, att)
    att = np.exp(att - att.max(-1, keepdims=True))
    att /= att.sum(-1, keepdims=True)
    o = np.einsum("hts,shd->thd", att, Vr).reshape(T, nq * hd)
    x = x + o @ W["wo"].T
    xn = rms(x, W["mn"])
    g, u = xn @ W["wg"].T, xn @ W["wu"].T
    x = x + (g / (1.0 + np.exp(-g)) * u) @ W["wd"].T
    return x, K, Vv


def random_layer(s, rng, constant=False):
    d, nq, nkv, hd, ffn = s["d"], s["nq"], s["nkv"], s["hd"], s["ffn"]
    if constant:  # timing only: values do not change BLAS cost, and filling is 100x cheaper
        f = lambda *shape: np.full(shape, 0.02, dtype=np.float32)  # noqa: E731
    else:
        f = lambda *shape: (rng.standard_normal(shape, dtype=np.float32) * 0.02)  # noqa: E731
    return dict(an=np.ones(d, np.float32), mn=np.ones(d, np.float32), wqkv=f((nq + 2 * nkv) * hd, d),
                wo=f(d, nq * hd), wg=f(ffn, d), wu=f(ffn, d), wd=f(d, ffn))


def time_forward(name, rows, ctx, threads=None, lm_rows=None, seed=0):
    """Bounded CPU sample: wall seconds of one forward of `rows` new rows after `ctx` cached
    positions at the named shape (numpy fp32, BLAS threads = all host cores unless given).
    One layer's weights are materialised and reused for every layer (identical FLOPs and
    bytes per layer); the LM head is timed on `lm_rows` rows with a vocab-sized matrix."""
    if threads:
        os.environ["OMP_NUM_THREADS"] = str(threads)
    s = SHAPES[name]
    rng = np.random.default_rng(seed)
    W = random_layer(s, rng, constant=True)
    inv = inv_freq(s)
    x = rng.standard_normal((rows, s["d"]), dtype=np.float32)
    kv_k = rng.standard_normal((ctx, s["nkv"], s["hd"]), dtype=np.float32)
    kv_v = rng.standard_normal((ctx, s["nkv"], s["hd"]), dtype=np.float32)
    pos = np.arange(ctx, ctx + rows)
    layer_forward(x, pos, kv_k, kv_v, W, s, inv)  # warm
    t0 = time.perf_counter()
    layer_forward(x, pos, kv_k, kv_v, W, s, inv)
    t_layer = time.perf_counter() - t0
    lm = np.full((s["vocab"], s["d"]), 0.02, dtype=np.float32)
    xo = x[: (lm_rows or rows)]
    t0 = time.perf_counter()
    _ = rms(xo, 1.0) @ lm.T
    t_lm = time.perf_counter() - t0
    return t_layer * s["layers"] + t_lm
