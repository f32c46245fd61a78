"""Diagnostic: where does the batched forward leave the bf16-mirrored fp64 reference?
Per shape: layer-0 K/V pool contents vs the reference's, and logits at a few positions."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import llama_ref as lr  # noqa: E402
import paper_2602_18931_b200 as ws  # noqa: E402

lib = ws.lib()
lib.ws_model_create.argtypes = [C.c_char_p, C.c_uint64, C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
lib.ws_model_destroy.argtypes = [C.c_void_p]
lib.ws_model_copy_weight.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_void_p, C.c_int64]
lib.ws_model_forward.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                 C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]


def rel(a, b):
    return ((a - b).norm(dim=-1) / b.norm(dim=-1).clamp(min=1e-30)).max().item()


for name in sys.argv[1:] or ["tiny", "tiny128", "llama3.2-1b:L1", "llama3-8b:L1", "llama3-8b:L2"]:
    s = lr.shape(name)
    V, T = s["vocab"], 40
    h = C.c_void_p()
    assert lib.ws_model_create(name.encode(), 11, 64, 64, 0, C.byref(h)) == 0
    ref = lr.RefModel(lib, h, name)
    g = torch.Generator().manual_seed(3)
    toks = torch.randint(0, V, (T,), generator=g).tolist()
    i32 = lambda v: torch.tensor(v, dtype=torch.int32)  # noqa: E731
    outs = [0, 1, 17, T - 1]
    logits = torch.empty(len(outs), V, dtype=torch.bfloat16, device="cuda")
    keep = [i32(toks), i32(list(range(T))), i32([0, T, 0, 0, 0, T, 0]), torch.zeros(T, dtype=torch.int64), i32(outs)]
    rc = lib.ws_model_forward(h, T, keep[0].data_ptr(), keep[1].data_ptr(), keep[1].data_ptr(), 1, keep[2].data_ptr(),
                              T, keep[1].data_ptr(), keep[3].data_ptr(), len(outs), keep[4].data_ptr(),
                              logits.data_ptr(), None)
    assert rc == 0, (rc, C.string_at(lib.ws_last_error()))
    torch.cuda.synchronize()
    n = s["layers"] * 64 * s["nkv"] * s["hd"]
    kp = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    vp = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    assert lib.ws_model_copy_weight(h, b"k_pool", 0, kp.data_ptr(), n) == 0
    assert lib.ws_model_copy_weight(h, b"v_pool", 0, vp.data_ptr(), n) == 0
    kall = kp.view(s["layers"], 64, s["nkv"] * s["hd"])[:, :T].double()
    vall = vp.view(s["layers"], 64, s["nkv"] * s["hd"])[:, :T].double()
    kp, vp = kall[0], vall[0]
    # reference layer-0 k / v
    nq, nkv, hd = s["nq"], s["nkv"], s["hd"]
    Lw = ref.layers[0]
    x = ref.emb[torch.tensor(toks, device="cuda")].double()
    xb, rs = lr.bf(x), ref._rs(x)
    a = lr.f32(lr.f32(xb @ Lw["wqkv"].T) * rs)
    c, sn = ref._cs(torch.arange(T, device="cuda"))
    k = lr.bf(ref._rope(a[:, nq * hd:(nq + nkv) * hd].view(T, nkv, hd), c, sn)).reshape(T, -1)
    v = lr.bf(a[:, (nq + nkv) * hd:]).reshape(T, -1)
    exact = lambda t: (t == 0).float().mean().item()  # noqa: E731
    rl = ref.logits(toks, list(range(T)), lr.causal(T), outs)
    if s["layers"] > 1:  # layer-1 V per row: exposes layer-0 attention / MLP differences per row
        x = ref.emb[torch.tensor(toks, device="cuda")].double()
        allowed = lr.causal(T).cuda()
        xb, rs = lr.bf(x), ref._rs(x)
        a = lr.f32(lr.f32(xb @ Lw["wqkv"].T) * rs)
        q = lr.bf(ref._rope(a[:, :nq * hd].view(T, nq, hd), c, sn))
        kk = lr.bf(ref._rope(a[:, nq * hd:(nq + nkv) * hd].view(T, nkv, hd), c, sn))
        vv = lr.bf(a[:, (nq + nkv) * hd:].view(T, nkv, hd))
        G = nq // nkv
        o = ref._attention(q, kk.repeat_interleave(G, 1), vv.repeat_interleave(G, 1), allowed).reshape(T, nq * hd)
        x = lr.f32(x + lr.f32(o @ Lw["wo"].T))
        xb, rs = lr.bf(x), ref._rs(x)
        g_ = lr.f32(lr.f32(xb @ Lw["wg"].T) * rs)
        u_ = lr.f32(lr.f32(xb @ Lw["wu"].T) * rs)
        x = lr.f32(x + lr.f32(lr.bf(g_ / (1 + torch.exp(-g_)) * u_) @ Lw["wd"].T))
        L1 = ref.layers[1]
        xb, rs = lr.bf(x), ref._rs(x)
        a1 = lr.f32(lr.f32(xb @ L1["wqkv"].T) * rs)
        v1 = lr.bf(a1[:, (nq + nkv) * hd:])
        per = ((vall[1] - v1).norm(dim=-1) / v1.norm(dim=-1))
        print("  layer-1 V rel per row:", " ".join(f"{per[i].item():.1e}" for i in range(T)), flush=True)
    print(f"{name}: K rel {rel(kp, k):.2e} (equal {exact(kp - k):.4f}), V rel {rel(vp, v):.2e} "
          f"(equal {exact(vp - v):.4f}); logits rel per row "
          + " ".join(f"{((logits.double()[i] - rl[i]).norm() / rl[i].norm()).item():.2e}" for i in range(len(outs))),
          flush=True)
    del ref
    lib.ws_model_destroy(h)
    torch.cuda.empty_cache()
