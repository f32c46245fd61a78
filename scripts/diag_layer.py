"""Diagnostic: a one-layer model's intermediate activations (attention output, SwiGLU output,
final residual) against the bf16-mirrored fp64 reference, row by row."""
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


def per_row(a, b):
    return ((a - b).norm(dim=-1) / b.norm(dim=-1).clamp(min=1e-30))


def frac_equal(a, b):
    return (a == b).double().mean().item()


for name in sys.argv[1:] or ["tiny:L1", "llama3-8b:L1", "llama3.2-1b:L1"]:
    s = lr.shape(name)
    V, T, cap = s["vocab"], 24, 64
    d, nq, nkv, hd, ffn = s["d"], s["nq"], s["nkv"], s["hd"], s["ffn"]
    h = C.c_void_p()
    assert lib.ws_model_create(name.encode(), 11, 64, cap, 0, C.byref(h)) == 0
    ref = lr.RefModel(lib, h, name)
    g = torch.Generator().manual_seed(3)
    toks = torch.randint(0, V, (T,), generator=g).tolist()
    i32 = lambda v: torch.tensor(v, dtype=torch.int32)  # noqa: E731
    keep = [i32(toks), i32(list(range(T))), i32([0, T, 0, 0, 0, T, 0]), torch.zeros(T, dtype=torch.int64),
            i32([T - 1])]
    logits = torch.empty(1, V, dtype=torch.bfloat16, device="cuda")
    rc = lib.ws_model_forward(h, T, keep[0].data_ptr(), keep[1].data_ptr(), keep[1].data_ptr(), 1, keep[2].data_ptr(),
                              T, keep[1].data_ptr(), keep[3].data_ptr(), 1, keep[4].data_ptr(), logits.data_ptr(), None)
    assert rc == 0, C.string_at(lib.ws_last_error())
    torch.cuda.synchronize()

    def grab(which, n, dt):
        t = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        assert lib.ws_model_copy_weight(h, which, 0, t.data_ptr(), n) == 0
        return t.view(dt) if dt != torch.bfloat16 else t
    xk = grab(b"ws_x", 2 * cap * d, torch.float32).view(cap, d)[:T].double()
    ak = grab(b"ws_attn", cap * nq * hd, torch.bfloat16).view(cap, nq * hd)[:T].double()
    hk = grab(b"ws_h", cap * ffn, torch.bfloat16).view(cap, ffn)[:T].double()
    Lw = ref.layers[0]
    x = ref.emb[torch.tensor(toks, device="cuda")].double()
    c, sn = ref._cs(torch.arange(T, device="cuda"))
    xb, rs = lr.bf(x), ref._rs(x)
    a = lr.f32(lr.f32(xb @ Lw["wqkv"].T) * rs)
    q = lr.bf(ref._rope(a[:, :nq * hd].view(T, nq, hd), c, sn))
    kk = lr.bf(ref._rope(a[:, nq * hd:(nq + nkv) * hd].view(T, nkv, hd), c, sn))
    vv = lr.bf(a[:, (nq + nkv) * hd:].view(T, nkv, hd))
    G = nq // nkv
    o = ref._attention(q, kk.repeat_interleave(G, 1), vv.repeat_interleave(G, 1), lr.causal(T).cuda()).reshape(T, -1)
    print(f"{name}: attn rel max {per_row(ak, o).max().item():.2e} equal {frac_equal(ak, o):.4f}", flush=True)
    x1 = lr.f32(x + lr.f32(ak @ Lw["wo"].T))  # continue from the KERNEL's attention output
    xb, rs = lr.bf(x1), ref._rs(x1)
    g_ = lr.f32(lr.f32(xb @ Lw["wg"].T) * rs)
    u_ = lr.f32(lr.f32(xb @ Lw["wu"].T) * rs)
    hh = lr.bf(g_ / (1 + torch.exp(-g_)) * u_)
    print(f"  swiglu h rel max {per_row(hk, hh).max().item():.2e} equal {frac_equal(hk, hh):.4f}", flush=True)
    x2 = lr.f32(x1 + lr.f32(hk @ Lw["wd"].T))  # from the kernel's h
    print(f"  residual x rel max {per_row(xk, x2).max().item():.2e} equal {frac_equal(xk, x2):.4f}; "
          f"|x| {x2.norm(dim=-1).mean().item():.3f}, |x1| {x1.norm(dim=-1).mean().item():.3f}", flush=True)
    # pieces: x1 alone and the down-projection output
    lib.ws_model_destroy(h)
    del ref
    torch.cuda.empty_cache()
