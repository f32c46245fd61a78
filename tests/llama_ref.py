"""Test-side reference of the batched Llama forward that rounds where the kernels round.

The reference (arxiv 2602.18931) has no model: its verify/draft arithmetic is a
position-indexed table (oracle.hpp:88-139). The model path is therefore checked against this
restatement of the same architecture on the same weights, in float64 with a rounding to bf16 /
fp32 at every point where the sm_100a kernels store a narrower value:

  x (residual)         fp32      embed_rows / O and down epilogues (fp32 +=, gemm_tc.cu)
  xb = bf16(x)         bf16      A operand of the normed projections (NormEpi producer)
  rs = rsqrt(sum x^2 / d + eps)  per-row fused RMSNorm scale (NormEpi consumer); norm weights
                                 are folded into Wqkv / Wgu at load (fold_norm_weight)
  q, k = bf16(rope(fp32(acc) * rs)), v = bf16(fp32(acc) * rs)   QKV epilogue (cos/sin fp32
                                 table from fp64 angles of fp32 inverse frequencies)
  attn = bf16(o / l)   K2's online softmax, mirrored tile by tile (hd 128: two key slices, merged
                       at the end): keys in 32-position tiles
                       (the group's prefix, then its extras), s = fp32(q.k) * fp32(scale log2 e),
                       running max per tile, p = exp2(s - max) in fp32, l += sum p (fp32),
                       o = o * corr + bf16(p) . v  (P is the bf16 A operand of the PV mma)
  h = bf16(silu(g) * u), g, u = fp32(acc) * rs   SwiGLU epilogue
  xo = bf16(x * rsqrt(mean x^2 + eps) * w_final)  rmsnorm_rows
  logits = bf16(xo W_lm^T)

Attention visibility is an explicit [T, T] boolean matrix, so one call covers causal prefill,
verify / catch-up groups over a cached prefix and masked tree groups (AttnGroup semantics,
csrc/kernels/llama_ops.cuh).
"""
import ctypes as C
import math

import torch

SHAPES = {  # mirrors shape_by_name (csrc/model/llama.cu); ":L<n>" truncates the layer count
    "llama3-8b": dict(layers=32, d=4096, nq=32, nkv=8, hd=128, ffn=14336, vocab=128256, theta=500000.0,
                      factor=8.0, tied=False),
    "llama3.2-1b": dict(layers=16, d=2048, nq=32, nkv=8, hd=64, ffn=8192, vocab=128256, theta=500000.0,
                        factor=32.0, tied=True),
    "llama3-70b": dict(layers=80, d=8192, nq=64, nkv=8, hd=128, ffn=28672, vocab=128256, theta=500000.0,
                       factor=8.0, tied=False),
    "tiny": dict(layers=2, d=256, nq=4, nkv=2, hd=64, ffn=512, vocab=1000, theta=10000.0, factor=0.0, tied=False),
    "tiny128": dict(layers=2, d=512, nq=4, nkv=1, hd=128, ffn=1024, vocab=2000, theta=500000.0, factor=8.0,
                    tied=False),
}
EPS = 1e-5


def shape(name):
    base, _, rest = name.partition(":L")
    s = dict(SHAPES[base])
    if rest:
        s["layers"] = int(rest)
    return s


def inv_freq_f32(s):
    """llama3_inv_freq (csrc/model/llama.cu): fp64 formula, stored as fp32."""
    hd = s["hd"]
    out = []
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
        out.append(inv)
    return torch.tensor(out, dtype=torch.float32)


def bf(t):
    return t.to(torch.bfloat16).to(torch.float64)


def f32(t):
    return t.to(torch.float32).to(torch.float64)


class RefModel:
    def __init__(self, lib, h, name):
        self.s = s = shape(name)
        d, nq, nkv, hd, ffn, V = s["d"], s["nq"], s["nkv"], s["hd"], s["ffn"], s["vocab"]
        lib.ws_model_copy_weight.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_void_p, C.c_int64]

        def get(wname, layer, n, shp, dt=torch.float64):
            t = torch.empty(n, dtype=torch.bfloat16, device="cuda")
            assert lib.ws_model_copy_weight(h, wname.encode(), layer, t.data_ptr(), n) == 0
            return t.view(*shp).to(dt)
        self.emb = get("embed", 0, V * d, (V, d), torch.bfloat16)
        self.lm = get("lm_head", 0, V * d, (V, d))
        self.fn = get("final_norm", 0, d, (d,))
        self.layers = []
        for layer in range(s["layers"]):
            qkv = (nq + 2 * nkv) * hd
            wgu = get("wgu", layer, 2 * ffn * d, (2 * ffn, d)).view(ffn // 16, 2, 16, d)
            self.layers.append(dict(
                wqkv=get("wqkv", layer, qkv * d, (qkv, d)), wo=get("wo", layer, d * nq * hd, (d, nq * hd)),
                wg=wgu[:, 0].reshape(ffn, d).contiguous(), wu=wgu[:, 1].reshape(ffn, d).contiguous(),
                wd=get("wdown", layer, d * ffn, (d, ffn))))
        inv = inv_freq_f32(s).double()
        self.inv = inv.cuda()

    def _cs(self, pos):
        ang = pos.double()[:, None] * self.inv[None, :]
        return f32(torch.cos(ang)), f32(torch.sin(ang))  # the fp32 table of the QKV epilogue

    def _rope(self, x, c, s_):  # x [T, H, hd]
        hd = x.shape[-1]
        a, b = x[..., :hd // 2], x[..., hd // 2:]
        c, s_ = c[:, None, :], s_[:, None, :]
        return torch.cat([a * c - b * s_, b * c + a * s_], dim=-1)

    @staticmethod
    def _attention(q, k, v, allowed, tile=32):
        """attn_mma_kernel (csrc/kernels/attention.cu) restated: 32-key tiles; hd 128 runs two key
        slices (slice ks takes tiles ks, ks+2, ...; the slices' states merge in slice order at the
        end), hd 64 one."""
        hd = q.shape[-1]
        slices = 2 if hd == 128 else 1
        sl2 = torch.tensor(1.0 / math.sqrt(hd), dtype=torch.float32) * torch.tensor(1.4426950408889634,
                                                                                     dtype=torch.float32)
        s = f32(torch.einsum("thd,shd->hts", q, k)) * sl2.double()
        s = f32(s).masked_fill(~allowed[None], float("-inf"))  # [H, Tq, Tk]
        H, Tq, Tk = s.shape
        vh = v.permute(1, 0, 2)  # [H, Tk, hd]
        states = []
        for ks in range(slices):
            m = torch.full((H, Tq), float("-inf"), dtype=torch.float64, device=s.device)
            lsum = torch.zeros(H, Tq, dtype=torch.float64, device=s.device)
            o = torch.zeros(H, Tq, hd, dtype=torch.float64, device=s.device)
            for t0 in range(ks * tile, Tk, slices * tile):
                st = s[:, :, t0:t0 + tile]
                nmax = torch.maximum(m, st.max(-1).values)
                base = torch.where(nmax == float("-inf"), torch.zeros_like(nmax), nmax)
                corr = torch.exp2(m - base)
                p = f32(torch.exp2(st - base[..., None]))
                lsum = f32(lsum * corr + p.sum(-1))
                o = o * corr[..., None] + torch.einsum("hts,hsd->htd", bf(p), vh[:, t0:t0 + tile])
                m = nmax
            states.append((m, lsum, o))
        m, lsum, o = states[0]
        for om, ol, oo in states[1:]:
            nm = torch.maximum(m, om)
            b = torch.where(nm == float("-inf"), torch.zeros_like(nm), nm)
            ca, cb = f32(torch.exp2(m - b)), f32(torch.exp2(om - b))
            lsum = f32(lsum * ca + ol * cb)
            o = o * ca[..., None] + oo * cb[..., None]
            m = nm
        inv = torch.where(lsum > 0, 1.0 / lsum, torch.zeros_like(lsum))
        return bf(o * inv[..., None]).permute(1, 0, 2)

    @staticmethod
    def _rs(x):
        return 1.0 / torch.sqrt((x * x).sum(-1, keepdim=True) / x.shape[-1] + EPS)

    def head(self, x):
        """Final RMSNorm + LM head from fp32 residual rows x [n, d] (rmsnorm_rows + the bf16 GEMM)."""
        xo = bf(x * torch.rsqrt((x * x).mean(-1, keepdim=True) + EPS) * self.fn)
        return bf(xo @ self.lm.T)

    def kv0(self, tokens, pos):
        """Layer-0 K (rotated) and V rows [T, n_kv * hd] of the given tokens (QKV epilogue)."""
        s = self.s
        nq, nkv, hd = s["nq"], s["nkv"], s["hd"]
        T = len(tokens)
        x = self.emb[torch.tensor(tokens, device="cuda")].double()
        c, s_ = self._cs(torch.tensor(pos, device="cuda"))
        a = f32(f32(bf(x) @ self.layers[0]["wqkv"].T) * self._rs(x))
        k = bf(self._rope(a[:, nq * hd:(nq + nkv) * hd].view(T, nkv, hd), c, s_)).reshape(T, -1)
        return k, bf(a[:, (nq + nkv) * hd:])

    def logits(self, tokens, pos, allowed, out_idx):
        """tokens/pos: length-T lists; allowed: [T, T] bool (row attends column); out_idx: the rows
        whose logits are returned (bf16-rounded, as float64 [n_out, V])."""
        s = self.s
        nq, nkv, hd = s["nq"], s["nkv"], s["hd"]
        T = len(tokens)
        tok = torch.tensor(tokens, device="cuda")
        p = torch.tensor(pos, device="cuda")
        allowed = allowed.to("cuda")
        c, s_ = self._cs(p)
        x = self.emb[tok].double()
        G = nq // nkv
        for Lw in self.layers:
            xb, rs = bf(x), self._rs(x)
            a = f32(f32(xb @ Lw["wqkv"].T) * rs)
            q = a[:, :nq * hd].view(T, nq, hd)
            k = a[:, nq * hd:(nq + nkv) * hd].view(T, nkv, hd)
            v = bf(a[:, (nq + nkv) * hd:].view(T, nkv, hd))
            q, k = bf(self._rope(q, c, s_)), bf(self._rope(k, c, s_))
            k = k.repeat_interleave(G, dim=1)
            v = v.repeat_interleave(G, dim=1)
            o = self._attention(q, k, v, allowed).reshape(T, nq * hd)
            x = f32(x + f32(o @ Lw["wo"].T))
            xb, rs = bf(x), self._rs(x)
            g = f32(f32(xb @ Lw["wg"].T) * rs)
            u = f32(f32(xb @ Lw["wu"].T) * rs)
            hh = bf(g / (1.0 + torch.exp(-g)) * u)
            x = f32(x + f32(hh @ Lw["wd"].T))
        return self.head(x[torch.tensor(out_idx, device="cuda")])


def causal(T):
    return torch.ones(T, T, dtype=torch.bool).tril()


def entropy64(logits):
    """entropy_of (oracle.hpp:21-33) of softmax(logits), float64, nats."""
    lp = torch.log_softmax(logits.double(), dim=-1)
    return -(lp.exp() * lp).sum(-1)
