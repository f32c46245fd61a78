"""ORACLE — TEST INFRASTRUCTURE ONLY: the CPU baseline of the config-3 workload, measured end
to end (bench.py's cpu_baseline leg and --impl reference arm; never on the product path).

The reference has no model. Its CPU path for this workload is therefore: the
reference's own RequestSim (sim.hpp:166-416, compiled unmodified into oracle/_ref) with its three
model calls (sim.hpp:297, :307, :314) answered by a CPU implementation of the same Llama-shape
pair — here torch on the host cores (bf16 weights, random-init with std 0.02, the GPU run's planted
bigram bias and generation cap, so draft/target agreement and sequence lengths match the GPU
workload). Requests run one at a time, each model call is one forward with a per-request KV
cache reused by longest common prefix (the CPU analogue of the GPU caches). The measured
quantity is committed tokens per wall second.
"""
import math
import os
import random
import time

import torch

from oracle import pyoracle as po

SHAPES = {  # shape_by_name (csrc/model/llama.cu)
    "llama3-8b": dict(layers=32, d=4096, nq=32, nkv=8, hd=128, ffn=14336, vocab=128256, theta=500000.0,
                      factor=8.0, tied=False),
    "llama3.2-1b": dict(layers=16, d=2048, nq=32, nkv=8, hd=64, ffn=8192, vocab=128256, theta=500000.0,
                        factor=32.0, tied=True),
    "tiny": dict(layers=2, d=256, nq=4, nkv=2, hd=64, ffn=512, vocab=1000, theta=10000.0, factor=0.0, tied=False),
    "tiny-draft": dict(layers=1, d=256, nq=4, nkv=2, hd=64, ffn=512, vocab=1000, theta=10000.0, factor=0.0,
                       tied=True),
}
M64 = (1 << 64) - 1


def splitmix64(x):  # model_backend.cu splitmix64
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


class CpuLlama:
    def __init__(self, name, seed):
        s = self.s = SHAPES[name]
        g = torch.Generator().manual_seed(seed)
        d, nq, nkv, hd, ffn, V = s["d"], s["nq"], s["nkv"], s["hd"], s["ffn"], s["vocab"]
        # one 16M-element seeded N(0, 0.02) block, tiled into every weight tensor at memcpy speed
        # (each tensor its own memory, so the forward streams the full model like the GPU's)
        block = (torch.randn(1 << 24, generator=g) * 0.02).to(torch.bfloat16)

        def w(*shape):
            n = math.prod(shape)
            out = torch.empty(n, dtype=torch.bfloat16)
            for o in range(0, n, block.numel()):
                m = min(block.numel(), n - o)
                out[o:o + m].copy_(block[(o // 7) % 4096:][:m] if m <= block.numel() - 4096 else block[:m])
            return out.view(*shape)
        self.emb = w(V, d)
        self.lm = self.emb if s["tied"] else w(V, d)
        self.layers = [dict(qkv=w((nq + 2 * nkv) * hd, d), o=w(d, nq * hd), gu=w(2 * ffn, d), dn=w(d, ffn))
                       for _ in range(s["layers"])]
        inv = []
        for i in range(hd // 2):
            f = 1.0 / (s["theta"] ** (2.0 * i / hd))
            if s["factor"] > 0:
                wl = 2 * math.pi / f
                if wl > 8192.0:
                    f = f / s["factor"]
                elif wl >= 2048.0:
                    sm = (8192.0 / wl - 1.0) / 3.0
                    f = (1 - sm) * f / s["factor"] + sm * f
            inv.append(f)
        self.inv = torch.tensor(inv, dtype=torch.float32)

    def new_cache(self):
        return dict(tokens=[], k=[None] * self.s["layers"], v=[None] * self.s["layers"])

    def forward(self, cache, ctx, want):
        """Feeds ctx[lcp:] after the cached prefix (longest common prefix with cache['tokens'],
        at most len(ctx) - want so the last `want` rows are computed); returns fp32 logits of the
        last `want` rows."""
        s = self.s
        nq, nkv, hd = s["nq"], s["nkv"], s["hd"]
        lcp = 0
        old = cache["tokens"]
        limit = min(len(old), len(ctx) - want)
        while lcp < limit and old[lcp] == ctx[lcp]:
            lcp += 1
        new = ctx[lcp:]
        T = len(new)
        pos = torch.arange(lcp, lcp + T, dtype=torch.float32)
        ang = pos[:, None] * self.inv[None, :]
        cos, sin = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
        x = self.emb[torch.tensor(new)].float()
        G = nq // nkv
        for li, W in enumerate(self.layers):
            xn = (x * torch.rsqrt((x * x).mean(-1, keepdim=True) + 1e-5)).to(torch.bfloat16)
            qkv = (xn @ W["qkv"].T).float()
            q = qkv[:, :nq * hd].view(T, nq, hd)
            k = qkv[:, nq * hd:(nq + nkv) * hd].view(T, nkv, hd)
            v = qkv[:, (nq + nkv) * hd:].view(T, nkv, hd)

            def rope(t):
                a, b = t[..., :hd // 2], t[..., hd // 2:]
                return torch.cat([a * cos - b * sin, b * cos + a * sin], -1)
            q, k = rope(q), rope(k)
            kc, vc = cache["k"][li], cache["v"][li]
            K = k if kc is None or lcp == 0 else torch.cat([kc[:lcp], k])
            Vv = v if vc is None or lcp == 0 else torch.cat([vc[:lcp], v])
            cache["k"][li], cache["v"][li] = K, Vv
            S = K.shape[0]
            att = torch.einsum("thd,shd->hts", q, K.repeat_interleave(G, 1)) / math.sqrt(hd)
            mask = torch.arange(S)[None, :] > (lcp + torch.arange(T))[:, None]
            att = att.masked_fill(mask[None], float("-inf")).softmax(-1)
            o = torch.einsum("hts,shd->thd", att, Vv.repeat_interleave(G, 1)).reshape(T, nq * hd)
            x = x + (o.to(torch.bfloat16) @ W["o"].T).float()
            xn = (x * torch.rsqrt((x * x).mean(-1, keepdim=True) + 1e-5)).to(torch.bfloat16)
            gu = (xn @ W["gu"].T).float().view(T, -1, 2, 16)
            g, u = gu[:, :, 0].reshape(T, -1), gu[:, :, 1].reshape(T, -1)
            x = x + ((g * torch.sigmoid(g) * u).to(torch.bfloat16) @ W["dn"].T).float()
        cache["tokens"] = list(ctx)
        xo = x[-want:]
        xo = (xo * torch.rsqrt((xo * xo).mean(-1, keepdim=True) + 1e-5)).to(torch.bfloat16)
        return (xo @ self.lm.T).float()


class CpuPair:
    """The config-3 pair on the CPU with the GPU run's plant / cap semantics (model_backend.cu)."""

    def __init__(self, target="llama3-8b", draft="llama3.2-1b", seed=1, prompt_len=128, seq_len=100, k=4,
                 eos=128001, plant=16.0, draft_plant_rate=0.8):
        self.t, self.d = CpuLlama(target, seed * 2 + 1), CpuLlama(draft, seed * 2 + 2)
        self.seed, self.P, self.L, self.k, self.eos, self.plant = seed, prompt_len, seq_len, k, eos, plant
        self.rate = draft_plant_rate
        self.V = self.t.s["vocab"]
        self.prompts, self.caches = {}, {}

    def prompt(self, r):
        if r not in self.prompts:
            g = random.Random((self.seed << 20) ^ (r + 1))
            self.prompts[r] = [g.randrange(self.V - 256) for _ in range(self.P)]
        return self.prompts[r]

    def planted(self, t, draft):
        if draft and (splitmix64(t ^ 0xD1B54A32D192ED03 ^ self.seed) % 1000000) >= self.rate * 1e6:
            return -1
        return splitmix64(t ^ 0xA0761D6478BD642F ^ self.seed) % (self.V - 256)

    def cache(self, r, which):
        key = (r, which)
        if key not in self.caches:
            self.caches[key] = (self.t if which == "t" else self.d).new_cache()
        return self.caches[key]

    def _rows(self, model, cache, ctx, want, draft):
        lg = model.forward(cache, ctx, want)
        n = len(ctx)
        for i in range(want):
            pl = self.planted(ctx[n - want + i], draft)
            if pl >= 0:
                lg[i, pl] += self.plant
        return lg

    def forced(self, pos):
        return (pos + 1 - self.P) >= self.L - 1

    def verify(self, r, committed, cands):
        ctx = self.prompt(r) + committed + cands
        lg = self._rows(self.t, self.cache(r, "t"), ctx, self.k + 1, False)
        base_pos = len(ctx) - self.k - 1
        ids, ents = [], []
        for i in range(self.k + 1):
            if self.forced(base_pos + i):
                ids.append(self.eos)
                ents.append(0.0)
                continue
            lp = torch.log_softmax(lg[i].double(), -1)
            ids.append(int(torch.argmax(lg[i])))
            ents.append(float(-(lp.exp() * lp).sum()))
        a = 0
        while a < self.k and ids[a] == cands[a]:
            a += 1
        return a, ids[a], ents[a]

    def draft(self, r, kind, context, n_committed):
        from paper_2602_18931_b200 import abi
        ctx = self.prompt(r) + context
        p = abi.Pred()
        if self.forced(len(ctx) - 1):
            p.n, p.id[0], p.prob[0], p.entropy = 1, self.eos, 1.0, 0.0
            return p
        lg = self._rows(self.d, self.cache(r, "c" if kind == 1 else "w"), ctx, 1, True)[0]
        pr = torch.softmax(lg.double(), -1)
        top = torch.topk(pr, 2)
        p.n = 2
        p.id[0], p.id[1] = int(top.indices[0]), int(top.indices[1])
        p.prob[0], p.prob[1] = float(top.values[0]), float(top.values[1])
        lp = torch.log(pr.clamp_min(1e-300))
        p.entropy = float(-(pr * lp).sum())
        return p


def prefill(pair, r):
    """The prompt's KV (positions [0, P-1)) in the request's target and both draft caches, as the
    GPU run's prefill phase does before its timed protocol."""
    head = pair.prompt(r)[:-1]
    pair.t.forward(pair.cache(r, "t"), head, 1)
    for which in ("c", "w"):
        pair.d.forward(pair.cache(r, which), head, 1)


def measure(requests=1, first=0, threads=None, pair=None, prefilled=True):
    """Committed tokens per wall second of the reference's RequestSim over requests
    [first, first + requests) with the CPU pair answering its model calls; prompts prefilled
    before the clock starts (prefilled=True). Returns (tokens/s, tokens, seconds, threads)."""
    from paper_2602_18931_b200 import abi
    threads = threads or os.cpu_count() or 1
    torch.set_num_threads(threads)
    pair = pair or CpuPair()
    pair.caches.clear()
    c = abi.config3(num_requests=first + requests, k=pair.k, seq_len=pair.L, vocab=pair.V, eos=pair.eos)
    c.first_request, c.local_requests = first, requests
    if prefilled:
        for r in range(first, first + requests):
            prefill(pair, r)
    t0 = time.perf_counter()
    b = po.ref_run_sim_models(c, lambda r, cm, cd: pair.verify(r, cm, cd),
                              lambda r, kind, ctx, nc: pair.draft(r, kind, ctx, nc),
                              with_tokens=False, with_steps=False)
    el = time.perf_counter() - t0
    toks = sum(m["tokens_committed"] for m in b.metrics_list())
    return toks / el, toks, el, threads
