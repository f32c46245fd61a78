"""The batched Llama forward (K1 GEMMs + K2 attention + K6 plumbing) vs a plain PyTorch fp32
reference of the same architecture on the same weights: prefill, verify-style causal groups
over a cached prefix, and tree-style groups (prefix + explicit ancestor slots)."""
import ctypes as C
import math

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

SHAPES = {  # mirrors shape_by_name (csrc/model/llama.cu)
    "tiny": dict(layers=2, d=256, nq=4, nkv=2, hd=64, ffn=512, vocab=1000, theta=10000.0, factor=0.0, tied=False),
    "tiny128": dict(layers=2, d=512, nq=4, nkv=1, hd=128, ffn=1024, vocab=2000, theta=500000.0, factor=8.0,
                    tied=False),
}


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_18931_b200 as ws
    lib = ws.lib()
    lib.ws_model_create.argtypes = [C.c_char_p, C.c_uint64, C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
    lib.ws_model_destroy.argtypes = [C.c_void_p]
    lib.ws_model_copy_weight.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_void_p, C.c_int64]
    lib.ws_model_forward.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                     C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    return lib


def inv_freq(s):
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


class Ref:
    def __init__(self, lib, h, s):
        self.s = s
        d, nq, nkv, hd, ffn, V = s["d"], s["nq"], s["nkv"], s["hd"], s["ffn"], s["vocab"]

        def get(name, layer, n, shape):
            t = torch.empty(n, dtype=torch.bfloat16, device="cuda")
            assert lib.ws_model_copy_weight(h, name.encode(), layer, t.data_ptr(), n) == 0
            return t.view(*shape).float()
        self.emb = get("embed", 0, V * d, (V, d))
        self.lm = get("lm_head", 0, V * d, (V, d))
        self.fn = get("final_norm", 0, d, (d,))
        self.layers = []
        for l in range(s["layers"]):
            qkv = (nq + 2 * nkv) * hd
            wgu = get("wgu", l, 2 * ffn * d, (2 * ffn, d)).view(ffn // 16, 2, 16, d)
            self.layers.append(dict(
                an=get("attn_norm", l, d, (d,)), wqkv=get("wqkv", l, qkv * d, (qkv, d)),
                wo=get("wo", l, d * nq * hd, (d, nq * hd)), mn=get("mlp_norm", l, d, (d,)),
                wg=wgu[:, 0].reshape(ffn, d), wu=wgu[:, 1].reshape(ffn, d),
                wd=get("wdown", l, d * ffn, (d, ffn))))
        self.inv = inv_freq(s).cuda()

    def rms(self, x, w):
        return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + 1e-5) * w

    def rope(self, x, pos):  # x [T, H, hd]
        hd = x.shape[-1]
        ang = pos.float()[:, None] * self.inv[None, :]
        c, s_ = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
        a, b = x[..., :hd // 2], x[..., hd // 2:]
        return torch.cat([a * c - b * s_, b * c + a * s_], dim=-1)

    def logits(self, tokens):
        s = self.s
        nq, nkv, hd = s["nq"], s["nkv"], s["hd"]
        T = len(tokens)
        pos = torch.arange(T, device="cuda")
        x = self.emb[torch.tensor(tokens, device="cuda")]
        mask = torch.full((T, T), float("-inf"), device="cuda").triu(1)
        for Lw in self.layers:
            xn = self.rms(x, Lw["an"])
            qkv = xn @ Lw["wqkv"].T
            q = qkv[:, :nq * hd].view(T, nq, hd)
            k = qkv[:, nq * hd:(nq + nkv) * hd].view(T, nkv, hd)
            v = qkv[:, (nq + nkv) * hd:].view(T, nkv, hd)
            q, k = self.rope(q, pos), self.rope(k, pos)
            G = nq // nkv
            k = k.repeat_interleave(G, dim=1)
            v = v.repeat_interleave(G, dim=1)
            att = torch.einsum("thd,shd->hts", q, k) / math.sqrt(hd) + mask
            o = torch.einsum("hts,shd->thd", att.softmax(-1), v).reshape(T, nq * hd)
            x = x + o @ Lw["wo"].T
            xn = self.rms(x, Lw["mn"])
            h = torch.nn.functional.silu(xn @ Lw["wg"].T) * (xn @ Lw["wu"].T)
            x = x + h @ Lw["wd"].T
        return self.rms(x, self.fn) @ self.lm.T


def forward(lib, h, rows, groups, extra, out_rows, vocab, masks=None):
    i32 = lambda v: torch.tensor(v, dtype=torch.int32)  # noqa: E731
    tok, pos, slot = (i32([r[k] for r in rows]) for k in range(3))
    g = i32([x for grp in groups for x in (tuple(grp) + (0,) * (7 - len(grp)))])
    mk = torch.tensor(masks if masks else [0] * len(rows), dtype=torch.int64)
    ex = i32(extra if extra else [0])
    orows = i32(out_rows)
    out = torch.empty(len(out_rows), vocab, dtype=torch.bfloat16, device="cuda")
    rc = lib.ws_model_forward(h, len(rows), tok.data_ptr(), pos.data_ptr(), slot.data_ptr(), len(groups),
                              g.data_ptr(), len(extra), ex.data_ptr(), mk.data_ptr(), len(out_rows), orows.data_ptr(),
                              out.data_ptr(), None)
    assert rc == 0
    return out.float()


def check(got, ref):
    err = ((got - ref).norm(dim=-1) / ref.norm(dim=-1)).max().item()
    assert err < 3e-2, err
    top = ref.topk(2, dim=-1)
    clear = (top.values[:, 0] - top.values[:, 1]) > 0.05
    assert (got.argmax(-1)[clear] == ref.argmax(-1)[clear]).all()


@pytest.fixture(scope="module")
def tiny_pair():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_18931_b200 as ws
    from paper_2602_18931_b200 import abi
    ctx = ws.Context(0)
    ctx.load_models(abi.model_cfg("tiny", "tiny-draft", prompt_len=16, max_requests=8, max_ctx=64,
                                  plant_target=6.0, plant_draft=6.0, draft_plant_rate=0.8))
    yield ctx
    ctx.close()


def test_model_sim_speculative_equals_greedy(tiny_pair):
    """§8c contract 3: the speculative stream equals the plain greedy stream of the same target
    (batch-invariant kernels: a row's logits do not depend on the batch it is computed in)."""
    from paper_2602_18931_b200 import abi
    c = abi.config3(num_requests=6, k=4, seq_len=30, vocab=1000, eos=999)
    spec = tiny_pair.run_model_sim(c)
    base = abi.config3(num_requests=6, k=4, seq_len=30, vocab=1000, eos=999)
    base.mode = abi.WS_MODE_BASELINE
    greedy = tiny_pair.run_model_sim(base)
    assert spec.ctrl_outputs() == greedy.ctrl_outputs()
    assert spec.wrk_outputs() == spec.ctrl_outputs()
    for m in spec.metrics_list():
        assert m["tokens_committed"] == 30
    again = tiny_pair.run_model_sim(c)
    assert again.metrics_list() == spec.metrics_list()
    st = tiny_pair.model_stats()
    assert st["target_forwards"] > 0 and st["draft_forwards"] > 0


def test_model_sim_protocol_threads_equal_one_thread(tiny_pair):
    """host_threads protocol threads (each its own verify/draft streams and workspaces over a
    contiguous request range, forwards running concurrently) give the one-thread results."""
    from paper_2602_18931_b200 import abi
    c1 = abi.config3(num_requests=8, k=4, seq_len=30, vocab=1000, eos=999)
    one = tiny_pair.run_model_sim(c1)
    for t in (2, 3):
        ct = abi.config3(num_requests=8, k=4, seq_len=30, vocab=1000, eos=999)
        ct.host_threads = t
        many = tiny_pair.run_model_sim(ct)
        assert many.metrics_list() == one.metrics_list()
        assert many.ctrl_outputs() == one.ctrl_outputs()


def test_model_sim_k8_and_accept_stats(tiny_pair):
    from paper_2602_18931_b200 import abi
    c = abi.config3(num_requests=8, k=8, seq_len=36, vocab=1000, eos=999)
    b = tiny_pair.run_model_sim(c)
    steps = b.step_list()
    assert steps and all(0 <= s[3] <= 8 for s in steps)
    # resync points are consistent with the accept lengths (controller.hpp:246-252)
    for s in steps:
        assert bool(s[6] & abi.WS_STEP_SYNC_STALL) == (s[3] < 8)


@pytest.mark.parametrize("name", ["tiny", "tiny128"])
def test_forward_prefill_verify_tree(L, name):
    s = SHAPES[name]
    h = C.c_void_p()
    assert L.ws_model_create(name.encode(), 7, 64, 64, 0, C.byref(h)) == 0
    try:
        ref = Ref(L, h, s)
        V = s["vocab"]
        g = torch.Generator().manual_seed(3)
        A = torch.randint(0, V, (6,), generator=g).tolist()
        B = torch.randint(0, V, (3,), generator=g).tolist()
        Cc = torch.randint(0, V, (1,), generator=g).tolist()
        D = torch.randint(0, V, (4,), generator=g).tolist()
        # 1) prefill A into slots 0..5 (one causal group)
        rows = [(A[p], p, p) for p in range(6)]
        got = forward(L, h, rows, [(0, 6, 0, 0, 0, 6)], list(range(6)), list(range(6)), V)
        check(got, ref.logits(A))
        # 2) verify-style group over the cached prefix + a fresh prefill of D in the same batch
        rows = [(B[i], 6 + i, 6 + i) for i in range(3)] + [(D[p], p, 30 + p) for p in range(4)]
        groups = [(0, 3, 0, 6, 0, 3), (3, 4, 30, 0, 3, 4)]
        extra = [6, 7, 8, 30, 31, 32, 33]
        got = forward(L, h, rows, groups, extra, list(range(7)), V)
        check(got[:3], ref.logits(A + B)[6:9])
        check(got[3:], ref.logits(D))
        # 3) tree-style: prefix A (slots 0..5) + ancestor B[0] (slot 6) + own token at slot 20
        rows = [(Cc[0], 7, 20)]
        got = forward(L, h, rows, [(0, 1, 0, 6, 0, 2)], [6, 20], [0], V)
        check(got, ref.logits(A + [B[0], Cc[0]])[7:8])
        # 4) masked shared-prefix tree group: leaf X at pos 6 (slot 40) sees only itself; leaf Y
        #    at pos 7 (slot 41) sees ancestor B[0] (slot 6) and itself — one pass over prefix A
        X, Y = D[0], D[1]
        rows = [(X, 6, 40), (Y, 7, 41)]
        got = forward(L, h, rows, [(0, 2, 0, 6, 0, 3, 1)], [6, 40, 41], [0, 1], V, masks=[0b010, 0b101])
        check(got[0:1], ref.logits(A + [X])[6:7])
        check(got[1:2], ref.logits(A + [B[0], Y])[7:8])
    finally:
        L.ws_model_destroy(h)


def test_model_sim_split_placement_equals_shared():
    """Split placement (draft model on a second GPU) gives the same per-request
    results as both models on one GPU. Needs two GPUs."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import paper_2602_18931_b200 as ws
    from paper_2602_18931_b200 import abi
    outs = []
    for draft_dev in (-1, 1):
        ctx = ws.Context(0)
        ctx.load_models(abi.model_cfg("tiny", "tiny-draft", prompt_len=16, max_requests=8, max_ctx=64,
                                      plant_target=6.0, plant_draft=6.0, draft_plant_rate=0.8),
                        draft_device=draft_dev)
        b = ctx.run_model_sim(abi.config3(num_requests=8, k=4, seq_len=30, vocab=1000, eos=999))
        outs.append((b.metrics_list(), b.ctrl_outputs()))
        ctx.close()
    assert outs[0] == outs[1]


@pytest.mark.parametrize("lanes", ["2", "3"])
def test_model_sim_draft_lanes(tiny_pair, monkeypatch, lanes):
    """Several draft lanes per protocol thread (the next draft batch planned and launched while
    another runs on its own stream and workspace) give the one-lane per-request results."""
    import paper_2602_18931_b200 as ws
    from paper_2602_18931_b200 import abi
    c = abi.config3(num_requests=8, k=4, seq_len=30, vocab=1000, eos=999)
    ref = tiny_pair.run_model_sim(c)
    monkeypatch.setenv("WS_DRAFT_LANES", lanes)
    ctx = ws.Context(0)  # backends read the switch when created
    try:
        ctx.load_models(abi.model_cfg("tiny", "tiny-draft", prompt_len=16, max_requests=8, max_ctx=64,
                                      plant_target=6.0, plant_draft=6.0, draft_plant_rate=0.8))
        got = ctx.run_model_sim(c)
        assert got.ctrl_outputs() == ref.ctrl_outputs()
        assert got.metrics_list() == ref.metrics_list()
    finally:
        ctx.close()
