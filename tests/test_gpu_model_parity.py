"""Model-path parity at the real shapes the bench runs (VERDICT r01 "what's weak" 1).

The batched forward of the Llama-3.1-8B shape (truncated to its first two layers: d 4096,
32/8 heads, hd 128, ffn 14336, V 128256) and of the full Llama-3.2-1B shape (16 layers, d 2048,
hd 64, ffn 8192, tied head) against tests/llama_ref.py, a float64 restatement that rounds to
bf16 / fp32 where the kernels do, on the same weights:

  * prefill: 104 requests' prompts of 128..227 tokens in ONE forward (104 causal groups, every
    context >= 4 of K2's 32-position KV tiles);
  * verify + catch-up: 104 groups over the cached prefixes in one forward — k+1 = 5 verify rows,
    and every fifth request a 40-row catch-up group (several vector-warp passes of K2);
  * worker tree groups: per request, speculative nodes written through one masked group, then
    four leaves with 64-bit ancestor masks in a second (the shared-prefix tree group of
    model_backend.cu submit_draft).

Two levels of comparison, because bf16 storage makes the end-to-end one noisy by construction:

* stage by stage (the kernels' own numerics), each stage fed the kernels' own inputs: layer-0
  K/V in the pool (K1 QKV GEMM + fused norm/RoPE/KV-append epilogue) from the embeddings; the
  last layer's attention output (K2) from the kernels' q and KV pool with the group's exact
  visibility; the logits (final norm + LM-head GEMM) from the kernels' final residual, and K3's
  entropy / argmax on them. Bar: 1e-3 relative per row (north_star), >= 99% of the bf16
  values bit-equal where the inputs are identical;
* end to end against the full float64 reference: every bf16 rounding point flips a few
  percent of its values whenever its fp32 input differs in the last bits (tensor-core
  accumulation order), and the next GEMM turns those flips into ~1e-4 relative input noise for
  the following rounding point. The measured end-to-end spread is therefore
  bounded, not 1e-3: logits E2E_TOL relative per row, entropy E2E_H_TOL relative, top-1 equal
  wherever the reference's top-2 margin exceeds E2E_MARGIN logits.
"""
import ctypes as C
import os
import random

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import llama_ref as lr  # noqa: E402  (tests/ is on sys.path under pytest)
from paper_2602_18931_b200 import abi  # noqa: E402

N_REQ = 104
S = 320          # slots per request: linear prefix [0, 280), tree nodes [280, 320)
TRIE0 = 280
STAGE_TOL = float(os.environ.get("WS_STAGE_TOL", "1e-3"))  # north_star: logits and entropy within 1e-3 relative
# Stage S3 is split in two so each kernel is checked on its own inputs: the final norm (bf16 rows
# from the kernels' fp32 residual) and the LM head (bf16 logits from the kernels' own final-norm
# rows). Both outputs are bf16: against the bf16-rounded fp64 reference an element differs by one
# ulp when the fp32 and fp64 values straddle a rounding boundary. Checked: no element more than one
# ulp off (plus, for logits near zero, 2^-10 of the row RMS: the fp32 and fp64 sums differ by more
# than their tiny ulp), the row error under 1e-3, and the bit-equal fractions. (Fed the fp64 norm
# instead, one flipped final-norm element of a large residual component moves a whole logit row by
# ~1e-3: measured 1.11e-3 on the 1B once its residual stream changed in the last bits.)
E2E_TOL = 3e-2     # end-to-end bf16 spread bound (see the module docstring)
E2E_H_TOL = 1e-3   # measured 1.2e-4 (8B:L2), 3.2e-5 (1B): the entropy meets the 1e-3 bar end to end
E2E_MARGIN = 0.25


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_18931_b200 as ws
    lib = ws.lib()
    lib.ws_model_create.argtypes = [C.c_char_p, C.c_uint64, C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
    lib.ws_model_destroy.argtypes = [C.c_void_p]
    lib.ws_model_forward.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                     C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.ws_op_row_stats_workspace_bytes.restype = C.c_size_t
    lib.ws_op_row_stats_workspace_bytes.argtypes = [C.c_uint32] * 3
    lib.ws_op_row_stats_bf16.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_float,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    return lib


class Batch:
    def __init__(self):
        self.tok, self.pos, self.slot, self.groups, self.extra, self.masks, self.out = [], [], [], [], [], [], []

    def group(self, rows, prefix_slot, prefix_len, extra_slots, masks=None):
        """rows: [(token, position, slot)]; extra_slots: the group's explicit slots (ancestors
        then its own rows' slots); masks: per-row bit masks over extra_slots (masked group)."""
        row0 = len(self.tok)
        for t, p, s in rows:
            self.tok.append(t)
            self.pos.append(p)
            self.slot.append(s)
        self.groups.append((row0, len(rows), prefix_slot, prefix_len, len(self.extra), len(extra_slots),
                            1 if masks else 0))
        self.extra += extra_slots
        self.masks += masks if masks else [0] * len(rows)
        return row0

    def run(self, lib, h, vocab):
        i32 = lambda v: torch.tensor(v, dtype=torch.int32)  # noqa: E731
        tok, pos, slot = i32(self.tok), i32(self.pos), i32(self.slot)
        g = i32([x for grp in self.groups for x in grp])
        ex = i32(self.extra or [0])
        mk = torch.tensor([m if m < 2 ** 63 else m - 2 ** 64 for m in self.masks], dtype=torch.int64)
        orows = i32(self.out)
        out = torch.empty(len(self.out), vocab, dtype=torch.bfloat16, device="cuda")
        rc = lib.ws_model_forward(h, len(self.tok), tok.data_ptr(), pos.data_ptr(), slot.data_ptr(),
                                  len(self.groups), g.data_ptr(), len(self.extra), ex.data_ptr(), mk.data_ptr(),
                                  len(self.out), orows.data_ptr(), out.data_ptr(), None)
        assert rc == 0
        torch.cuda.synchronize()
        return out


def k3_entropy(lib, logits):
    rows, V = logits.shape
    ws = torch.zeros(lib.ws_op_row_stats_workspace_bytes(rows, V, 0), dtype=torch.uint8, device="cuda")
    out = torch.zeros(rows * C.sizeof(abi.Pred), dtype=torch.uint8, device="cuda")
    assert lib.ws_op_row_stats_bf16(logits.data_ptr(), rows, V, V, 1.0, out.data_ptr(), None, ws.data_ptr(),
                                    torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    arr = (abi.Pred * rows).from_buffer_copy(out.cpu().numpy().tobytes())
    return [(p.id[0], p.entropy) for p in arr]


def rel_rows(a, b):
    return (a - b).norm(dim=-1) / b.norm(dim=-1).clamp(min=1e-30)


class Stages:
    """Runs one forward and checks it stage by stage and end to end (see the module docstring)."""

    def __init__(self, lib, h, name, ref):
        self.lib, self.h, self.ref = lib, h, ref
        self.s = lr.shape(name)
        self.worst = {"kv0": 0.0, "attn": 0.0, "norm": 0.0, "head": 0.0, "k3_h": 0.0, "e2e": 0.0, "e2e_h": 0.0}
        self.eq = {"kv0": [], "attn": [], "norm": [], "head": []}
        self.rows = 0

    def grab(self, which, n):
        t = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        assert self.lib.ws_model_copy_weight(self.h, which.encode(), 0, t.data_ptr(), n) == 0
        return t

    def run(self, b):
        s = self.s
        V, d, nq, nkv, hd, nl = s["vocab"], s["d"], s["nq"], s["nkv"], s["hd"], s["layers"]
        logits = b.run(self.lib, self.h, V)
        n = len(b.tok)
        pool_n = nl * N_REQ * S * nkv * hd
        kp = self.grab("k_pool", pool_n).view(nl, N_REQ * S, nkv * hd)
        vp = self.grab("v_pool", pool_n).view(nl, N_REQ * S, nkv * hd)
        cap = self.cap  # the workspace's row capacity (max rows of any forward so far)
        x = self.grab("ws_x", 2 * cap * d).view(torch.float32).view(cap, d)[:n].double()
        q = self.grab("ws_q", cap * nq * hd).view(cap, nq, hd)[:n].double()
        at = self.grab("ws_attn", cap * nq * hd).view(cap, nq * hd)[:n].double()
        # S1: layer-0 K/V of every written row from its embedding
        k0, v0 = self.ref.kv0(b.tok, b.pos)
        slots = torch.tensor(b.slot, device="cuda")
        for got, want in ((kp[0, slots].double(), k0), (vp[0, slots].double(), v0)):
            r = rel_rows(got, want).max().item()
            self.worst["kv0"] = max(self.worst["kv0"], r)
            self.eq["kv0"].append((got == want).double().mean().item())
            assert r < STAGE_TOL, ("kv0", r)
        # S2: last-layer attention from the kernels' q and KV pool, group by group
        G = nq // nkv
        for (row0, nr, ps, pl, eo, el, masked) in b.groups:
            keys = list(range(ps, ps + pl)) + b.extra[eo:eo + el]
            ks = torch.tensor(keys, device="cuda")
            K = kp[nl - 1, ks].double().view(len(keys), nkv, hd).repeat_interleave(G, 1)
            Vv = vp[nl - 1, ks].double().view(len(keys), nkv, hd).repeat_interleave(G, 1)
            allowed = torch.zeros(nr, len(keys), dtype=torch.bool)
            allowed[:, :pl] = True
            xi = torch.arange(el)[None, :]
            if masked:
                mk = torch.tensor(b.masks[row0:row0 + nr], dtype=torch.int64)[:, None]
                allowed[:, pl:] = ((mk >> xi) & 1) == 1
            else:
                allowed[:, pl:] = xi <= (el - nr + torch.arange(nr))[:, None]
            want = self.ref._attention(q[row0:row0 + nr], K, Vv, allowed.cuda()).reshape(nr, nq * hd)
            got = at[row0:row0 + nr]
            r = rel_rows(got, want).max().item()
            self.worst["attn"] = max(self.worst["attn"], r)
            self.eq["attn"].append((got == want).double().mean().item())
            assert r < STAGE_TOL, ("attn", row0, r)
        # S3a: final norm from the kernels' residual rows — bf16 rows, one-ulp flips only
        n_out = len(b.out)
        # the workspace's output-row capacity: 256 at creation, grown to the largest n_out so far
        self.cap_out = max(getattr(self, "cap_out", 256), n_out)
        xo = self.grab("ws_xo", self.cap_out * d).view(self.cap_out, d)[:n_out].double()
        xs = x[torch.tensor(b.out, device="cuda")]
        xo_want = lr.bf(xs * torch.rsqrt((xs * xs).mean(-1, keepdim=True) + lr.EPS) * self.ref.fn)
        r = rel_rows(xo, xo_want).max().item()
        self.worst["norm"] = max(self.worst["norm"], r)
        self.eq["norm"].append((xo == xo_want).double().mean().item())
        ulp_n = torch.exp2(torch.floor(torch.log2(torch.maximum(xo.abs(), xo_want.abs()).clamp(min=1e-30))) - 7)
        assert bool(((xo - xo_want).abs() <= ulp_n * 1.0001).all()), ("norm", "more than one bf16 ulp")
        assert r < STAGE_TOL, ("norm", r)
        # S3b: LM head from the kernels' own final-norm rows, then K3 on our logits
        want = lr.bf(xo @ self.ref.lm.T)
        got_l = logits.double()
        r = rel_rows(got_l, want).max().item()
        self.worst["head"] = max(self.worst["head"], r)
        # one bf16 ulp of the value, plus the fp32-vs-fp64 accumulation difference for logits near
        # zero (cancellation), bounded at 2^-10 of the row's RMS
        ulp = torch.exp2(torch.floor(torch.log2(torch.maximum(got_l.abs(), want.abs()).clamp(min=1e-30))) - 7)
        slack = want.pow(2).mean(-1, keepdim=True).sqrt() * 2.0 ** -10
        excess = (got_l - want).abs() - ulp * 1.0001 - slack
        worst_x = excess.max().item()
        if worst_x > 0:
            bad = (excess > 0).nonzero()[:5].tolist()
            info = [(i, j, got_l[i, j].item(), want[i, j].item(), ulp[i, j].item(), slack[i, 0].item(),
                     rel_rows(got_l[i:i + 1], want[i:i + 1]).item()) for i, j in bad]
            raise AssertionError(("head", "logits more than one bf16 ulp off", int((excess > 0).sum().item()), info))
        self.eq["head"].append((got_l == want).double().mean().item())
        assert r < STAGE_TOL, ("head", r)
        ours = k3_entropy(self.lib, logits)
        h_ref = lr.entropy64(want)
        top = want.topk(2, dim=-1)
        clear = (top.values[:, 0] - top.values[:, 1]) > top.values[:, 0].abs() * 2.0 ** -7
        for i, (id0, hh) in enumerate(ours):
            e = abs(hh - h_ref[i].item()) / max(h_ref[i].item(), 1e-12)
            self.worst["k3_h"] = max(self.worst["k3_h"], e)
            assert e < STAGE_TOL, ("k3 entropy", i, hh, h_ref[i].item())
            if clear[i]:
                assert id0 == top.indices[i, 0].item(), ("k3 argmax", i)
        self.rows += len(b.out)
        return logits, ours

    def end_to_end(self, got, ours, want, what):
        r = rel_rows(got.double(), want)
        self.worst["e2e"] = max(self.worst["e2e"], r.max().item())
        assert r.max().item() < E2E_TOL, (what, r.max().item())
        h_ref = lr.entropy64(want)
        top = want.topk(2, dim=-1)
        for i, (id0, hh) in enumerate(ours):
            e = abs(hh - h_ref[i].item()) / max(h_ref[i].item(), 1e-12)
            self.worst["e2e_h"] = max(self.worst["e2e_h"], e)
            assert e < E2E_H_TOL, (what, i, hh, h_ref[i].item())
            if (top.values[i, 0] - top.values[i, 1]).item() > E2E_MARGIN:
                assert id0 == top.indices[i, 0].item(), (what, "argmax", i)


@pytest.mark.parametrize("name", ["llama3-8b:L2", "llama3.2-1b"])
def test_forward_real_shapes(L, name):
    s = lr.shape(name)
    V = s["vocab"]
    h = C.c_void_p()
    assert L.ws_model_create(name.encode(), 11, N_REQ * S, 256, 0, C.byref(h)) == 0
    try:
        ref = lr.RefModel(L, h, name)
        st = Stages(L, h, name, ref)
        rng = random.Random(1234)
        P = [128 + (r * 37) % 100 for r in range(N_REQ)]
        prompt = [[rng.randrange(V) for _ in range(P[r])] for r in range(N_REQ)]

        # ---- (1) prefill: one causal group per request, all in one forward ----
        b = Batch()
        want = []
        for r in range(N_REQ):
            base = r * S
            row0 = b.group([(prompt[r][p], p, base + p) for p in range(P[r])], base, 0,
                           [base + p for p in range(P[r])])
            picks = [P[r] - 1, P[r] // 2] if r % 4 else [P[r] - 1, P[r] // 2, 0, 31, 32, 100]
            for p in picks:
                b.out.append(row0 + p)
            want.append((r, picks))
        st.cap = max(256, len(b.tok))
        got, ours = st.run(b)
        o = 0
        for r, picks in want:
            ref_l = ref.logits(prompt[r], list(range(P[r])), lr.causal(P[r]), picks)
            st.end_to_end(got[o:o + len(picks)], ours[o:o + len(picks)], ref_l, f"prefill r{r}")
            o += len(picks)

        # ---- (2) verify (k+1 = 5 rows) and catch-up (40 rows) groups over the cached prefixes ----
        b = Batch()
        new = {}
        for r in range(N_REQ):
            n = 40 if r % 5 == 0 else 5
            base = r * S
            toks = [rng.randrange(V) for _ in range(n)]
            new[r] = toks
            row0 = b.group([(toks[i], P[r] + i, base + P[r] + i) for i in range(n)], base, P[r],
                           [base + P[r] + i for i in range(n)])
            b.out += [row0 + i for i in range(n)]
        got, ours = st.run(b)
        o = 0
        for r in range(N_REQ):
            n = len(new[r])
            T = P[r] + n
            ref_l = ref.logits(prompt[r] + new[r], list(range(T)), lr.causal(T), list(range(P[r], T)))
            st.end_to_end(got[o:o + n], ours[o:o + n], ref_l, f"verify r{r}")
            o += n

        # ---- (3) worker tree: speculative nodes, then leaves with ancestor masks ----
        # nodes (token, depth, parent): n0 (d0), n1 (d1, parent n0), n2 (d0, sibling of n0);
        # leaves: l0 under n1, l1 under n2, l2 at the root, l3 under n0
        par = [-1, 0, -1, 1, 2, -1, 0]  # n0 n1 n2 | l0 l1 l2 l3
        depth = [0, 1, 0, 2, 1, 0, 1]

        def mask_of(i):
            m = 0
            while i >= 0:
                m |= 1 << i
                i = par[i]
            return m
        tree = {}
        b1, b2 = Batch(), Batch()
        for r in range(N_REQ):
            base, t0 = r * S, r * S + TRIE0
            tk = [rng.randrange(V) for _ in range(7)]
            slots = [t0 + i for i in range(7)]
            tree[r] = tk
            row0 = b1.group([(tk[i], P[r] + depth[i], slots[i]) for i in range(3)], base, P[r], slots[:3],
                            masks=[mask_of(i) for i in range(3)])
            b1.out += [row0 + i for i in range(3)]
            # the leaf group's extras: the three ancestors, then the four leaves' own slots
            row0 = b2.group([(tk[i], P[r] + depth[i], slots[i]) for i in range(3, 7)], base, P[r], slots,
                            masks=[mask_of(i) for i in range(3, 7)])
            b2.out += [row0 + i for i in range(4)]
        got1, ours1 = st.run(b1)
        got2, ours2 = st.run(b2)
        for r in range(N_REQ):
            tk = tree[r]
            T = P[r] + 7
            allowed = torch.zeros(T, T, dtype=torch.bool)
            allowed[:P[r], :P[r]] = lr.causal(P[r])
            for i in range(7):
                allowed[P[r] + i, :P[r]] = True
                j = i
                while j >= 0:
                    allowed[P[r] + i, P[r] + j] = True
                    j = par[j]
            ref_l = ref.logits(prompt[r] + tk, list(range(P[r])) + [P[r] + dd for dd in depth], allowed,
                               list(range(P[r], T)))
            st.end_to_end(got1[3 * r:3 * r + 3], ours1[3 * r:3 * r + 3], ref_l[:3], f"tree nodes r{r}")
            st.end_to_end(got2[4 * r:4 * r + 4], ours2[4 * r:4 * r + 4], ref_l[3:], f"tree leaves r{r}")
        eq = {k: min(v) for k, v in st.eq.items()}
        print(f"\n{name}: {st.rows} output rows; worst relative error per stage "
              + ", ".join(f"{k} {v:.2e}" for k, v in st.worst.items())
              + "; min bit-equal fraction " + ", ".join(f"{k} {v:.4f}" for k, v in eq.items()))
        assert eq["kv0"] >= 0.99 and eq["attn"] >= 0.95 and eq["norm"] >= 0.99 and eq["head"] >= 0.95, eq
    finally:
        L.ws_model_destroy(h)


def test_model_sim_plant_off_speculative_equals_greedy():
    """A config-3 slice at the real shapes with the planted bias OFF: every argmax then depends
    on the forward (no +16 logit decides it), so spec == greedy exercises the kernels' batch
    invariance on the bench shapes rather than the plant (§8c contract 3)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_18931_b200 as ws
    ctx = ws.Context(0)
    try:
        ctx.load_models(abi.model_cfg("llama3-8b", "llama3.2-1b", max_requests=12, max_ctx=192,
                                      plant_target=0.0, plant_draft=0.0))
        c = abi.config3(num_requests=12, k=4, seq_len=24)
        spec = ctx.run_model_sim(c)
        base = abi.config3(num_requests=12, k=4, seq_len=24)
        base.mode = abi.WS_MODE_BASELINE
        greedy = ctx.run_model_sim(base)
        assert spec.ctrl_outputs() == greedy.ctrl_outputs()
        assert spec.wrk_outputs() == spec.ctrl_outputs()
        assert all(m["tokens_committed"] == 24 for m in spec.metrics_list())
        # with no shared bias the random-init pair rarely agrees: most verify steps reject
        steps = spec.step_list()
        assert steps and sum(1 for s in steps if s[3] < 4) > len(steps) // 2
    finally:
        ctx.close()


def test_split_k_row_slices_with_fused_norm():
    """GEMM split-K row slicing (workspace too small for one launch) with the fused
    RMSNorm on must give the logits of the unsliced cluster split-K (bit for bit). Run in
    subprocesses: the GEMM switches are read once per process."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = os.path.join(root, "tests", "_split_slice_probe.py")
    outs = []
    for extra in ({}, {"WS_GEMM_DSMEM": "0", "WS_GEMM_WS_ROWS": "128"}):
        env = dict(os.environ, WS_GEMM_CSPLIT="1", **extra)
        r = subprocess.run([sys.executable, script], capture_output=True, text=True, env=env, cwd=root,
                           timeout=600)
        assert r.returncode == 0, r.stderr
        outs.append(r.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1], outs
