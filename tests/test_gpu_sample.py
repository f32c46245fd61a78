"""K4R — speculative rejection sampling on the model path (north_star 3; an extension the
reference does not have: SPEC.md:102 keeps it greedy-only, so parity is pinned by the plain-C
restatement oracle/restate.c or_model_rejection_verify, written from kernels/sample.cuh's rule).

Bar: accept lengths and sampled bonus ids bit-exact, final entropy within 1e-12 relative, on
synthetic rows (planted peaks, -inf-free ties, forced point-mass rows, top-p nuclei,
temperatures) and on real-model logits (ws_model_forward of the tiny and Llama-3.2-1B shapes);
plus whole runs in rejection mode: deterministic, independent of the batching (protocol
threads), and the Philox draw keyed by (seed, request, step, position) only.
"""
import ctypes as C
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import pyoracle as po  # noqa: E402
from paper_2602_18931_b200 import abi  # noqa: E402


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_18931_b200 as ws
    lib = ws.lib()
    lib.ws_op_verify_rejection_bf16.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                                C.c_float, C.c_float, C.c_void_p, C.c_void_p, C.c_uint64,
                                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    return lib


def run_gpu(L, logits, k, cands, probs, seed, reqs, steps, inv_temp, top_p, forced=None):
    n = len(reqs)
    V = logits.shape[1]
    dc = torch.tensor(cands, dtype=torch.int32, device="cuda")
    dp = torch.tensor(probs, dtype=torch.float64, device="cuda")
    dr = torch.tensor(reqs, dtype=torch.int64, device="cuda")
    ds = torch.tensor(steps, dtype=torch.int32, device="cuda")
    df = torch.tensor(forced, dtype=torch.int32, device="cuda") if forced is not None else None
    out = torch.zeros(n * C.sizeof(abi.VerifyOut), dtype=torch.uint8, device="cuda")
    rc = L.ws_op_verify_rejection_bf16(logits.data_ptr(), n, k, V, logits.stride(0), inv_temp, top_p, dc.data_ptr(),
                                       dp.data_ptr(), seed, dr.data_ptr(), ds.data_ptr(),
                                       df.data_ptr() if df is not None else None, out.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    arr = (abi.VerifyOut * n).from_buffer_copy(out.cpu().numpy().tobytes())
    return [(o.accepted, o.bonus, o.final_entropy) for o in arr]


def check(L, logits, k, cands, probs, seed, reqs, steps, inv_temp=1.0, top_p=1.0, forced=None):
    got = run_gpu(L, logits, k, cands, probs, seed, reqs, steps, inv_temp, top_p, forced)
    rows = logits.float().cpu().numpy()
    for j, (a, b, h) in enumerate(got):
        blk = rows[j * (k + 1):(j + 1) * (k + 1)]
        f = forced[j * (k + 1):(j + 1) * (k + 1)] if forced is not None else None
        wa, wb, wh = po.model_rejection_verify(blk, k, cands[j * k:(j + 1) * k], probs[j * k:(j + 1) * k], seed,
                                               reqs[j], steps[j], inv_temp, top_p, f)
        assert (a, b) == (wa, wb), (j, (a, b), (wa, wb))
        assert h == pytest.approx(wh, rel=1e-12, abs=1e-15)
    return got


def synth_case(V, n, k, seed, scale=2.0, greedy_frac=0.6):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(n * (k + 1), V, device="cuda", generator=g) * scale
    rng = random.Random(seed)
    peaks = [rng.randrange(V) for _ in range(n * (k + 1))]
    x[torch.arange(n * (k + 1)), torch.tensor(peaks, device="cuda")] += 14.0
    logits = x.to(torch.bfloat16)
    cands, probs = [], []
    for j in range(n):
        for i in range(k):
            row = j * (k + 1) + i
            cands.append(peaks[row] if rng.random() < greedy_frac else rng.randrange(V))
            probs.append(rng.choice([rng.random(), 1.0, 0.05]))
    reqs = [rng.randrange(1 << 40) for _ in range(n)]
    steps = [rng.randrange(1000) for _ in range(n)]
    return logits, cands, probs, reqs, steps, peaks


@pytest.mark.parametrize("V", [1000, 32768, 128256])
@pytest.mark.parametrize("top_p,inv_temp", [(1.0, 1.0), (0.9, 1.0), (0.5, 1.4), (1.0, 0.7)])
def test_rejection_vs_restatement(L, V, top_p, inv_temp):
    n, k = 12, 4
    logits, cands, probs, reqs, steps, _ = synth_case(V, n, k, V + int(top_p * 100))
    got = check(L, logits, k, cands, probs, 0x1234ABCD9876, reqs, steps, inv_temp, top_p)
    assert any(a > 0 for a, _, _ in got) and any(a < k for a, _, _ in got)


def test_rejection_forced_rows_and_ties(L):
    """Forced rows (point masses: the generation cap's EOS) and flat rows (many equal logits:
    the inverse CDF's id order and the nucleus' kept ties decide)."""
    n, k, V = 8, 4, 4096
    logits, cands, probs, reqs, steps, peaks = synth_case(V, n, k, 7)
    logits[3 * (k + 1):4 * (k + 1)] = 0.0  # a request with all-flat rows
    forced = [-1] * (n * (k + 1))
    for j in range(n):
        if j % 3 == 0:
            forced[j * (k + 1) + 2] = V - 1
            cands[j * k + 2] = V - 1 if j % 2 else cands[j * k + 2]
    for top_p in (1.0, 0.7):
        check(L, logits, k, cands, probs, 99, reqs, steps, 1.0, top_p, forced)


def test_rejection_on_real_model_logits(L):
    """The same bar on logits of real forwards (tiny and Llama-3.2-1B shapes, 2 layers)."""
    import paper_2602_18931_b200 as ws
    lib = ws.lib()
    lib.ws_model_create.argtypes = [C.c_char_p, C.c_uint64, C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
    lib.ws_model_destroy.argtypes = [C.c_void_p]
    lib.ws_model_forward.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                     C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    for name, V in (("tiny", 1000), ("llama3.2-1b:L2", 128256)):
        h = C.c_void_p()
        assert lib.ws_model_create(name.encode(), 3, 512, 64, 0, C.byref(h)) == 0
        try:
            n, k, T = 6, 4, 24
            rng = random.Random(11)
            toks = [rng.randrange(V) for _ in range(n * T)]
            i32 = lambda v: torch.tensor(v, dtype=torch.int32)  # noqa: E731
            pos = [p for _ in range(n) for p in range(T)]
            slot = list(range(n * T))
            groups = [x for j in range(n) for x in (j * T, T, j * T, 0, j * T, T, 0)]
            outs = [j * T + T - (k + 1) + i for j in range(n) for i in range(k + 1)]
            keep = [i32(toks), i32(pos), i32(slot), i32(groups), i32(slot), torch.zeros(n * T, dtype=torch.int64),
                    i32(outs)]
            logits = torch.empty(len(outs), V, dtype=torch.bfloat16, device="cuda")
            assert lib.ws_model_forward(h, n * T, keep[0].data_ptr(), keep[1].data_ptr(), keep[2].data_ptr(), n,
                                        keep[3].data_ptr(), n * T, keep[4].data_ptr(), keep[5].data_ptr(), len(outs),
                                        keep[6].data_ptr(), logits.data_ptr(), None) == 0
            torch.cuda.synchronize()
            am = logits.float().argmax(-1).tolist()
            cands = [am[j * (k + 1) + i] if rng.random() < 0.7 else rng.randrange(V) for j in range(n)
                     for i in range(k)]
            probs = [rng.random() for _ in range(n * k)]
            for top_p in (1.0, 0.8):
                check(L, logits, k, cands, probs, 5, list(range(n)), [1] * n, 1.0, top_p)
        finally:
            lib.ws_model_destroy(h)


def test_model_run_rejection_mode_deterministic():
    """Whole config-3-style runs in rejection mode on small shapes: identical per-request results
    across repeated runs and across protocol-thread counts (the draws depend only on the key
    and (request, step, position), the kernels are batch-invariant); every request completes."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_18931_b200 as ws
    ctx = ws.Context(0)
    try:
        ctx.load_models(abi.model_cfg("tiny", "tiny-draft", prompt_len=16, max_requests=8, max_ctx=64,
                                      plant_target=4.0, plant_draft=4.0, draft_plant_rate=0.8))

        def cfg(threads=1, top_p=1.0, seed=77):
            c = abi.config3(num_requests=8, k=4, seq_len=30, vocab=1000, eos=999)
            c.verify = abi.WS_VERIFY_REJECTION
            c.sample_seed = seed
            c.top_p = top_p
            c.host_threads = threads
            return c
        a = ctx.run_model_sim(cfg())
        b = ctx.run_model_sim(cfg())
        t = ctx.run_model_sim(cfg(threads=3))
        for x in (b, t):
            assert x.metrics_list() == a.metrics_list()
            assert x.ctrl_outputs() == a.ctrl_outputs()
            assert x.step_list() == a.step_list()
        assert all(m["tokens_committed"] == 30 for m in a.metrics_list())
        steps = a.step_list()
        assert any(s[3] > 0 for s in steps) and any(s[3] < 4 for s in steps)
        other = ctx.run_model_sim(cfg(seed=78))
        assert other.ctrl_outputs() != a.ctrl_outputs()  # the key matters
        nuc = ctx.run_model_sim(cfg(top_p=0.5))
        assert all(m["tokens_committed"] == 30 for m in nuc.metrics_list())
    finally:
        ctx.close()
