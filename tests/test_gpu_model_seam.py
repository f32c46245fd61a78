"""The drop-in at the reference's own seam (SURVEY §8b, §8c contract 2).

The reference's RequestSim (sim.hpp:166-416, compiled unmodified into oracle/_ref) runs its
own controller / worker state machines, scheduler and token trees; only its three model calls
(run_target_step at sim.hpp:297, draft_prediction at :307 and :314) are answered by the GPU
models through the per-call C ABI (ws_model_verify / ws_model_draft), via the fold-back seam
hooks of oracle/ref_shim.cpp. Its committed streams, per-request metrics, accept lengths,
bonus tokens, final entropies and resync / entropy-reset flags must equal ws_run_model_sim's
(our batched driver over the same models) bit for bit: the per-row predictions the GPU exports
drive the reference's state machines to exactly the run the B200 build produced.
"""
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import pyoracle as po  # noqa: E402
from paper_2602_18931_b200 import abi  # noqa: E402

CASES = [  # (target, draft, vocab, prompt_len, requests, seq_len, k, plant)
    ("tiny", "tiny-draft", 1000, 16, 6, 30, 4, 6.0),
    ("tiny", "tiny-draft", 1000, 16, 4, 36, 8, 6.0),
    ("llama3-8b:L2", "llama3.2-1b:L2", 128256, 32, 4, 24, 4, 16.0),
]


@pytest.mark.parametrize("target,draft,vocab,prompt,nreq,seq_len,k,plant", CASES)
def test_reference_requestsim_through_gpu_models(target, draft, vocab, prompt, nreq, seq_len, k, plant):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not po.ref_available():
        pytest.skip("oracle/_ref not built")
    import paper_2602_18931_b200 as ws
    ctx = ws.Context(0)
    try:
        ctx.load_models(abi.model_cfg(target, draft, prompt_len=prompt, max_requests=nreq, max_ctx=prompt + seq_len + 16,
                                      plant_target=plant, plant_draft=plant, draft_plant_rate=0.8))
        eos = vocab - 1 if vocab < 128256 else abi.LLAMA_EOS
        cfg = abi.config3(num_requests=nreq, k=k, seq_len=seq_len, vocab=vocab, eos=eos)
        ours = ctx.run_model_sim(cfg)

        ctx.model_open(k, seq_len, eos)
        ctx.model_prefill(list(range(nreq)))
        calls = {"verify": 0, "draft": 0}

        def verify_fn(req, committed, cands):
            calls["verify"] += 1
            return ctx.model_verify([(req, committed, cands)])[0]

        def draft_fn(req, kind, context, n_committed):
            calls["draft"] += 1
            return ctx.model_draft([(req, kind, context, n_committed)])[0]

        ref = po.ref_run_sim_models(cfg, verify_fn, draft_fn)
        assert calls["verify"] > 0 and calls["draft"] > 0
        assert ref.metrics_list() == ours.metrics_list()
        assert ref.ctrl_outputs() == ours.ctrl_outputs()
        assert ref.wrk_outputs() == ours.wrk_outputs()
        assert ref.step_list() == ours.step_list()
        assert sum(m["target_steps"] for m in ref.metrics_list()) == calls["verify"]
    finally:
        ctx.close()


def test_per_call_verify_rows_and_batching():
    """ws_model_verify over several jobs in one forward equals one job per call (batch
    invariance of the per-call path), and its exported rows are the walk's inputs: the accept
    length is the first row whose argmax differs from the candidate (run_target_step,
    oracle.hpp:127-139), bonus = that row's argmax, final entropy = its entropy."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import random

    import paper_2602_18931_b200 as ws
    ctx = ws.Context(0)
    try:
        ctx.load_models(abi.model_cfg("tiny", "tiny-draft", prompt_len=16, max_requests=8, max_ctx=64,
                                      plant_target=6.0, plant_draft=6.0, draft_plant_rate=0.8))
        k = 4
        ctx.model_open(k, 40, 999)
        rng = random.Random(5)
        jobs = [(r, [rng.randrange(1000) for _ in range(rng.randrange(0, 12))],
                 [rng.randrange(1000) for _ in range(k)]) for r in range(8)]
        # make some candidates the model's own greedy choice so accepts > 0 occur
        for i in range(0, 8, 2):
            r, committed, cands = jobs[i]
            for j in range(k):
                (_, bonus, _), = ctx.model_verify([(r, committed + cands[:j], [0] * k)])
                cands[j] = bonus
        batched, rows = ctx.model_verify(jobs, with_rows=True)
        single = [ctx.model_verify([j])[0] for j in jobs]
        assert batched == single
        for i, ((r, committed, cands), (a, b, h)) in enumerate(zip(jobs, batched)):
            rr = rows[i * (k + 1):(i + 1) * (k + 1)]
            acc = 0
            while acc < k and rr[acc].id[0] == cands[acc]:
                acc += 1
            assert (a, b, h) == (acc, rr[acc].id[0], rr[acc].entropy)
        assert any(a > 0 for a, _, _ in batched)
        # draft: batched == single; evict forgets the KV but not the answer
        djobs = [(r, abi.WS_JOB_WORKER_DRAFT, c + x[:2], len(c)) for r, c, x in jobs]
        db = [(p.n, tuple(p.id), p.entropy) for p in ctx.model_draft(djobs)]
        ds = [(p.n, tuple(p.id), p.entropy) for j in djobs for p in ctx.model_draft([j])]
        assert db == ds
        ctx.model_evict(3)
        again = ctx.model_draft([djobs[3]])[0]
        assert (again.n, tuple(again.id), again.entropy) == db[3]
    finally:
        ctx.close()
