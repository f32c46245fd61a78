"""Wall-clock mode (the reference's networked runtime brought in-box, runtime.hpp:153-386):
controller and worker state machines against real time, model steps completing with their GPU
work, proposals / validations on host queues delayed by rtt/2 (LatencyEmulator, net.hpp:149-163).

* Greedy verify makes the committed stream independent of timing: every request's stream equals
  the plain greedy stream of the same target (§8c contract 3) whatever the RTT.
* The decision log replays through the REFERENCE's own controller (oracle/_ref,
  ref_replay_model_log, the replay_decision_log pattern of runtime.hpp:404-454): every launch the
  reference makes equals the logged one, t_update matches after every turn, and the replayed
  committed streams and controller counters equal the run's.
"""
import os

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import pyoracle as po  # noqa: E402
from paper_2602_18931_b200 import abi  # noqa: E402

CASES = [("tiny", "tiny-draft", 1000, 16, 6.0, 20000), ("tiny", "tiny-draft", 1000, 16, 6.0, 60000),
         ("llama3-8b:L2", "llama3.2-1b:L2", 128256, 32, 16.0, 20000)]


@pytest.mark.parametrize("target,draft,vocab,prompt,plant,rtt", CASES)
def test_wallclock_run_replays_in_reference(target, draft, vocab, prompt, plant, rtt, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_18931_b200 as ws
    ctx = ws.Context(0)
    try:
        nreq, seq_len = 6, 30
        ctx.load_models(abi.model_cfg(target, draft, prompt_len=prompt, max_requests=nreq, max_ctx=prompt + seq_len + 16,
                                      plant_target=plant, plant_draft=plant, draft_plant_rate=0.8))
        eos = vocab - 1 if vocab < 128256 else abi.LLAMA_EOS
        c = abi.config3(num_requests=nreq, k=4, seq_len=seq_len, vocab=vocab, eos=eos)
        c.rtt, c.r_estimate = rtt, -1
        log = str(tmp_path / "decisions.ndjson")
        run = ctx.run_model_wallclock(c, decision_log=log)
        base = abi.config3(num_requests=nreq, k=4, seq_len=seq_len, vocab=vocab, eos=eos)
        base.mode = abi.WS_MODE_BASELINE
        greedy = ctx.run_model_sim(base)
        assert run.ctrl_outputs() == greedy.ctrl_outputs()
        m = run.metrics_list()
        assert all(x["tokens_committed"] == seq_len for x in m)
        assert all(x["latency"] > 0 for x in m)
        if not po.ref_available():
            pytest.skip("oracle/_ref not built")
        rep, turns = po.ref_replay_model_log(c, log)
        with open(log) as f:
            assert turns == sum(1 for line in f if line.strip())
        assert rep.ctrl_outputs() == run.ctrl_outputs()
        keys = ("tokens_committed", "target_steps", "ctrl_draft_passes", "ctrl_local_draft_steps",
                "ctrl_catchup_batches", "sync_stalls", "entropy_resets", "stale_specs")
        for a, b in zip(rep.metrics_list(), m):
            assert {k: a[k] for k in keys} == {k: b[k] for k in keys}
    finally:
        ctx.close()


def test_wallclock_baseline_mode_uses_local_drafts_only():
    """Baseline mode in wall-clock time: no worker, every draft is the controller's own."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_18931_b200 as ws
    ctx = ws.Context(0)
    try:
        ctx.load_models(abi.model_cfg("tiny", "tiny-draft", prompt_len=16, max_requests=4, max_ctx=64,
                                      plant_target=6.0, plant_draft=6.0, draft_plant_rate=0.8))
        c = abi.config3(num_requests=4, k=4, seq_len=24, vocab=1000, eos=999)
        c.mode = abi.WS_MODE_BASELINE
        b = ctx.run_model_wallclock(c)
        assert all(x["worker_draft_steps"] == 0 and x["ctrl_draft_passes"] > 0 for x in b.metrics_list())
    finally:
        ctx.close()
