"""Teacher-forced trace export: the GPU model pair's behaviour written in the
reference's NDJSON trace format, checked three ways — the format's validation rules, our own
model run commits exactly the exported greedy path, and the reference's trace oracle
(oracle/_ref, OracleKind::trace) replays the file with the same per-request results as our K9
path replaying the records it dealt."""
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

L = 30       # generated tokens of the model run (the cap: index L-1 is EOS)
N = 6
EOS = 999


def expected_commit(greedy):
    out = []
    for t in greedy:
        out.append(t)
        if t == EOS:
            return out
    return out + [EOS]


@pytest.fixture(scope="module")
def pair():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_18931_b200 as ws
    from paper_2602_18931_b200 import abi
    ctx = ws.Context(0)
    ctx.load_models(abi.model_cfg("tiny", "tiny-draft", prompt_len=16, max_requests=8, max_ctx=64,
                                  plant_target=6.0, plant_draft=6.0, draft_plant_rate=0.8))
    yield ctx
    ctx.close()


def test_trace_export_roundtrip(pair, tmp_path):
    from paper_2602_18931_b200 import abi, trace
    recs = pair.export_trace(0, N, L - 1)
    lines = trace.records_to_ndjson(recs, N, L - 1)
    for line in lines:
        trace.check_line(line, 1000)
    path = str(tmp_path / "pair.ndjson")
    trace.write_trace(path, recs, N, L - 1)
    greedy = [[recs[s * (L - 1) + i].target_token for i in range(L - 1)] for s in range(N)]

    # our model run commits exactly the exported greedy path (spec == greedy, §8c)
    c = abi.config3(num_requests=N, k=4, seq_len=L, vocab=1000, eos=EOS)
    b = pair.run_model_sim(c)
    assert b.ctrl_outputs() == [expected_commit(g) for g in greedy]

    from oracle import pyoracle as po
    if not po.ref_available():
        pytest.skip("reference not built (oracle/_ref)")
    c2 = abi.config3(num_requests=N, k=4, seq_len=L - 1, vocab=1000, eos=EOS)
    ref = po.ref_run_sim_trace(c2, path)
    dealt, lens = po.ref_trace_deal(c2.oracle, path, N, L - 1)
    assert lens == [L - 1] * N
    dealt_greedy = [[dealt[s * (L - 1) + i].target_token for i in range(L - 1)] for s in range(N)]
    assert sorted(dealt_greedy) == sorted(greedy)  # the reference deals a seeded shuffle
    assert ref.ctrl_outputs() == [expected_commit(g) for g in dealt_greedy]
    # our K9 path on the records the reference dealt: identical per-request results
    pair.load_oracle(dealt, N, c2.oracle)
    k9 = pair.run_sim_full(c2, resident=True)
    assert k9.metrics_list() == ref.metrics_list()
    assert k9.ctrl_outputs() == ref.ctrl_outputs()
    assert k9.wrk_outputs() == ref.wrk_outputs()
