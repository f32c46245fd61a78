"""GPU parity for the tiny-pair path (K9 kernel + batched driver), through the C ABI, against
the oracle (oracle/restate.c), the committed golden fixtures, and — where present — the
reference itself (oracle/_ref). Bit-exact: token ids, accept lengths, resync points,
entropies (f64), virtual latencies and every counter."""
import random

import pytest

import paper_2602_18931_b200 as ws
from oracle import pyoracle as po
from paper_2602_18931_b200 import abi

pytestmark = pytest.mark.gpu


def fingerprint(b):
    steps = b.step_list()
    return {
        "metrics": b.metrics_list(),
        "ctrl_fnv": "%016x" % po.fnv_tokens(b.ctrl_outputs()),
        "wrk_fnv": "%016x" % po.fnv_tokens(b.wrk_outputs()),
        "ctrl_len": [len(x) for x in b.ctrl_outputs()],
        "steps_fnv": "%016x" % po.fnv_tokens([[s[0], s[1], s[2] & 0xFFFFFFFF, s[3], s[4], s[6]]
                                              for s in steps]),
        "n_steps": len(steps),
    }


@pytest.fixture(scope="module")
def tables(gpu_ctx):
    o = abi.oracle_cfg(seed=21, vocab_size=512, eos_id=511, sequence_length=60)
    n = 8
    recs = po.synth(o, n)
    gpu_ctx.load_oracle(recs, n, o)
    return o, n, recs


def test_verify_matches_oracle(gpu_ctx, tables):
    o, n, recs = tables
    L = o.sequence_length
    rnd = random.Random(1)
    for k in (1, 4, 8):
        seq, base, cands = [], [], []
        for _ in range(3000):
            s, b = rnd.randrange(n), rnd.randrange(L + 10)
            row = []
            for i in range(k):
                p = b + i
                t = recs[s * L + p].target_token if p < L else o.eos_id
                row.append(t if rnd.random() < 0.85 else rnd.randrange(o.vocab_size))
            seq.append(s)
            base.append(b)
            cands.append(row)
        got = gpu_ctx.run_target_step(seq, base, cands)
        for j in range(len(seq)):
            assert got[j] == po.run_target_step(recs, seq[j], L, o.eos_id, base[j], cands[j])


def test_rejection_matches_oracle(gpu_ctx, tables):
    o, n, recs = tables
    L = o.sequence_length
    rnd = random.Random(2)
    k = 6
    seq, req, step, base, cands = [], [], [], [], []
    for j in range(4000):
        s, b = rnd.randrange(n), rnd.randrange(L + 4)
        row = []
        for i in range(k):
            p = b + i
            if p < L:
                r = recs[s * L + p]
                row.append(rnd.choice([r.draft_top1, r.draft_top2, r.target_token,
                                       rnd.randrange(o.vocab_size)]))
            else:
                row.append(o.eos_id)
        seq.append(s)
        req.append(rnd.randrange(1 << 40))
        step.append(rnd.randrange(200))
        base.append(b)
        cands.append(row)
    seed = 0xC0FFEE1234
    got = gpu_ctx.rejection_verify(seq, req, step, base, cands, seed)
    for j in range(len(seq)):
        want = po.rejection_verify(recs, seq[j], L, o.eos_id, o.vocab_size, seed, req[j], step[j],
                                   base[j], cands[j])
        assert got[j] == want, j


def test_draft_matches_oracle(gpu_ctx, tables):
    o, n, recs = tables
    L = o.sequence_length
    rnd = random.Random(3)
    seq = [rnd.randrange(n) for _ in range(5000)]
    pos = [rnd.randrange(L + 8) for _ in range(5000)]
    got = gpu_ctx.draft_prediction(seq, pos)
    for j in range(len(seq)):
        assert got[j] == po.draft_prediction(recs, seq[j], L, o.eos_id, pos[j])


def test_run_sim_golden(gpu_ctx, golden):
    for case in golden["cases"]:
        c = abi.sim_cfg_from_dict(case["config"])
        b = gpu_ctx.run_sim_full(c)
        got = fingerprint(b)
        for key in ("metrics", "ctrl_fnv", "wrk_fnv", "ctrl_len", "steps_fnv", "n_steps"):
            assert got[key] == case[key], (case["name"], key)
        assert b.out.gpu_launches > 0 and b.out.gpu_launches == b.out.rounds


def test_config1_per_step(gpu_ctx, golden):
    case = next(c for c in golden["cases"] if c["name"] == "config1")
    b = gpu_ctx.run_sim_full(abi.sim_cfg_from_dict(case["config"]))
    assert [[s[0], s[1], s[2], s[3], s[4], s[5], s[6]] for s in b.step_list()] == case["steps"]


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_config2_host_threads(gpu_ctx, golden, threads):
    for name in ("config2", "config2_rejection"):
        case = next(c for c in golden["cases"] if c["name"] == name)
        c = abi.sim_cfg_from_dict(case["config"])
        c.host_threads = threads
        got = fingerprint(gpu_ctx.run_sim_full(c))
        for key in ("metrics", "ctrl_fnv", "wrk_fnv", "steps_fnv"):
            assert got[key] == case[key], (name, threads, key)


def test_resident_path_and_shards(gpu_ctx, golden):
    case = next(c for c in golden["cases"] if c["name"] == "config2")
    c = abi.sim_cfg_from_dict(case["config"])
    recs = ws.oracle_synth(c.oracle, c.num_requests)
    gpu_ctx.load_oracle(recs, c.num_requests, c.oracle)
    metrics = []
    for first, n in ((0, 20), (20, 44)):
        s = abi.sim_cfg_from_dict(case["config"])
        s.first_request, s.local_requests = first, n
        metrics += gpu_ctx.run_sim_full(s, resident=True).metrics_list()
    assert metrics == case["metrics"]


@pytest.mark.skipif(not po.ref_available(), reason="reference not built")
def test_live_vs_reference(gpu_ctx):
    for seed in (6, 7):
        for verify in (abi.WS_VERIFY_GREEDY, abi.WS_VERIFY_REJECTION):
            c = abi.config2(seed=seed, num_requests=32, verify=verify)
            c.host_threads = 4
            assert fingerprint(gpu_ctx.run_sim_full(c)) == fingerprint(po.ref_run_sim(c))
