"""Host-logic parity: the product's C++ state machines and batched event driver
(controller/worker/SpecTree/RequestRun in libwanspec_b200.so) driven through the model seam
(ws_run_sim_with_model) by the CPU oracle, against the reference's own RequestSim — live via
oracle/_ref where it exists and against the committed golden fixtures everywhere.
No GPU involved: these pin the host half of the hot path."""
import pytest

import paper_2602_18931_b200 as ws
from oracle import pyoracle as po
from paper_2602_18931_b200 import abi

ref = pytest.mark.skipif(not po.ref_available(), reason="reference not built (oracle/_ref)")


def run_host(c):
    return ws.run_sim_with_model(c, po.model_round_fn(c))


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


def test_golden_cases(golden):
    for case in golden["cases"]:
        c = abi.sim_cfg_from_dict(case["config"])
        got = fingerprint(run_host(c))
        for key in ("metrics", "ctrl_fnv", "wrk_fnv", "ctrl_len", "steps_fnv", "n_steps"):
            assert got[key] == case[key], (case["name"], key)


def test_golden_cases_lanes_driver(golden, monkeypatch):
    """The continuous-batching driver (two asynchronous lanes, completions returned in a
    scrambled order) reproduces every golden case: per-request results cannot depend on how
    jobs are grouped into batches or on which lane finishes first."""
    monkeypatch.setenv("WS_EMULATE_LANES", "1")
    for case in golden["cases"]:
        c = abi.sim_cfg_from_dict(case["config"])
        got = fingerprint(run_host(c))
        for key in ("metrics", "ctrl_fnv", "wrk_fnv", "ctrl_len", "steps_fnv", "n_steps"):
            assert got[key] == case[key], (case["name"], key)


def test_config1_per_step_log(golden):
    case = next(c for c in golden["cases"] if c["name"] == "config1")
    b = run_host(abi.sim_cfg_from_dict(case["config"]))
    steps = [[s[0], s[1], s[2], s[3], s[4], s[5], s[6]] for s in b.step_list()]
    assert steps == case["steps"]
    assert [s[3] for s in steps] == [4, 1, 4, 2, 4, 0, 4, 1, 4, 1, 4, 4, 1, 2, 3, 4, 4, 4, 4, 2,
                                     4, 4, 4, 0, 4, 1]  # SURVEY §8c fingerprint
    assert b.ctrl_outputs() == case["ctrl_outputs"]
    m = b.metrics_list()[0]
    assert m["latency"] == 1325900 and m["target_steps"] == 26


def test_closed_forms():
    """test_sim.cpp:33-47 (baseline closed form) and :58-99 (hand-traced schedule)."""
    for k, want in ((1, 1545000), (2, 1305600), (4, 1068000)):
        c = abi.sim_cfg(mode=abi.WS_MODE_BASELINE, k=k, seed=3, match_prob=1.0)
        m = run_host(c).metrics_list()[0]
        assert m["latency"] == want
        cycles = (100 + k) // (k + 1)
        assert m["target_steps"] == cycles and m["ctrl_draft_passes"] == cycles * k
    c = abi.apply_stage(abi.sim_cfg(k=2, rtt=0, seed=1, match_prob=1.0, sequence_length=10), "plain")
    m = run_host(c).metrics_list()[0]
    assert (m["latency"], m["target_steps"], m["worker_draft_steps"]) == (108600, 4, 15)
    c = abi.apply_stage(abi.sim_cfg(k=2, rtt=0, seed=1, match_prob=1.0), "plain")
    m = run_host(c).metrics_list()[0]
    assert m["latency"] == 2 * 7500 + 34 * 23400 and m["ctrl_draft_passes"] == 0


def test_committed_equals_greedy_every_mode():
    """acceptance criterion 1 (acceptance_main.cpp:47-76), reduced seeds."""
    for rtt in (0, 20000, 70000):
        for stage in ("plain", "branching", "branching_theta", "full"):
            c = abi.apply_stage(abi.sim_cfg(rtt=rtt, num_requests=4, seed=rtt + 1), stage)
            fn = po.model_round_fn(c)
            b = ws.run_sim_with_model(c, fn)
            recs = fn.records
            L = c.oracle.sequence_length
            for r, (co, wo) in enumerate(zip(b.ctrl_outputs(), b.wrk_outputs())):
                greedy = [recs[r * L + i].target_token for i in range(L)]
                assert co == greedy and wo == greedy


def test_extreme_rtt_collapses_to_baseline():  # test_sim.cpp:140-156
    wan = abi.apply_stage(abi.sim_cfg(seed=5, rtt=10_000_000), "plain")
    base = abi.apply_stage(abi.sim_cfg(seed=5, rtt=10_000_000), "plain")
    base.mode = abi.WS_MODE_BASELINE
    a, b = run_host(wan).metrics_list()[0], run_host(base).metrics_list()[0]
    assert (a["latency"], a["ctrl_draft_passes"], a["target_steps"]) == \
        (b["latency"], b["ctrl_draft_passes"], b["target_steps"])


def test_config2_livelock_at_default_max_nodes():
    """config 2 at max_nodes=64 exceeds the event budget in the reference; the
    new driver must detect the same livelock (sim.hpp:198) rather than spin."""
    c = abi.config2(num_requests=27, max_nodes=64)
    c.first_request, c.local_requests = 26, 1  # the first stalling request (seed 1)
    with pytest.raises(ws.WanspecError) as e:
        run_host(c)
    assert "event budget" in str(e.value)


@ref
@pytest.mark.parametrize("seed", [4, 5])
def test_live_vs_reference_config2(seed):
    for verify in (abi.WS_VERIFY_GREEDY, abi.WS_VERIFY_REJECTION):
        c = abi.config2(seed=seed, num_requests=16, verify=verify)
        assert fingerprint(run_host(c)) == fingerprint(po.ref_run_sim(c))


@ref
def test_live_vs_reference_jitter_backstop_sweep():
    for seed in range(1, 6):
        for rtt in (0, 15000, 40000):
            c = abi.apply_stage(abi.sim_cfg(k=3, rtt=rtt, jitter=2500, seed=seed, num_requests=2,
                                            wait_backstop=bool(seed % 2), max_nodes=32), "full")
            assert fingerprint(run_host(c)) == fingerprint(po.ref_run_sim(c)), (seed, rtt)


def test_sharded_equals_full():
    """Requests are independent: any shard of the dealt stream reproduces those requests."""
    c = abi.config2(num_requests=12)
    full = run_host(c)
    parts = []
    for first, n in ((0, 5), (5, 4), (9, 3)):
        s = abi.config2(num_requests=12)
        s.first_request, s.local_requests = first, n
        parts.append(run_host(s))
    assert sum((p.metrics_list() for p in parts), []) == full.metrics_list()
    assert sum((p.ctrl_outputs() for p in parts), []) == full.ctrl_outputs()


def test_config_errors_map_to_configerror():
    for bad in (dict(k=0), dict(b=3), dict(s=0), dict(rtt=-1), dict(num_requests=0),
                dict(vocab_size=1), dict(eos_id=40000), dict(match_prob=1.5)):
        c = abi.sim_cfg(**bad)
        with pytest.raises(ws.ConfigError):
            ws.run_sim_with_model(c, lambda *a: 0)
