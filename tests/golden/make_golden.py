"""Generates tests/golden/*.json from the reference itself (oracle/_ref/libwanspec_ref.so,
compiled from /root/reference/proj/include by oracle/Makefile). Run here, where the
reference exists; the JSON travels with the repo so the GPU box needs no reference.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2602_18931_b200 import abi  # noqa: E402
from oracle import pyoracle as po  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def cfg_dict(c):
    d = {n: getattr(c, n) for n, _ in abi.SimCfg._fields_ if n != "oracle"}
    d["oracle"] = {n: getattr(c.oracle, n) for n, _ in abi.OracleCfg._fields_}
    return d


def run_case(name, c, full_steps=False):
    b = po.ref_run_sim(c)
    steps = b.step_list()
    case = {
        "name": name,
        "config": cfg_dict(c),
        "metrics": b.metrics_list(),
        "ctrl_fnv": "%016x" % po.fnv_tokens(b.ctrl_outputs()),
        "wrk_fnv": "%016x" % po.fnv_tokens(b.wrk_outputs()),
        "ctrl_len": [len(x) for x in b.ctrl_outputs()],
        "steps_fnv": "%016x" % po.fnv_tokens([[s[0], s[1], s[2] & 0xFFFFFFFF, s[3], s[4], s[6]]
                                              for s in steps]),
        "n_steps": len(steps),
    }
    if full_steps:
        case["steps"] = [[s[0], s[1], s[2], s[3], s[4], s[5], s[6]] for s in steps]
        case["ctrl_outputs"] = b.ctrl_outputs()
    return case


def main():
    po.build()
    cases = []
    cases.append(run_case("config1", abi.config1(), full_steps=True))
    cases.append(run_case("config2", abi.config2()))
    cases.append(run_case("config2_rejection", abi.config2(verify=abi.WS_VERIFY_REJECTION)))
    for seed in (2, 3):
        cases.append(run_case(f"config2_seed{seed}", abi.config2(seed=seed)))
    # acceptance criterion 1 shape (acceptance_main.cpp:47-76): modes × RTTs, seeds 1..3
    for rtt in (0, 10000, 30000, 70000):
        for stage in ("plain", "branching", "branching_theta", "full"):
            c = abi.apply_stage(abi.sim_cfg(rtt=rtt, num_requests=3), stage)
            cases.append(run_case(f"accept1_{stage}_{rtt}", c))
        c = abi.sim_cfg(rtt=rtt, num_requests=3, mode=abi.WS_MODE_BASELINE)
        cases.append(run_case(f"accept1_baseline_{rtt}", c))
    # closed forms (test_sim.cpp:33-99) and jitter determinism (:101-111)
    for k in (1, 2, 4):
        c = abi.sim_cfg(mode=abi.WS_MODE_BASELINE, k=k, seed=3, match_prob=1.0)
        cases.append(run_case(f"baseline_closed_form_k{k}", c))
    c = abi.apply_stage(abi.sim_cfg(k=2, rtt=0, seed=1, match_prob=1.0, sequence_length=10), "plain")
    cases.append(run_case("hand_traced_10", c, full_steps=True))
    c = abi.sim_cfg(rtt=20000, jitter=1500, seed=42, num_requests=3)
    cases.append(run_case("jitter_42", c))
    c = abi.apply_stage(abi.sim_cfg(k=2, rtt=20000, seed=5, wait_backstop=True, num_requests=2), "full")
    cases.append(run_case("backstop_5", c))
    c = abi.apply_stage(abi.sim_cfg(k=4, rtt=20000, seed=9, catchup_batch_limit=2, num_requests=2), "full")
    cases.append(run_case("catchup_limit2", c))

    synth = []
    for seed in (1, 7, 1234):
        o = abi.oracle_cfg(seed=seed)
        recs = po.synth(o, 4, use_ref=True)
        synth.append({"seed": seed, "n_seq": 4, "bytes_fnv": "%016x" % po.fnv_tokens(
            [list(memoryview(bytes(recs)).cast("I"))])})
    with open(os.path.join(OUT, "sim_cases.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py (reference via oracle/_ref)",
                   "cases": cases, "synth": synth}, f, indent=1)
    print(f"wrote {len(cases)} cases")


if __name__ == "__main__":
    main()
