"""Experiment front-end (experiment.hpp:25-596) vs the reference's own.

tests/golden/experiments/ holds the reference front-end's outputs (oracle/_ref: parse_experiment
-> run_experiment -> render_csv / render_per_seed_csv / render_manifest) on its experiment files
(shrunk grids; generator tests/golden/make_experiment_golden.py). Our front-end
(paper_2602_18931_b200/experiment.py) must reproduce all three files byte for byte:
  * on CPU, with the batched host driver over the restated tiny pair (ws_run_sim_with_model +
    oracle/restate.c — the host-logic seam the CPU suite uses);
  * on the GPU (-m gpu), with the K9 path (Context.run_sim_full).
Parser errors carry the reference's messages and line numbers.
"""
import os

import pytest

from paper_2602_18931_b200 import experiment as ex

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "experiments")
NAMES = ["single_baseline", "ablation", "phi_sweep"]


def gold(name, ext):
    with open(os.path.join(GOLD, name + ext)) as f:
        return f.read()


def tiny_entropies(c):
    """phi_quantiles' sample (sim.hpp:578-586): the target entropies of num_requests sequences."""
    import paper_2602_18931_b200 as ws
    recs = ws.oracle_synth(c.oracle, c.num_requests)
    return [r.target_entropy for r in recs]


def check(name, runner):
    cfg = ex.parse_experiment(gold(name, ".exp"))
    r = ex.run_experiment(cfg, 1, runner, entropies=tiny_entropies)
    assert ex.render_csv(r) == gold(name, ".csv")
    assert ex.render_per_seed_csv(r) == gold(name, "_per_seed.csv")
    assert ex.render_manifest(r) == gold(name, ".manifest.json")


@pytest.mark.parametrize("name", NAMES)
def test_frontend_matches_reference_cpu_seam(name):
    import paper_2602_18931_b200 as ws
    from oracle import pyoracle as po

    def runner(c):
        return ws.run_sim_with_model(c, po.model_round_fn(c), with_tokens=False, with_steps=False)
    check(name, runner)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_frontend_matches_reference_gpu(name, gpu_ctx):
    def runner(c):
        return gpu_ctx.run_sim_full(c, with_tokens=False, with_steps=False)
    check(name, runner)


def test_manifest_roundtrip_and_parse_errors():
    cfg = ex.config_from_manifest(gold("ablation", ".manifest.json"))
    assert cfg.suite == "ablation" and cfg.seed == 1 and cfg.iterations == 3
    bad = [("[experiment]\nsuite = nope\n", 'line 2: unknown suite "nope"'),
           ("[bogus]\n", "line 1: unknown section [bogus]"),
           ("[protocol]\nk = 1.5\n", "line 2: expected a non-negative integer"),
           ("k = 2\n", "line 1: key before any [section]"),
           ("[grid]\nrtt_ms = 10,,20\n", "line 2: empty list element"),
           ("[timing]\nprofile = custom\n", 'timing profile "custom" needs t_target_ms and t_draft_ms')]
    for text, msg in bad:
        with pytest.raises(ex.ParseError) as e:
            ex.parse_experiment(text)
        assert str(e.value) == msg
