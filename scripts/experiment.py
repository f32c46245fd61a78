"""The experiment CLI (the reference's `wanspec run <file.exp>`, tools/wanspec.cpp:39-68) over the
B200 path: parses a reference experiment file, runs its suite and writes the CSV, per-seed CSV and
manifest (paper_2602_18931_b200/experiment.py).

  python scripts/experiment.py FILE.exp [--harness sim|model|wallclock] [--target llama3-8b]
                               [--draft llama3.2-1b] [--out DIR] [--seed N]

harness sim: the tiny oracle pair on the K9 path (per-request metrics equal the reference's).
harness model / wallclock: the Llama-shape pair (random-init bf16, planted bias; config 3's
workload); seed i of a suite selects the i-th block of `requests` prompts; the sequence length
is the file's; `model` runs on the virtual clock with the l40s/swiftspec step times, `wallclock`
in real time with the B200's step times (latency columns in real µs).
WANSPEC_SEED overrides the seed (tools/wanspec.cpp:49-54).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2602_18931_b200 as ws  # noqa: E402
from paper_2602_18931_b200 import abi  # noqa: E402
from paper_2602_18931_b200 import experiment as ex  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("file")
    p.add_argument("--harness", choices=["sim", "model", "wallclock"], default="sim")
    p.add_argument("--target", default="llama3-8b")
    p.add_argument("--draft", default="llama3.2-1b")
    p.add_argument("--out", default=".")
    p.add_argument("--seed", type=int, default=None)
    a = p.parse_args()
    with open(a.file) as f:
        cfg = ex.parse_experiment(f.read())
    seed = a.seed if a.seed is not None else int(os.environ.get("WANSPEC_SEED", cfg.seed))
    ctx = ws.Context(0)
    if a.harness == "sim":
        def runner(c):
            return ctx.run_sim_full(c, with_tokens=False, with_steps=False)

        def entropies(c):
            return [r.target_entropy for r in ws.oracle_synth(c.oracle, c.num_requests)]
    else:
        n_blocks = cfg.iterations
        seq = cfg.oracle["sequence_length"]
        ctx.load_models(abi.model_cfg(a.target, a.draft, max_requests=n_blocks * cfg.requests,
                                      max_ctx=128 + seq + cfg.k + 8))

        def runner(c):
            i = c.oracle.seed - seed
            c.oracle.vocab_size, c.oracle.eos_id = abi.LLAMA_VOCAB, abi.LLAMA_EOS
            c.first_request, c.local_requests = i * cfg.requests, cfg.requests
            c.num_requests = (i + 1) * cfg.requests
            run = ctx.run_model_wallclock if a.harness == "wallclock" else ctx.run_model_sim
            return run(c, with_tokens=False, with_steps=False)

        def entropies(c):
            recs = ctx.export_trace(0, cfg.requests, seq)
            return [r.target_entropy for r in recs]
    r = ex.run_experiment(cfg, seed, runner, harness=a.harness, entropies=entropies)
    os.makedirs(a.out, exist_ok=True)
    ex.write_outputs(r, a.out)
    sys.stdout.write(ex.render_csv(r))
    ctx.close()


if __name__ == "__main__":
    main()
