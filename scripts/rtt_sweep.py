"""BASELINE configs[3] — RTT sweep: controller fallback to local draft vs worker proposals.

For each RTT (ms) the same requests run in WANSpec mode and in the baseline mode (the
controller drafts everything locally, SimConfig.baseline); offload % = 1 − controller draft
passes (WANSpec) / controller draft passes (baseline) on the same seeds (sim.hpp:503-504,
experiment.hpp:419-423). Two model pairs:

  * the reference's tiny oracle pair on the GPU (K9 path), beside the reference itself
    (oracle/_ref run_sim_full) when it is built — per-request metrics must be identical;
  * the Llama-3.1-8B / 3.2-1B shapes (random-init bf16 + planted bias) on the GPU.

    python scripts/rtt_sweep.py [--requests 16] [--rtts 10,15,20,30,50,70,100,150,200] [--md out.md]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2602_18931_b200 as ws  # noqa: E402
from paper_2602_18931_b200 import abi  # noqa: E402


def totals(b):
    ms = b.metrics_list()
    keys = ("ctrl_draft_passes", "ctrl_local_draft_steps", "worker_draft_steps", "target_steps",
            "tokens_committed", "sync_stalls")
    out = {k: sum(m[k] for m in ms) for k in keys}
    out["mean_latency_ms"] = sum(m["latency"] for m in ms) / len(ms) / 1e3
    return out


def sweep_tiny(ctx, rtts, n, k):
    from oracle import pyoracle as po
    rows = []
    for rtt in rtts:
        res = {}
        for mode in ("wanspec", "baseline"):
            c = abi.apply_stage(abi.sim_cfg(k=k, rtt=int(rtt * 1000), num_requests=n, max_nodes=256), "full")
            if mode == "baseline":
                c.mode = abi.WS_MODE_BASELINE
            b = ctx.run_sim_full(c, with_tokens=False, with_steps=False)
            res[mode] = totals(b)
            if po.ref_available():
                r = po.ref_run_sim(c, with_tokens=False, with_steps=False)
                res[mode]["ref_identical"] = r.metrics_list() == b.metrics_list()
        rows.append((rtt, res))
    return rows


def sweep_llama(ctx, rtts, n, k):
    ctx.run_model_sim(abi.config3(num_requests=n, k=k), with_tokens=False, with_steps=False)  # warm-up
    rows = []
    for rtt in rtts:
        res = {}
        for mode in ("wanspec", "baseline"):
            c = abi.config3(num_requests=n, k=k)
            c.rtt = int(rtt * 1000)
            c.r_estimate = -1
            if mode == "baseline":
                c.mode = abi.WS_MODE_BASELINE
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            b = ctx.run_model_sim(c, with_tokens=False, with_steps=False)
            torch.cuda.synchronize()
            res[mode] = totals(b)
            res[mode]["wall_s"] = time.perf_counter() - t0
        rows.append((rtt, res))
    return rows


def table(title, rows, ref_col):
    lines = [f"### {title}", "",
             "| RTT ms | offload % | ctrl draft passes (WANSpec / baseline) | ctrl local draft steps | worker draft "
             "steps | target steps | mean virtual latency ms (WANSpec / baseline) |"
             + (" = reference |" if ref_col else " wall tokens/s (WANSpec run) |"),
             "|---:|---:|---|---:|---:|---:|---|" + ("---|" if ref_col else "---:|")]
    for rtt, r in rows:
        w, bl = r["wanspec"], r["baseline"]
        off = 100.0 * (1.0 - w["ctrl_draft_passes"] / max(1, bl["ctrl_draft_passes"]))
        extra = (" %s |" % ("yes" if w.get("ref_identical") and bl.get("ref_identical") else "NO")) if ref_col else \
            " %.0f |" % (w["tokens_committed"] / w["wall_s"])
        lines.append(f"| {rtt:g} | {off:.1f} | {w['ctrl_draft_passes']} / {bl['ctrl_draft_passes']} | "
                     f"{w['ctrl_local_draft_steps']} | {w['worker_draft_steps']} | {w['target_steps']} | "
                     f"{w['mean_latency_ms']:.1f} / {bl['mean_latency_ms']:.1f} |" + extra)
    return "\n".join(lines) + "\n"


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--requests", type=int, default=16)
    p.add_argument("--k", type=int, default=4)
    p.add_argument("--rtts", default="10,15,20,30,50,70,100,150,200")
    p.add_argument("--md", default="")
    p.add_argument("--skip-llama", action="store_true")
    a = p.parse_args()
    rtts = [float(x) for x in a.rtts.split(",")]
    ctx = ws.Context(0)
    out = ["# r01 — config 4: RTT sweep (controller fallback vs worker proposals)", "",
           f"{a.requests} requests, k={a.k}, b=2, s=4, θ=φ=0.5, max_nodes=256, stage `full`; offload % = 1 − controller "
           "draft passes in WANSpec mode / in baseline mode on the same seeds (sim.hpp:503-504). Command: "
           f"`python scripts/rtt_sweep.py --requests {a.requests} --k {a.k}`.", ""]
    tiny = sweep_tiny(ctx, rtts, a.requests, a.k)
    for rtt, r in tiny:
        print(json.dumps({"pair": "tiny", "rtt_ms": rtt, **r}))
    out.append(table("Tiny oracle pair (K9 on the GPU; last column: per-request metrics identical to the "
                     "reference's run_sim_full)", tiny, True))
    if not a.skip_llama:
        ctx.load_models(abi.model_cfg(max_requests=max(16, a.requests)))
        llama = sweep_llama(ctx, rtts, a.requests, a.k)
        for rtt, r in llama:
            print(json.dumps({"pair": "llama", "rtt_ms": rtt, **r}))
        out.append(table("Llama-3.1-8B / 3.2-1B shapes (random-init bf16, planted bias; model path on the GPU)",
                         llama, False))
    if a.md:
        with open(a.md, "w") as f:
            f.write("\n".join(out))
    ctx.close()


if __name__ == "__main__":
    main()
