"""Benchmark of the WANSpec verify/draft hot path on B200 (contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1]): the tiny draft/target pair, 64 requests
per GPU (weak scaling: rank r runs requests [64r, 64r+64) of one dealt stream), k=8, b=2, s=4,
theta=phi=0.5, RTT 20 ms, max_nodes=256 (the reference livelocks at 64), greedy
verify by default (--verify rejection for the Philox extension). One "step" = every request of
the shard decoded to EOS through the batched driver; metric = accepted (committed) tokens/s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "accepted tokens/s (tiny pair, 64 req/GPU, k=8, b=2, s=4, RTT 20 ms)"
UNIT = "tokens/s"
REQ_PER_GPU = 64


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--verify", choices=["greedy", "rejection"], default="greedy")
    p.add_argument("--host-threads", type=int, default=0)
    p.add_argument("--cpu-sample-s", type=float, default=6.0)
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def workload_cfg(world, rank, verify):
    from paper_2602_18931_b200 import abi
    c = abi.config2(verify=abi.WS_VERIFY_REJECTION if verify == "rejection" else abi.WS_VERIFY_GREEDY,
                    num_requests=REQ_PER_GPU * world)
    c.first_request, c.local_requests = REQ_PER_GPU * rank, REQ_PER_GPU
    return c


def config_block(args, world, host_threads):
    return {"workload": "BASELINE configs[1]: tiny draft/target pair (oracle tables, V=32768), "
                        f"{REQ_PER_GPU} requests/GPU, k=8, b=2, s=4, theta=phi=0.5, RTT 20 ms, "
                        "max_nodes=256",
            "verify": args.verify, "requests_total": REQ_PER_GPU * world,
            "parallelism": f"requests sharded over {world} GPU(s), no collective",
            "host_threads_per_gpu": host_threads,
            "l2": "inputs (460 KB tables) are L2-resident by design; L2 flushed (256 MB write) "
                  "before every timed step"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_gpu{index}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except Exception:
            return None
        if not rows:
            return None
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3:7]) if v.strip() == "Active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def k9_algorithmic_bytes(out, k):
    """Algorithmic bytes of the K9 launches of one run (SURVEY §8d units):
    verify job: 32 B job + 4k B candidates + 4(k+1) B target ids + 8 B entropy read, 16 B out;
    draft row: 16 B job + 8 B ids + 24 B probs/entropy read, 40 B out."""
    v, d = out.verify_rows, out.draft_rows
    return v * (32 + 4 * k + 4 * (k + 1) + 8 + 16) + d * (16 + 8 + 24 + 40)


def cpu_reference_sample(world, verify, seconds, threads):
    """The reference's own run_sim_full (oracle/_ref) on this host's cores: bounded sample."""
    from oracle import pyoracle as po
    cfg = workload_cfg(1, 0, verify)
    cfg.num_requests = REQ_PER_GPU * world
    cfg.first_request, cfg.local_requests = 0, 0
    toks, t0, runs = 0, time.perf_counter(), 0
    while True:
        b = po.ref_run_sim(cfg, threads=threads, with_tokens=False, with_steps=False)
        toks += sum(m["tokens_committed"] for m in b.metrics_list())
        runs += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return toks / el, runs, el


def run_reference(args, rank, world):
    if rank != 0:
        return
    from oracle import pyoracle as po
    if not po.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
        return
    threads = os.cpu_count() or 1
    cfg = workload_cfg(1, 0, args.verify)
    cfg.num_requests = REQ_PER_GPU * world
    cfg.first_request, cfg.local_requests = 0, 0
    for _ in range(args.warmup):
        po.ref_run_sim(cfg, threads=threads, with_tokens=False, with_steps=False)
    toks = 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        b = po.ref_run_sim(cfg, threads=threads, with_tokens=False, with_steps=False)
        toks += sum(m["tokens_committed"] for m in b.metrics_list())
    el = time.perf_counter() - t0
    value = toks / el
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * el / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference", "config": config_block(args, world, threads),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{args.steps} full runs of {REQ_PER_GPU * world} requests "
                                       "(run_sim_full via oracle/_ref, requests partitioned over threads)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    args = parse()
    rank, local_rank, world = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import paper_2602_18931_b200 as ws
    from paper_2602_18931_b200 import abi

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    ncpu = os.cpu_count() or 1
    host_threads = args.host_threads or max(1, min(16, ncpu // max(1, world)))
    cfg = workload_cfg(world, rank, args.verify)
    cfg.host_threads = host_threads
    ctx = ws.Context(local_rank)
    recs = ws.oracle_synth(cfg.oracle, cfg.num_requests)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident path: tables in HBM before the timed region ----
    ctx.load_oracle(recs, cfg.num_requests, cfg.oracle)
    for _ in range(args.warmup):
        ctx.run_sim_full(cfg, with_tokens=False, with_steps=False, resident=True)
    tokens, total_ms, launches, kernel_ms, alg_bytes = 0, 0.0, 0, 0.0, 0
    barrier()
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b = ctx.run_sim_full(cfg, with_tokens=False, with_steps=False, resident=True)
            e1.record()
            torch.cuda.synchronize()
            total_ms += e0.elapsed_time(e1)
            tokens += sum(m["tokens_committed"] for m in b.metrics_list())
            launches += b.out.gpu_launches
            kernel_ms += b.out.kernel_ms
            alg_bytes += k9_algorithmic_bytes(b.out, cfg.k)
    barrier()

    # ---- end to end through the public C-ABI call: host tables -> HBM, results -> host ----
    e2e_ms, e2e_tokens, h2d, d2h = 0.0, 0, 0, 0
    for i in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.load_oracle(recs, cfg.num_requests, cfg.oracle)
        b = ctx.run_sim_full(cfg, with_tokens=True, with_steps=False, resident=True)
        e1.record()
        torch.cuda.synchronize()
        e2e_ms += e0.elapsed_time(e1)
        e2e_tokens += sum(m["tokens_committed"] for m in b.metrics_list())
        h2d += b.out.h2d_bytes + cfg.num_requests * cfg.oracle.sequence_length * 64  # SoA tables
        d2h += b.out.d2h_bytes
    barrier()

    stats = torch.tensor([total_ms, float(tokens), e2e_ms, float(e2e_tokens), float(launches)],
                         dtype=torch.float64, device="cuda")
    if dist:
        mx = stats.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = stats.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        total_ms_max, e2e_ms_max = mx[0].item(), mx[2].item()
        tokens_all, e2e_tokens_all, launches_all = sm[1].item(), sm[3].item(), sm[4].item()
    else:
        total_ms_max, e2e_ms_max = total_ms, e2e_ms
        tokens_all, e2e_tokens_all, launches_all = float(tokens), float(e2e_tokens), float(launches)

    if rank == 0:
        peak, peak_kind = measured_peak_hbm()
        avg_kernel_s = (kernel_ms / 1000.0) / max(1, launches)
        achieved = (alg_bytes / max(1, launches)) / avg_kernel_s / 1e9 if avg_kernel_s > 0 else 0.0
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "k9_traffic.json")) as f:
                traffic = json.load(f).get("bytes_per_launch")
        except Exception:
            pass
        cpu_value, runs, el = cpu_reference_sample(1, args.verify, args.cpu_sample_s, ncpu) \
            if world == 1 else (None, 0, 0)
        value = tokens_all / (total_ms_max / 1000.0)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(args, world, host_threads),
            "e2e": {"value": e2e_tokens_all / (e2e_ms_max / 1000.0), "unit": UNIT,
                    "h2d_bytes_per_step": h2d // max(1, args.steps),
                    "d2h_bytes_per_step": d2h // max(1, args.steps)},
            "gpu_launches": int(launches_all),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "k9_round", "peak_kind": peak_kind,
                         "note": "K9 moves ~100 KB/launch: latency-bound by construction"},
            "clocks": clk.summary(),
        }
        if cpu_value is not None:
            line["cpu_baseline"] = {"value": cpu_value, "unit": UNIT, "cores": ncpu, "kind": "reference",
                                    "sample": f"{runs} runs of 64 requests in {el:.1f} s "
                                              "(reference run_sim_full via oracle/_ref, all host cores)"}
        print(json.dumps(line))
    ctx.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
