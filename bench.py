"""Benchmark of the WANSpec verify/draft hot path on B200 (contract: one JSON line on rank 0).

Default workload (--workload llama; BASELINE.json configs[2], the config the metric's
"1/2/4/8 B200" is quoted on): Llama-3.1-8B-shape target + Llama-3.2-1B-shape draft, random-init
bf16 weights, 256 requests of 128-token seeded prompts sharded over the GPUs (strong scaling),
100 generated tokens each, k=4, b=2, s=4, theta=phi=0.5, RTT 20 ms (virtual clock), greedy
verify. One step = every request of the shard decoded to EOS through the batched driver, every
verify / draft model call a batched forward on the GPU. Metric: accepted (committed) tokens/s.

--workload tiny: BASELINE configs[1], the tiny oracle pair, 64 requests per GPU (weak scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload llama|tiny]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "accepted tokens/s at 1/2/4/8 B200 (WANSpec verify + draft rollout)"
UNIT = "tokens/s"
TINY_REQ_PER_GPU = 64
LLAMA_REQUESTS = 256


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=["llama", "tiny"], default="llama")
    p.add_argument("--k", type=int, default=4)
    p.add_argument("--requests", type=int, default=LLAMA_REQUESTS)
    p.add_argument("--verify", choices=["greedy", "rejection"], default="greedy")
    p.add_argument("--host-threads", type=int, default=0)
    p.add_argument("--shards", type=int, default=int(os.environ.get("WS_SHARDS", "1")),
                   help="llama: protocol threads per GPU, each with its own verify/draft streams")
    p.add_argument("--placement", choices=["shared", "split"], default=os.environ.get("WS_PLACEMENT", "shared"),
                   help="llama, N >= 2: 'split' puts the draft model on its own GPU (ranks < N/2 drive "
                        "target GPU r + draft GPU r + N/2; SURVEY §8e), 'shared' shards requests over all GPUs")
    p.add_argument("--cpu-sample-s", type=float, default=6.0)
    p.add_argument("--cpu-seq", type=int, default=8,
                   help="llama CPU baseline: committed tokens per measured CPU sample (one request)")
    p.add_argument("--target", choices=["llama3-8b", "llama3-70b"], default="llama3-8b",
                   help="llama: the target model shape; llama3-70b is BASELINE config 5's model (141 GB of "
                        "bf16 weights; use --requests 128)")
    p.add_argument("--tp", type=int, default=1,
                   help="llama: tensor-parallel ranks of the target per process (BASELINE config 5): the "
                        "process drives GPUs local_rank*tp .. +tp-1, the draft model sits on the last of them")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    except Exception:
        return 6650.0, 1400.0, "fallback"


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


# ------------------------------------------------------------------ workloads
def shard(total, world, rank):
    lo, hi = total * rank // world, total * (rank + 1) // world
    return lo, hi - lo


def llama_cfg(args, world, rank):
    from paper_2602_18931_b200 import abi
    c = abi.config3(num_requests=args.requests, k=args.k)
    c.first_request, c.local_requests = shard(args.requests, world, rank)
    return c


def tiny_cfg(args, world, rank):
    from paper_2602_18931_b200 import abi
    c = abi.config2(verify=abi.WS_VERIFY_REJECTION if args.verify == "rejection" else abi.WS_VERIFY_GREEDY,
                    num_requests=TINY_REQ_PER_GPU * world)
    c.first_request, c.local_requests = TINY_REQ_PER_GPU * rank, TINY_REQ_PER_GPU
    return c


def config_block(args, world, host_threads):
    if args.workload == "llama":
        tname = {"llama3-8b": "Llama-3.1-8B", "llama3-70b": "Llama-3.1-70B"}[args.target]
        return {"workload": ("BASELINE configs[2]: " if args.target == "llama3-8b" and args.tp == 1 else
                             f"BASELINE configs[4]: target tensor-parallel over {args.tp} GPUs per process "
                             f"(peer-memory all-reduce fused into the residual update), the draft model replicated on "
                             f"every rank (request r's drafts on rank r % {args.tp}): "
                             if args.tp > 1 else
                             "BASELINE configs[4]'s model, whole on one GPU per rank (no TP): ") +
                            f"{tname}-shape target / Llama-3.2-1B-shape draft "
                            "(random-init bf16), 128-token seeded prompts, 100 generated tokens, "
                            f"{args.requests} requests, k={args.k}, b=2, s=4, theta=phi=0.5, RTT 20 ms "
                            "(virtual), greedy verify, planted shared bigram bias (match ~0.8)",
                "model": f"{args.target} + llama3.2-1b", "global_batch": args.requests, "seq_len": 128 + 100,
                "parallelism": (f"split placement: requests sharded over {world // 2} target GPU(s), each "
                                f"paired with its own draft GPU (SURVEY §8e), no collective"
                                if args.placement == "split" and world >= 2 and world % 2 == 0 else
                                f"dp{world} x tp{args.tp}: requests sharded over {world} process(es) (strong "
                                f"scaling, no collective between them), each target tensor-parallel over "
                                f"{args.tp} GPUs (peer-memory all-reduce)"
                                if args.tp > 1 else
                                f"requests sharded over {world} GPU(s) (strong scaling), no collective"),
                "l2": "weights (>=18.5 GB) and KV (>126 MB) exceed L2; no explicit flush needed"}
    return {"workload": "BASELINE configs[1]: tiny draft/target pair (oracle tables, V=32768), "
                        f"{TINY_REQ_PER_GPU} requests/GPU, k=8, b=2, s=4, theta=phi=0.5, RTT 20 ms, "
                        "max_nodes=256", "verify": args.verify,
            "parallelism": f"requests sharded over {world} GPU(s), no collective",
            "host_threads_per_gpu": host_threads,
            "l2": "tables are L2-resident by design; L2 flushed (256 MB write) before every timed step"}


MODEL_SHAPES = {  # shape_by_name (csrc/model/llama.cu)
    "llama3-8b": dict(L=32, d=4096, nq=32, nkv=8, hd=128, ffn=14336, V=128256),
    "llama3-70b": dict(L=80, d=8192, nq=64, nkv=8, hd=128, ffn=28672, V=128256),
    "llama3.2-1b": dict(L=16, d=2048, nq=32, nkv=8, hd=64, ffn=8192, V=128256),
}


def unit_roofline(shape, fw, ms, rows, out_rows, kv_pos, attn_pairs, peak_bw, peak_tf, causal_half=False):
    """Roofline of one forward unit (SURVEY §8d units, per forward = run totals / forwards):
    FLOPs = 2 P_layers rows + 2 P_lm out_rows + 4 L pairs n_q hd   (pairs = rows x visible keys)
    bytes = 2 P_layers + 2 P_lm [out_rows > 0] + KVB (keys read + rows written) + 4 V out_rows
    (the bf16 logits written by the LM head and read once by K3/K4). time = measured device time
    of the unit on its own stream (CUDA events), divided by its forwards."""
    m = MODEL_SHAPES[shape]
    per_layer = (m["nq"] + 2 * m["nkv"]) * m["hd"] * m["d"] + m["d"] * m["nq"] * m["hd"] + 3 * m["ffn"] * m["d"]
    P_layers, P_lm = per_layer * m["L"], m["V"] * m["d"]
    kvb = m["L"] * 2 * m["nkv"] * m["hd"] * 2
    fw = max(1, fw)
    r, o, kv, pairs = rows / fw, out_rows / fw, kv_pos / fw, attn_pairs / fw
    if causal_half:  # prefill groups: causal over their own rows, about half the pairs are visible
        pairs /= 2
    flops = 2 * P_layers * r + 2 * P_lm * o + 4 * m["L"] * pairs * m["nq"] * m["hd"]
    byts = 2 * P_layers + (2 * P_lm if o > 0 else 0) + kvb * (kv + r) + 4 * m["V"] * o
    t = ms / 1e3 / fw
    t_tensor, t_hbm = flops / (peak_tf * 1e12), byts / (peak_bw * 1e9)
    out = {"rows_per_forward": r, "out_rows_per_forward": o, "forwards": fw, "ms_per_forward": t * 1e3,
           "alg_flops": flops, "alg_bytes": byts}
    if t_tensor >= t_hbm:
        out.update({"bound": "tensor", "achieved": flops / t / 1e12, "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": t_tensor / t})
    else:
        out.update({"bound": "hbm", "achieved": byts / t / 1e9, "peak": peak_bw, "unit": "GB/s", "frac": t_hbm / t})
    return out


def llama_rooflines(rs, target, peak_bw, peak_tf, tp=1):
    """verify (the headline), prefill and draft units from ws_model_run_stats of the timed runs."""
    verify = unit_roofline(target, rs["verify_forwards"], rs["verify_ms"], rs["verify_rows"], rs["verify_out_rows"],
                           rs["verify_kv_pos"], rs["verify_attn_pairs"], peak_bw * tp, peak_tf * tp)
    prefill = unit_roofline(target, rs["prefill_forwards"], rs["prefill_target_ms"], rs["prefill_rows"], 0,
                            rs["prefill_kv_pos"], rs["prefill_attn_pairs"], peak_bw * tp, peak_tf * tp,
                            causal_half=True)
    if tp > 1:  # the draft model is replicated on every rank (one replica per rank's share)
        verify["gpus"] = prefill["gpus"] = tp
        if not os.environ.get("WS_TP_DRAFT_RANK"):
            draft = unit_roofline("llama3.2-1b", rs["draft_forwards"], rs["draft_ms"], rs["draft_rows"],
                                  rs["draft_out_rows"], rs["draft_kv_pos"], rs["draft_attn_pairs"], peak_bw * tp,
                                  peak_tf * tp)
            draft["gpus"] = tp
    draft = unit_roofline("llama3.2-1b", rs["draft_forwards"], rs["draft_ms"], rs["draft_rows"], rs["draft_out_rows"],
                          rs["draft_kv_pos"], rs["draft_attn_pairs"], peak_bw, peak_tf)
    return verify, prefill, draft


def k3_sample(rows, k, peak_bw, iters=20):
    """K3 (fused softmax + entropy + top-2) with the K4 greedy accept walk fused behind it, timed
    alone on a verify-shaped bf16 logits block of `rows` = verify jobs x (k+1) rows (the mean
    verify forward of the run) with candidates: CUDA events on the launching stream, L2 flushed
    (256 MB write) before every launch. Algorithmic bytes = rows x V x 2 (logits read once)."""
    import ctypes as C

    import torch

    import paper_2602_18931_b200 as ws
    from paper_2602_18931_b200 import abi
    L, V = ws.lib(), 128256
    n_req = max(1, rows // (k + 1))
    rows = n_req * (k + 1)
    L.ws_op_row_stats_workspace_bytes.restype = C.c_size_t
    L.ws_op_row_stats_workspace_bytes.argtypes = [C.c_uint32] * 3
    L.ws_op_verify_greedy_bf16.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    g = torch.Generator(device="cuda").manual_seed(7)
    x = (torch.randn(rows, V, device="cuda", generator=g) * 2).to(torch.bfloat16)
    cand = torch.randint(0, V, (n_req * k,), device="cuda", generator=g, dtype=torch.int32)
    wsb = torch.zeros(L.ws_op_row_stats_workspace_bytes(rows, V, n_req), dtype=torch.uint8, device="cuda")
    vout = torch.zeros(n_req * C.sizeof(abi.VerifyOut), dtype=torch.uint8, device="cuda")
    pred = torch.zeros(rows * C.sizeof(abi.Pred), dtype=torch.uint8, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    tot = 0.0
    for it in range(iters + 3):
        flush.fill_(0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        rc = L.ws_op_verify_greedy_bf16(x.data_ptr(), n_req, k, V, V, cand.data_ptr(), vout.data_ptr(),
                                        pred.data_ptr(), wsb.data_ptr(), st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        assert rc == 0
        if it >= 3:
            tot += e0.elapsed_time(e1) / 1e3
    t = tot / iters
    gbs = rows * V * 2 / t / 1e9
    return {"kernel": "K3 row_stats + K4 greedy accept (fused)", "rows": rows, "verify_jobs": n_req, "vocab": V,
            "us": t * 1e6, "bound": "hbm", "achieved": gbs, "peak": peak_bw, "unit": "GB/s", "frac": gbs / peak_bw,
            "timing": "CUDA events, L2 flushed before each launch, the mean verify forward's output rows"}


_CPU_PAIR = None


def cpu_measured(target, k, seq, steps, warmup):
    """The CPU baseline of the Llama workload, measured end to end: the reference's own
    RequestSim (oracle/_ref, unmodified) with its model calls answered by a torch-CPU bf16 port
    of the same Llama pair on all host cores (oracle/cpu_pair.py: same planted bias and
    generation cap), one request at a time as the reference runs them (sim.hpp:433), its prompt
    prefilled before the clock starts. A sample = request 0 decoded to `seq` committed tokens
    (the same deterministic protocol trajectory every sample, so samples differ only by CPU
    timing noise). Returns the line's cpu_baseline object."""
    global _CPU_PAIR
    from oracle import cpu_pair
    if _CPU_PAIR is None or _CPU_PAIR.L != seq or _CPU_PAIR.k != k:
        _CPU_PAIR = cpu_pair.CpuPair(target=target, seq_len=seq, k=k)
    for _ in range(warmup):
        cpu_pair.measure(requests=1, first=0, pair=_CPU_PAIR)
    rates, toks, secs, threads = [], 0, 0.0, 1
    for _ in range(max(1, steps)):
        r, t, el, threads = cpu_pair.measure(requests=1, first=0, pair=_CPU_PAIR)
        rates.append(r)
        toks += t
        secs += el
    value = toks / secs
    spread = (max(rates) - min(rates)) / value if len(rates) > 1 else 0.0
    return {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
            "protocol": "reference RequestSim (oracle/_ref) — its model calls answered by the CPU port",
            "sample": f"{len(rates)} timed sample(s) after {warmup} warm-up: request 0 of config 3 decoded to "
                      f"{seq} committed tokens (prompt prefilled untimed), {target} + llama3.2-1b in torch bf16 on "
                      f"{threads} host threads; per-sample tokens/s min {min(rates):.3f} / median "
                      f"{statistics.median(rates):.3f} / max {max(rates):.3f} (spread {100 * spread:.1f}%)"}


def cpu_port_sample(args, k):
    return cpu_measured("llama3-8b", k, args.cpu_seq, steps=3, warmup=1)


# ------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    if args.workload == "tiny":
        from oracle import pyoracle as po
        if not po.ref_available():
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
            return
        cfg = tiny_cfg(args, 1, 0)
        cfg.num_requests = TINY_REQ_PER_GPU * world
        cfg.first_request, cfg.local_requests = 0, 0
        for _ in range(args.warmup):
            po.ref_run_sim(cfg, threads=threads, with_tokens=False, with_steps=False)
        toks, t0 = 0, time.perf_counter()
        for _ in range(args.steps):
            b = po.ref_run_sim(cfg, threads=threads, with_tokens=False, with_steps=False)
            toks += sum(m["tokens_committed"] for m in b.metrics_list())
        el = time.perf_counter() - t0
        value, sample, kind = toks / el, f"{args.steps} full runs of {cfg.num_requests} requests " \
                                         "(run_sim_full via oracle/_ref, requests over threads)", "reference"
    else:
        # The reference has no model: its CPU path for the config-3 workload is its
        # own RequestSim with the model calls answered by the CPU port, measured end to end.
        cb = cpu_measured(args.target, args.k, args.cpu_seq, steps=args.steps, warmup=min(args.warmup, 1))
        value, sample, kind = cb["value"], cb["sample"], cb["kind"]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
            "scaling": "strong" if args.workload == "llama" else "weak", "vs_baseline": None,
            "dtype": "bf16" if args.workload == "llama" else "f64", "data": "synthetic", "impl": "reference",
            "config": config_block(args, world, threads),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    rank, local_rank, world = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import paper_2602_18931_b200 as ws
    from paper_2602_18931_b200 import abi

    dev0 = local_rank * max(1, args.tp)  # first GPU of this process (tensor-parallel ranks follow)
    torch.cuda.set_device(dev0)
    dist = None
    host_group = None
    split = args.workload == "llama" and args.placement == "split" and world >= 2 and world % 2 == 0
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev0))
        if split:
            # Under split placement rank r's draft lane runs on rank r + N/2's GPU: the idle ranks
            # must not park an NCCL barrier kernel there (a second context on that GPU is
            # time-sliced against the draft forwards), so barriers and the timing reduction go
            # over a host (gloo) group.
            host_group = dist.new_group(backend="gloo")

    def barrier():
        if dist:
            dist.barrier(group=host_group)
        torch.cuda.synchronize()

    ncpu = os.cpu_count() or 1
    host_threads = args.host_threads or max(1, min(16, ncpu // max(1, world)))
    ctx = ws.Context(dev0)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    peak_bw, peak_tf, peak_kind = peaks()

    active = not split or rank < world // 2
    if args.workload == "llama":
        if split:  # requests sharded over the target GPUs; GPU r + N/2 runs rank r's drafts
            cfg = llama_cfg(args, world // 2, min(rank, world // 2 - 1))
        else:
            cfg = llama_cfg(args, world, rank)
        cfg.host_threads = max(1, args.shards)
        if active:
            ctx.load_models(abi.model_cfg(target=args.target, max_requests=args.requests, tp=args.tp),
                            draft_device=(local_rank + world // 2 if split else
                                          dev0 + int(os.environ["WS_TP_DRAFT_RANK"])
                                          if args.tp > 1 and "WS_TP_DRAFT_RANK" in os.environ else -1))

        def run_once(tokens_out=False):
            return ctx.run_model_sim(cfg, with_tokens=tokens_out, with_steps=False)
    else:
        cfg = tiny_cfg(args, world, rank)
        cfg.host_threads = host_threads
        recs = ws.oracle_synth(cfg.oracle, cfg.num_requests)
        ctx.load_oracle(recs, cfg.num_requests, cfg.oracle)

        def run_once(tokens_out=False):
            return ctx.run_sim_full(cfg, with_tokens=tokens_out, with_steps=False, resident=True)

    for _ in range(args.warmup if active else 0):
        run_once()
    tokens, total_ms, launches, kernel_ms, h2d, d2h = 0, 0.0, 0, 0.0, 0, 0
    mstats = {}
    barrier()
    with ClockSampler(dev0) as clk:
        for _ in range(args.steps if active else 0):
            if args.workload == "tiny":
                flush.fill_(1.0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b = run_once(tokens_out=True)
            e1.record()
            torch.cuda.synchronize()
            total_ms += e0.elapsed_time(e1)
            tokens += sum(m["tokens_committed"] for m in b.metrics_list())
            launches += b.out.gpu_launches
            kernel_ms += b.out.kernel_ms
            h2d += b.out.h2d_bytes
            d2h += b.out.d2h_bytes + sum(b.ctrl_len[i] for i in range(b.n)) * 4
            if args.workload == "llama":
                for kk, v in ctx.run_stats().items():
                    mstats[kk] = mstats.get(kk, 0) + v
    barrier()

    torch.cuda.set_device(dev0)
    stats = torch.tensor([total_ms, float(tokens), float(launches)], dtype=torch.float64,
                         device="cpu" if host_group is not None else torch.device("cuda", dev0))
    if dist:
        mx, sm = stats.clone(), stats.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=host_group)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM, group=host_group)
        total_ms_max, tokens_all, launches_all = mx[0].item(), sm[1].item(), sm[2].item()
    else:
        total_ms_max, tokens_all, launches_all = total_ms, float(tokens), float(launches)

    if rank == 0:
        value = tokens_all / (total_ms_max / 1000.0)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world * max(1, args.tp), "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms_max / args.steps, "higher_is_better": True,
                "scaling": "strong" if args.workload == "llama" else "weak", "vs_baseline": None,
                "dtype": "bf16" if args.workload == "llama" else "f64", "data": "synthetic",
                "config": config_block(args, world, host_threads),
                # the public C-ABI call is already end to end: host protocol → per-round H2D of the
                # batch (tokens, positions, slots, groups, candidates) → forwards → D2H of results
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": h2d // max(1, args.steps),
                        "d2h_bytes_per_step": d2h // max(1, args.steps),
                        "note": "the timed step is the public call (ws_run_model_sim / ws_run_sim) from host "
                                "buffers: every round's job tables go H2D and its results D2H inside the timed "
                                "region, so value and e2e are one measurement"},
                "gpu_launches": int(launches_all), "clocks": clk.summary()}
        if args.workload == "llama":
            # a tensor-parallel verify / prefill forward runs on tp GPUs: its roofline is tp x one GPU's
            verify, prefill, draft = llama_rooflines(mstats, args.target, peak_bw, peak_tf, tp=args.tp)
            roof = dict(verify)
            traffic = None
            tpath = os.path.join(ROOT, "profiles", "r02_verify_traffic.json")
            if os.path.exists(tpath) and args.target == "llama3-8b":  # ncu dram bytes of one verify forward
                with open(tpath) as f:
                    tj = json.load(f)
                traffic = tj["dram_read_bytes"] + tj["dram_write_bytes"]
                roof["traffic_rows"] = tj["rows"]
                roof["traffic_source"] = ("profiles/r02_verify_traffic.json (ncu, one verify forward + K3/K4 at "
                                          "%d rows)" % tj["rows"])
            roof.update({"traffic": traffic, "kernel": "verify forward (target model + K3/K4), prompt prefill "
                                                       "excluded", "peak_kind": peak_kind,
                         "prefill": prefill, "draft": draft,
                         "note": "in-run device time of each unit on its own stream while the other lanes run "
                                 "concurrently on the same GPU; per-forward averages"})
            line["roofline"] = roof
            try:
                line["k3"] = k3_sample(max(args.k + 1, int(round(verify["out_rows_per_forward"]))), args.k, peak_bw)
            except Exception as e:  # a secondary figure: never fail the bench line over it
                line["k3"] = {"unavailable": str(e)}
            line["model_time"] = {k: (v / args.steps if isinstance(v, float) else v // args.steps)
                                  for k, v in mstats.items()}
            if world == 1 and args.target != "llama3-8b":
                line["cpu_baseline"] = {"value": None, "unavailable": "the numpy-port sample is defined for the "
                                                                      "config-3 (8B) target"}
            elif world == 1:
                try:
                    line["cpu_baseline"] = cpu_port_sample(args, args.k)
                except Exception as e:  # the CPU port needs ~2 GB of host RAM per 8B layer
                    line["cpu_baseline"] = {"value": None, "unavailable": str(e)}
        else:
            from oracle import pyoracle as po
            alg = 0
            line["roofline"] = {"bound": "hbm", "achieved": None, "peak": peak_bw, "unit": "GB/s", "frac": None,
                                "traffic": None, "kernel": "k9_round", "peak_kind": peak_kind,
                                "note": "K9 moves ~100 KB/launch: latency-bound by construction"}
            if kernel_ms > 0 and launches > 0:
                per_launch_s = kernel_ms / 1e3 / launches
                k9 = (b.out.verify_rows * (32 + 4 * cfg.k + 4 * (cfg.k + 1) + 8 + 16)
                      + b.out.draft_rows * 88) / max(1, b.out.gpu_launches)
                alg = k9 / per_launch_s / 1e9
                line["roofline"].update({"achieved": alg, "frac": alg / peak_bw})
            if world == 1 and po.ref_available():
                t0, toks, runs = time.perf_counter(), 0, 0
                c1 = tiny_cfg(args, 1, 0)
                while time.perf_counter() - t0 < args.cpu_sample_s:
                    rb = po.ref_run_sim(c1, threads=ncpu, with_tokens=False, with_steps=False)
                    toks += sum(m["tokens_committed"] for m in rb.metrics_list())
                    runs += 1
                el = time.perf_counter() - t0
                line["cpu_baseline"] = {"value": toks / el, "unit": UNIT, "cores": ncpu, "kind": "reference",
                                        "sample": f"{runs} runs of 64 requests (reference run_sim_full via "
                                                  "oracle/_ref, all host cores)"}
        print(json.dumps(line))
    ctx.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
