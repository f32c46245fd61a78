"""Experiment front-end: the reference's INI experiment files, suites, CSV,
per-seed CSV and manifest (experiment.hpp:25-596, sim.hpp:469-645), driving the B200 path.

Same file format and errors (parse_experiment, experiment.hpp:168-282: unknown sections / keys
rejected with their line numbers), the same suites over paired seeds (single, ablation,
phi_sweep; median ratios of per-seed totals, sim.hpp:469-522; phi grid = quantiles of the
observed target entropy, sim.hpp:574-606), byte-identical CSV rendering (kCsvHeader /
kPerSeedCsvHeader, experiment.hpp:322-390) and a manifest embedding the source text
(experiment.hpp:409-442). Every run goes through a `runner(cfg) -> RunBuffers`:

  * harness "sim" (the tiny oracle pair): Context.run_sim_full — the K9 path on the GPU, whose
    per-request metrics equal the reference's run_sim_full; tests/test_experiment_frontend.py
    renders the reference's own suites (oracle/_ref) beside ours and compares the CSVs byte for byte;
  * harness "model": the loaded Llama-shape pair (Context.run_model_sim), seed i selecting the
    i-th block of `requests` prompts; phi grid from the pair's teacher-forced target entropies;
  * harness "wallclock": the same pair in wall-clock mode (Context.run_model_wallclock; real µs).

The deploy suite's networked rows (TCP loopback, runtime.hpp:506-528) are out of scope: the WAN
is modelled in-box; its "runtime" rows are rendered with status "skipped".
"""
import json
import math

from . import abi

KCSV_HEADER = ("suite,harness,mode,rtt_ms,phi,theta,b,s,k,seed,requests,iterations,"
               "median_latency_us,baseline_median_latency_us,median_latency_ratio,"
               "median_ctrl_draft_passes,baseline_median_ctrl_draft_passes,"
               "median_ctrl_draft_ratio,median_sync_stalls,median_worker_draft_steps,status")
KPER_SEED_HEADER = ("suite,harness,mode,rtt_ms,phi,seed,requests,latency_us,ctrl_draft_passes,"
                    "sync_stalls,worker_draft_steps,tokens_committed,baseline_latency_us,"
                    "baseline_ctrl_draft_passes")
RATIO_DEFINITION = ("median over paired seeds of (wanspec total / baseline total); totals are "
                    "summed over the run's requests; ctrl draft passes count every controller "
                    "draft forward pass including catch-up batches; the baseline denominator "
                    "counts all baseline draft forward passes")
SUITES = ("single", "ablation", "phi_sweep", "deploy")
STAGES = ("wanspec_plain", "wanspec_branch", "wanspec_branch_theta", "wanspec_full")


class ParseError(ValueError):
    """ParseError (types.hpp:39)."""


def ms_to_us(ms):  # types.hpp:22-24 (llround)
    x = ms * 1000.0
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


class ExperimentConfig:
    """ExperimentConfig (experiment.hpp:25-95) with its defaults."""

    def __init__(self):
        self.suite = "single"
        self.mode = "wanspec_full"
        self.seed = 1
        self.iterations = 20
        self.requests = 3
        self.oracle = dict(kind="stochastic", seed=1, vocab_size=32768, eos_id=32767, match_prob=0.8,
                           entropy_low=0.3, entropy_high=1.5, second_correct_prob=0.3, sequence_length=100,
                           trace_path="")
        self.profile = "l40s"
        self.t_target, self.t_draft = 23400, 7500
        self.k, self.b, self.s = 2, 2, 4
        self.theta, self.phi = 0.5, 0.5
        self.catchup_batch_limit = 32
        self.max_nodes = 64
        self.wait_backstop = False
        self.rtt_us = [0]
        self.phi_points = 100
        self.jitter = 0
        self.csv_path = "results.csv"
        self.per_seed_csv_path = ""
        self.manifest_path = ""
        self.source_text = ""

    def to_sim(self):
        """ExperimentConfig::to_sim (experiment.hpp:68-86) as a ws_sim_cfg."""
        o = self.oracle
        c = abi.sim_cfg(t_target=self.t_target, t_draft=self.t_draft, k=self.k, b=self.b, s=self.s,
                        theta=self.theta, phi=self.phi, catchup_batch_limit=self.catchup_batch_limit,
                        max_nodes=self.max_nodes, wait_backstop=self.wait_backstop, num_requests=self.requests,
                        jitter=self.jitter,
                        oracle=abi.oracle_cfg(seed=self.seed, vocab_size=o["vocab_size"], eos_id=o["eos_id"],
                                              match_prob=o["match_prob"], entropy_low=o["entropy_low"],
                                              entropy_high=o["entropy_high"],
                                              second_correct_prob=o["second_correct_prob"],
                                              sequence_length=o["sequence_length"]))
        return c


def _copy(c):
    d = abi.SimCfg()
    C_memmove(d, c)
    return d


def C_memmove(dst, src):
    import ctypes
    ctypes.memmove(ctypes.addressof(dst), ctypes.addressof(src), ctypes.sizeof(src))


_STAGE = {"wanspec_plain": "plain", "wanspec_branch": "branching", "wanspec_branch_theta": "branching_theta",
          "wanspec_full": "full"}


def apply_stage(c, stage):
    """apply_stage (sim.hpp:97-119) on a copy; stage names as stage_name (sim.hpp:86-93)."""
    return abi.apply_stage(_copy(c), _STAGE[stage])


def apply_mode(c, mode):
    """apply_mode (experiment.hpp:99-109)."""
    if mode == "baseline":
        d = _copy(c)
        d.mode = abi.WS_MODE_BASELINE
        return d
    if mode in ("wanspec", "wanspec_full"):
        return apply_stage(c, "wanspec_full")
    if mode in STAGES:
        return apply_stage(c, mode)
    raise ValueError(f'experiment: unknown mode "{mode}"')


class _Parser:
    def __init__(self):
        self.lineno = 0

    def fail(self, msg):
        raise ParseError(f"line {self.lineno}: {msg}")

    def number(self, v):
        try:
            return float(v)
        except ValueError:
            self.fail(f'expected a number, got "{v}"')

    def integer(self, v):
        d = self.number(v)
        if d < 0 or int(d) != d:
            self.fail("expected a non-negative integer")
        return int(d)

    def boolean(self, v):
        if v in ("true", "on", "1"):
            return True
        if v in ("false", "off", "0"):
            return False
        self.fail("expected true/false")

    def list(self, v):
        out = []
        for item in v.split(","):
            item = item.strip(" \t\r")
            if not item:
                self.fail("empty list element")
            out.append(self.number(item))
        return out


def parse_experiment(text):
    """parse_experiment (experiment.hpp:168-282): same sections, keys, defaults and errors."""
    cfg = ExperimentConfig()
    cfg.source_text = text
    p = _Parser()
    section = ""
    custom_tt = custom_td = False
    for raw in text.split("\n"):
        p.lineno += 1
        line = raw.split("#", 1)[0].strip(" \t\r")
        if not line:
            continue
        if line[0] == "[":
            if line[-1] != "]":
                p.fail("unterminated section header")
            section = line[1:-1]
            if section not in ("experiment", "oracle", "timing", "protocol", "grid", "output"):
                p.fail(f"unknown section [{section}]")
            continue
        if "=" not in line:
            p.fail("expected key = value")
        key, val = (x.strip(" \t\r") for x in line.split("=", 1))
        if not key or not val:
            p.fail("empty key or value")
        if not section:
            p.fail("key before any [section]")
        o = cfg.oracle
        if section == "experiment":
            if key == "suite":
                if val not in SUITES:
                    p.fail(f'unknown suite "{val}"')
                cfg.suite = val
            elif key == "mode":
                cfg.mode = val
            elif key == "seed":
                cfg.seed = p.integer(val)
            elif key == "iterations":
                cfg.iterations = p.integer(val)
            elif key == "requests":
                cfg.requests = p.integer(val)
            else:
                p.fail(f'unknown key "{key}" in [experiment]')
        elif section == "oracle":
            if key == "kind":
                if val not in ("stochastic", "trace"):
                    p.fail(f'unknown oracle kind "{val}"')
                o["kind"] = val
            elif key in ("match_prob", "entropy_low", "entropy_high", "second_correct_prob"):
                o[key] = p.number(val)
            elif key in ("sequence_length", "vocab_size", "eos_id"):
                o[key] = p.integer(val)
            elif key == "trace_path":
                o["trace_path"] = val
            else:
                p.fail(f'unknown key "{key}" in [oracle]')
        elif section == "timing":
            if key == "profile":
                cfg.profile = val
                if val == "l40s":
                    cfg.t_target, cfg.t_draft = 23400, 7500
                elif val == "swiftspec":
                    cfg.t_target, cfg.t_draft = 6000, 1000
                elif val != "custom":
                    p.fail(f'unknown profile "{val}" (l40s, swiftspec, custom)')
            elif key == "t_target_ms":
                cfg.t_target, custom_tt = ms_to_us(p.number(val)), True
            elif key == "t_draft_ms":
                cfg.t_draft, custom_td = ms_to_us(p.number(val)), True
            else:
                p.fail(f'unknown key "{key}" in [timing]')
        elif section == "protocol":
            if key in ("k", "b", "s", "catchup_batch_limit", "max_nodes"):
                setattr(cfg, key, p.integer(val))
            elif key in ("theta", "phi"):
                setattr(cfg, key, p.number(val))
            elif key == "wait_backstop":
                cfg.wait_backstop = p.boolean(val)
            else:
                p.fail(f'unknown key "{key}" in [protocol]')
        elif section == "grid":
            if key == "rtt_ms":
                cfg.rtt_us = [ms_to_us(ms) for ms in p.list(val)]
            elif key == "phi_points":
                cfg.phi_points = p.integer(val)
            elif key == "jitter_ms":
                cfg.jitter = ms_to_us(p.number(val))
            else:
                p.fail(f'unknown key "{key}" in [grid]')
        elif section == "output":
            if key == "csv":
                cfg.csv_path = val
            elif key == "per_seed_csv":
                cfg.per_seed_csv_path = val
            elif key == "manifest":
                cfg.manifest_path = val
    if cfg.profile == "custom" and not (custom_tt and custom_td):
        raise ParseError('timing profile "custom" needs t_target_ms and t_draft_ms')

    def stem(path):
        return path.rsplit(".", 1)[0] if "." in path else path
    if not cfg.per_seed_csv_path:
        cfg.per_seed_csv_path = stem(cfg.csv_path) + "_per_seed.csv"
    if not cfg.manifest_path:
        cfg.manifest_path = stem(cfg.csv_path) + ".manifest.json"
    if cfg.iterations < 1:
        raise ValueError("experiment: iterations must be >= 1")
    if cfg.suite == "phi_sweep" and cfg.phi_points < 2:
        raise ValueError("experiment: phi_points must be >= 2")
    apply_mode(cfg.to_sim(), cfg.mode)  # reject bad single-suite modes early
    return cfg


# ---------------------------------------------------------------- paired runs (sim.hpp:469-522)
def _totals(bufs):
    ms = bufs.metrics_list()
    return dict(latency=sum(m["latency"] for m in ms), passes=sum(m["ctrl_draft_passes"] for m in ms),
                stalls=sum(m["sync_stalls"] for m in ms), wsteps=sum(m["worker_draft_steps"] for m in ms),
                tokens=sum(m["tokens_committed"] for m in ms))


def median(v):  # sim.hpp:157-162
    v = sorted(v)
    n = len(v)
    if not n:
        return 0.0
    return v[n // 2] if n % 2 else 0.5 * (v[n // 2 - 1] + v[n // 2])


def paired_ratios(runs, baselines):
    r = dict(median_latency_ratio=median([w["latency"] / b["latency"] for w, b in zip(runs, baselines)]),
             median_token_ratio=median([w["passes"] / b["passes"] for w, b in zip(runs, baselines)]),
             median_latency_us=median([float(w["latency"]) for w in runs]),
             median_ctrl_passes=median([float(w["passes"]) for w in runs]),
             baseline_median_latency_us=median([float(b["latency"]) for b in baselines]),
             baseline_median_ctrl_passes=median([float(b["passes"]) for b in baselines]),
             median_sync_stalls=median([float(w["stalls"]) for w in runs]),
             median_worker_steps=median([float(w["wsteps"]) for w in runs]))
    return r


class Result:
    def __init__(self, cfg, effective_seed):
        self.config = cfg
        self.effective_seed = effective_seed
        self.rows = []
        self.per_seed = []
        self.ok = True


def _seeded(c, seed):
    d = _copy(c)
    d.oracle.seed = seed
    return d


def _baselines(runner, base, iterations):
    out = []
    for i in range(iterations):
        c = _copy(base)
        c.mode = abi.WS_MODE_BASELINE
        c.rtt, c.jitter = 0, 0
        c.oracle.seed = base.oracle.seed + i
        out.append(_totals(runner(c)))
    return out


def _row(res, harness, mode, c, rtt, phi, ratios, status="ok"):
    res.rows.append(dict(harness=harness, mode=mode, rtt=rtt, phi=phi, theta=c.theta, b=c.b, s=c.s, k=c.k,
                         ratios=ratios, status=status))


def _per_seed(res, harness, mode, rtt, phi, base_seed, runs, baselines):
    for i, (w, b) in enumerate(zip(runs, baselines)):
        res.per_seed.append(dict(harness=harness, mode=mode, rtt=rtt, phi=phi, seed=base_seed + i, run=w, base=b))


def phi_quantiles(entropies, points):
    """phi_quantiles (sim.hpp:574-594) over an observed target entropy list."""
    e = sorted(entropies)
    return [e[int((i * (len(e) - 1)) / (points - 1) + 0.5)] for i in range(points)]


def run_experiment(cfg, effective_seed, runner, harness="sim", entropies=None):
    """run_experiment (experiment.hpp:573-596) with `runner(ws_sim_cfg) -> RunBuffers`.
    entropies(base_cfg) -> the observed target entropies (phi grid) for the phi sweep."""
    res = Result(cfg, effective_seed)
    base = cfg.to_sim()
    base.oracle.seed = effective_seed
    baselines = _baselines(runner, base, cfg.iterations)
    if cfg.suite in ("single", "deploy"):
        mode_cfg = apply_mode(base, cfg.mode)
        for rtt in cfg.rtt_us:
            runs = []
            for i in range(cfg.iterations):
                c = _seeded(mode_cfg, base.oracle.seed + i)
                c.rtt = rtt
                runs.append(_totals(runner(c)))
            _row(res, harness, cfg.mode, mode_cfg, rtt, mode_cfg.phi, paired_ratios(runs, baselines))
            _per_seed(res, harness, cfg.mode, rtt, mode_cfg.phi, base.oracle.seed, runs, baselines)
            if cfg.suite == "deploy":
                _row(res, "runtime", cfg.mode, mode_cfg, rtt, mode_cfg.phi, paired_ratios([], []),
                     "skipped: TCP loopback out of scope (in-box WAN; use harness wallclock)")
    elif cfg.suite == "ablation":
        for rtt in cfg.rtt_us:
            for stage in STAGES:
                st = apply_stage(base, stage)
                runs = []
                for i in range(cfg.iterations):
                    c = _seeded(st, base.oracle.seed + i)
                    c.rtt = rtt
                    runs.append(_totals(runner(c)))
                _row(res, harness, stage, st, rtt, st.phi, paired_ratios(runs, baselines))
                _per_seed(res, harness, stage, rtt, st.phi, base.oracle.seed, runs, baselines)
    elif cfg.suite == "phi_sweep":
        ent = entropies(base) if entropies else None
        if ent is None:
            raise ValueError("phi sweep needs the observed target entropies")
        for rtt in cfg.rtt_us:
            for phi in phi_quantiles(ent, cfg.phi_points):
                runs = []
                for i in range(cfg.iterations):
                    c = _seeded(base, base.oracle.seed + i)
                    c.mode = abi.WS_MODE_WANSPEC
                    c.rtt, c.phi = rtt, phi
                    runs.append(_totals(runner(c)))
                pc = _copy(base)
                pc.phi = phi
                _row(res, harness, "wanspec_full", pc, rtt, phi, paired_ratios(runs, baselines))
                _per_seed(res, harness, "wanspec_full", rtt, phi, base.oracle.seed, runs, baselines)
    return res


# ---------------------------------------------------------------- rendering (experiment.hpp:322-426)
def _f(v):
    return "%.6f" % v


def _fms(us):
    return "%.3f" % (us / 1000.0)


def render_csv(r):
    c = r.config
    out = [KCSV_HEADER]
    for w in r.rows:
        q = w["ratios"]
        out.append(",".join([c.suite, w["harness"], w["mode"], _fms(w["rtt"]), _f(w["phi"]), _f(w["theta"]),
                             str(w["b"]), str(w["s"]), str(w["k"]), str(r.effective_seed), str(c.requests),
                             str(c.iterations), _f(q["median_latency_us"]), _f(q["baseline_median_latency_us"]),
                             _f(q["median_latency_ratio"]), _f(q["median_ctrl_passes"]),
                             _f(q["baseline_median_ctrl_passes"]), _f(q["median_token_ratio"]),
                             _f(q["median_sync_stalls"]), _f(q["median_worker_steps"]), w["status"]]))
    return "\n".join(out) + "\n"


def render_per_seed_csv(r):
    c = r.config
    out = [KPER_SEED_HEADER]
    for p in r.per_seed:
        w, b = p["run"], p["base"]
        out.append(",".join([c.suite, p["harness"], p["mode"], _fms(p["rtt"]), _f(p["phi"]), str(p["seed"]),
                             str(c.requests), str(w["latency"]), str(w["passes"]), str(w["stalls"]),
                             str(w["wsteps"]), str(w["tokens"]), str(b["latency"]), str(b["passes"])]))
    return "\n".join(out) + "\n"


def render_manifest(r):
    m = {"tool": "wanspec", "format": 1, "suite": r.config.suite, "effective_seed": r.effective_seed,
         "csv": r.config.csv_path, "per_seed_csv": r.config.per_seed_csv_path, "csv_columns": KCSV_HEADER,
         "per_seed_columns": KPER_SEED_HEADER, "ratio_definition": RATIO_DEFINITION,
         "source": r.config.source_text}
    return json.dumps(m, indent=2, ensure_ascii=False) + "\n"


def config_from_manifest(text):
    """config_from_manifest (experiment.hpp:430-442): the embedded file with its seed pinned."""
    m = json.loads(text)
    if "source" not in m or "effective_seed" not in m:
        raise ParseError("manifest: missing source or effective_seed")
    cfg = parse_experiment(m["source"])
    cfg.seed = m["effective_seed"]
    return cfg


def write_outputs(r, directory="."):
    import os
    for path, text in ((r.config.csv_path, render_csv(r)), (r.config.per_seed_csv_path, render_per_seed_csv(r)),
                       (r.config.manifest_path, render_manifest(r))):
        with open(os.path.join(directory, path), "w") as f:
            f.write(text)
