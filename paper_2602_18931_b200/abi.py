"""ctypes mirror of include/wanspec_b200.h (the C ABI's POD layouts and status codes).

Field names follow the reference structs they restate: OracleConfig (oracle.hpp:37-47),
SimConfig (sim.hpp:28-80), RequestMetrics (sim.hpp:121-134), TokenRecord (types.hpp:67-72),
Prediction (types.hpp:56-63).
"""
import ctypes as C

WS_OK = 0
WS_ECONFIG = -1
WS_EPARSE = -2
WS_EPROTO = -3
WS_ELOGIC = -4
WS_ECUDA = -5
WS_EARG = -6

WS_VERIFY_GREEDY = 0
WS_VERIFY_REJECTION = 1
WS_MODE_BASELINE = 0
WS_MODE_WANSPEC = 1

WS_STEP_SYNC_STALL = 1
WS_STEP_ENTROPY_RESET = 2


class TokenRecord(C.Structure):
    _fields_ = [
        ("target_token", C.c_uint32), ("target_top2", C.c_uint32),
        ("target_p1", C.c_double), ("target_p2", C.c_double), ("target_entropy", C.c_double),
        ("draft_top1", C.c_uint32), ("draft_top2", C.c_uint32),
        ("draft_p1", C.c_double), ("draft_p2", C.c_double), ("draft_entropy", C.c_double),
    ]


class Pred(C.Structure):
    _fields_ = [("n", C.c_uint32), ("id", C.c_uint32 * 2), ("pad", C.c_uint32),
                ("prob", C.c_double * 2), ("entropy", C.c_double)]


class VerifyOut(C.Structure):
    """ws_verify_out: one run_target_step result (oracle.hpp:127-139)."""
    _fields_ = [("accepted", C.c_uint32), ("bonus", C.c_uint32), ("final_entropy", C.c_double)]


class OracleCfg(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64), ("vocab_size", C.c_uint32), ("eos_id", C.c_uint32),
        ("match_prob", C.c_double), ("entropy_low", C.c_double), ("entropy_high", C.c_double),
        ("second_correct_prob", C.c_double), ("sequence_length", C.c_uint32), ("pad", C.c_uint32),
    ]


class SimCfg(C.Structure):
    _fields_ = [
        ("mode", C.c_int32), ("verify", C.c_int32),
        ("rtt", C.c_int64), ("jitter", C.c_int64), ("r_estimate", C.c_int64),
        ("t_target", C.c_int64), ("t_draft", C.c_int64),
        ("k", C.c_uint32), ("b", C.c_uint32), ("s", C.c_uint32),
        ("catchup_batch_limit", C.c_uint32),
        ("theta", C.c_double), ("phi", C.c_double),
        ("max_nodes", C.c_uint32), ("wait_backstop", C.c_int32),
        ("num_requests", C.c_uint32), ("first_request", C.c_uint32),
        ("local_requests", C.c_uint32), ("host_threads", C.c_uint32),
        ("sample_seed", C.c_uint64),
        ("oracle", OracleCfg),
        ("top_p", C.c_float), ("temperature", C.c_float),
    ]


class RequestMetrics(C.Structure):
    _fields_ = [(n, C.c_int64 if n == "latency" else C.c_uint64) for n in (
        "latency", "tokens_committed", "target_steps", "ctrl_draft_passes",
        "ctrl_local_draft_steps", "ctrl_catchup_batches", "worker_draft_steps",
        "sync_stalls", "entropy_resets", "stale_specs")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class StepLog(C.Structure):
    _fields_ = [("request", C.c_uint32), ("step", C.c_uint32), ("base", C.c_uint64),
                ("accepted", C.c_uint32), ("bonus", C.c_uint32), ("final_entropy", C.c_double),
                ("time", C.c_int64), ("flags", C.c_uint32), ("pad", C.c_uint32)]


class RunOut(C.Structure):
    _fields_ = [
        ("metrics", C.POINTER(RequestMetrics)),
        ("ctrl_tokens", C.POINTER(C.c_uint32)), ("ctrl_len", C.POINTER(C.c_uint32)),
        ("wrk_tokens", C.POINTER(C.c_uint32)), ("wrk_len", C.POINTER(C.c_uint32)),
        ("max_len", C.c_uint32), ("pad", C.c_uint32),
        ("steps", C.POINTER(StepLog)), ("max_steps", C.c_uint64), ("n_steps", C.c_uint64),
        ("rounds", C.c_uint64), ("gpu_launches", C.c_uint64), ("verify_rows", C.c_uint64),
        ("draft_rows", C.c_uint64), ("kernel_ms", C.c_double),
        ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
    ]


class ModelCfg(C.Structure):
    _fields_ = [("target", C.c_char_p), ("draft", C.c_char_p), ("seed", C.c_uint64),
                ("prompt_len", C.c_uint32), ("max_requests", C.c_uint32), ("max_ctx", C.c_uint32),
                ("trie_slots", C.c_uint32), ("plant_target", C.c_float), ("plant_draft", C.c_float),
                ("draft_plant_rate", C.c_float), ("tp", C.c_uint32)]


def model_cfg(target="llama3-8b", draft="llama3.2-1b", seed=1, prompt_len=128, max_requests=256,
              max_ctx=256, trie_slots=512, plant_target=16.0, plant_draft=16.0, draft_plant_rate=0.8, tp=1):
    """The config-3 model pair (random-init Llama shapes + planted shared bigram bias); tp > 1
    splits the target over GPUs device .. device + tp - 1 (BASELINE config 5)."""
    return ModelCfg(target.encode(), draft.encode(), seed, prompt_len, max_requests, max_ctx, trie_slots,
                    plant_target, plant_draft, draft_plant_rate, tp)


LLAMA_VOCAB = 128256
LLAMA_EOS = 128001


def config3(num_requests=256, k=4, seq_len=100, vocab=LLAMA_VOCAB, eos=LLAMA_EOS):
    """BASELINE configs[2]: 256 requests, k in {4, 8}, b=2, s=4, theta=phi=0.5, RTT 20 ms,
    100 generated tokens; max_nodes=256 as config 2."""
    return apply_stage(sim_cfg(k=k, rtt=20000, num_requests=num_requests, max_nodes=256,
                               vocab_size=vocab, eos_id=eos, sequence_length=seq_len), "full")


def oracle_cfg(seed=1, vocab_size=32768, eos_id=32767, match_prob=0.8, entropy_low=0.3,
               entropy_high=1.5, second_correct_prob=0.3, sequence_length=100):
    """OracleConfig defaults (oracle.hpp:37-47)."""
    return OracleCfg(seed, vocab_size, eos_id, match_prob, entropy_low, entropy_high,
                     second_correct_prob, sequence_length, 0)


def sim_cfg(mode=WS_MODE_WANSPEC, verify=WS_VERIFY_GREEDY, rtt=0, jitter=0, r_estimate=-1,
            t_target=23400, t_draft=7500, k=2, b=2, s=4, theta=0.5, phi=0.5,
            catchup_batch_limit=32, max_nodes=64, wait_backstop=False, num_requests=1,
            first_request=0, local_requests=0, host_threads=1, sample_seed=0, oracle=None, **oracle_kw):
    """SimConfig defaults (sim.hpp:28-45); oracle_kw forwarded to oracle_cfg."""
    c = SimCfg()
    c.mode, c.verify = mode, verify
    c.rtt, c.jitter, c.r_estimate = rtt, jitter, r_estimate
    c.t_target, c.t_draft = t_target, t_draft
    c.k, c.b, c.s = k, b, s
    c.catchup_batch_limit = catchup_batch_limit
    c.theta, c.phi = theta, phi
    c.max_nodes = max_nodes
    c.wait_backstop = 1 if wait_backstop else 0
    c.num_requests, c.first_request, c.local_requests = num_requests, first_request, local_requests
    c.host_threads = host_threads
    c.sample_seed = sample_seed
    c.oracle = oracle if oracle is not None else oracle_cfg(**oracle_kw)
    return c


def apply_stage(c, stage):
    """apply_stage (sim.hpp:97-119): cumulative ablation stages."""
    c.mode = WS_MODE_WANSPEC
    if stage == "plain":
        c.b, c.theta, c.phi = 1, 0.0, 0.0
    elif stage == "branching":
        c.b, c.theta, c.phi = 2, 0.0, 0.0
    elif stage == "branching_theta":
        c.b, c.phi = 2, 0.0
    elif stage == "full":
        c.b = 2
    else:
        raise ValueError(stage)
    return c


def config1():
    """BASELINE configs[0]: default single-request simulation, k=4, wanspec_full, RTT 20 ms
    (SURVEY §8d row 1)."""
    return apply_stage(sim_cfg(k=4, rtt=20000, num_requests=1), "full")


def config2(verify=WS_VERIFY_GREEDY, num_requests=64, seed=1, max_nodes=256):
    """BASELINE configs[1]: 64 requests, k=8, b=2, s=4, theta=phi=0.5, RTT 20 ms;
    max_nodes=256 (the reference livelocks at its default 64)."""
    c = apply_stage(sim_cfg(k=8, rtt=20000, num_requests=num_requests, max_nodes=max_nodes,
                            verify=verify, sample_seed=0x5EED, seed=seed), "full")
    return c


def sim_cfg_from_dict(d):
    """Inverse of the golden fixtures' config dicts."""
    c = SimCfg()
    for k, v in d.items():
        if k == "oracle":
            o = OracleCfg()
            for kk, vv in v.items():
                setattr(o, kk, vv)
            c.oracle = o
        else:
            setattr(c, k, v)
    return c


def sim_cfg_to_dict(c):
    d = {n: getattr(c, n) for n, _ in SimCfg._fields_ if n != "oracle"}
    d["oracle"] = {n: getattr(c.oracle, n) for n, _ in OracleCfg._fields_}
    return d


class RunBuffers:
    """Caller-owned output buffers for ws_run_sim / ref_run_sim."""

    def __init__(self, cfg, with_tokens=True, with_steps=True):
        n = cfg.local_requests or (cfg.num_requests - cfg.first_request)
        self.n = n
        self.max_len = cfg.oracle.sequence_length + 2 * cfg.k + 4
        self.metrics = (RequestMetrics * n)()
        self.ctrl_len = (C.c_uint32 * n)()
        self.wrk_len = (C.c_uint32 * n)()
        self.ctrl_tokens = (C.c_uint32 * (n * self.max_len))() if with_tokens else None
        self.wrk_tokens = (C.c_uint32 * (n * self.max_len))() if with_tokens else None
        self.max_steps = n * (self.max_len + 4) if with_steps else 0
        self.steps = (StepLog * self.max_steps)() if with_steps else None
        self.out = RunOut()
        o = self.out
        o.metrics = self.metrics
        o.ctrl_len, o.wrk_len = self.ctrl_len, self.wrk_len
        o.ctrl_tokens = self.ctrl_tokens if with_tokens else None
        o.wrk_tokens = self.wrk_tokens if with_tokens else None
        o.max_len = self.max_len
        o.steps = self.steps if with_steps else None
        o.max_steps = self.max_steps

    def ctrl_outputs(self):
        return [list(self.ctrl_tokens[i * self.max_len:i * self.max_len + self.ctrl_len[i]])
                for i in range(self.n)]

    def wrk_outputs(self):
        return [list(self.wrk_tokens[i * self.max_len:i * self.max_len + self.wrk_len[i]])
                for i in range(self.n)]

    def metrics_list(self):
        return [self.metrics[i].as_dict() for i in range(self.n)]

    def step_list(self):
        n = min(self.out.n_steps, self.max_steps)
        return [(s.request, s.step, s.base, s.accepted, s.bonus, s.final_entropy, s.flags)
                for s in self.steps[:n]]


class RunStats(C.Structure):
    """ws_run_stats (include/wanspec_b200.h): per-unit device time of the last model run."""
    _fields_ = [("verify_ms", C.c_double), ("draft_ms", C.c_double), ("prefill_target_ms", C.c_double),
                ("prefill_draft_ms", C.c_double), ("verify_rows", C.c_uint64), ("verify_out_rows", C.c_uint64),
                ("verify_forwards", C.c_uint64), ("draft_rows", C.c_uint64), ("draft_out_rows", C.c_uint64),
                ("draft_forwards", C.c_uint64), ("prefill_rows", C.c_uint64), ("prefill_forwards", C.c_uint64),
                ("verify_kv_pos", C.c_uint64), ("verify_attn_pairs", C.c_uint64), ("draft_kv_pos", C.c_uint64),
                ("draft_attn_pairs", C.c_uint64), ("prefill_kv_pos", C.c_uint64), ("prefill_attn_pairs", C.c_uint64)]


WS_JOB_VERIFY, WS_JOB_CTRL_DRAFT, WS_JOB_WORKER_DRAFT = 0, 1, 2


class ModelJob(C.Structure):
    """ws_model_job: one per-call model job (request, kind, committed / context lengths)."""
    _fields_ = [("request", C.c_uint32), ("kind", C.c_uint32), ("n_committed", C.c_uint32), ("len", C.c_uint32),
                ("off", C.c_uint64)]


class WireMsg(C.Structure):
    """ws_wire_msg (include/wanspec_b200.h): one protocol message, flat."""
    _fields_ = [("kind", C.c_uint32), ("n_path", C.c_uint32), ("request_id", C.c_uint64), ("seq_no", C.c_uint64),
                ("base", C.c_uint64), ("config_digest", C.c_uint64), ("final_length", C.c_uint64),
                ("n_cands", C.c_uint32), ("cand_token", C.c_uint32 * 2), ("cand_prob", C.c_double * 2),
                ("cand_entropy", C.c_double * 2), ("n_accepted", C.c_uint32), ("bonus", C.c_uint32),
                ("final_entropy", C.c_double), ("path", C.c_uint32 * 1024), ("accepted", C.c_uint32 * 255),
                ("pad", C.c_uint32)]

