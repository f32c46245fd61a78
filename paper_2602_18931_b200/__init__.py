"""B200-native WANSpec verify / draft hot path (arxiv 2602.18931), Python host mirror.

The product is the native library `_lib/libwanspec_b200.so` (C ABI in
include/wanspec_b200.h): host C++ controller/worker state machines and a batched event
driver calling hand-written sm_100a kernels. This module only loads it and mirrors the
reference's names (run_sim_full, run_target_step, draft_prediction, SimConfig fields) so
tests and benchmarks read like the reference's. There is no CPU fallback: a missing library
raises, and every model call needs a CUDA device.
"""
import ctypes as C
import os

from . import abi
from .abi import (WS_ECONFIG, WS_ECUDA, WS_EARG, WS_ELOGIC, WS_EPROTO, WS_OK,  # noqa: F401
                  WS_VERIFY_GREEDY, WS_VERIFY_REJECTION, WS_MODE_BASELINE, WS_MODE_WANSPEC,
                  apply_stage, config1, config2, oracle_cfg, sim_cfg)

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "_lib", "libwanspec_b200.so")
_P = C.POINTER
_lib = None


class WanspecError(RuntimeError):
    """A negative WS_E* status from the C ABI (types.hpp:35-45 error classes)."""

    def __init__(self, code, msg):
        super().__init__(f"{_CODE_NAMES.get(code, code)}: {msg}")
        self.code = code


class ConfigError(WanspecError):
    pass


_CODE_NAMES = {WS_ECONFIG: "ConfigError", WS_EPROTO: "ProtocolError", WS_ELOGIC: "LogicError",
               WS_ECUDA: "CudaError", WS_EARG: "ArgumentError", abi.WS_EPARSE: "ParseError"}

MODEL_ROUND_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p,
                             C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_uint64)


def lib():
    """Load the native library (built in-tree by build.py / __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"native library missing: {LIB_PATH} (run __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    L.ws_last_error.restype = C.c_char_p
    L.ws_device_count.argtypes = [_P(C.c_int)]
    L.ws_create.argtypes = [C.c_int, _P(C.c_void_p)]
    L.ws_destroy.argtypes = [C.c_void_p]
    L.ws_oracle_synth.argtypes = [_P(abi.OracleCfg), C.c_uint32, _P(abi.TokenRecord)]
    L.ws_load_oracle.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                 _P(abi.TokenRecord)]
    L.ws_verify.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, _P(C.c_uint32), _P(C.c_uint64),
                            _P(C.c_uint32), _P(C.c_uint32), _P(C.c_uint32), _P(C.c_double)]
    L.ws_verify_rejection.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint64,
                                      _P(C.c_uint32), _P(C.c_uint64), _P(C.c_uint32),
                                      _P(C.c_uint64), _P(C.c_uint32), _P(C.c_uint32),
                                      _P(C.c_uint32), _P(C.c_double)]
    L.ws_draft.argtypes = [C.c_void_p, C.c_uint32, _P(C.c_uint32), _P(C.c_uint64), _P(abi.Pred)]
    L.ws_run_sim.argtypes = [C.c_void_p, _P(abi.SimCfg), _P(abi.RunOut)]
    L.ws_run_sim_resident.argtypes = [C.c_void_p, _P(abi.SimCfg), _P(abi.RunOut)]
    L.ws_run_sim_with_model.argtypes = [_P(abi.SimCfg), MODEL_ROUND_FN, C.c_void_p, _P(abi.RunOut)]
    L.ws_model_load.argtypes = [C.c_void_p, _P(abi.ModelCfg)]
    L.ws_model_load_split.argtypes = [C.c_void_p, _P(abi.ModelCfg), C.c_int]
    L.ws_model_export_trace.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, _P(abi.TokenRecord)]
    L.ws_run_model_sim.argtypes = [C.c_void_p, _P(abi.SimCfg), _P(abi.RunOut)]
    L.ws_model_stats.argtypes = [C.c_void_p, _P(C.c_double), _P(C.c_double), _P(C.c_uint64), _P(C.c_uint64),
                                 _P(C.c_uint64), _P(C.c_uint64)]
    _lib = L
    return L


def _check(rc):
    if rc != WS_OK:
        msg = lib().ws_last_error().decode(errors="replace")
        if rc == WS_ECONFIG:
            raise ConfigError(rc, msg)
        raise WanspecError(rc, msg)


def device_count():
    n = C.c_int()
    _check(lib().ws_device_count(C.byref(n)))
    return n.value


def oracle_synth(ocfg, n_seq):
    """Oracle::open + n_seq × next_sequence (oracle.hpp:264-290) on the host."""
    recs = (abi.TokenRecord * (n_seq * ocfg.sequence_length))()
    _check(lib().ws_oracle_synth(C.byref(ocfg), n_seq, recs))
    return recs


class Context:
    """One GPU's hot-path context (ws_ctx): device tables, streams, staging buffers."""

    def __init__(self, device=0):
        self._h = C.c_void_p()
        _check(lib().ws_create(device, C.byref(self._h)))
        self.device = device

    def close(self):
        if self._h:
            lib().ws_destroy(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- tiny pair tables (K9) --
    def load_oracle(self, records, n_seq, ocfg):
        _check(lib().ws_load_oracle(self._h, n_seq, ocfg.sequence_length, ocfg.vocab_size,
                                    ocfg.eos_id, records))

    def run_target_step(self, seq, base, cands):
        """Batched run_target_step (oracle.hpp:127-139): seq/base lists, cands list of lists."""
        n = len(seq)
        k = len(cands[0]) if n else 0
        s = (C.c_uint32 * n)(*seq)
        b = (C.c_uint64 * n)(*base)
        c = (C.c_uint32 * max(1, n * k))(*[t for row in cands for t in row])
        a, bo, h = (C.c_uint32 * n)(), (C.c_uint32 * n)(), (C.c_double * n)()
        _check(lib().ws_verify(self._h, n, k, s, b, c, a, bo, h))
        return [(a[i], bo[i], h[i]) for i in range(n)]

    def rejection_verify(self, seq, request, step, base, cands, sample_seed):
        n = len(seq)
        k = len(cands[0]) if n else 0
        s = (C.c_uint32 * n)(*seq)
        r = (C.c_uint64 * n)(*request)
        st = (C.c_uint32 * n)(*step)
        b = (C.c_uint64 * n)(*base)
        c = (C.c_uint32 * max(1, n * k))(*[t for row in cands for t in row])
        a, bo, h = (C.c_uint32 * n)(), (C.c_uint32 * n)(), (C.c_double * n)()
        _check(lib().ws_verify_rejection(self._h, n, k, sample_seed, s, r, st, b, c, a, bo, h))
        return [(a[i], bo[i], h[i]) for i in range(n)]

    def draft_prediction(self, seq, pos):
        """Batched SequenceTrace::draft_prediction (oracle.hpp:96-98)."""
        n = len(seq)
        s = (C.c_uint32 * n)(*seq)
        p = (C.c_uint64 * n)(*pos)
        out = (abi.Pred * n)()
        _check(lib().ws_draft(self._h, n, s, p, out))
        return [(o.n, tuple(o.id[:o.n]), tuple(o.prob[:o.n]), o.entropy) for o in out]

    # -- real-model pair (config 3) --
    def load_models(self, mcfg, draft_device=-1):
        """Allocate + seed-initialise the target/draft models and their KV pools on this GPU
        (the draft model on `draft_device` under split placement)."""
        self._mcfg = mcfg  # keep the C strings alive
        _check(lib().ws_model_load_split(self._h, C.byref(mcfg), int(draft_device)))

    def export_trace(self, first_request, n, length):
        """Teacher-forced records of the loaded pair (ws_model_export_trace): n * length
        TokenRecords, request-major (see trace.py for the reference's NDJSON format)."""
        recs = (abi.TokenRecord * (n * length))()
        _check(lib().ws_model_export_trace(self._h, first_request, n, length, recs))
        return recs

    def run_model_sim(self, cfg, with_tokens=True, with_steps=True):
        """run_sim_full with the verify/draft model calls on the loaded models."""
        bufs = abi.RunBuffers(cfg, with_tokens, with_steps)
        _check(lib().ws_run_model_sim(self._h, C.byref(cfg), C.byref(bufs.out)))
        return bufs

    def run_model_wallclock(self, cfg, decision_log=None, with_tokens=True, with_steps=True):
        """Wall-clock mode (ws_run_model_wallclock): real time, GPU completions, injected RTT/2
        queues; optional NDJSON decision log for the reference replay."""
        bufs = abi.RunBuffers(cfg, with_tokens, with_steps)
        _check(lib().ws_run_model_wallclock(self._h, C.byref(cfg), C.byref(bufs.out),
                                            decision_log.encode() if decision_log else None))
        return bufs

    def model_stats(self):
        v = [C.c_double(), C.c_double(), C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()]
        _check(lib().ws_model_stats(self._h, *[C.byref(x) for x in v]))
        keys = ("target_ms", "draft_ms", "target_rows", "draft_rows", "target_forwards", "draft_forwards")
        return {k: x.value for k, x in zip(keys, v)}

    # -- per-call model boundary (include/wanspec_b200.h "per-call model boundary") --
    def model_open(self, k, sequence_length, eos_id):
        _check(lib().ws_model_open(self._h, k, sequence_length, eos_id))
        self._call_k = k

    def model_prefill(self, requests):
        r = (C.c_uint32 * max(1, len(requests)))(*requests)
        _check(lib().ws_model_prefill(self._h, len(requests), r))

    def model_verify(self, jobs, with_rows=False):
        """jobs: [(request, committed tokens, candidates)] -> [(accepted, bonus, entropy)] (and
        the per-row predictions when with_rows)."""
        n, k = len(jobs), self._call_k
        js = (abi.ModelJob * max(1, n))()
        toks, cand = [], []
        for j, (req, committed, cands) in enumerate(jobs):
            js[j].request, js[j].kind, js[j].n_committed, js[j].len, js[j].off = (
                req, abi.WS_JOB_VERIFY, len(committed), len(committed), len(toks))
            toks += committed
            assert len(cands) == k
            cand += cands
        t = (C.c_uint32 * max(1, len(toks)))(*toks)
        c = (C.c_uint32 * max(1, len(cand)))(*cand)
        out = (abi.VerifyOut * max(1, n))()
        rows = (abi.Pred * (n * (k + 1))) () if with_rows else None
        _check(lib().ws_model_verify(self._h, n, js, t, c, out, rows))
        res = [(o.accepted, o.bonus, o.final_entropy) for o in out[:n]]
        return (res, list(rows)) if with_rows else res

    def model_draft(self, jobs):
        """jobs: [(request, kind, context tokens, n_committed)] -> [abi.Pred]."""
        n = len(jobs)
        js = (abi.ModelJob * max(1, n))()
        toks = []
        for j, (req, kind, context, n_committed) in enumerate(jobs):
            js[j].request, js[j].kind, js[j].n_committed, js[j].len, js[j].off = (
                req, kind, n_committed, len(context), len(toks))
            toks += context
        t = (C.c_uint32 * max(1, len(toks)))(*toks)
        out = (abi.Pred * max(1, n))()
        _check(lib().ws_model_draft(self._h, n, js, t, out))
        return list(out[:n])

    def model_evict(self, request):
        _check(lib().ws_model_evict(self._h, request))

    def run_stats(self):
        """ws_model_run_stats: verify / draft / prefill device time and rows of the last run."""
        st = abi.RunStats()
        _check(lib().ws_model_run_stats(self._h, C.byref(st)))
        return {f: getattr(st, f) for f, _ in abi.RunStats._fields_}

    # -- whole runs --
    def run_sim_full(self, cfg, with_tokens=True, with_steps=True, resident=False):
        """run_sim_full (sim.hpp:429-442) through the batched GPU driver; returns RunBuffers."""
        bufs = abi.RunBuffers(cfg, with_tokens, with_steps)
        fn = lib().ws_run_sim_resident if resident else lib().ws_run_sim
        _check(fn(self._h, C.byref(cfg), C.byref(bufs.out)))
        return bufs


def run_sim_with_model(cfg, round_fn, with_tokens=True, with_steps=True):
    """The driver with a caller-supplied model round (host-logic tests). round_fn receives
    (n_verify, verify_jobs_ptr, cands_ptr, n_draft, draft_jobs_ptr, verify_out_ptr,
    draft_out_ptr, mode, seed) as raw addresses and returns 0."""
    bufs = abi.RunBuffers(cfg, with_tokens, with_steps)

    def tramp(user, nv, vj, cands, nd, dj, vo, do, mode, seed):
        try:
            return round_fn(nv, vj, cands, nd, dj, vo, do, mode, seed)
        except Exception:  # surfaced as a driver error
            import traceback
            traceback.print_exc()
            return 1

    cb = MODEL_ROUND_FN(tramp)
    _check(lib().ws_run_sim_with_model(C.byref(cfg), cb, None, C.byref(bufs.out)))
    return bufs
