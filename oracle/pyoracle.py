"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes access to (a) the plain-C restatement oracle/_build/liboracle.so (restate.c) and
(b) the reference itself compiled into oracle/_ref/libwanspec_ref.so (ref_shim.cpp over
/root/reference/proj/include). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module, and only as the checker.
"""
import ctypes as C
import os
import subprocess

from paper_2602_18931_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIBORACLE = os.path.join(HERE, "_build", "liboracle.so")
LIBREF = os.path.join(HERE, "_ref", "libwanspec_ref.so")
REF_INCLUDE = "/root/reference/proj/include"

_P = C.POINTER


def build(ref=True):
    """Build the checker (restatement always; the reference when its sources are here)."""
    targets = [LIBORACLE]
    if ref and os.path.isdir(REF_INCLUDE):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + [t for t in targets], check=True)


def _load_oracle():
    lib = C.CDLL(LIBORACLE)
    lib.or_synth.argtypes = [_P(abi.OracleCfg), C.c_uint32, _P(abi.TokenRecord)]
    lib.or_entropy_of.argtypes = [_P(C.c_double), C.c_size_t, _P(C.c_double)]
    lib.or_run_target_step.argtypes = [_P(abi.TokenRecord), C.c_uint32, C.c_uint32, C.c_uint64,
                                       _P(C.c_uint32), C.c_uint32, _P(C.c_uint32),
                                       _P(C.c_uint32), _P(C.c_double)]
    lib.or_run_target_step.restype = None
    lib.or_draft_prediction.argtypes = [_P(abi.TokenRecord), C.c_uint32, C.c_uint32, C.c_uint64,
                                        _P(abi.Pred)]
    lib.or_draft_prediction.restype = None
    lib.or_target_prediction.argtypes = lib.or_draft_prediction.argtypes
    lib.or_target_prediction.restype = None
    lib.or_philox4x32_10.argtypes = [_P(C.c_uint32), _P(C.c_uint32), _P(C.c_uint32)]
    lib.or_philox4x32_10.restype = None
    lib.or_rejection_verify.argtypes = [_P(abi.TokenRecord), C.c_uint32, C.c_uint32, C.c_uint32,
                                        C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64,
                                        _P(C.c_uint32), C.c_uint32, _P(C.c_uint32),
                                        _P(C.c_uint32), _P(C.c_double)]
    lib.or_rejection_verify.restype = None
    lib.or_fnv1a_tokens.argtypes = [C.c_uint64, _P(C.c_uint32), C.c_size_t]
    lib.or_fnv1a_tokens.restype = C.c_uint64
    lib.or_row_stats.argtypes = [_P(C.c_float), C.c_uint32, C.c_double, _P(abi.Pred)]
    lib.or_row_stats.restype = None
    lib.or_model_round.argtypes = [_P(abi.TokenRecord), C.c_uint32, C.c_uint32, C.c_uint32,
                                   C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_int, C.c_uint64]
    lib.or_model_round.restype = None
    lib.or_mt64_seed.argtypes = [C.c_void_p, C.c_uint64]
    lib.or_mt64_seed.restype = None
    lib.or_mt64_next.argtypes = [C.c_void_p]
    lib.or_mt64_next.restype = C.c_uint64
    return lib


def _load_ref():
    lib = C.CDLL(LIBREF)
    lib.ref_run_sim.argtypes = [_P(abi.SimCfg), C.c_int, _P(abi.RunOut), C.c_char_p, C.c_size_t]
    lib.ref_oracle_synth.argtypes = [_P(abi.OracleCfg), C.c_uint32, _P(abi.TokenRecord)]
    lib.ref_target_step.argtypes = [_P(abi.TokenRecord), C.c_uint32, C.c_uint32, C.c_uint64,
                                    _P(C.c_uint32), C.c_uint32, _P(C.c_uint32), _P(C.c_uint32),
                                    _P(C.c_double)]
    lib.ref_draft_prediction.argtypes = [_P(abi.TokenRecord), C.c_uint32, C.c_uint32,
                                         C.c_uint64, _P(abi.Pred)]
    lib.ref_entropy_of.argtypes = [_P(C.c_double), C.c_size_t, _P(C.c_double)]
    lib.ref_set_trace_path.argtypes = [C.c_char_p]
    lib.ref_trace_deal.argtypes = [_P(abi.OracleCfg), C.c_char_p, C.c_uint32, C.c_uint32, _P(abi.TokenRecord),
                                   _P(C.c_uint32), C.c_char_p, C.c_size_t]
    return lib


_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        _oracle = _load_oracle()
    return _oracle


def ref_available():
    return os.path.exists(LIBREF)


def ref_lib():
    global _ref
    if _ref is None:
        _ref = _load_ref()
    return _ref


# ---------------- convenience wrappers ----------------
def synth(ocfg, n_seq, use_ref=False):
    recs = (abi.TokenRecord * (n_seq * ocfg.sequence_length))()
    lib = ref_lib() if use_ref else oracle_lib()
    fn = lib.ref_oracle_synth if use_ref else lib.or_synth
    rc = fn(C.byref(ocfg), n_seq, recs)
    if rc != 0:
        raise ValueError(f"synth failed rc={rc}")
    return recs


def entropy_of(probs, use_ref=False):
    arr = (C.c_double * len(probs))(*probs)
    out = C.c_double()
    lib = ref_lib() if use_ref else oracle_lib()
    fn = lib.ref_entropy_of if use_ref else lib.or_entropy_of
    rc = fn(arr, len(probs), C.byref(out))
    if rc != 0:
        raise ValueError("entropy_of: invalid distribution")
    return out.value


def run_target_step(recs, seq_index, seq_len, eos, base, cands, use_ref=False):
    arr = (C.c_uint32 * max(1, len(cands)))(*cands)
    a, b, h = C.c_uint32(), C.c_uint32(), C.c_double()
    ptr = C.cast(C.byref(recs, seq_index * seq_len * C.sizeof(abi.TokenRecord)),
                 _P(abi.TokenRecord))
    if use_ref:
        ref_lib().ref_target_step(ptr, seq_len, eos, base, arr, len(cands), C.byref(a),
                                  C.byref(b), C.byref(h))
    else:
        oracle_lib().or_run_target_step(ptr, seq_len, eos, base, arr, len(cands), C.byref(a),
                                        C.byref(b), C.byref(h))
    return a.value, b.value, h.value


def draft_prediction(recs, seq_index, seq_len, eos, pos, use_ref=False):
    p = abi.Pred()
    ptr = C.cast(C.byref(recs, seq_index * seq_len * C.sizeof(abi.TokenRecord)),
                 _P(abi.TokenRecord))
    if use_ref:
        ref_lib().ref_draft_prediction(ptr, seq_len, eos, pos, C.byref(p))
    else:
        oracle_lib().or_draft_prediction(ptr, seq_len, eos, pos, C.byref(p))
    return (p.n, tuple(p.id[:p.n]), tuple(p.prob[:p.n]), p.entropy)


def rejection_verify(recs, seq_index, seq_len, eos, vocab, seed, request, step, base, cands):
    arr = (C.c_uint32 * max(1, len(cands)))(*cands)
    a, b, h = C.c_uint32(), C.c_uint32(), C.c_double()
    ptr = C.cast(C.byref(recs, seq_index * seq_len * C.sizeof(abi.TokenRecord)),
                 _P(abi.TokenRecord))
    oracle_lib().or_rejection_verify(ptr, seq_len, eos, vocab, seed, request, step, base, arr,
                                     len(cands), C.byref(a), C.byref(b), C.byref(h))
    return a.value, b.value, h.value


def philox(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    oracle_lib().or_philox4x32_10(c, k, o)
    return tuple(o)


def fnv_tokens(streams):
    h = C.c_uint64(0xCBF29CE484222325).value
    lib = oracle_lib()
    for s in streams:
        arr = (C.c_uint32 * max(1, len(s)))(*s)
        h = lib.or_fnv1a_tokens(h, arr, len(s))
    return h


def row_stats(row, inv_temp=1.0):
    """K3 restatement (fp64) for one float32 row (sequence or numpy array)."""
    import numpy as np
    x = np.ascontiguousarray(np.asarray(row, dtype=np.float32))
    p = abi.Pred()
    oracle_lib().or_row_stats(x.ctypes.data_as(_P(C.c_float)), x.size, inv_temp, C.byref(p))
    return (p.n, tuple(p.id[:p.n]), tuple(p.prob[:p.n]), p.entropy)


def model_rejection_verify(rows, k, cands, cand_probs, seed, request, step, inv_temp=1.0, top_p=1.0, forced=None):
    """K4R restatement (oracle/restate.c or_model_rejection_verify) over one request's k+1
    float32 rows (numpy [k+1, V]): returns (accepted, bonus, final_entropy)."""
    import numpy as np
    x = np.ascontiguousarray(np.asarray(rows, dtype=np.float32))
    V = x.shape[1]
    c = (C.c_uint32 * max(1, k))(*cands)
    q = (C.c_double * max(1, k))(*cand_probs)
    f = (C.c_int32 * (k + 1))(*forced) if forced is not None else None
    a, b, h = C.c_uint32(), C.c_uint32(), C.c_double()
    lib = oracle_lib()
    lib.or_model_rejection_verify.argtypes = [_P(C.c_float), C.c_uint32, C.c_uint32, C.c_uint32, C.c_float,
                                              C.c_float, _P(C.c_uint32), _P(C.c_double), C.c_uint64, C.c_uint64,
                                              C.c_uint32, _P(C.c_int32), _P(C.c_uint32), _P(C.c_uint32),
                                              _P(C.c_double)]
    lib.or_model_rejection_verify(x.ctypes.data_as(_P(C.c_float)), k, V, V, inv_temp, top_p, c, q, seed, request,
                                  step, f, C.byref(a), C.byref(b), C.byref(h))
    return a.value, b.value, h.value


def ref_run_sim(cfg, threads=1, with_tokens=True, with_steps=True):
    """The reference's run_sim_full over cfg's shard. Returns abi.RunBuffers."""
    bufs = abi.RunBuffers(cfg, with_tokens, with_steps)
    err = C.create_string_buffer(512)
    rc = ref_lib().ref_run_sim(C.byref(cfg), threads, C.byref(bufs.out), err, 512)
    if rc != 0:
        raise RuntimeError(f"ref_run_sim rc={rc}: {err.value.decode()}")
    return bufs


REF_VERIFY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.POINTER(C.c_uint32), C.c_uint32,
                            C.POINTER(C.c_uint32), C.c_uint32, C.POINTER(abi.VerifyOut))
REF_DRAFT_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32), C.c_uint32,
                           C.c_uint32, C.POINTER(abi.Pred))


def ref_run_sim_models(cfg, verify_fn, draft_fn, with_tokens=True, with_steps=True):
    """The reference's own RequestSim (sim.hpp:166-416) with its model calls answered by
    verify_fn(request, committed, cands) -> (accepted, bonus, final_entropy) and
    draft_fn(request, kind, context, n_committed) -> abi.Pred (ref_shim.cpp model mode)."""
    bufs = abi.RunBuffers(cfg, with_tokens, with_steps)
    err = C.create_string_buffer(512)

    def vtramp(user, req, committed, n, cand, k, out):
        try:
            a, b, h = verify_fn(req, [committed[i] for i in range(n)], [cand[i] for i in range(k)])
            out[0].accepted, out[0].bonus, out[0].final_entropy = a, b, h
            return 0
        except Exception:
            import traceback
            traceback.print_exc()
            return 1

    def dtramp(user, req, kind, context, n, n_committed, out):
        try:
            out[0] = draft_fn(req, kind, [context[i] for i in range(n)], n_committed)
            return 0
        except Exception:
            import traceback
            traceback.print_exc()
            return 1

    vcb, dcb = REF_VERIFY_FN(vtramp), REF_DRAFT_FN(dtramp)
    lib = ref_lib()
    lib.ref_run_sim_models.argtypes = [C.POINTER(abi.SimCfg), REF_VERIFY_FN, REF_DRAFT_FN, C.c_void_p,
                                       C.POINTER(abi.RunOut), C.c_char_p, C.c_size_t]
    rc = lib.ref_run_sim_models(C.byref(cfg), vcb, dcb, None, C.byref(bufs.out), err, 512)
    if rc != 0:
        raise RuntimeError(f"ref_run_sim_models rc={rc}: {err.value.decode()}")
    return bufs


def ref_replay_model_log(cfg, path):
    """The reference's controller state machine replaying a wall-clock decision log
    (ref_shim.cpp ref_replay_model_log): (RunBuffers with the replayed streams / counters, turns)."""
    bufs = abi.RunBuffers(cfg, True, False)
    err = C.create_string_buffer(1024)
    turns = C.c_uint64()
    lib = ref_lib()
    lib.ref_replay_model_log.argtypes = [C.POINTER(abi.SimCfg), C.c_char_p, C.POINTER(abi.RunOut),
                                         C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]
    rc = lib.ref_replay_model_log(C.byref(cfg), path.encode(), C.byref(bufs.out), C.byref(turns), err, 1024)
    if rc != 0:
        raise RuntimeError(f"ref_replay_model_log rc={rc}: {err.value.decode()}")
    return bufs, turns.value


def ref_run_sim_trace(cfg, path, threads=1, with_tokens=True, with_steps=True):
    """run_sim_full with the reference's trace oracle (OracleKind::trace) replaying `path`."""
    lib = ref_lib()
    lib.ref_set_trace_path(path.encode())
    try:
        return ref_run_sim(cfg, threads, with_tokens, with_steps)
    finally:
        lib.ref_set_trace_path(None)


def ref_trace_deal(ocfg, path, n, max_len):
    """The first n sequences the reference's trace oracle deals from `path` (its validation and
    seeded shuffle): (records n * max_len, lengths)."""
    recs = (abi.TokenRecord * (n * max_len))()
    lens = (C.c_uint32 * n)()
    err = C.create_string_buffer(512)
    rc = ref_lib().ref_trace_deal(C.byref(ocfg), path.encode(), n, max_len, recs, lens, err, 512)
    if rc != 0:
        raise RuntimeError(f"ref_trace_deal rc={rc}: {err.value.decode()}")
    return recs, list(lens)


def model_round_fn(cfg):
    """A CPU model round (the restated tiny pair) for ws_run_sim_with_model: the checker
    behind the host-logic parity tests. Synthesizes cfg.num_requests sequences first."""
    recs = synth(cfg.oracle, cfg.num_requests)
    lib = oracle_lib()
    L, eos, V = cfg.oracle.sequence_length, cfg.oracle.eos_id, cfg.oracle.vocab_size

    def fn(nv, vj, cands, nd, dj, vo, do, mode, seed):
        lib.or_model_round(recs, L, eos, V, nv, vj, cands, nd, dj, vo, do, mode, seed)
        return 0

    fn.records = recs
    return fn
