"""Pins the oracle (oracle/restate.c) before anything is checked against it: the reference's
own known-answer tests (proj/tests/unit/test_oracle.cpp), Random123's Philox KATs, and
bit-exact agreement with the reference compiled into oracle/_ref where it is available."""
import ctypes as C
import math

import pytest

from oracle import pyoracle as po
from paper_2602_18931_b200 import abi

ref = pytest.mark.skipif(not po.ref_available(), reason="reference not built (oracle/_ref)")


def small_cfg(seed):  # test_oracle.cpp:21-27
    return abi.oracle_cfg(seed=seed, vocab_size=256, eos_id=255)


# ---- entropy_of (test_oracle.cpp:31-73) ----
def test_entropy_known_answers():
    assert po.entropy_of([1.0]) == 0.0
    assert po.entropy_of([0.5, 0.5]) == pytest.approx(math.log(2.0), rel=1e-12)
    assert po.entropy_of([0.7, 0.2, 0.1]) == pytest.approx(0.80181855, rel=1e-7)
    assert po.entropy_of([0.25, 0.75, 0.0]) == po.entropy_of([0.0, 0.75, 0.25])
    assert po.entropy_of([0.25] * 4) == pytest.approx(math.log(4.0), rel=1e-12)


def test_entropy_rejects_bad_distributions():
    with pytest.raises(ValueError):
        po.entropy_of([0.5, 0.4])
    with pytest.raises(ValueError):
        po.entropy_of([1.2, -0.2])


@ref
def test_entropy_matches_reference_random():
    import random
    rnd = random.Random(5)
    for _ in range(500):  # acceptance_main.cpp:363-380 shape
        n = rnd.randint(1, 12)
        w = [rnd.random() + 1e-6 for _ in range(n)]
        s = sum(w)
        p = [x / s for x in w]
        assert po.entropy_of(p) == po.entropy_of(p, use_ref=True)


# ---- synthesis (test_oracle.cpp:75-195) ----
@ref
@pytest.mark.parametrize("seed", [1, 7, 42, 1234])
def test_synth_bit_exact_vs_reference(seed):
    o = abi.oracle_cfg(seed=seed)
    assert bytes(po.synth(o, 12)) == bytes(po.synth(o, 12, use_ref=True))


def test_synth_matches_golden_fingerprints(golden):
    for s in golden["synth"]:
        recs = po.synth(abi.oracle_cfg(seed=s["seed"]), s["n_seq"])
        got = "%016x" % po.fnv_tokens([list(memoryview(bytes(recs)).cast("I"))])
        assert got == s["bytes_fnv"], s["seed"]


def test_match_rate_calibrates():  # test_oracle.cpp:109-130
    for seed in (1, 7, 42, 1234):
        o = abi.oracle_cfg(seed=seed, match_prob=0.8)
        recs = po.synth(o, 100)
        m = sum(r.draft_top1 == r.target_token for r in recs)
        assert abs(m / len(recs) - 0.8) < 0.02


def test_records_well_formed():  # test_oracle.cpp:152-173
    o = abi.oracle_cfg(seed=5)
    recs = po.synth(o, 5)
    for i, r in enumerate(recs):
        assert r.target_p1 > r.target_p2 > 0 and r.target_p1 + r.target_p2 <= 1.0
        assert r.draft_p1 > r.draft_p2 > 0 and r.draft_p1 + r.draft_p2 <= 1.0
        assert r.target_entropy > 0 and r.draft_entropy > 0
        assert r.draft_top1 != r.draft_top2
        if i % 100 == 99:
            assert r.target_token == o.eos_id


def test_past_end_is_confident_eos():  # test_oracle.cpp:184-195
    o = small_cfg(3)
    o.sequence_length = 4
    recs = po.synth(o, 1)
    a, bonus, h = po.run_target_step(recs, 0, 4, o.eos_id, 100, [])
    assert (a, bonus, h) == (0, o.eos_id, 0.0)
    n, ids, probs, h = po.draft_prediction(recs, 0, 4, o.eos_id, 100)
    assert (n, ids, probs, h) == (1, (o.eos_id,), (1.0,), 0.0)


def test_run_target_step_known_answer():  # test_oracle.cpp:197-214
    o = small_cfg(4)
    o.sequence_length = 6
    recs = po.synth(o, 1)
    t = [recs[i].target_token for i in range(6)]
    a, bonus, _ = po.run_target_step(recs, 0, 6, o.eos_id, 0, [t[0], t[1]])
    assert (a, bonus) == (2, t[2])
    wrong = 8 if t[0] == 7 else 7
    a, bonus, _ = po.run_target_step(recs, 0, 6, o.eos_id, 0, [wrong, t[1]])
    assert (a, bonus) == (0, t[0])


@ref
def test_run_target_step_vs_reference_random():
    import random
    rnd = random.Random(11)
    o = abi.oracle_cfg(seed=3, vocab_size=64, eos_id=63, sequence_length=40)
    recs = po.synth(o, 3)
    for _ in range(2000):
        s = rnd.randrange(3)
        base = rnd.randrange(45)
        k = rnd.randint(0, 9)
        cands = []
        for i in range(k):
            pos = base + i
            tt = recs[s * 40 + pos].target_token if pos < 40 else 63
            cands.append(tt if rnd.random() < 0.8 else rnd.randrange(64))
        assert po.run_target_step(recs, s, 40, 63, base, cands) == \
            po.run_target_step(recs, s, 40, 63, base, cands, use_ref=True)
        pos = rnd.randrange(45)
        assert po.draft_prediction(recs, s, 40, 63, pos) == \
            po.draft_prediction(recs, s, 40, 63, pos, use_ref=True)


# ---- Philox4x32-10 (Random123 kat_vectors) ----
def test_philox_known_answers():
    assert po.philox((0, 0, 0, 0), (0, 0)) == (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)
    assert po.philox((0xffffffff,) * 4, (0xffffffff,) * 2) == \
        (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)
    assert po.philox((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0)) \
        == (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)


# ---- rejection rule (extension; parity unpinned by the reference) ----
def test_rejection_reduces_to_exact_match_for_identical_models():
    """With Pd == Pt every proposal with pt>0 is accepted (u*p < p for u<1)."""
    o = abi.oracle_cfg(seed=9, match_prob=1.0)
    recs = po.synth(o, 1)
    # match_prob 1: draft top-1 == target token, so the candidate has pd = p1_d, pt = p1_t
    L = o.sequence_length
    t = [recs[i].target_token for i in range(L)]
    acc_total = 0
    for step in range(50):
        a, b, h = po.rejection_verify(recs, 0, L, o.eos_id, o.vocab_size, 77, 0, step, 10, t[10:14])
        assert 0 <= a <= 4
        acc_total += a
    assert acc_total > 0


def test_rejection_distribution_matches_target_marginal():
    """Speculative sampling leaves the target distribution invariant: the first committed
    token (accepted candidate or residual draw) is distributed as the completed Pt."""
    o = abi.oracle_cfg(seed=13, vocab_size=8, eos_id=7, sequence_length=4)
    recs = po.synth(o, 1)
    r0 = recs[0]
    pt = {r0.target_token: r0.target_p1, r0.target_top2: r0.target_p2}
    tail = (1.0 - r0.target_p1 - r0.target_p2) / 6
    cand = r0.draft_top1
    counts = {}
    n = 40000
    for step in range(n):
        a, b, _ = po.rejection_verify(recs, 0, 4, 7, 8, 99, 0, step, 0, [cand])
        first = cand if a == 1 else b
        counts[first] = counts.get(first, 0) + 1
    for tok in range(8):
        expect = pt.get(tok, tail)
        assert abs(counts.get(tok, 0) / n - expect) < 0.012, (tok, counts.get(tok, 0) / n, expect)


def test_row_stats_restatement_small():
    import numpy as np
    x = np.array([0.0, 2.0, 2.0, -1.0], dtype=np.float32)
    n, ids, probs, h = po.row_stats(x)
    e = np.exp(x.astype(np.float64) - 2.0)
    p = e / e.sum()
    assert ids == (1, 2)  # tie → lower id first
    assert probs[0] == pytest.approx(p[1], rel=1e-14)
    assert h == pytest.approx(float(-(p * np.log(p)).sum()), rel=1e-12)


def test_unit_from_words_range():
    lib = po.oracle_lib()
    lib.or_unit_from_words.restype = C.c_double
    lib.or_unit_from_words.argtypes = [C.c_uint32, C.c_uint32]
    assert lib.or_unit_from_words(0, 0) == 0.0
    assert lib.or_unit_from_words(0xffffffff, 0xffffffff) < 1.0


def test_model_rejection_restatement_samples_the_target():
    """or_model_rejection_verify (the K4R checker): with no candidates (k = 0) the bonus is a
    draw from the target row p' — empirical frequencies over 20000 Philox counters match the
    softmax; with top_p, tokens outside the nucleus never appear; a candidate whose target
    probability is 1 is always accepted."""
    import math

    import numpy as np
    row = np.array([[2.0, 1.0, 0.5, 0.0, -1.0, 3.0, 0.25, 1.5]], dtype=np.float32)
    p = np.exp(row[0] - row[0].max())
    p /= p.sum()
    counts = np.zeros(8)
    for r in range(20000):
        a, b, h = po.model_rejection_verify(row, 0, [], [], 42, r, 0)
        assert a == 0
        counts[b] += 1
    assert np.abs(counts / 20000 - p).max() < 0.012
    assert h == pytest.approx(-(p * np.log(p)).sum(), rel=1e-12)
    order = np.argsort(-p)
    nucleus = set(order[:np.searchsorted(np.cumsum(p[order]), 0.6) + 1].tolist())
    for r in range(3000):
        _, b, _ = po.model_rejection_verify(row, 0, [], [], 7, r, 0, top_p=0.6)
        assert b in nucleus
    sharp = np.full((3, 8), -1e4, dtype=np.float32)
    sharp[:, 5] = 0.0
    for r in range(200):
        a, b, _ = po.model_rejection_verify(sharp, 2, [5, 5], [0.3, 1.0], 1, r, 3)
        assert (a, b) == (2, 5)
    assert math.isfinite(h)
