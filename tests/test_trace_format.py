"""The NDJSON trace writer (paper_2602_18931_b200/trace.py) against the reference's trace
validation rules (oracle.hpp trace_io): canonical field order, candidate order, probability
ranges, entropy-zero iff certain — including the edge cases a real model's records hit."""
import json

from paper_2602_18931_b200 import abi, trace


def rec(t, t2, p1, p2, h, d, d2, q1, q2, hd):
    r = abi.TokenRecord()
    r.target_token, r.target_top2, r.target_p1, r.target_p2, r.target_entropy = t, t2, p1, p2, h
    r.draft_top1, r.draft_top2, r.draft_p1, r.draft_p2, r.draft_entropy = d, d2, q1, q2, hd
    return r


def test_trace_lines_follow_the_reference_rules():
    recs = [rec(5, 7, 0.9, 0.05, 0.4, 5, 9, 0.6, 0.3, 0.9),       # ordinary
            rec(3, 4, 1.0, 1e-9, 0.0, 3, 1, 0.5, 0.5, 0.7),        # certain target, tie in the draft
            rec(8, 2, 0.999, 0.0, 0.0, 8, 6, 0.999999, 1e-7, 0.0),  # underflow / zero entropy < 1
            rec(1, 0, 0.7, 0.3000001, 0.6, 1, 0, 0.5, 0.2, 0.9)]    # top-2 sum rounding over 1
    lines = trace.records_to_ndjson(recs, 2, 2)
    assert len(lines) == 2
    for line in lines:
        trace.check_line(line, 16)
    first = json.loads(lines[0])["tokens"]
    assert [list(t) for t in first] == [["t", "tp", "te", "dp", "de"]] * 2
    assert first[0]["tp"] == [[5, 0.9], [7, 0.05]] and first[0]["te"] == 0.4
    # certain prediction: zero entropy, vanishing runner-up; draft tie canonicalised by id
    assert first[1]["tp"][0] == [3, 1.0] and first[1]["te"] == 0.0 and 0.0 < first[1]["tp"][1][1] <= 1e-300
    assert first[1]["dp"] == [[1, 0.5], [3, 0.5]]
