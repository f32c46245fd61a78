"""Teacher-forced trace export of the GPU model pair in the reference's NDJSON trace format
(docs/trace_format.md of the reference: one line per sequence, {"tokens": [{"t", "tp", "te",
"dp", "de"}, ...]}, field order fixed), so the reference's own trace oracle
(OracleKind::trace, oracle.hpp:183-290) replays real-model behaviour.

The records come from ws_model_export_trace: the target's greedy path, with the target's and
the draft's top-2 and entropy on each committed context. The format's validation rules
(oracle.hpp trace_io::parse_prediction) are enforced here: probabilities in (0, 1], top-2 sum
<= 1, entropy zero exactly when the top probability is 1.
"""
import json
import math

_TINY = 1e-300


def _pair_block(top1, top2, p1, p2, h):
    p1 = min(max(p1, _TINY), 1.0)
    if p1 >= 1.0:  # a certain prediction: zero entropy, a vanishing runner-up
        p1, h = 1.0, 0.0
        p2 = min(max(p2, _TINY), 1e-300)
    else:
        p2 = min(max(p2, _TINY), p1, 1.0 - p1)
        if not h > 0.0:
            h = 5e-324 if h == 0.0 else abs(h)  # the top is < 1, so the entropy is not zero
    if p2 == p1 and top2 < top1:  # canonical order: ties by ascending id
        top1, top2 = top2, top1
    return [[int(top1), p1], [int(top2), p2]], h


def records_to_ndjson(records, n, length):
    """records: n * length ws_token_record (request-major) -> list of NDJSON lines."""
    lines = []
    for s in range(n):
        toks = []
        for i in range(length):
            r = records[s * length + i]
            tp, te = _pair_block(r.target_token, r.target_top2, r.target_p1, r.target_p2, r.target_entropy)
            dp, de = _pair_block(r.draft_top1, r.draft_top2, r.draft_p1, r.draft_p2, r.draft_entropy)
            toks.append({"t": int(tp[0][0]), "tp": tp, "te": te, "dp": dp, "de": de})
        lines.append(json.dumps({"tokens": toks}, separators=(",", ":")))
    return lines


def write_trace(path, records, n, length):
    with open(path, "w") as f:
        for line in records_to_ndjson(records, n, length):
            f.write(line + "\n")


def check_line(line, vocab):
    """The reference's validation rules for one trace line (trace_io, oracle.hpp:145-230)."""
    obj = json.loads(line)
    assert list(obj) == ["tokens"] and obj["tokens"]
    for tok in obj["tokens"]:
        assert list(tok) == ["t", "tp", "te", "dp", "de"]
        for key, h in (("tp", tok["te"]), ("dp", tok["de"])):
            pr = tok[key]
            assert len(pr) >= 2
            for a, b in zip(pr, pr[1:]):
                assert a[1] > b[1] or (a[1] == b[1] and a[0] < b[0])
            assert all(0.0 < p <= 1.0 and 0 <= i < vocab for i, p in pr)
            assert pr[0][1] + pr[1][1] <= 1.0 + 1e-12
            assert h >= 0.0 and (h == 0.0) == (pr[0][1] == 1.0) and math.isfinite(h)
        assert tok["t"] == tok["tp"][0][0]
