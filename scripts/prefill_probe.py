"""Per-class device time of prompt-prefill forwards (the bench's prefill phase): n_req groups of
P-1 = 127 causal rows for the Llama-3.1-8B target and the Llama-3.2-1B draft (8 128 rows at 64).

    WS_PROFILE_MODEL=1 python scripts/prefill_probe.py [n_req] [iters]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import forward_probe as fp  # noqa: E402

P = 128


def prefill_batch(n_req, slots_per_req):
    tok, pos, slot, groups, extra, mask, outr = [], [], [], [], [], [], []
    for r in range(n_req):
        row0, eoff = len(tok), len(extra)
        base = r * slots_per_req
        for p in range(P - 1):
            tok.append((r * 7919 + p * 104729) % (fp.V - 256))
            pos.append(p)
            slot.append(base + p)
            extra.append(base + p)
        groups.append((row0, P - 1, base, 0, eoff, P - 1, 0))
        mask += [0] * (P - 1)
    outr.append(len(tok) - 1)
    return tok, pos, slot, groups, extra, mask, outr


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    L = fp.bind()
    for name in ("llama3-8b", "llama3.2-1b"):
        print(json.dumps(fp.run(L, name, prefill_batch(n, 256), n * 256, iters)), flush=True)
