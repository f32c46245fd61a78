"""Per-class device time of single forwards at a range of batch sizes (the small-M regime of the
draft chain and of strong scaling): Llama-3.2-1B draft rows as worker tree leaves (4 per request)
over 176-position prefixes, and Llama-3.1-8B verify rows (k+1 = 5 per request). Env switches of
the GEMM (WS_GEMM_PAIR, WS_GEMM_*) apply, so variants can be compared in one call.

    WS_PROFILE_MODEL=1 python scripts/gemm_probe.py [iters] [draft_rows,...] [verify_reqs,...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import forward_probe as fp  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    drows = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "48,96,192,384,768").split(",")]
    vreqs = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "32,64,107").split(",")]
    L = fp.bind()
    for r in drows:
        n_wrk = max(1, r // 4)
        res = fp.run(L, "llama3.2-1b", fp.draft_batch(n_wrk=n_wrk, leaves=4, n_ctrl=0), n_wrk * 1024, iters)
        print(json.dumps({"tag": os.environ.get("TAG", ""), **res}), flush=True)
    for n in vreqs:
        res = fp.run(L, "llama3-8b", fp.verify_batch(n_req=n), n * 256, iters)
        print(json.dumps({"tag": os.environ.get("TAG", ""), **res}), flush=True)


if __name__ == "__main__":
    main()
