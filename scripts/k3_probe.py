"""K3+K4 (row statistics + the greedy accept walk) alone at a verify-shaped batch: n_req x (k+1)
bf16 logits rows of V = 128256 (the bench's `k3` figure; the short command for ncu captures).

    python scripts/k3_probe.py [n_req] [k]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

if __name__ == "__main__":
    n_req = int(sys.argv[1]) if len(sys.argv) > 1 else 107
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    bw, _, _ = bench.peaks()
    print(json.dumps(bench.k3_sample(n_req * (k + 1), k, bw, iters=5)))
