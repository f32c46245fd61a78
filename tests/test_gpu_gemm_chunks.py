"""K1 canonical K chunks (gemm_tc.cu pick_chunks / SplitArgs.chunks): a shape with C chunks
accumulates each K chunk from zero in its own TMEM columns and sums the chunks in order, either
all in one CTA (large batches) or as C split units whose partials are reduced in split order
(small batches: through distributed shared memory on CTA pairs for C = 2, else global memory).
Both give identical bits, so the split can follow the batch size without breaking batch
invariance (the property behind speculative stream == greedy stream).

The chunk rules are read once per process (WS_GEMM_CHUNKS), so the check runs in a child process.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2602_18931_b200 import ops
torch.manual_seed(0)
out = []
for (N, K) in [(2048, 8192), (2048, 2048), (4096, 4096), (4096, 14336)]:
    W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    A = torch.randn(1200, K, device="cuda").to(torch.bfloat16)
    R = torch.randn(1200, N, device="cuda")
    ref = None
    for M in (1200, 520, 200, 48, 5):
        for epi in (0, 1):
            o = R[:M].clone() if epi == 1 else None
            y = ops.gemm(A[:M].contiguous(), W, out=o, epi=epi, splits=0)
            torch.cuda.synchronize()
            if M == 1200:
                if epi == 0:
                    ref0 = y.clone()
                else:
                    ref1 = y.clone()
                continue
            want = ref0[:M] if epi == 0 else ref1[:M]
            same = torch.equal(y.view(torch.int16) if epi == 0 else y.view(torch.int32),
                               want.view(torch.int16) if epi == 0 else want.view(torch.int32))
            out.append((N, K, M, epi, bool(same)))
    # against the unchunked product (fp32 reference): the chunk sums stay within fp32 noise
    full = A.float() @ W.float().t()
    err = ((ref1 - R) - full).abs().max().item() / full.abs().max().item()
    out.append((N, K, "err", err))
print(out)
"""


@pytest.mark.gpu
def test_chunked_split_equals_in_cta_chunks():
    env = dict(os.environ, WS_GEMM_CHUNKS="2048:8192:2,2048:2048:4,4096:4096:2,4096:14336:2")
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = eval(r.stdout.strip().splitlines()[-1])
    for item in res:
        if item[2] == "err":
            assert item[3] < 1e-3, item
        else:
            assert item[4], item
