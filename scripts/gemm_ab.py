import os, sys, torch, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_2602_18931_b200 import ops
res = {}
for (N, K) in [(4096, 14336), (2048, 8192)]:
    W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    for M in (48, 160, 320, 535):
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        X = torch.zeros(M, N, device="cuda")
        for _ in range(3): ops.gemm(A, W, out=X, epi=1, splits=0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(40): ops.gemm(A, W, out=X, epi=1, splits=0)
        e1.record(); torch.cuda.synchronize()
        res[f"{N}x{K} M={M}"] = round(e0.elapsed_time(e1) / 40 * 1e3, 1)
print(json.dumps(res))
