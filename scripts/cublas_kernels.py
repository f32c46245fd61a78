"""Which cuBLAS kernels (tile configs) torch.matmul picks for the model path's projection
shapes — the library baseline our K1 GEMM is compared against (scripts/bench_kernels.py)."""
import json
import sys

import torch
from torch.profiler import ProfilerActivity, profile

SHAPES = [(530, 6144, 4096, "8B qkv"), (530, 4096, 4096, "8B o"), (530, 28672, 4096, "8B gate_up"),
          (530, 4096, 14336, "8B down"), (655, 3072, 2048, "1B qkv"), (655, 2048, 2048, "1B o"),
          (655, 16384, 2048, "1B gate_up"), (655, 2048, 8192, "1B down")]


def main():
    for (M, N, K, name) in SHAPES:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        for _ in range(3):
            torch.matmul(A, W.T)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            torch.matmul(A, W.T)
            torch.cuda.synchronize()
        names = [(e.name, e.device_time) for e in prof.events() if e.device_time > 0]
        print(json.dumps({"shape": name, "M": M, "N": N, "K": K, "kernels": names}))
        sys.stdout.flush()


if __name__ == "__main__":
    main()
