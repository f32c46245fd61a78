"""Kernel-level timings (CUDA events, warm, L2-flushed) for the model-path kernels.

    python scripts/bench_kernels.py gemm
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2602_18931_b200 import ops  # noqa: E402

PEAK_TF = 1634.9
PEAK_GBS = 6544.3


def timeit(fn, iters=20, flush=None):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(iters):
        if flush is not None:
            flush.fill_(0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / iters / 1e3


def gemm():
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    res = []
    for (M, N, K, name) in [(1280, 6144, 4096, "8B qkv"), (1280, 4096, 4096, "8B o"),
                            (1280, 28672, 4096, "8B gate_up"), (1280, 4096, 14336, "8B down"),
                            (1280, 128256, 4096, "8B lm_head"), (160, 28672, 4096, "8B gate_up R32"),
                            (2304, 28672, 4096, "8B gate_up k8"), (1024, 16384, 2048, "1B gate_up")]:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        for bn in (0, 64, 128, 256):
            t = timeit(lambda: ops.gemm(A, W, out=out, bn=bn), flush=flush)
            fl = 2.0 * M * N * K
            by = 2.0 * (M * K + N * K + M * N)
            rt = max(fl / (PEAK_TF * 1e12), by / (PEAK_GBS * 1e9))
            res.append({"shape": name, "M": M, "N": N, "K": K, "bn": bn or ops_pick(M, N), "ms": t * 1e3,
                        "tflops": fl / t / 1e12, "gbs": by / t / 1e9, "roofline_frac": rt / t})
        t = timeit(lambda: torch.matmul(A, W.T), flush=flush)
        res.append({"shape": name, "impl": "torch(cuBLAS)", "ms": t * 1e3, "tflops": 2.0 * M * N * K / t / 1e12})
        del A, W, out
    for r in res:
        print(json.dumps(r))


def gemm_model():
    """The model path's projections at the measured mean batch rows (8B verify ~530 rows,
    1B draft ~655 rows): every tile width (BN multiple of 16), against cuBLAS on the same
    operands. One JSON line per shape: {bn: us}, the default pick and cuBLAS."""
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    shapes = [(530, 6144, 4096, "8B qkv"), (530, 4096, 4096, "8B o"), (530, 28672, 4096, "8B gate_up"),
              (530, 4096, 14336, "8B down"), (655, 3072, 2048, "1B qkv"), (655, 2048, 2048, "1B o"),
              (655, 16384, 2048, "1B gate_up"), (655, 2048, 8192, "1B down"), (300, 128256, 2048, "1B lm_head"),
              (140, 128256, 4096, "8B lm_head")]
    only = os.environ.get("SHAPES")
    for (M, N, K, name) in shapes:
        if only and name not in only.split(","):
            continue
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        fl = 2.0 * M * N * K
        per = {}
        for bn in range(64, 257, 32):
            per[bn] = round(timeit(lambda: ops.gemm(A, W, out=out, bn=bn), flush=flush) * 1e6, 1)
        t_def = timeit(lambda: ops.gemm(A, W, out=out), flush=flush)
        t_cub = timeit(lambda: torch.matmul(A, W.T), flush=flush)
        best = min(per, key=per.get)
        print(json.dumps({"shape": name, "M": M, "N": N, "K": K, "default_us": round(t_def * 1e6, 1),
                          "cublas_us": round(t_cub * 1e6, 1), "best_bn": best, "best_us": per[best],
                          "tflops_default": round(fl / t_def / 1e12), "per_bn": per}))
        sys.stdout.flush()
        del A, W, out


def overhead():
    """Fixed cost of one GEMM launch: K sweep at the 8B O-projection shape, with and without an
    L2 flush (a different kernel) in front, 10 back-to-back launches per event pair."""
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    M, N = 530, 4096
    for K in (64, 512, 4096):
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        t_f = timeit(lambda: ops.gemm(A, W, out=out, bn=160), flush=flush)

        def ten():
            for _ in range(10):
                ops.gemm(A, W, out=out, bn=160)
        t_10 = timeit(ten) / 10
        print(json.dumps({"K": K, "us_after_flush": round(t_f * 1e6, 1), "us_back_to_back": round(t_10 * 1e6, 1)}))


def rowstats():
    import ctypes as C
    import paper_2602_18931_b200 as ws
    L = ws.lib()
    L.ws_op_row_stats_workspace_bytes.restype = C.c_size_t
    L.ws_op_row_stats_workspace_bytes.argtypes = [C.c_uint32] * 3
    L.ws_op_row_stats_bf16.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_float,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    for rows, V in [(1280, 128256), (2304, 128256), (160, 128256), (1024, 128256), (4096, 32768)]:
        x = (torch.randn(rows, V, device="cuda") * 2).to(torch.bfloat16)
        wsb = torch.zeros(L.ws_op_row_stats_workspace_bytes(rows, V, 0), dtype=torch.uint8, device="cuda")
        out = torch.zeros(rows * 40, dtype=torch.uint8, device="cuda")
        st = torch.cuda.current_stream().cuda_stream

        def fn():
            L.ws_op_row_stats_bf16(x.data_ptr(), rows, V, V, 1.0, out.data_ptr(), None, wsb.data_ptr(), st)
        t = timeit(fn, flush=flush)
        by = rows * V * 2 + rows * 40
        print(json.dumps({"kernel": "row_stats_bf16", "rows": rows, "V": V, "ms": t * 1e3,
                          "gbs": by / t / 1e9, "frac_hbm": by / t / 1e9 / PEAK_GBS}))


def one_gemm():
    """One realistic verify-batch GEMM (8B gate/up + SwiGLU; M = the mean verify batch, 990 rows
    under verify batching, override with WS_ONE_GEMM_M), for ncu --set full."""
    M, N, K = int(os.environ.get("WS_ONE_GEMM_M", "990")), 28672, 4096
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    out = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
    for _ in range(4):
        ops.gemm(A, W, out=out, epi=ops.EPI_SWIGLU)
    torch.cuda.synchronize()
    t = timeit(lambda: ops.gemm(A, W, out=out, epi=ops.EPI_SWIGLU))
    print(json.dumps({"kernel": "gemm gate_up+swiglu", "M": M, "N": N, "K": K, "ms": t * 1e3,
                      "tflops": 2.0 * M * N * K / t / 1e12}))


def one_split():
    """One cluster split-K GEMM (1B down at 655 rows, 2 K halves, BN 192) and its one-pass
    counterpart, for ncu side by side."""
    M, N, K = 655, 2048, 8192
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    os.environ["WS_GEMM_PAIR"] = "2"
    for _ in range(3):
        ops.gemm(A, W, out=out, epi=1, bn=192, splits=2)
        ops.gemm(A, W, out=out, epi=1)
    torch.cuda.synchronize()
    ops.gemm(A, W, out=out, epi=1, bn=192, splits=2)
    ops.gemm(A, W, out=out, epi=1)
    torch.cuda.synchronize()


def one_add():
    """One residual-epilogue GEMM (1B down projection at 655 rows, out fp32 += acc), for ncu."""
    M, N, K = 655, 2048, 8192
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    for _ in range(4):
        ops.gemm(A, W, out=out, epi=1)
    torch.cuda.synchronize()
    t = timeit(lambda: ops.gemm(A, W, out=out, epi=1))
    ob = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    tb = timeit(lambda: ops.gemm(A, W, out=ob))
    print(json.dumps({"kernel": "gemm down+residual", "M": M, "N": N, "K": K, "us": t * 1e6,
                      "bf16_out_us": tb * 1e6}))


def splitk_pair():
    """Split-K on CTA pairs vs one pass (default tile pick), residual epilogue, L2 flushed: the
    narrow projections are L2-throughput-bound (every N tile re-reads the activation rows)."""
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    for (M, N, K, name) in [(655, 2048, 8192, "1B down"), (655, 2048, 2048, "1B o"), (530, 4096, 14336, "8B down"),
                            (530, 4096, 4096, "8B o"), (160, 2048, 8192, "1B down M=160"),
                            (150, 4096, 14336, "8B down M=150")]:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        X = torch.zeros(M, N, device="cuda")
        os.environ.pop("WS_GEMM_PAIR", None)
        res = {"1": round(timeit(lambda: ops.gemm(A, W, out=X, epi=1), flush=flush) * 1e6, 1)}
        os.environ["WS_GEMM_PAIR"] = "2"
        for sp in (2, 3, 4):
            for bn in (128, 192, 256):
                res[f"{sp}x{bn}"] = round(timeit(lambda: ops.gemm(A, W, out=X, epi=1, bn=bn, splits=sp),
                                                 flush=flush) * 1e6, 1)
        os.environ.pop("WS_GEMM_PAIR", None)
        best = min(res, key=res.get)
        print(json.dumps({"shape": name, "M": M, "N": N, "K": K, "best": best, "us": res}))
        sys.stdout.flush()


def pair(shape="8B o"):
    """One launch each of our GEMM and cuBLAS on one model shape (for an ncu side-by-side)."""
    dims = {"8B o": (530, 4096, 4096), "8B gate_up": (530, 28672, 4096), "1B lm_head": (300, 128256, 2048),
            "1B down": (655, 2048, 8192)}[shape]
    M, N, K = dims
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    for _ in range(3):
        ops.gemm(A, W, out=out)
        torch.matmul(A, W.T)
    torch.cuda.synchronize()
    flush.fill_(0)
    ops.gemm(A, W, out=out)
    flush.fill_(0)
    torch.matmul(A, W.T)
    torch.cuda.synchronize()


def ops_pick(M, N):
    bm = (M + 127) // 128
    if bm * ((N + 255) // 256) >= 296:
        return 256
    if bm * ((N + 127) // 128) >= 148:
        return 128
    return 64


def timeline():
    """WS_GEMM_ABLATE=8: per-phase timeline (ns from kernel entry) of CTA 0's first unit, for
    small and large M at the 1B O / 8B gate-up shapes, back to back after a warm-up."""
    import ctypes as C
    import paper_2602_18931_b200 as ws
    L = ws.lib()
    L.ws_debug_gemm_trace.argtypes = [C.c_void_p]
    names = ["entry", "prologue", "dep_wait", "first_full", "last_mma", "acc_ready", "epi_done", "exit"]
    for (M, N, K, epi, name) in [(160, 2048, 2048, 1, "1B o M=160"), (655, 2048, 2048, 1, "1B o M=655"),
                                 (655, 2048, 8192, 1, "1B down M=655"), (530, 4096, 14336, 1, "8B down M=530"),
                                 (655, 16384, 2048, 2, "1B gate_up M=655"),
                                 (160, 28672, 4096, 2, "8B gate_up M=160"), (530, 28672, 4096, 2, "8B gate_up M=530")]:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        out = torch.zeros(M, N, device="cuda", dtype=torch.float32) if epi == 1 else None
        for _ in range(3):
            ops.gemm(A, W, out=out, epi=epi)
        torch.cuda.synchronize()
        ops.gemm(A, W, out=out, epi=epi)
        torch.cuda.synchronize()
        buf = (C.c_ulonglong * 8)()
        assert L.ws_debug_gemm_trace(buf) == 0
        t0 = buf[0]
        print(json.dumps({"gemm": name, **{n: (buf[i] - t0) for i, n in enumerate(names)}}))


def timeline_split():
    """WS_GEMM_ABLATE=8 timeline of CTA 0 for the cluster split-K (pairs, 2 K halves) vs one pass."""
    import ctypes as C
    import paper_2602_18931_b200 as ws
    L = ws.lib()
    L.ws_debug_gemm_trace.argtypes = [C.c_void_p]
    names = ["entry", "prologue", "dep_wait", "first_full", "last_mma", "acc_ready", "epi_done", "exit"]
    for (M, N, K, sp, bn, name) in [(160, 2048, 8192, 1, 0, "1B down M=160 one pass"),
                                    (160, 2048, 8192, 2, 128, "1B down M=160 split 2 bn128"),
                                    (655, 2048, 8192, 1, 0, "1B down M=655 one pass"),
                                    (655, 2048, 8192, 2, 192, "1B down M=655 split 2 bn192")]:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        out = torch.zeros(M, N, device="cuda", dtype=torch.float32)
        os.environ["WS_GEMM_PAIR"] = "2"
        for _ in range(3):
            ops.gemm(A, W, out=out, epi=1, bn=bn, splits=sp)
        torch.cuda.synchronize()
        ops.gemm(A, W, out=out, epi=1, bn=bn, splits=sp)
        torch.cuda.synchronize()
        buf = (C.c_ulonglong * 8)()
        assert L.ws_debug_gemm_trace(buf) == 0
        t0 = buf[0]
        print(json.dumps({"gemm": name, **{n: (buf[i] - t0) for i, n in enumerate(names)}}))
        os.environ.pop("WS_GEMM_PAIR", None)


def splitk():
    """Deterministic split-K (fixed split count, last split sums the partials in order) vs one
    pass, for the narrow projections at small (N = 8 GPUs) and full (N = 1) batch rows."""
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    for (N, K, name) in [(2048, 2048, "1B o"), (2048, 8192, "1B down"), (4096, 4096, "8B o"),
                         (4096, 14336, "8B down")]:
        for M in (80, 160, 530, 655):
            A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
            X = torch.zeros(M, N, device="cuda")
            res = {}
            for sp in (1, 2, 4, 8):
                if K // 64 < 2 * sp:
                    continue
                best = None
                for bn in (64, 128, 256) if sp > 1 else (0,):
                    t = timeit(lambda: ops.gemm(A, W, out=X, epi=1, bn=bn, splits=sp), flush=flush) * 1e6
                    best = t if best is None or t < best[0] else best
                    best = (t, bn) if isinstance(best, float) else best
                res[sp] = (round(best[0], 1), best[1])
            print(json.dumps({"shape": name, "M": M, "split_us_bn": res}))
            sys.stdout.flush()


if __name__ == "__main__":
    if sys.argv[1] == "pair":
        pair(" ".join(sys.argv[2:]) or "8B o")
    else:
        {"gemm": gemm, "gemm_model": gemm_model, "rowstats": rowstats, "one_gemm": one_gemm, "overhead": overhead,
         "timeline": timeline, "splitk": splitk, "one_add": one_add, "splitk_pair": splitk_pair, "timeline_split": timeline_split, "one_split": one_split}[sys.argv[1]]()
