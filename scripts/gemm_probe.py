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




def timeline_small():
    """WS_GEMM_ABLATE=8: per-phase timeline (ns from CTA 0's entry) of small-M GEMMs at the 1B
    shapes, each measured after a warm-up: where a ~13 µs small GEMM spends its time."""
    import ctypes as C

    import torch

    import paper_2602_18931_b200 as ws
    from paper_2602_18931_b200 import ops
    L = ws.lib()
    L.ws_debug_gemm_trace.argtypes = [C.c_void_p]
    names = ["entry", "prologue", "dep_wait", "first_full", "last_mma", "acc_ready", "epi_done", "exit"]
    shapes = [(3072, 2048, 0, "1B qkv(bf16 epi)"), (2048, 2048, 1, "1B o"), (2048, 8192, 1, "1B down"),
              (16384, 2048, 2, "1B gate_up")]
    if os.environ.get("WS_TIMELINE_8B"):
        shapes = [(6144, 4096, 0, "8B qkv(bf16 epi)"), (4096, 4096, 1, "8B o"), (4096, 14336, 1, "8B down"),
                  (28672, 4096, 2, "8B gate_up")]
    for M in [int(x) for x in os.environ.get("WS_TIMELINE_M", "48,160,512").split(",")]:
        for (N, K, epi, name) in shapes:
            A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
            out = torch.zeros(M, N, device="cuda", dtype=torch.float32) if epi == 1 else None
            for _ in range(3):
                ops.gemm(A, W, out=out, epi=epi)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ops.gemm(A, W, out=out, epi=epi)
            e1.record()
            torch.cuda.synchronize()
            buf = (C.c_ulonglong * 8)()
            assert L.ws_debug_gemm_trace(buf) == 0
            t0 = buf[0]
            print(json.dumps({"gemm": f"{name} M={M}", "event_us": round(e0.elapsed_time(e1) * 1e3, 1),
                              **{n: round((buf[i] - t0) / 1e3, 2) for i, n in enumerate(names)}}), flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "timeline":
    timeline_small()
    sys.exit(0)


if __name__ == "__main__":
    main()
