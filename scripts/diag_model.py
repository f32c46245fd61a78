"""Diagnostics for the config-3 model pair: logit scale vs the planted bias, draft/target
agreement, and per-step accept statistics of a short run.

    python scripts/diag_model.py [target] [draft] [requests]
"""
import collections
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2602_18931_b200 as ws  # noqa: E402
from paper_2602_18931_b200 import abi  # noqa: E402


def logits_probe(name, V):
    L = ws.lib()
    L.ws_model_create.argtypes = [C.c_char_p, C.c_uint64, C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
    L.ws_model_forward.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                   C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ws_model_destroy.argtypes = [C.c_void_p]
    h = C.c_void_p()
    assert L.ws_model_create(name.encode(), 3, 64, 64, 0, C.byref(h)) == 0
    T = 16
    tok = torch.randint(0, V - 256, (T,), dtype=torch.int32)
    pos = torch.arange(T, dtype=torch.int32)
    grp = torch.tensor([0, T, 0, 0, 0, T], dtype=torch.int32)
    out = torch.empty(T, V, dtype=torch.bfloat16, device="cuda")
    rc = L.ws_model_forward(h, T, tok.data_ptr(), pos.data_ptr(), pos.data_ptr(), 1, grp.data_ptr(), T,
                            pos.data_ptr(), T, pos.data_ptr(), out.data_ptr(), None)
    assert rc == 0, ws.lib().ws_last_error()
    x = out.float()
    print(json.dumps({"model": name, "logit_std": x.std().item(), "logit_absmax": x.abs().max().item(),
                      "finite": bool(torch.isfinite(x).all().item()),
                      "row_max_mean": x.max(dim=1).values.mean().item()}))
    L.ws_model_destroy(h)


def main():
    target = sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"
    draft = sys.argv[2] if len(sys.argv) > 2 else "llama3.2-1b"
    nreq = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    V = 128256 if target.startswith("llama") else 1000
    logits_probe(target, V)
    logits_probe(draft, V)
    ctx = ws.Context(0)
    ctx.load_models(abi.model_cfg(target, draft, max_requests=max(8, nreq)))
    c = abi.config3(num_requests=nreq, k=4)
    b = ctx.run_model_sim(c)
    steps = b.step_list()
    acc = collections.Counter(s[3] for s in steps)
    print(json.dumps({"metrics0": b.metrics_list()[0], "accept_hist": dict(sorted(acc.items())),
                      "mean_accept": sum(s[3] for s in steps) / max(1, len(steps)),
                      "first_tokens": b.ctrl_outputs()[0][:12], "model_stats": ctx.model_stats()}))


if __name__ == "__main__":
    main()
