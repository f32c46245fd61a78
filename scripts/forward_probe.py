"""One representative verify forward (Llama-3.1-8B shape) and one representative draft forward
(Llama-3.2-1B shape) through the C ABI (ws_model_forward), at the mean batch shapes measured
in the config-3 run (verify: 105 requests x k+1 = 5 rows over ~176-position prefixes; draft:
256 worker tree groups of 2 leaf rows + 150 controller rows). Small footprint and few launches:
the short command for the ncu launch list and per-kernel captures under profiles/.

    python scripts/forward_probe.py [iters]
"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2602_18931_b200 as ws  # noqa: E402

V = 128256
PREFIX = 176


def bind():
    L = ws.lib()
    L.ws_model_create.argtypes = [C.c_char_p, C.c_uint64, C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
    L.ws_model_forward.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                   C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ws_model_destroy.argtypes = [C.c_void_p]
    return L


def verify_batch(n_req=105, rows=5, slots_per_req=256):
    tok, pos, slot, groups, extra, outr = [], [], [], [], [], []
    for r in range(n_req):
        row0, eoff = len(tok), len(extra)
        for j in range(rows):
            p = PREFIX + j
            tok.append((r * 7919 + j * 104729) % (V - 256))
            pos.append(p)
            slot.append(r * slots_per_req + p)
            extra.append(r * slots_per_req + p)
            outr.append(row0 + j)
        groups.append((row0, rows, r * slots_per_req, PREFIX, eoff, rows, 0))
    return tok, pos, slot, groups, extra, [0] * len(tok), outr


def draft_batch(n_wrk=256, leaves=2, n_ctrl=150, slots_per_req=1024):
    tok, pos, slot, groups, extra, mask, outr = [], [], [], [], [], [], []
    for r in range(n_wrk):  # worker tree group: leaves see their own slot only (masked)
        row0, eoff = len(tok), len(extra)
        for j in range(leaves):
            s = r * slots_per_req + 600 + j
            tok.append((r * 31 + j) % (V - 256))
            pos.append(PREFIX + 1)
            slot.append(s)
            extra.append(s)
            mask.append(1 << j)
            outr.append(row0 + j)
        groups.append((row0, leaves, r * slots_per_req + 256, PREFIX + 1, eoff, leaves, 1))
    for r in range(n_ctrl):  # controller local draft: one causal row over its linear cache
        row0, eoff = len(tok), len(extra)
        s = r * slots_per_req + PREFIX + 1
        tok.append((r * 17) % (V - 256))
        pos.append(PREFIX + 1)
        slot.append(s)
        extra.append(s)
        mask.append(0)
        outr.append(row0)
        groups.append((row0, 1, r * slots_per_req, PREFIX + 1, eoff, 1, 0))
    return tok, pos, slot, groups, extra, mask, outr


def run(L, name, batch, n_slots, iters, device=0):
    h = C.c_void_p()
    rc = L.ws_model_create(name.encode(), 7, n_slots, 2048, device, C.byref(h))
    assert rc == 0, L.ws_last_error()
    tok, pos, slot, groups, extra, mask, outr = batch
    i32 = lambda v: torch.tensor(v, dtype=torch.int32)  # noqa: E731
    t_tok, t_pos, t_slot = i32(tok), i32(pos), i32(slot)
    t_grp = i32([x for g in groups for x in g])
    t_ext, t_out = i32(extra), i32(outr)
    t_msk = torch.tensor(mask, dtype=torch.int64)
    logits = torch.empty(len(outr), V, dtype=torch.bfloat16, device=torch.device("cuda", device))
    st = torch.cuda.current_stream(device)

    def fwd():
        rc = L.ws_model_forward(h, len(tok), t_tok.data_ptr(), t_pos.data_ptr(), t_slot.data_ptr(), len(groups),
                                t_grp.data_ptr(), len(extra), t_ext.data_ptr(), t_msk.data_ptr(), len(outr),
                                t_out.data_ptr(), logits.data_ptr(), C.c_void_p(st.cuda_stream))
        assert rc == 0, L.ws_last_error()

    for _ in range(2):
        fwd()
    torch.cuda.synchronize(device)
    ms = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.device(device):
            e0.record(st)
            fwd()
            e1.record(st)
        torch.cuda.synchronize(device)
        ms.append(e0.elapsed_time(e1))
    L.ws_model_destroy(h)
    return {"model": name, "device": device, "rows": len(tok), "groups": len(groups), "out_rows": len(outr),
            "ms_median": sorted(ms)[len(ms) // 2], "ms_all": [round(x, 3) for x in ms]}


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    L = bind()
    devs = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0"])]
    for dev in devs:
        nv = int(os.environ.get("WS_PROBE_VERIFY_REQ", "105"))  # 198 = the mean batch under verify batching
        only = os.environ.get("WS_PROBE_ONLY", "")  # "verify" / "draft": one of the two forwards
        if only != "draft":
            print(json.dumps(run(L, "llama3-8b", verify_batch(n_req=nv), nv * 256, iters, dev)))
        if only != "verify":
            print(json.dumps(run(L, "llama3.2-1b", draft_batch(), 256 * 1024, iters, dev)))


if __name__ == "__main__":
    main()
