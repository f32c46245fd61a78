"""Subprocess probe of test_split_k_row_slices_with_fused_norm: one 600-row forward of a
2-layer Llama-3.2-1B-shape model (O / down GEMMs K >= 1024, so WS_GEMM_CSPLIT splits them);
prints a hash of the logits."""
import ctypes as C
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_18931_b200 as ws  # noqa: E402

lib = ws.lib()
lib.ws_model_create.argtypes = [C.c_char_p, C.c_uint64, C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
lib.ws_model_forward.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                 C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
h = C.c_void_p()
assert lib.ws_model_create(b"llama3.2-1b:L2", 5, 1024, 64, 0, C.byref(h)) == 0
g = torch.Generator().manual_seed(0)
n = 600
tok = torch.randint(0, 128000, (n,), generator=g, dtype=torch.int32)
pos = torch.tensor([i % 200 for i in range(n)], dtype=torch.int32)
slot = torch.arange(n, dtype=torch.int32)
groups = torch.tensor([0, 200, 0, 0, 0, 200, 0,
                       200, 200, 200, 0, 200, 200, 0,
                       400, 200, 400, 0, 400, 200, 0], dtype=torch.int32)
extra = torch.arange(n, dtype=torch.int32)
masks = torch.zeros(n, dtype=torch.int64)
out_rows = torch.arange(0, n, 7, dtype=torch.int32)
logits = torch.empty(len(out_rows), 128256, dtype=torch.bfloat16, device="cuda")
rc = lib.ws_model_forward(h, n, tok.data_ptr(), pos.data_ptr(), slot.data_ptr(), 3, groups.data_ptr(), n,
                          extra.data_ptr(), masks.data_ptr(), len(out_rows), out_rows.data_ptr(), logits.data_ptr(),
                          None)
assert rc == 0, ws.last_error() if hasattr(ws, "last_error") else rc
torch.cuda.synchronize()
print(hashlib.sha256(logits.view(torch.int16).cpu().numpy().tobytes()).hexdigest())
