"""torch-tensor conveniences over the device-pointer kernel entry points (ws_op_*).

torch supplies device memory and the current stream only; every op runs the library's own
sm_100a kernels. Used by the GPU kernel tests and the model-path harness.
"""
import ctypes as C

from . import _check, lib

_P = C.c_void_p
_bound = False


def _bind():
    global _bound
    if _bound:
        return
    L = lib()
    L.ws_op_gemm_bf16.argtypes = [_P, _P, _P] + [C.c_int] * 9 + [_P]
    _bound = True


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


EPI_BF16, EPI_ADD_F32, EPI_SWIGLU = 0, 1, 2


def gemm(A, W, out=None, epi=EPI_BF16, bn=0, splits=1):
    """out = A @ W.T (bf16 in, fp32 accumulate) with the chosen fused epilogue."""
    import torch
    _bind()
    M, K = A.shape
    N = W.shape[0]
    assert W.shape[1] == K and A.dtype == torch.bfloat16 and W.dtype == torch.bfloat16
    if out is None:
        if epi == EPI_ADD_F32:
            out = torch.zeros(M, N, dtype=torch.float32, device=A.device)
        elif epi == EPI_SWIGLU:
            out = torch.empty(M, N // 2, dtype=torch.bfloat16, device=A.device)
        else:
            out = torch.empty(M, N, dtype=torch.bfloat16, device=A.device)
    _check(lib().ws_op_gemm_bf16(A.data_ptr(), W.data_ptr(), out.data_ptr(), M, N, K, A.stride(0),
                                 W.stride(0), out.stride(0), epi, bn, splits, _stream()))
    return out


def interleave_gate_up(w_gate, w_up, block=16):
    """Rows [g0..g15, u0..u15, g16..g31, ...] — the SwiGLU epilogue's expected weight layout."""
    import torch
    F, K = w_gate.shape
    g = w_gate.view(F // block, block, K)
    u = w_up.view(F // block, block, K)
    return torch.stack([g, u], dim=1).reshape(2 * F, K).contiguous()
