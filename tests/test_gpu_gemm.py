"""K1 tcgen05 GEMM vs a plain PyTorch fp32 reference of the same op (bf16 inputs)."""
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_18931_b200 import ops as o
    return o


def rel_err(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30)).item()


SHAPES = [(128, 256, 64), (37, 1000, 128), (200, 4096, 4096), (1280, 6144, 4096), (160, 4096, 14336),
          (513, 2048, 8192)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("bn", [64, 80, 128, 144, 240, 256])
def test_gemm_bf16(ops, shape, bn):
    M, N, K = shape
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    out = ops.gemm(A, W, bn=bn)
    ref = A.float() @ W.float().T
    assert rel_err(out, ref) < 4e-3, (shape, bn)


@pytest.mark.parametrize("bn", [64, 144, 176, 256])
def test_gemm_add_f32(ops, bn):
    M, N, K = 300, 4096, 2048
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    X = torch.randn(M, N, device="cuda")
    ref = X + A.float() @ W.float().T
    ops.gemm(A, W, out=X, epi=ops.EPI_ADD_F32, bn=bn)
    assert rel_err(X, ref) < 1e-5


@pytest.mark.parametrize("bn", [64, 96, 128, 192, 224, 256])
def test_gemm_swiglu(ops, bn):
    M, F, K = 260, 1024, 1024
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    Wg = (torch.randn(F, K, device="cuda") * 0.03).to(torch.bfloat16)
    Wu = (torch.randn(F, K, device="cuda") * 0.03).to(torch.bfloat16)
    Wgu = ops.interleave_gate_up(Wg, Wu)
    h = ops.gemm(A, Wgu, epi=ops.EPI_SWIGLU, bn=bn)
    g = A.float() @ Wg.float().T
    u = A.float() @ Wu.float().T
    ref = torch.nn.functional.silu(g) * u
    assert rel_err(h, ref) < 6e-3


def test_gemm_batch_and_tile_invariance(ops):
    """A row's output is bit-identical whatever the batch (M) and the N-tile width: each output
    element's K reduction runs in the same order in every configuration (no split-K) — the
    property behind "speculative stream == greedy stream" (SURVEY §8c contract 3)."""
    M, N, K = 700, 4096, 4096
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    ref = ops.gemm(A, W, bn=256)
    for bn in (64, 96, 128, 144, 208, 0):
        assert torch.equal(ops.gemm(A, W, bn=bn), ref)
    for lo, hi in ((0, 1), (5, 37), (128, 300), (690, 700)):
        assert torch.equal(ops.gemm(A[lo:hi].contiguous(), W, bn=64), ref[lo:hi])


@pytest.mark.parametrize("epi", [0, 1, 2])
@pytest.mark.parametrize("splits", [2, 4])
def test_gemm_split_k(ops, epi, splits):
    """Deterministic split-K (last split sums the partials in split order): correct, repeatable,
    and row-invariant across batch sizes at a fixed split count."""
    M, N, K = 333, 2048, 4096
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    if epi == 2:
        Wg, Wu = W[:N // 2], W[N // 2:]
        W = ops.interleave_gate_up(Wg.contiguous(), Wu.contiguous())
        ref = torch.nn.functional.silu(A.float() @ Wg.float().T) * (A.float() @ Wu.float().T)
    else:
        ref = A.float() @ W.float().T
    if epi == 1:
        X0 = torch.randn(M, N, device="cuda")
        out = X0.clone()
        ops.gemm(A, W, out=out, epi=1, splits=splits)
        assert rel_err(out, X0 + ref) < 1e-5
        return
    out = ops.gemm(A, W, epi=epi, splits=splits)
    assert rel_err(out, ref) < 6e-3
    again = ops.gemm(A, W, epi=epi, splits=splits)
    assert torch.equal(out, again)
    part = ops.gemm(A[100:140].contiguous(), W, epi=epi, splits=splits, bn=64)
    assert torch.equal(part, out[100:140])


def test_gemm_large_throughput_smoke(ops):
    """8B-shape gate/up at 1280 verify rows: correct and finishes."""
    M, N, K = 1280, 28672, 4096
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    out = ops.gemm(A, W)
    idx = torch.randint(0, N, (64,), device="cuda")
    ref = A.float() @ W[idx].float().T
    assert rel_err(out[:, idx], ref) < 4e-3


@pytest.mark.parametrize("epi", [0, 1, 2])
@pytest.mark.parametrize("shape", [(530, 4096, 4096), (655, 2048, 2048), (100, 1024, 512), (300, 3072, 1024)])
def test_gemm_cta_pair(ops, monkeypatch, epi, shape):
    """CTA-pair tiles (cta_group::2, 256 x BN over two SMs) against the fp32 reference and,
    bit for bit, against single-CTA tiles: the pair issues the same K-ordered MMA chain."""
    M, N, K = shape
    g = torch.Generator(device="cuda").manual_seed(M + N + K + epi)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    if epi == 2:
        Wg, Wu = W[:N // 2].contiguous(), W[N // 2:].contiguous()
        W = ops.interleave_gate_up(Wg, Wu)
        ref = torch.nn.functional.silu(A.float() @ Wg.float().T) * (A.float() @ Wu.float().T)
    else:
        ref = A.float() @ W.float().T
    outs = {}
    for mode in ("0", "2"):
        monkeypatch.setenv("WS_GEMM_PAIR", mode)
        if epi == 1:
            X = torch.ones(M, N, device="cuda")
            ops.gemm(A, W, out=X, epi=1)
            outs[mode] = X - 1.0
        else:
            outs[mode] = ops.gemm(A, W, epi=epi)
        torch.cuda.synchronize()
    assert rel_err(outs["2"], ref) < 6e-3
    assert torch.equal(outs["2"], outs["0"])


@pytest.mark.parametrize("epi", [0, 1])
@pytest.mark.parametrize("splits", [2, 3])
def test_gemm_cta_pair_split_k(ops, monkeypatch, epi, splits):
    """Split-K on CTA pairs: two K halves in a cluster of four reduced through distributed shared
    memory, or (other counts / WS_GEMM_DSMEM=0) each CTA publishing its rows' partial and the
    last split summing them in split order — bit for bit the single-CTA split-K result at the
    same split count, also with an odd number of 128-row blocks (the pair's padding block)."""
    M, N, K = 655, 2048, 8192
    g = torch.Generator(device="cuda").manual_seed(splits * 7 + epi)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    ref = A.float() @ W.float().T
    outs = {}
    for mode, bn, dsmem in (("0", 128, "1"), ("2", 256, "1"), ("2", 96, "1"), ("2", 128, "0"), ("2", 192, "1")):
        # splits == 2 on pairs reduces through distributed shared memory unless WS_GEMM_DSMEM=0
        monkeypatch.setenv("WS_GEMM_PAIR", mode)
        monkeypatch.setenv("WS_GEMM_DSMEM", dsmem)
        if epi == 1:
            X = torch.ones(M, N, device="cuda")
            ops.gemm(A, W, out=X, epi=1, splits=splits, bn=bn)
            outs[(mode, bn, dsmem)] = X - 1.0
        else:
            outs[(mode, bn, dsmem)] = ops.gemm(A, W, epi=epi, splits=splits, bn=bn)
        torch.cuda.synchronize()
    base = outs[("0", 128, "1")]
    assert rel_err(base, ref) < 6e-3
    for k, v in outs.items():
        assert torch.equal(v, base), k
