"""K3 (fused softmax/entropy/top-2) and K4 (greedy verify epilogue) vs the fp64 oracle
restatement (oracle/restate.c or_row_stats) on the same bf16 logits. Ids are bit-exact
(argmax over exact bf16 values, ties to the lower id); probabilities and entropy within 1e-3
relative (fp32 reductions)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import pyoracle as po  # noqa: E402
from paper_2602_18931_b200 import abi  # noqa: E402


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_18931_b200 as ws
    lib = ws.lib()
    lib.ws_op_row_stats_workspace_bytes.restype = C.c_size_t
    lib.ws_op_row_stats_workspace_bytes.argtypes = [C.c_uint32] * 3
    lib.ws_op_row_stats_bf16.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_float,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.ws_op_verify_greedy_bf16.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    return lib


def preds_from(buf, n):
    arr = (abi.Pred * n).from_buffer_copy(buf.cpu().numpy().tobytes())
    return [(p.n, tuple(p.id[:p.n]), tuple(p.prob[:p.n]), p.entropy) for p in arr]


def run_stats(L, logits, inv_temp=1.0):
    rows, V = logits.shape
    ws = torch.zeros(L.ws_op_row_stats_workspace_bytes(rows, V, 0), dtype=torch.uint8, device="cuda")
    out = torch.zeros(rows * C.sizeof(abi.Pred), dtype=torch.uint8, device="cuda")
    st = torch.zeros(rows, 4, dtype=torch.float32, device="cuda")
    rc = L.ws_op_row_stats_bf16(logits.data_ptr(), rows, V, logits.stride(0), inv_temp, out.data_ptr(),
                                st.data_ptr(), ws.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    return preds_from(out, rows), st


def make_logits(rows, V, scale, seed, planted=None):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(rows, V, device="cuda", generator=g) * scale
    if planted is not None:
        idx = torch.randint(0, V, (rows,), device="cuda", generator=g)
        x[torch.arange(rows), idx] += planted
    return x.to(torch.bfloat16)


@pytest.mark.parametrize("V", [7, 1000, 32768, 32769, 128256])
@pytest.mark.parametrize("scale", [0.5, 4.0])
def test_row_stats_vs_oracle(L, V, scale):
    rows = 37
    x = make_logits(rows, V, scale, V + int(scale * 10), planted=6.0)
    got, _ = run_stats(L, x)
    xf = x.float().cpu().numpy()
    for r in range(rows):
        n, ids, probs, h = po.row_stats(xf[r])
        assert got[r][1] == ids, r
        assert got[r][2] == pytest.approx(probs, rel=1e-3)
        assert got[r][3] == pytest.approx(h, rel=1e-3, abs=1e-6)


def test_ties_resolve_to_lower_id(L):
    V = 70000
    x = torch.zeros(3, V, device="cuda", dtype=torch.bfloat16)
    x[0, [5, 40000, 69999]] = 3.0
    x[1, [65536, 32768]] = 2.0
    x[2, :] = 1.0
    got, _ = run_stats(L, x)
    assert got[0][1] == (5, 40000)
    assert got[1][1] == (32768, 65536)
    assert got[2][1] == (0, 1)
    assert got[2][3] == pytest.approx(np.log(V), rel=1e-4)


def test_top2_vector_and_thread_placements(L):
    """K3 keeps each lane's two best 8-element vectors (by vector maximum), merges them over the
    warp and rescans the tile's best two. Plant the top-2 where that could go wrong: both in one
    vector, in two vectors of one lane (ids 256 apart inside an 8192-wide tile), ties inside one
    lane, ties between a same-vector element and another lane's, across tiles, in the short last
    tile (and the round-1 64K-chunk geometry: ids 2048 / 65536 apart)."""
    V = 128256
    x = (torch.randn(16, V, device="cuda", generator=torch.Generator(device="cuda").manual_seed(11)) * 0.1)
    plants = [
        {100: 5.0, 103: 4.0},                      # same vector
        {5: 5.0, 5 + 2048 * 3: 4.0},               # same thread, different vectors
        {7: 5.0, 7 + 2048: 5.0, 3: 4.5},           # tie for first in one thread; 3rd in 1st's vector
        {1 + 2048 * 5: 5.0, 1 + 2048 * 2: 5.0, 1: 5.0},  # three-way tie in one thread
        {16: 5.0, 17: 4.0, 24: 4.0},               # tie for second: same vector (17) vs thread 3 (24)
        {40: 5.0, 47: 4.0, 8: 4.0},                # tie for second: lower id in another thread wins
        {65536 + 10: 5.0, 10: 5.0},                # tie across chunks
        {128255: 5.0, 128254: 5.0},                # last vector of the row
        {5: 5.0, 5 + 256 * 3: 4.0},                # same lane, different vectors
        {9: 5.0, 9 + 256: 5.0, 12: 4.5},           # tie for first in one lane; 3rd in 1st's vector
        {8192 + 3: 5.0, 3: 5.0},                   # tie across tiles
        {8192 * 15 + 5000: 5.0, 8192 * 15 + 4999: 4.9},  # short last tile
        {300: 5.0, 301: 4.0, 300 + 8: 4.0},        # tie for second: same vector vs the next lane's
    ]
    want = [(100, 103), (5, 5 + 2048 * 3), (7, 7 + 2048), (1, 1 + 2048 * 2), (16, 17), (40, 8),
            (10, 65546), (128254, 128255), (5, 5 + 256 * 3), (9, 9 + 256), (3, 8195),
            (8192 * 15 + 5000, 8192 * 15 + 4999), (300, 301)]
    for r, pl in enumerate(plants):
        for i, v in pl.items():
            x[r, i] = v
    x = x.to(torch.bfloat16)
    got, _ = run_stats(L, x)
    xf = x.float().cpu().numpy()
    for r in range(len(plants)):
        assert got[r][1] == want[r], (r, got[r][1])
        _, ids, probs, h = po.row_stats(xf[r])
        assert ids == want[r]
        assert got[r][2] == pytest.approx(probs, rel=1e-3)
        assert got[r][3] == pytest.approx(h, rel=1e-3)


def test_temperature(L):
    x = make_logits(16, 32000, 2.0, 5)
    got, _ = run_stats(L, x, inv_temp=1.0 / 0.7)
    xf = x.float().cpu().numpy()
    for r in range(16):
        _, ids, probs, h = po.row_stats(xf[r], 1.0 / 0.7)
        assert got[r][1] == ids
        assert got[r][3] == pytest.approx(h, rel=1e-3)


def test_batch_invariance(L):
    """A row's statistics are bit-identical whatever the batch it is computed in."""
    x = make_logits(300, 128256, 3.0, 9, planted=4.0)
    full, _ = run_stats(L, x)
    one, _ = run_stats(L, x[123:124].contiguous())
    part, _ = run_stats(L, x[100:160].contiguous())
    assert one[0] == full[123]
    assert part[23] == full[123]


def test_workspace_reuse_across_row_counts(L):
    """The self-resetting tickets live at fixed offsets: one workspace serves launches of any
    size in any order (the model backend reuses it every round)."""
    V = 128256
    ws = torch.zeros(L.ws_op_row_stats_workspace_bytes(600, V, 0), dtype=torch.uint8, device="cuda")
    for rows in (600, 37, 255, 1, 600, 90):
        x = make_logits(rows, V, 3.0, rows, planted=5.0)
        out = torch.zeros(rows * C.sizeof(abi.Pred), dtype=torch.uint8, device="cuda")
        rc = L.ws_op_row_stats_bf16(x.data_ptr(), rows, V, V, 1.0, out.data_ptr(), None, ws.data_ptr(),
                                    torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        torch.cuda.synchronize()
        got = preds_from(out, rows)
        want = x.float().argmax(dim=1).cpu().tolist()
        assert [g[1][0] for g in got] == want


@pytest.mark.parametrize("k", [1, 4, 8])
def test_verify_greedy_epilogue(L, k):
    n_req, V = 50, 128256
    rows = n_req * (k + 1)
    x = make_logits(rows, V, 1.0, 100 + k, planted=8.0)
    argmax = x.float().argmax(dim=1).view(n_req, k + 1).cpu()
    rnd = np.random.default_rng(k)
    cand = argmax[:, :k].clone()
    for j in range(n_req):  # corrupt a random suffix
        cut = rnd.integers(0, k + 1)
        if cut < k:
            cand[j, cut] = (cand[j, cut] + 1) % V
    cand_d = cand.to(torch.int32).cuda()
    ws = torch.zeros(L.ws_op_row_stats_workspace_bytes(rows, V, n_req), dtype=torch.uint8, device="cuda")
    out = torch.zeros(n_req * 16, dtype=torch.uint8, device="cuda")
    rowp = torch.zeros(rows * C.sizeof(abi.Pred), dtype=torch.uint8, device="cuda")
    for _ in range(2):  # second launch checks the self-resetting tickets
        rc = L.ws_op_verify_greedy_bf16(x.data_ptr(), n_req, k, V, V, cand_d.data_ptr(), out.data_ptr(),
                                        rowp.data_ptr(), ws.data_ptr(), torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        torch.cuda.synchronize()
        o = np.frombuffer(out.cpu().numpy().tobytes(), dtype=[("a", "<u4"), ("b", "<u4"), ("h", "<f8")])
        preds = preds_from(rowp, rows)
        for j in range(n_req):
            a = 0
            while a < k and int(cand[j, a]) == int(argmax[j, a]):
                a += 1
            assert int(o["a"][j]) == a
            assert int(o["b"][j]) == int(argmax[j, a])
            assert float(o["h"][j]) == preds[j * (k + 1) + a][3]


@pytest.mark.parametrize("V", [1000, 128256, 128257])
def test_masked_minus_inf_columns(L, V):
    """-inf logits (masked vocabulary) carry probability 0 and add 0 to the entropy
    (entropy_of's 0 ln 0 = 0, oracle.hpp:21-33) instead of turning it into NaN; ids, probs and
    entropy match the fp64 oracle on the same masked rows, in vector chunks and the scalar tail."""
    rows = 9
    x = make_logits(rows, V, 2.0, 11 + V, planted=5.0)
    g = torch.Generator(device="cuda").manual_seed(5)
    mask = torch.rand(rows, V, device="cuda", generator=g) < 0.5
    mask[1] = True
    mask[1, [3, V - 1]] = False  # two survivors, one in the scalar tail when V % 8
    mask[2, :] = False
    mask[2, V - 3:] = True       # only the tail masked
    x = x.masked_fill(mask, float("-inf"))
    got, st = run_stats(L, x)
    xf = x.float().cpu().numpy()
    for r in range(rows):
        n, ids, probs, h = po.row_stats(xf[r])
        assert np.isfinite(got[r][3]), r
        assert got[r][1] == ids, r
        assert got[r][2] == pytest.approx(probs, rel=1e-3, abs=1e-9)
        assert got[r][3] == pytest.approx(h, rel=1e-3, abs=1e-6)
