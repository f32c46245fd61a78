"""CPU check of K3's top-2 decomposition (paper_2602_18931_b200/csrc/kernels/rowstats.cu).

The kernel does not insert every element into a running top-2. A row is cut into 8192-wide
tiles, one warp per tile; lane l streams the tile's 8-element vectors l, l + 32, ... and keeps,
branch-free, its two best vectors ranked by (vector max desc, vector index asc). The warp merges
the lanes' pairs (xor butterfly, same ranking) and rescans only the tile's two best vectors;
elements past the last whole vector are inserted one by one. Tile results merge into the row's
top-2. This test restates that partition in Python. On tie-heavy rows it must give exactly the
Prediction tie rule's top-2 (types.hpp:54-55: descending value, ties to the lower id), which a
brute-force sort provides. The GPU kernel itself is checked against the oracle in
tests/test_gpu_rowstats.py.
"""
import numpy as np
import pytest

TILE, LANES = 8192, 32
NONE = 2**32 - 1


def better(v, i, w, j):
    return v > w or (v == w and i < j)


def insert(top, v, i):
    (v1, i1), (v2, i2) = top
    if better(v, i, v2, i2):
        if better(v, i, v1, i1):
            return [(v, i), (v1, i1)]
        return [(v1, i1), (v, i)]
    return top


def merge2(a, b):
    return insert(insert(a, *b[0]), *b[1])


def kernel_top2(x):
    empty = [(-np.inf, NONE), (-np.inf, NONE)]
    row_top = empty
    for lo in range(0, len(x), TILE):
        hi = min(len(x), lo + TILE)
        nvec = (hi - lo) // 8
        warp_best = empty  # the tile's two best vectors: (vector max, first element id)
        tail = empty
        for lane in range(LANES):
            b = empty
            for vi in range(lane, nvec, LANES):  # the lane's branch-free two-best-vectors update
                id0 = lo + 8 * vi
                mx = float(x[id0:id0 + 8].max())
                p1, p2 = mx > b[0][0], mx > b[1][0]
                b = [(mx, id0), b[0]] if p1 else ([b[0], (mx, id0)] if p2 else b)
            warp_best = merge2(warp_best, b)
            for e in range(lo + nvec * 8 + lane, hi, LANES):  # element-wise tail
                tail = insert(tail, float(x[e]), e)
        top = tail
        for _, id0 in warp_best:  # rescan the tile's two best vectors
            if id0 != NONE:
                for j in range(8):
                    top = insert(top, float(x[id0 + j]), id0 + j)
        row_top = merge2(row_top, top)
    return row_top[0][1], row_top[1][1]


def brute_top2(x):
    order = sorted(range(len(x)), key=lambda i: (-float(x[i]), i))
    return order[0], order[1]


@pytest.mark.parametrize("V,levels,seed", [(4100, 3, 1), (70001, 5, 2), (8192 * 2 + 24, 2, 3), (256 * 8 + 5, 4, 4)])
def test_best2_rescan_matches_brute_force(V, levels, seed):
    rng = np.random.default_rng(seed)
    for _ in range(3):
        # few distinct values -> heavy ties inside vectors, lanes and tiles
        x = rng.integers(0, levels, size=V).astype(np.float32)
        assert kernel_top2(x) == brute_top2(x)


def test_best2_same_vector_and_same_lane():
    x = np.zeros(20000, dtype=np.float32)
    x[100], x[103] = 5, 4                     # both in one vector
    assert kernel_top2(x) == (100, 103)
    x[:] = 0
    x[5], x[5 + 256 * 3] = 5, 4               # one lane, two vectors
    assert kernel_top2(x) == (5, 5 + 256 * 3)
    x[:] = 0
    x[40], x[47], x[8] = 5, 4, 4              # tie for second: another lane's lower id wins
    assert kernel_top2(x) == (40, 8)
    x[:] = 0
    x[8192 + 3], x[3] = 5, 5                  # tie across tiles
    assert kernel_top2(x) == (3, 8195)
