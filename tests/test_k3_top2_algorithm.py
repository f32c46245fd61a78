"""CPU check of K3's top-2 decomposition (paper_2602_18931_b200/csrc/kernels/rowstats.cu, Best2).

The kernel does not insert every element into a running top-2. Each thread keeps its two best
8-element vectors ranked by (vector max desc, vector index asc) and afterwards rescans only
those two. This test restates that thread partition in Python: 65536-wide chunks, 256 threads,
and thread t owning vectors t, t + 256, ... of its chunk. On tie-heavy rows the restatement must
give exactly the Prediction tie rule's top-2 (types.hpp:54-55: descending value, ties to the
lower id), which a brute-force sort provides. The GPU kernel itself is checked against the oracle
in tests/test_gpu_rowstats.py.
"""
import numpy as np
import pytest

CHUNK, THREADS = 65536, 256


def better(v, i, w, j):
    return v > w or (v == w and i < j)


def insert(top, v, i):
    (v1, i1), (v2, i2) = top
    if better(v, i, v2, i2):
        if better(v, i, v1, i1):
            return [(v, i), (v1, i1)]
        return [(v1, i1), (v, i)]
    return top


def kernel_top2(x):
    empty = [(-np.inf, 2**32 - 1), (-np.inf, 2**32 - 1)]
    row_top = empty
    for lo in range(0, len(x), CHUNK):
        hi = min(len(x), lo + CHUNK)
        nvec = (hi - lo) // 8
        for t in range(THREADS):
            top = empty
            b = [(-np.inf, None), (-np.inf, None)]  # Best2: (vector max, first element id)
            for vi in range(t, nvec, THREADS):
                id0 = lo + 8 * vi
                mx = float(x[id0:id0 + 8].max())
                p1 = b[0][1] is None or mx > b[0][0]
                p2 = b[1][1] is None or mx > b[1][0]
                if p1:
                    b = [(mx, id0), b[0]]
                elif p2:
                    b = [b[0], (mx, id0)]
            for _, id0 in b:
                if id0 is not None:
                    for j in range(8):
                        top = insert(top, float(x[id0 + j]), id0 + j)
            for e in range(lo + nvec * 8 + t, hi, THREADS):  # scalar tail
                top = insert(top, float(x[e]), e)
            for v, i in top:
                row_top = insert(row_top, v, i)
    return row_top[0][1], row_top[1][1]


def brute_top2(x):
    order = sorted(range(len(x)), key=lambda i: (-float(x[i]), i))
    return order[0], order[1]


@pytest.mark.parametrize("V,levels,seed", [(4100, 3, 1), (70001, 5, 2), (65536 + 24, 2, 3), (2048 * 8 + 5, 4, 4)])
def test_best2_rescan_matches_brute_force(V, levels, seed):
    rng = np.random.default_rng(seed)
    for _ in range(3):
        # few distinct values -> heavy ties inside vectors, threads and chunks
        x = rng.integers(0, levels, size=V).astype(np.float32)
        assert kernel_top2(x) == brute_top2(x)


def test_best2_same_vector_and_same_thread():
    x = np.zeros(70000, dtype=np.float32)
    x[100], x[103] = 5, 4                     # both in one vector
    assert kernel_top2(x) == (100, 103)
    x[:] = 0
    x[5], x[5 + 2048 * 3] = 5, 4              # one thread, two vectors
    assert kernel_top2(x) == (5, 5 + 2048 * 3)
    x[:] = 0
    x[40], x[47], x[8] = 5, 4, 4              # tie for second: another thread's lower id wins
    assert kernel_top2(x) == (40, 8)
