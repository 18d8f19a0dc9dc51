"""The hand-written stable merge sort of the K3 small-job sorts
(csrc/msort.cuh) against a stable sort on the host: random, few-distinct and
all-equal keys, sizes around the tile (1792) and merge-pass boundaries."""
import numpy as np
import pytest

import paper_2403_05821_b200 as po

pytestmark = pytest.mark.gpu


def _sort(a, b, v):
    lib = po._abi.cuda_lib()
    n = len(a)
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    v = np.ascontiguousarray(v, dtype=np.uint32)
    oa, ob = np.empty(max(n, 1), np.uint64), np.empty(max(n, 1), np.uint64)
    ov = np.empty(max(n, 1), np.uint32)
    lib.check(lib.debug_merge_sort(a.ctypes.data, b.ctypes.data, v.ctypes.data, n, oa.ctypes.data,
                                   ob.ctypes.data, ov.ctypes.data))
    return oa[:n], ob[:n], ov[:n]


@pytest.mark.parametrize("n", [0, 1, 2, 7, 8, 1791, 1792, 1793, 3584, 3585, 10_000, 100_003, 600_000])
@pytest.mark.parametrize("kind", ["random", "few", "equal", "sorted", "reversed"])
def test_merge_sort_is_stable_and_ordered(n, kind):
    rng = np.random.default_rng(n * 7 + len(kind))
    if kind == "random":
        a = rng.integers(0, 2**64 - 1, n, dtype=np.uint64)
        b = rng.integers(0, 2**64 - 1, n, dtype=np.uint64)
    elif kind == "few":
        a = rng.integers(0, 3, n).astype(np.uint64)
        b = rng.integers(0, 5, n).astype(np.uint64) << np.uint64(60)
    elif kind == "equal":
        a = np.full(n, 42, np.uint64)
        b = np.full(n, 7, np.uint64)
    elif kind == "sorted":
        a = np.arange(n, dtype=np.uint64) // 3
        b = np.zeros(n, np.uint64)
    else:
        a = (np.arange(n, dtype=np.uint64)[::-1] // 5).copy()
        b = np.zeros(n, np.uint64)
    v = np.arange(n, dtype=np.uint32)
    oa, ob, ov = _sort(a, b, v)
    order = np.lexsort((v, b, a))  # stable by (a, b): ties in input (= v) order
    assert np.array_equal(oa, a[order]) and np.array_equal(ob, b[order])
    assert np.array_equal(ov, v[order])
