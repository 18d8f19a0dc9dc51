"""The hand-written onesweep radix sort of the K8 row-key sorts (csrc/radix.cu)
against a stable sort on the host: random, skewed, constant and all-equal
digits, every bit range width, sizes around the tile boundaries."""
import random

import numpy as np
import pytest

import paper_2403_05821_b200 as po

pytestmark = pytest.mark.gpu


def _sort(keys, vals, lo, hi):
    lib = po._abi.cuda_lib()
    n = len(keys)
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    v = np.ascontiguousarray(vals, dtype=np.uint32)
    ok = np.empty(max(n, 1), np.uint64)
    ov = np.empty(max(n, 1), np.uint32)
    lib.check(lib.debug_radix_sort(k.ctypes.data, v.ctypes.data, n, lo, hi, ok.ctypes.data,
                                   ov.ctypes.data))
    return ok[:n], ov[:n]


def _expect(keys, vals, lo, hi):
    mask = np.uint64((1 << (hi - lo)) - 1) if hi - lo < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
    digit = (keys >> np.uint64(lo)) & mask if hi > lo else np.zeros_like(keys)
    order = np.argsort(digit, kind="stable")
    return keys[order], vals[order]


@pytest.mark.parametrize("n", [0, 1, 5, 2047, 2048, 2049, 100_000, 1_000_003])
def test_radix_sort_matches_stable_sort(n):
    rng = np.random.default_rng(n)
    for lo, hi in [(0, 64), (0, 13), (3, 40), (32, 64), (0, 8), (7, 7)]:
        for kind in ("random", "skewed", "constant"):
            if kind == "random":
                keys = rng.integers(0, 2**63, n, dtype=np.uint64) * np.uint64(2) + \
                    rng.integers(0, 2, n, dtype=np.uint64)
            elif kind == "skewed":
                keys = (rng.zipf(1.3, n).astype(np.uint64) << np.uint64(lo)) | \
                    rng.integers(0, 4, n, dtype=np.uint64)
            else:
                keys = np.full(n, 0x1234_5678_9ABC_DEF0, np.uint64)
            vals = np.arange(n, dtype=np.uint32)
            gk, gv = _sort(keys, vals, lo, hi)
            ek, ev = _expect(keys, vals, lo, hi)
            assert np.array_equal(gv, ev), (n, lo, hi, kind)
            assert np.array_equal(gk, ek), (n, lo, hi, kind)
