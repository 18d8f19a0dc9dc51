"""FD validation / discovery on the GPU dictionary (po_fd_compare, csrc/fd.cu)
against the compiled reference (oracle/_ref: the reference's own
validate_fds / discover_fds, fd.hpp:66-141) and the reference's unit-test
known answers (test_table.cpp:166-227)."""
import random

import pytest

import paper_2403_05821_b200 as po
from fd_cases import known_fd_cases
from oracle.pyoracle import available, oracle
from paper_2403_05821_b200 import gen
from tables import ALPHABETS, random_table

pytestmark = pytest.mark.gpu


def _ref():
    return oracle("reference" if available("reference") else "port")


def test_fd_known_answers_gpu():
    for name, check in known_fd_cases():
        check(po)


@pytest.mark.parametrize("alpha", sorted(ALPHABETS))
def test_fd_random_tables_vs_reference(alpha):
    rng = random.Random(77)
    R = _ref()
    for _ in range(60):
        t = random_table(rng, 40, 6, ALPHABETS[alpha], max_len=rng.randint(1, 3))
        assert po.discover_fds(t, 1000) == R.discover_fds(t, 1000)
        names = [t.field_name(f) for f in range(t.field_count())]
        rng.shuffle(names)
        cuts = sorted(rng.sample(range(len(names) + 1), 2))
        groups = [g for g in (names[:cuts[0]], names[cuts[0]:cuts[1]], names[cuts[1]:]) if g]
        assert po.validate_fds(t, groups) == R.validate_fds(t, groups)


def test_fd_copied_columns_large():
    # columns that are exact copies / renamings of each other at 30K rows
    rng = random.Random(5)
    vals = [bytes([rng.randrange(256) for _ in range(rng.randint(0, 6))]) for _ in range(900)]
    rows = []
    for _ in range(30_000):
        v = rng.randrange(len(vals))
        rows.append([vals[v], b"k" + str(v).encode(), vals[rng.randrange(len(vals))], vals[v][::-1]])
    t = po.Table([b"a", b"b", b"c", b"d"], rows)
    got = po.discover_fds(t, 100_000)
    assert got == oracle("port").discover_fds(t, 100_000)
    rep = po.validate_fds(t, [[b"a", b"c"], [b"b", b"d"]])
    assert rep == oracle("port").validate_fds(t, [[b"a", b"c"], [b"b", b"d"]])


def test_fd_c3_prefix():
    t = gen.generate(3, n_rows=20_000)
    fds = gen.fds(3)
    assert po.validate_fds(t, fds) == oracle("port").validate_fds(t, fds)
    assert po.discover_fds(t, 50_000) == oracle("port").discover_fds(t, 50_000)
