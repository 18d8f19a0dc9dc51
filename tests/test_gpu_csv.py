"""CSV ingest on the GPU (csrc/csv.cu: parallel 6-state reader) against the
reference's own load_csv (oracle/_ref, table.hpp:114-215): same table, or
same error class and message, on random byte soups over the reader's
special bytes, on tables written with the reference's quoting rule, with
LF / CRLF / CR line ends, and at scale (the C2 table written as CSV)."""
import random

import numpy as np
import pytest

import paper_2403_05821_b200 as po
from csv_util import SOUPS, outcome, to_csv
from oracle.pyoracle import available, oracle
from paper_2403_05821_b200 import gen
from tables import ALPHABETS, random_table

pytestmark = pytest.mark.gpu


def _ref():
    return oracle("reference" if available("reference") else "port")


def test_csv_byte_soups():
    rng = random.Random(99)
    R = _ref()
    for _ in range(1500):
        d = bytes(rng.choice(rng.choice(SOUPS)) for _ in range(rng.randint(0, 60)))
        assert outcome(po.load_csv, d) == outcome(R.load_csv, d), d


def test_csv_known_cases():
    R = _ref()
    for d in [b"", b"\n", b"a\n", b"a", b"a,b\n1,2", b"a,b\n1,2\n", b"a,b\n1,2\n\n", b"a,b\n\n1,2\n",
              b'a\n"x', b'"a\nb",c\n1,2\n', b'a,b\r\n"1""2",3\r\n', b"a,a\n", b",b\n", b'"a"x,b\n',
              b'a\n""\n', b"a\r\r", b"a\n1\r\n\r\n"]:
        assert outcome(po.load_csv, d) == outcome(R.load_csv, d), d


def test_csv_written_tables():
    rng = random.Random(7)
    R = _ref()
    for _ in range(120):
        t = random_table(rng, 30, 5, rng.choice(list(ALPHABETS.values())), max_len=8, min_len=0)
        d = to_csv(t, rng.choice([b"\n", b"\r\n", b"\r"]))
        assert outcome(po.load_csv, d) == outcome(R.load_csv, d)


def test_csv_chunk_boundaries():
    # quoted cells with embedded newlines / quotes straddling the 4 KB chunks
    rng = random.Random(3)
    rows = [[bytes(rng.choice(b'ab,"\n\r ') for _ in range(rng.randint(0, 300))) for _ in range(3)]
            for _ in range(400)]
    t = po.Table([b"x", b"y", b"z"], rows)
    d = to_csv(t, b"\r\n")
    got = po.load_csv(d)
    assert outcome(lambda _: got, d) == outcome(_ref().load_csv, d)


def test_csv_c2_scale():
    t = gen.generate(2, n_rows=200_000)
    d = to_csv(t)
    got = po.load_csv(d)
    assert got.field_names == t.field_names and got.row_count() == t.row_count()
    assert np.array_equal(got.offsets, t.offsets) and np.array_equal(got.arena[: got.cell_bytes],
                                                                     t.arena[: t.cell_bytes])


@pytest.mark.parametrize("seed", range(6))
def test_csv_block_paths(seed):
    # texts of 20-200 KB made mostly of quote-free 16-byte blocks with commas,
    # LF / CRLF line ends, blank lines, runs of empty cells and rare quoted
    # cells: the transition, count and emit passes take their 16-byte block
    # paths (and fall back to bytes around quotes and CRs) across many 4 KB
    # chunks; compared with the reference reader (table or error)
    rng = random.Random(1000 + seed)
    R = _ref()
    width = rng.randint(1, 7)
    eol = rng.choice([b"\n", b"\r\n"])
    # seeds 0, 3: blank lines; 1, 4: wrong widths (errors); 2, 5: clean tables
    p_blank = 0.03 if seed % 3 == 0 else 0.0
    p_wide = 0.03 if seed % 3 == 1 else 0.0
    lines = [b",".join(b"h%d" % i for i in range(width))]
    for _ in range(rng.randint(100, 1500)):
        if rng.random() < p_blank:
            lines.append(b"")  # a blank line (an error unless it is the last)
            continue
        cells = []
        for _ in range(width if rng.random() >= p_wide else rng.randint(1, width + 2)):
            k = rng.choice([0, 0, 1, 5, 15, 16, 17, 40, 120])
            v = bytes(rng.choice(b"abcdefghij klmnop") for _ in range(k))
            if rng.random() < 0.02:
                v = b'"' + v.replace(b'"', b'""') + b',"'
            cells.append(v)
        lines.append(b",".join(cells))
    d = eol.join(lines) + (eol if rng.random() < 0.7 else b"")
    assert outcome(po.load_csv, d) == outcome(R.load_csv, d)
