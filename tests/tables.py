"""Deterministic table families for the parity tests.

Python restatements of the reference test generators' SHAPES
(proj/tests/test_util.hpp:17-63, test_solver_greedy.cpp:28-44) plus byte-
class stress tables; the exact byte contents need not match the reference's
std::mt19937 streams because every comparison is differential (GPU vs the
oracle on the same table)."""
from __future__ import annotations

import random

from paper_2403_05821_b200 import Table

ALPHABETS = {
    "ab": b"ab",
    "esc": b'ab "\\\n\x01 \t',
    "all": bytes(range(256)),
    "ws": b"a b\t\n\x0b\x0c\r",
}


def random_table(rng: random.Random, max_rows: int, max_fields: int, alphabet: bytes = b"ab",
                 max_len: int = 3, min_len: int = 1, min_rows: int = 1) -> Table:
    n = rng.randint(min_rows, max_rows)
    m = rng.randint(1, max_fields)
    rows = [[bytes(rng.choice(alphabet) for _ in range(rng.randint(min_len, max_len)))
             for _ in range(m)] for _ in range(n)]
    return Table([f"f{i}" for i in range(m)], rows)


def distinct_first_table(n: int, m: int) -> Table:
    rows = [[bytes([ord("a") + r])] + [bytes([ord("A") + f]) for f in range(1, m)]
            for r in range(n)]
    return Table([f"f{i}" for i in range(m)], rows)


def group_per_field_table(x: int, m: int) -> Table:
    n = m * x
    nxt = [ord("a")]

    def fresh():
        v = bytes([nxt[0]])
        nxt[0] += 1
        return v

    gv = [fresh() for _ in range(m)]
    rows = []
    for r in range(n):
        g = r // x
        rows.append([gv[g] if f == g else fresh() for f in range(m)])
    return Table([f"f{i}" for i in range(m)], rows)


def fd_covered_table(rng: random.Random, max_rows: int, max_fields: int) -> Table:
    n = rng.randint(2, max_rows)
    m = rng.randint(2, max_fields)
    ents = rng.randint(1, n)
    tuples = [[bytes([ord("a") + (e * m + f) % 26]) * rng.randint(1, 3) + str(e).encode()
               for f in range(m)] for e in range(ents)]
    rows = [list(tuples[rng.randrange(ents)]) for _ in range(n)]
    return Table([f"f{i}" for i in range(m)], rows)


def skewed_table(rng: random.Random, n: int, cards: list[int], lens: list[int],
                 alphabet: bytes = b"abcdefgh ") -> Table:
    """Columns with controlled cardinality and value length (C1-like)."""
    pools = []
    for card, ln in zip(cards, lens):
        pool = set()
        while len(pool) < card:
            pool.add(bytes(rng.choice(alphabet) for _ in range(rng.randint(max(1, ln // 2), ln))))
        pools.append(sorted(pool))
    rows = []
    for _ in range(n):
        rows.append([p[min(int(rng.paretovariate(1.2)) - 1, len(p) - 1)] if rng.random() < 0.7
                     else rng.choice(p) for p in pools])
    return Table([f"col{i}" for i in range(len(cards))], rows)
